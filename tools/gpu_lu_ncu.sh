#!/bin/bash
# usage: bash tools/gpu_lu_ncu.sh TAG -- LU kernel launch list (one factorization, n=512, prec 256/768, K=64)
TAG=${1:-r}
mkdir -p gpurun_out
CMD="python tools/bench_lu.py --n 512 --precs 256,512,768 --Ks 64"
timeout 600 $CMD > gpurun_out/lu_plain_$TAG.json 2>&1 || { echo "plain failed"; tail gpurun_out/lu_plain_$TAG.json; exit 1; }
cat gpurun_out/lu_plain_$TAG.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_launches_$TAG.csv $CMD > gpurun_out/lu_ncu_$TAG.log 2>&1
echo "ncu rc=$?"
