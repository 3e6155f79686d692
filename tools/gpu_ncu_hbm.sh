#!/bin/bash
# usage: bash tools/gpu_ncu_hbm.sh TAG -- ncu --set full of the HBM-bound kernels (split A, split B, fold) of the bench step
TAG=${1:-r}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_hbm_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_hbm_$TAG.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fold_normalize|split_kernel" -s 3 -c 3 -o gpurun_out/prof_hbm_$TAG $CMD > gpurun_out/ncu_hbm_$TAG.log 2>&1; echo "ncu rc=$?"
