#!/bin/bash
# usage: bash tools/gpu_ncu_full.sh TAG  -- ncu --set full of the top kernels (1 GPU)
TAG=${1:-r}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_full_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_full_$TAG.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:slicegemm_tc -s 1 -c 1 -o gpurun_out/prof_gemm_$TAG $CMD > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fold_normalize|split_tma_kernel" -s 0 -c 3 -o gpurun_out/prof_hbm_$TAG $CMD > gpurun_out/ncu_hbm_$TAG.log 2>&1; echo "ncu hbm rc=$?"
ls -la gpurun_out/*.ncu-rep
