#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_fold.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fold_normalize" -s 0 -c 1 -o gpurun_out/prof_fold_$TAG $CMD > gpurun_out/ncu_fold_$TAG.log 2>&1; echo "ncu rc=$?"
