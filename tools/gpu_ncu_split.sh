#!/bin/bash
# usage: bash tools/gpu_ncu_split.sh TAG -- ncu --set full of the two split launches of one bench step
TAG=${1:-r}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_split_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_tma" -s 2 -c 2 -o gpurun_out/prof_split_$TAG $CMD > gpurun_out/ncu_split_$TAG.log 2>&1; echo "ncu rc=$?"
