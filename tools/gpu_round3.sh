#!/bin/bash
# checkpoint: final suite + bench + ncu (gpu_final.sh), then all configs and small-call latency
TAG=${1:-r}
bash tools/gpu_final.sh $TAG
timeout 1200 python tools/bench_configs.py > gpurun_out/configs_$TAG.json 2>/dev/null; echo "configs rc=$?"
timeout 600 python tools/call_latency.py > gpurun_out/lat_$TAG.json 2>&1; echo "latency rc=$?"; tail -1 gpurun_out/lat_$TAG.json
