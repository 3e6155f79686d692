#!/bin/bash
# GPU suite, then small-call latency (call_latency.py) and the per-kernel launch list of small calls
TAG=${1:-r}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python tools/call_latency.py > gpurun_out/lat_$TAG.json 2>&1; echo "latency rc=$?"; tail -1 gpurun_out/lat_$TAG.json
bash tools/gpu_small_ncu.sh $TAG
