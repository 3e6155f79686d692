#!/bin/bash
# device-rule tests (fused small pre-pass and the tcgen05 T GEMM path), small-call latency, launch list
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_rule.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pt_$TAG.log 2>&1; tail -2 gpurun_out/pt_$TAG.log
timeout 600 python tools/call_latency.py > gpurun_out/lat_$TAG.json 2>&1; echo "latency rc=$?"; tail -1 gpurun_out/lat_$TAG.json
MPCGEMM_PREPASS_SMALL=0 timeout 600 python tools/call_latency.py > gpurun_out/lat0_$TAG.json 2>&1; echo "latency(small=0) rc=$?"; tail -1 gpurun_out/lat0_$TAG.json
bash tools/gpu_small_ncu.sh $TAG 2>&1 | head -40
