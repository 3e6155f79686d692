#!/bin/bash
# usage: bash tools/gpu_devrule.sh TAG -- device-rule tests + per-call latency of the small configs
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_rule.py tests/test_gpu_counts.py -q -p no:cacheprovider -x > gpurun_out/pytest_dr_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dr_$TAG.log
tail -30 gpurun_out/pytest_dr_$TAG.log
timeout 600 python tools/call_latency.py > gpurun_out/latency_$TAG.json 2> gpurun_out/latency_$TAG.err; echo "lat rc=$?"
cat gpurun_out/latency_$TAG.json | head -8; tail -5 gpurun_out/latency_$TAG.err
