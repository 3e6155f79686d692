#!/bin/bash
# usage: bash tools/gpu_devrule2.sh TAG -- device-rule tests, latency of small configs, ncu full of the cfg1 GEMM + fold
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_rule.py tests/test_gpu_counts.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_dr_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dr_$TAG.log
tail -3 gpurun_out/pytest_dr_$TAG.log
timeout 600 python tools/call_latency.py > gpurun_out/latency_$TAG.json 2> gpurun_out/latency_$TAG.err; echo "lat rc=$?"
head -6 gpurun_out/latency_$TAG.json; tail -3 gpurun_out/latency_$TAG.err
timeout 600 ncu --set full --clock-control none -k regex:"fold_normalize|slicegemm_tc_kernel" -s 2 -c 2 -o gpurun_out/prof_small_$TAG python tools/small_calls.py 1 > gpurun_out/ncu_small_$TAG.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_small_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_small_$TAG.csv 2>/dev/null
python tools/ncu_raw_summary.py gpurun_out/raw_small_$TAG.csv 2>&1 | head -50
