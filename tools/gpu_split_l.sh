#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_lu.py -q -p no:cacheprovider -x > gpurun_out/pytest_sl_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_sl_$TAG.log
for cfg in "X=0" "MPCGEMM_SPLIT_V1=1"; do env $cfg timeout 300 python tools/call_latency.py 2>/dev/null | grep "cfg5" | head -2; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"split" --csv --log-file gpurun_out/ncu_sl_$TAG.csv python tools/small_calls.py j1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_sl_$TAG.csv | tail -8
