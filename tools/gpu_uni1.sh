#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_u1_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_u1_$TAG.log
for cfg in "X=0" "MPCGEMM_FOLD_NOUNI1=1"; do env $cfg timeout 300 python tools/call_latency.py 2>/dev/null | grep "cfg2_3M\|cfg5" | head -3; done
for cfg in "X=0" "MPCGEMM_FOLD_NOUNI1=1"; do
env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"fold_normalize" --csv --log-file gpurun_out/ncu_u1_$TAG.csv python tools/small_calls.py j1 > /dev/null 2>&1
echo "[$cfg]"; python tools/ncu_summary.py gpurun_out/ncu_u1_$TAG.csv | tail -3
done
