#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_hn_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_hn_$TAG.log
for cfg in "X=0" "MPCGEMM_HALFN=0" "X=0" "MPCGEMM_HALFN=0"; do env $cfg timeout 300 python tools/call_latency.py 2>/dev/null | grep "cfg5_3M" | head -1; done
