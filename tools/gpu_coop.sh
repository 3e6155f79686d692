#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_device_rule.py -x -q -p no:cacheprovider > gpurun_out/coop_pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/coop_pt.log
timeout 300 python tools/call_latency.py > gpurun_out/lat_coop.json 2>&1; echo "latency rc=$?"; tail -1 gpurun_out/lat_coop.json
timeout 300 python tools/small_calls.py 1 > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/small_calls.py 1 2>/dev/null | grep -E "duration" | tail -4 | awk -F'"' '{print $(NF-1), substr($10,1,50)}'
