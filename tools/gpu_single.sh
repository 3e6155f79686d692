#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_rule.py -x -q -p no:cacheprovider > gpurun_out/single_pt.log 2>&1; tail -3 gpurun_out/single_pt.log
timeout 600 python tools/call_latency.py > gpurun_out/lat_single.json 2>&1; echo "latency rc=$?"; tail -1 gpurun_out/lat_single.json
timeout 300 python tools/small_calls.py 1 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/small_calls.py 1 2>/dev/null | grep -E "duration" | tail -5 | awk -F'"' '{print $(NF-1), substr($10,1,60)}'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prepass_single -s 3 -c 1 -o gpurun_out/prof_single python tools/small_calls.py 1 > /dev/null 2>&1; echo "ncu rc=$?"
