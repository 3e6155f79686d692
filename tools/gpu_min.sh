#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_device_rule.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/min_pt.log 2>&1; tail -2 gpurun_out/min_pt.log
for w in j1 2; do
timeout 300 python tools/small_calls.py $w > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/small_calls.py $w 2>/dev/null | grep -E "duration" | tail -7 | awk -F'"' '{print $(NF-1), substr($10,1,50)}'
done
MPCGEMM_PREPASS_SMALL=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/small_calls.py 2 2>/dev/null | grep -E "prepass_min" | tail -1 | awk -F'"' '{print "cfg2 min (T GEMM path)", $(NF-1)}'
timeout 600 python tools/bench_configs.py > gpurun_out/configs_min.json 2>/dev/null; python -c "
import json
for r in json.load(open('gpurun_out/configs_min.json'))['configs']: print(r['config'], r['method'], round(r['ms'],4), round(r['gemm_ms'],4))"
