#!/bin/bash
# full GPU suite, small-call latency, all configs, then a short bench line
TAG=${1:-r}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python tools/call_latency.py > gpurun_out/lat_$TAG.json 2>&1; echo "latency rc=$?"; tail -1 gpurun_out/lat_$TAG.json
timeout 1200 python tools/bench_configs.py > gpurun_out/configs_$TAG.json 2>/dev/null; echo "configs rc=$?"
python -c "
import json
for r in json.load(open('gpurun_out/configs_$TAG.json'))['configs']: print(r['config'], r['method'], round(r['ms'],4), round(r['gemm_ms'],4))"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'clk', d['clocks']['sm_mhz'])"
