#!/bin/bash
# usage: bash tools/gpu_fold2.sh TAG -- fold: parity tests, bench fold time, cfg5 latency, ncu fold instructions
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_fuzz.py tests/test_gpu_device_rule.py tests/test_gpu_lu.py -q -p no:cacheprovider -x > gpurun_out/pytest_fold_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_fold_$TAG.log
for cfg in "X=0" "X=0"; do
  env $cfg timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/fab_$TAG.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/fab_$TAG.json').read().strip().splitlines()[-1])
print('[$cfg] step', round(d['ms_per_step'],2), 'fold', d['stages_ms']['ms_fold'], 'split', d['stages_ms']['ms_split'], 'gemm', d['stages_ms']['ms_gemm'], 'MHz', d['clocks']['sm_mhz'])"
done
timeout 600 python tools/call_latency.py > gpurun_out/latency_$TAG.json 2> gpurun_out/latency_$TAG.err; echo "lat rc=$?"
head -6 gpurun_out/latency_$TAG.json
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,sm__issue_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"fold_normalize" -s 1 -c 1 --csv --log-file gpurun_out/ncu_fold_$TAG.csv $CMD > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_fold_$TAG.csv | tail -5
