#!/bin/bash
# usage: bash tools/gpu_round2.sh TAG -- full GPU suite (with durations), bench, ncu launch list
TAG=${1:-r}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -25 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'clk', d['clocks'])
print('roof', {k: d['roofline'][k] for k in ('achieved','peak','frac','frac_vs_in_run_mma_ceiling','ceilings_in_run') if k in d['roofline']})
for h in d['hbm_kernels']: print(h['kernel'], h['ms'], h['frac'])
print('4M', d.get('method_4M')); print('e2e', d.get('e2e',{}).get('ms_per_step'), d.get('e2e',{}).get('blocking_ms_per_step'))
print('cpu', d.get('cpu_baseline'))
"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
