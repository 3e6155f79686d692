#!/bin/bash
# usage: bash tools/gpu_iter2.sh TAG [pytest -k expr] -- GPU suite, bench, ncu launch list + HBM kernels
TAG=${1:-r}
K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$K" > gpurun_out/pytest_gpu_$TAG.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'e2e', round(d.get('e2e',{}).get('ms_per_step',0),1), 'clk', d['clocks'].get('sm_mhz'))
for h in d['hbm_kernels']: print(h['kernel'], h['ms'], h['frac'])
" 2>&1 | tail -4
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fold_normalize|split_tma" --csv --log-file gpurun_out/ncu_hbm2_$TAG.csv $CMD > gpurun_out/ncu_hbm2_$TAG.log 2>&1
echo "ncu rc=$?"; python tools/ncu_summary.py gpurun_out/ncu_hbm2_$TAG.csv 2>&1 | tail -12
