#!/bin/bash
# usage: bash tools/gpu_ncu_split2.sh TAG -- bench + ncu --set full of the split kernels and the fold
TAG=${1:-r}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_split_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_split_$TAG.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'stages', d['stages_ms'], 'clk', d['clocks'].get('sm_mhz'))
for h in d['hbm_kernels']: print(h['kernel'], h['ms'], h['frac'])
"
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fold_normalize|split_tma_kernel" -s 0 -c 3 -o gpurun_out/prof_hbm_$TAG $CMD > gpurun_out/ncu_hbm_$TAG.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_hbm_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_hbm_$TAG.csv 2>/dev/null
python tools/ncu_raw_summary.py gpurun_out/raw_hbm_$TAG.csv 2>&1 | head -60
