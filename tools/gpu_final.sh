#!/bin/bash
# usage: bash tools/gpu_final.sh TAG -- GPU suite, bench line, ncu launch list, ncu --set full of the GEMM / split / fold
TAG=${1:-r}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'value', d['value'], 'stages', d['stages_ms'], 'clk', d['clocks'])
print('roof', {k: d['roofline'][k] for k in ('achieved','peak','frac','frac_vs_in_run_mma_ceiling','ceilings_in_run') if k in d['roofline']})
for h in d['hbm_kernels']: print(h['kernel'], h['ms'], h['frac'])
print('4M', d.get('method_4M')); print('e2e', d.get('e2e',{}).get('ms_per_step'), d.get('e2e',{}).get('blocking_ms_per_step'))
print('launches', d['gpu_launches'], 'cpu', d.get('cpu_baseline',{}).get('value'))
"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:slicegemm_tc2 -s 1 -c 1 -o gpurun_out/prof_gemm_$TAG $CMD > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fold_normalize|split2?_tma_kernel" -s 0 -c 3 -o gpurun_out/prof_hbm_$TAG $CMD > gpurun_out/ncu_hbmf_$TAG.log 2>&1; echo "ncu hbm rc=$?"
for f in gemm hbm; do ncu -i gpurun_out/prof_${f}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${f}_$TAG.csv 2>/dev/null; python tools/ncu_raw_summary.py gpurun_out/raw_${f}_$TAG.csv > gpurun_out/sum_${f}_$TAG.txt 2>&1; done
cat gpurun_out/sum_gemm_$TAG.txt | head -24
