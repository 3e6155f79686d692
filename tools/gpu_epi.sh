#!/bin/bash
# slice-GEMM epilogue change: parity, config 5 stages, config 4 bench, old (HEAD lib) vs new
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_counts.py tests/test_gpu_determinism.py -x -q > gpurun_out/epi_pt.log 2>&1; tail -2 gpurun_out/epi_pt.log
for v in old new; do
  unset MPCGEMM_LIB; [ $v = old ] && export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so
  timeout 600 python tools/cfg5_stages.py | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v cfg5', d['total'])"
done
for it in 1 2; do
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
done
unset MPCGEMM_LIB
CONFIGS=1,2,3 timeout 900 python tools/bench_configs.py > gpurun_out/cfg_epi.json 2>/dev/null
python -c "
import json
for r in json.load(open('gpurun_out/cfg_epi.json'))['configs']: print(r['config'], r['method'], round(r['ms'],4), round(r['gemm_ms'],4))"
