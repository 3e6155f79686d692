#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/epi2_pt.log 2>&1; tail -2 gpurun_out/epi2_pt.log
for v in old new; do
  unset MPCGEMM_LIB; [ $v = old ] && export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so
  timeout 600 python tools/cfg5_stages.py | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v cfg5', d['total'], [r['ms_gemm'] for r in d['gemms']][-4:])"
  CONFIGS=1,2 timeout 900 python tools/bench_configs.py > gpurun_out/cfg_epi.json 2>/dev/null
  python -c "
import json
for r in json.load(open('gpurun_out/cfg_epi.json'))['configs']: print('$v', r['config'], r['method'], round(r['ms'],4), round(r['gemm_ms'],4))"
done
