#!/bin/bash
# A/B of the current tree vs MPCGEMM_PBLK=0 (no p-blocks, no lead stages): parity, bench GEMM ms
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -1
for T in a b a b; do
  timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/kp_$T.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/kp_$T.json')); print('$T', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])"
done
