#!/bin/bash
# power experiment (results invalid when MPCGEMM_DBG != 0): slice-GEMM time / clock with the partial
# stores off (1), operands from one L2 tile (2), ~1 MB of varying L2-resident operands (4), no operand
# traffic after the first ring fill (8)
for D in 0 2 8 10 0; do
  MPCGEMM_DBG=$D timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/pow_$D.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pow_$D.json')); print('dbg=$D', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks'])"
done
