#!/bin/bash
# power experiment: slice-GEMM time / clock / power with the partial stores off (1), operands L2-resident (2), both (3)
for D in 0 4 5 2 0; do
  MPCGEMM_DBG=$D timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/pow_$D.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pow_$D.json')); print('dbg=$D', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks'])"
done
