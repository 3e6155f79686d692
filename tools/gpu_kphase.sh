#!/bin/bash
# full GPU suite with the defaults (k-phase hints, p-blocks of 32), then serpentine / p-block A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
run() {  # tag env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/kp_$tag.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/kp_$tag.json')); print('$tag', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])"
}
run def
run serp0 MPCGEMM_SERPENTINE=0
run pb40 MPCGEMM_PBLK=40
run def2
run serp0b MPCGEMM_SERPENTINE=0
run pb28 MPCGEMM_PBLK=28
