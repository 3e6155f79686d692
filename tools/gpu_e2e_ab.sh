#!/bin/bash
# e2e A/B: TMA split vs the per-thread split, twice each (bench line e2e ms and step ms)
for V in 0 1 0 1; do
  if [ $V = 1 ]; then export MPCGEMM_SPLIT_V1=1; else unset MPCGEMM_SPLIT_V1; fi
  timeout 600 python bench.py --no-cpu > gpurun_out/e2e_ab_$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_ab_$V.json')); print('split_v1=$V', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['stages_ms']['ms_split'], d['clocks']['sm_mhz'])"
done
