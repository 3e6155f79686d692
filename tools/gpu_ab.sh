#!/bin/bash
# A/B: bench with the old library then the new, alternating, same box
mkdir -p gpurun_out
for it in 1 2; do
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_${v}_$it.json 2>gpurun_out/ab_${v}_$it.err
  python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$it.json'));print('$v', d['ms_per_step'], d['stages_ms'], d['clocks'])"
done
done
