#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_unic2.log 2>&1; tail -2 gpurun_out/pt_unic2.log
for it in 1 2; do
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  for meth in 3M 4M; do
    timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra --method $meth > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v $meth', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
  done
done
done
