#!/bin/bash
# usage: bash tools/gpu_env_ab.sh "ENV=val ..." "ENV=val ..."   -- bench under two env settings, twice each
mkdir -p gpurun_out
for it in 1 2; do
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/envab.json 2>gpurun_out/envab.err
  python -c "import json;d=json.load(open('gpurun_out/envab.json'));print('[$cfg]', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'], d['roofline']['achieved'])" || tail -3 gpurun_out/envab.err
done
done
