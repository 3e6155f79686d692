#!/bin/bash
# split A/B: HEAD library (libmpcgemm_ab_old.so) vs the working tree, in-step split ms (bench) and ncu split time
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/split_pt.log 2>&1; tail -2 gpurun_out/split_pt.log
for it in 1 2; do
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
done
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:split2_tma -c 2 --csv \
    python bench.py --no-e2e --no-cpu --no-extra --steps 1 --warmup 0 2>/dev/null | grep -E "duration|inst_exec" | awk -F'"' -v t=$v '{print t, $(NF-5), $(NF-1)}'
done
unset MPCGEMM_LIB
