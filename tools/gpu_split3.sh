#!/bin/bash
# split: PTX carry chains + 4x4 byte transposes vs HEAD lib
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -x -q > gpurun_out/s3_pt.log 2>&1; tail -2 gpurun_out/s3_pt.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
for v in new old; do
  unset MPCGEMM_LIB; [ $v = old ] && export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"split2?_tma" -s 1 -c 1 --csv --log-file gpurun_out/ncu_s3_$v.csv $CMD > /dev/null 2>&1
  echo "== $v"; python tools/ncu_summary.py gpurun_out/ncu_s3_$v.csv | tail -6
done
unset MPCGEMM_LIB
for it in 1 2; do
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
done
