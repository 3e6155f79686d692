#!/bin/bash
# fold at 7 CTAs/SM vs HEAD lib: cfg4 ncu + in-step, cfg2 / cfg5 per-call
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -x -q > gpurun_out/f7_pt.log 2>&1; tail -1 gpurun_out/f7_pt.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
for v in old new; do
  unset MPCGEMM_LIB; [ $v = old ] && export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:fold_normalize -s 1 -c 1 --csv --log-file gpurun_out/ncu_f7_$v.csv $CMD > /dev/null 2>&1
  echo "== $v"; python tools/ncu_summary.py gpurun_out/ncu_f7_$v.csv | tail -4
  CONFIGS=2,5 timeout 900 python tools/bench_configs.py > gpurun_out/cfg_f7.json 2>/dev/null
  python -c "
import json
for r in json.load(open('gpurun_out/cfg_f7.json'))['configs']: print('$v', r['config'], r['method'], round(r['ms'],4), r['stages_ms']['ms_fold'])"
done
for it in 1 2; do
for v in old new; do
  if [ $v = old ]; then export MPCGEMM_LIB=$PWD/paper_2307_06072_b200/libmpcgemm_ab_old.so; else unset MPCGEMM_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],2), d['stages_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
done
