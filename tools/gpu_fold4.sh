#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -x -q > gpurun_out/f4_pt.log 2>&1; tail -2 gpurun_out/f4_pt.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
for v in 0 1; do
  MPCGEMM_FOLD_L2HINT=$v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:fold_normalize -s 1 -c 1 --csv --log-file gpurun_out/ncu_f4_$v.csv $CMD > /dev/null 2>&1
  echo "== L2HINT $v"; python tools/ncu_summary.py gpurun_out/ncu_f4_$v.csv | tail -7
done
bash tools/gpu_env_ab.sh "MPCGEMM_FOLD_L2HINT=0" "MPCGEMM_FOLD_L2HINT=1"
