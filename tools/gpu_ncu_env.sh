#!/bin/bash
# usage: bash tools/gpu_ncu_env.sh TAG "ENV=.. ENV=.." ...  -- targeted ncu metrics of the slice GEMM per env setting
TAG=$1; shift
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  i=$((i+1))
  CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
  env $cfg timeout 600 $CMD > gpurun_out/plain_env.log 2>&1 && \
  env $cfg timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"slicegemm_tc" -s 1 -c 1 --csv --log-file gpurun_out/ncu_env_${TAG}_$i.csv $CMD > /dev/null 2>&1
  echo "== [$cfg]"; python tools/ncu_summary.py gpurun_out/ncu_env_${TAG}_$i.csv | tail -7
done
