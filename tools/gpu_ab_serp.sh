#!/bin/bash
# A/B of the serpentine k order: targeted ncu metrics of the slice GEMM (DRAM reads, L2 hit, time, clock)
mkdir -p gpurun_out
for S in 1 0; do
  MPCGEMM_SERPENTINE=$S timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:slicegemm_tc2 -s 1 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu 2>/dev/null > gpurun_out/ab_serp_ncu_$S.csv
done
