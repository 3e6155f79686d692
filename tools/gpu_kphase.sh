#!/bin/bash
# TMA L2 promotion A/B for the digit-plane maps (MPCGEMM_L2PROMO): bench GEMM ms and DRAM bytes
mkdir -p gpurun_out
for V in 256 128 0 256 128 0; do
  MPCGEMM_L2PROMO=$V timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/kp_$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/kp_$V.json')); print('promo=$V', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])"
done
for V in 128 0; do
  MPCGEMM_L2PROMO=$V timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:slicegemm_tc2 -c 1 --csv \
    python bench.py --no-e2e --no-cpu --steps 1 --warmup 0 2>/dev/null | grep -E "dram__" | awk -F'"' -v t=$V '{print "promo=" t, $(NF-5), $(NF-1)}'
done
