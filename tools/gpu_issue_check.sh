#!/bin/bash
# slice GEMM issue-rate check per L2 promotion: bench GEMM ms, and one ncu launch with the IMMA-active and DRAM metrics
mkdir -p gpurun_out
for V in 128 128; do
  MPCGEMM_L2PROMO=$V timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/ic_$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ic_$V.json')); print('promo=$V bench', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])"
done
for V in 128; do
  MPCGEMM_L2PROMO=$V timeout 900 ncu --clock-control none --metrics sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    -k regex:slicegemm_tc2 -c 1 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 0 2>/dev/null | grep -E "imma|dram__|duration|per_second" | awk -F'"' -v t=$V '{print "promo=" t, $(NF-5), $(NF-1)}'
done
