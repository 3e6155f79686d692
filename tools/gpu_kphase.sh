#!/bin/bash
# k-phase hand-off A/B: parity, bench GEMM ms with MPCGEMM_HANDOFF=1/0, DRAM bytes of the slice GEMM
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -1
run() {  # tag env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/kp_$tag.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/kp_$tag.json')); print('$tag', round(d['ms_per_step'],1), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])"
}
ncurun() {
  local tag=$1; shift
  env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    -k regex:slicegemm_tc2 -c 1 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 0 > gpurun_out/kp_ncu_$tag.csv 2>/dev/null
  grep -E "dram__|hit_rate|duration" gpurun_out/kp_ncu_$tag.csv | awk -F'"' -v t=$tag '{print t, $(NF-5), $(NF-1)}'
}
run h1 MPCGEMM_HANDOFF=1
run h0 MPCGEMM_HANDOFF=0
run h1b MPCGEMM_HANDOFF=1
run h0b MPCGEMM_HANDOFF=0
ncurun h1 MPCGEMM_HANDOFF=1
ncurun h0 MPCGEMM_HANDOFF=0
