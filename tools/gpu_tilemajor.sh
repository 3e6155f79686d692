#!/bin/bash
# tile-major unit order + tile-wide k-phase hints (MPCGEMM_ORDER=3 MPCGEMM_KPHASE=3): parity under
# the new order, bench GEMM ms A/B against the default, ncu DRAM bytes of the slice GEMM
mkdir -p gpurun_out
MPCGEMM_ORDER=3 MPCGEMM_KPHASE=3 MPCGEMM_PBLK=32 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_counts.py tests/test_gpu_device_rule.py tests/test_gpu_adaptive.py -x -q -p no:cacheprovider > gpurun_out/tm_pt.log 2>&1; tail -2 gpurun_out/tm_pt.log
run() {  # tag order kphase pblk
  MPCGEMM_ORDER=$2 MPCGEMM_KPHASE=$3 MPCGEMM_PBLK=$4 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/tm.json 2>gpurun_out/tm.err
  python -c "import json;d=json.load(open('gpurun_out/tm.json'));print('$1', round(d['ms_per_step'],2), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tm.err
}
for it in 1 2; do
  run base 2 2 64
  run t3p32 3 3 32
  run t3p24 3 3 24
  run t3p64 3 3 64
  run t2p64 3 2 64
done
for cfg in "2 2 64" "3 3 32" "3 3 24"; do
  set -- $cfg
  MPCGEMM_ORDER=$1 MPCGEMM_KPHASE=$2 MPCGEMM_PBLK=$3 timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second -k regex:slicegemm_tc2 -c 1 --csv \
    python bench.py --no-e2e --no-cpu --no-extra --steps 1 --warmup 0 2>/dev/null | grep -E "dram__|duration|per_second" | awk -F'"' -v t="$cfg" '{print t, $(NF-5), $(NF-1)}'
done
