#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_device_rule.py -q -p no:cacheprovider -x > gpurun_out/pytest_split_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_split_$TAG.log
for cfg in "X=0" "MPCGEMM_SPLIT_BYTESTG=1" "X=0" "MPCGEMM_SPLIT_BYTESTG=1"; do
  env $cfg timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/sab_$TAG.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sab_$TAG.json').read().strip().splitlines()[-1])
print('[$cfg] step', round(d['ms_per_step'],2), 'split', d['stages_ms']['ms_split'], 'fold', d['stages_ms']['ms_fold'], 'gemm', d['stages_ms']['ms_gemm'], 'MHz', d['clocks']['sm_mhz'])"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
for cfg in "X=0" "MPCGEMM_SPLIT_BYTESTG=1"; do
env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"split_tma" -s 0 -c 2 --csv --log-file gpurun_out/ncu_split_$TAG.csv $CMD > /dev/null 2>&1
echo "[$cfg]"; python tools/ncu_summary.py gpurun_out/ncu_split_$TAG.csv | grep -v "^\[" 
done
