#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_pc_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_pc_$TAG.log
timeout 600 python tools/determinism.py 4 30 MPCGEMM_DBG=16
for cfg in "X=0" "MPCGEMM_FOLD_NOUNI1=1" "X=0" "MPCGEMM_FOLD_NOUNI1=1"; do
  env $cfg timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/pc_$TAG.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pc_$TAG.json').read().strip().splitlines()[-1])
print('[$cfg] step', round(d['ms_per_step'],2), 'fold', d['stages_ms']['ms_fold'], 'split', d['stages_ms']['ms_split'], 'gemm', d['stages_ms']['ms_gemm'], 'MHz', d['clocks']['sm_mhz'])"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
for cfg in "X=0" "MPCGEMM_FOLD_NOUNI1=1"; do
env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:"fold_normalize" -s 1 -c 1 --csv --log-file gpurun_out/ncu_pc_$TAG.csv $CMD > /dev/null 2>&1
echo "[$cfg]"; python tools/ncu_summary.py gpurun_out/ncu_pc_$TAG.csv | tail -4
done
