#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
MPCGEMM_FOLD_EPT=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/pytest_ept_$TAG.log 2>&1; echo "pytest ept4 rc=$?"; tail -1 gpurun_out/pytest_ept_$TAG.log
for cfg in "X=0" "MPCGEMM_FOLD_EPT=4" "X=0" "MPCGEMM_FOLD_EPT=4"; do
  env $cfg timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/fab_$TAG.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/fab_$TAG.json').read().strip().splitlines()[-1])
print('[$cfg] step', round(d['ms_per_step'],2), 'fold', d['stages_ms']['ms_fold'], 'gemm', d['stages_ms']['ms_gemm'], 'MHz', d['clocks']['sm_mhz'])"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
for cfg in "X=0" "MPCGEMM_FOLD_EPT=4"; do
env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"fold_normalize" -s 1 -c 1 --csv --log-file gpurun_out/ncu_ept_$TAG.csv $CMD > /dev/null 2>&1
echo "[$cfg]"; python tools/ncu_summary.py gpurun_out/ncu_ept_$TAG.csv | tail -3
done
for cfg in "X=0" "MPCGEMM_FOLD_EPT=4"; do env $cfg timeout 300 python tools/call_latency.py 2>/dev/null | grep cfg5_3M | head -1; done
