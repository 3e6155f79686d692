#!/bin/bash
# small-call latency under env variants (A/B of slice-GEMM unit shapes for small configs)
mkdir -p gpurun_out
for v in "X=0" "MPCGEMM_G2=0" "MPCGEMM_G2=0 MPCGEMM_BALANCE=2" "MPCGEMM_G2=0 MPCGEMM_BALANCE=4" "MPCGEMM_BALANCE=4" "X=1"; do
  env $v timeout 600 python tools/call_latency.py > gpurun_out/lat_env.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/lat_env.json').read().strip().splitlines()[-1])
print('$v', {k: (v['ms_device_rule_graph'], v.get('ms_slicegemm')) for k, v in d.items()})"
done
