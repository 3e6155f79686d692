#!/bin/bash
# small-call latency: fold variants x unit shapes (config 1 / 2)
mkdir -p gpurun_out
for v in "X=0" "MPCGEMM_FOLD_SFIX=1" "MPCGEMM_G2=1" "MPCGEMM_G2=1 MPCGEMM_FOLD_SFIX=1" "MPCGEMM_BALANCE=1 MPCGEMM_G2=0 MPCGEMM_FOLD_UNIC=0" "X=1"; do
  env $v timeout 600 python tools/call_latency.py > gpurun_out/lat_env.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/lat_env.json').read().strip().splitlines()[-1])
print('$v', {k: (v['ms_device_rule_graph'], v.get('ms_slicegemm')) for k, v in d.items() if 'cfg5' not in k})"
done
