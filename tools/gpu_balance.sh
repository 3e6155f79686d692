#!/bin/bash
for b in 4 1 2 8 4; do echo "BALANCE=$b"; MPCGEMM_BALANCE=$b CONFIGS=2,3,5 timeout 600 python tools/bench_configs.py 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print([(c['config'], c['method'], round(c['ms'],3)) for c in d['configs']])"; done
