#!/bin/bash
# new default schedule (ORDER=2, KPHASE=2, PBLK=64) vs round-2 (ORDER=1, KPHASE=1, PBLK=32)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_o2.log 2>&1; tail -2 gpurun_out/pt_o2.log
OLD="MPCGEMM_ORDER=1 MPCGEMM_KPHASE=1 MPCGEMM_PBLK=32"
bash tools/gpu_env_ab.sh "$OLD" "MPCGEMM_ORDER=2"
env $OLD CONFIGS=2,3,5 timeout 900 python tools/bench_configs.py > gpurun_out/cfg_old.json 2>gpurun_out/cfg_old.err
CONFIGS=2,3,5 timeout 900 python tools/bench_configs.py > gpurun_out/cfg_new.json 2>gpurun_out/cfg_new.err
python - << 'PY'
import json
for t in ("old","new"):
    for r in json.load(open(f"gpurun_out/cfg_{t}.json"))["configs"]:
        print(t, r["config"], r["method"], round(r["ms"], 3), round(r["gemm_ms"], 3))
PY
