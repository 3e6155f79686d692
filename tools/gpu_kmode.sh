#!/bin/bash
# class-grouped unit order (MPCGEMM_ORDER=2) and job-wide k-phase hints (MPCGEMM_KPHASE=2)
mkdir -p gpurun_out
MPCGEMM_ORDER=2 MPCGEMM_KPHASE=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py tests/test_gpu_fullsize.py -x -q > gpurun_out/kmode_pt.log 2>&1; tail -2 gpurun_out/kmode_pt.log
bash tools/gpu_env_ab.sh "MPCGEMM_ORDER=1 MPCGEMM_KPHASE=1" "MPCGEMM_ORDER=2 MPCGEMM_KPHASE=1" "MPCGEMM_ORDER=2 MPCGEMM_KPHASE=2"
bash tools/gpu_ncu_env.sh km "MPCGEMM_ORDER=2 MPCGEMM_KPHASE=1" "MPCGEMM_ORDER=2 MPCGEMM_KPHASE=2" "MPCGEMM_ORDER=2 MPCGEMM_KPHASE=2 MPCGEMM_PBLK=64"
