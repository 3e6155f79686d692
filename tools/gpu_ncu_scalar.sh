#!/bin/bash
# ncu source-level profile of the device MP scalar ops (mp_scalar_kernel, fms + recip at 256 / 768 bits)
mkdir -p gpurun_out
CNT=8192 timeout 300 python tools/mp_scalar_probe.py > gpurun_out/scalar_probe.log 2>&1 || exit 1
CNT=8192 timeout 900 ncu --set full --import-source on -k regex:mp_scalar -o gpurun_out/prof_scalar python tools/mp_scalar_probe.py > gpurun_out/ncu_scalar.log 2>&1; echo "ncu rc=$?"
