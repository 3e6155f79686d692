#!/bin/bash
# usage: bash tools/gpu_counts.sh TAG -- MMA-count tests, the GPU suite, ncu IMMA instruction count at config 4
TAG=${1:-r}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_counts.py -q -p no:cacheprovider > gpurun_out/pytest_counts_$TAG.log 2>&1; echo "counts rc=$?" >> gpurun_out/pytest_counts_$TAG.log
tail -5 gpurun_out/pytest_counts_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -5 gpurun_out/pytest_gpu_$TAG.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_cnt_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_imma.sum,sm__inst_executed_pipe_tensor.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"slicegemm_tc2" -s 1 -c 1 --csv --log-file gpurun_out/ncu_imma_$TAG.csv $CMD > gpurun_out/ncu_imma_$TAG.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/ncu_imma_$TAG.csv | tail -6
