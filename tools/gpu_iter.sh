#!/bin/bash
# usage: bash tools/gpu_iter.sh TAG [bench args]  -- gpu tests, bench, targeted ncu metrics of the slice GEMM
TAG=${1:-r}
shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu $@"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"slicegemm_tc|fold_norm|split_kernel" --csv --log-file gpurun_out/ncu_metrics_$TAG.csv $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
