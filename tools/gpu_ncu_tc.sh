#!/bin/bash
# tensor-core operand / TMEM metrics of the slice GEMM at config 4 (SURVEY 8(d) list)
TAG=${1:-r}
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_imma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_2cta.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__mem_tensor_reads_op_ldt.sum,sm__mem_tensor_writes_op_utcmma.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:slicegemm_tc2 -s 1 -c 1 --csv --log-file gpurun_out/ncu_tc_$TAG.csv $CMD > /dev/null 2>&1
echo rc=$?; python tools/ncu_summary.py gpurun_out/ncu_tc_$TAG.csv
