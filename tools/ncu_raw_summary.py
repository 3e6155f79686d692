"""Key metrics of an `ncu -i X.ncu-rep --page raw --csv` dump, one block per kernel launch."""
import csv
import re
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_imma.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed.sum", "smsp__inst_executed.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]
rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
idx = {k: h.index(k) for k in KEYS if k in h}
ki = h.index("Kernel Name")
for r in rows[2:]:
    print(f"== {r[ki][:70]}")
    for k, i in idx.items():
        print(f"   {k:85s} {r[i]:>18s} {units[i]}")
