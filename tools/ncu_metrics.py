"""Selected --set full metrics per launch of an ncu report (one line per kernel)."""
import csv
import subprocess
import sys

M = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,"
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,"
     "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,lts__t_sector_hit_rate.pct,"
     "launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,"
     "sm__inst_executed.avg.per_cycle_active,smsp__sass_inst_executed_op_local_ld.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", M], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h = r[0]
idx = [i for i, x in enumerate(h) if "__" in x]
for row in r[2:]:
    print(row[h.index("Kernel Name")][:40])
    print("   " + " | ".join(f"{h[i].split('.')[0][-24:]}={row[i]}" for i in idx))
