"""Prints the headline metrics and top stall reasons of an ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, rows = r[0], r[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second"]
for row in rows:
    for i, n in enumerate(h):
        if n in want:
            print(f"{n:70s} {row[i]}")
    st = [(float(row[i] or 0), n) for i, n in enumerate(h)
          if n.startswith("smsp__average_warp_latency_issue_stalled") and n.endswith(".ratio")]
    st = [(v, n) for v, n in st if v > 0]
    tot = sum(v for v, _ in st)
    for v, n in sorted(st, reverse=True)[:8]:
        print(f"  stall {n.split('stalled_')[1]:40s} {100*v/tot:5.1f}%")
