"""Key metrics + stall reasons of one kernel from an ncu report (raw page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__waves_per_multiprocessor", "launch__grid_size", "launch__block_size"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:60s} {v[i]} {rows[1][i]}")
out = []
for i, n in enumerate(h):
    if "smsp__average_warps_issue_stalled" in n and n.endswith("per_issue_active.ratio"):
        try:
            out.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(out)[::-1][:8]))
