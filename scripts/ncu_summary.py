"""Summarise an ncu --set full report: key metrics + top stall reasons per kernel."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("==", d.get("Kernel Name", "")[:90])
    for k in keys:
        if k in d:
            print(f"   {k:70s} {d[k]} {rows[1][h.index(k)]}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:6]))
