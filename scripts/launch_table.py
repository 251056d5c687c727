"""Per-kernel table (time, share, launches, DRAM GB) of the measured step from the ncu
metrics capture of scripts/one_step.py (same csv as scripts/traffic_capture.py):
  python scripts/launch_table.py gpurun_out/traffic.csv > profiles/r2_launches.md"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[ii], {"kernel": r[ki]})
    d[r[ni]] = float(r[vi].replace(",", ""))
launches = list(per.values())
step = launches[len(launches) // 2:]
agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
for d in step:
    m = re.search(r"\b(k_[A-Za-z0-9_]+(<[^>]*>)?)", d["kernel"])
    k = m.group(1) if m else d["kernel"]
    a = agg[k]
    a[0] += d.get("gpu__time_duration.sum", 0.0)
    a[1] += 1
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[0] for a in agg.values())
print(f"Kernels in step: {len(step)}; sum of kernel time {tot / 1e9:.3f} s.\n")
print("| kernel | time (s) | share | launches | DRAM GB |")
print("|---|---|---|---|---|")
for k, (t, c, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
    if t / tot < 0.003:
        continue
    print(f"| {k} | {t / 1e9:.4f} | {100 * t / tot:.1f}% | {c} | {b / 1e9:.2f} |")
