"""Per-kernel-class DRAM traffic of one C4 step from an ncu metrics capture
(dram__bytes_read/write.sum, gpu__time_duration.sum per launch) of
scripts/one_step.py: second half of the launches (the measured step)."""
import collections
import csv
import json
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
agg = collections.defaultdict(lambda: collections.Counter())
for d in step:
    k = d["kernel"].replace("hg::(anonymous namespace)::", "").split("(")[0]
    k = k.split("<")[0].replace("void ", "").replace("unnamed>::", "")
    agg[k]["launches"] += 1
    agg[k]["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    agg[k]["ns"] += d.get("gpu__time_duration.sum", 0)
out = {k: {"launches": v["launches"], "dram_bytes": v["bytes"], "dram_bytes_per_launch": v["bytes"] / v["launches"],
           "ms": v["ns"] / 1e6} for k, v in agg.items()}
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, v in sorted(out.items(), key=lambda x: -x[1]["ms"]):
    print(f"{k:24s} {v['launches']:5d} {v['ms']:9.2f} ms {v['dram_bytes'] / 1e9:9.2f} GB")
