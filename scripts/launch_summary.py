"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
scripts/one_step.py (two MLE steps): per-kernel totals of the second step."""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[vi]]
half = data[len(data) // 2:]
agg = collections.defaultdict(lambda: [0.0, 0])
for k, v in half:
    k = k.replace("hg::(anonymous namespace)::", "").replace("hg::<unnamed>::", "").split("(")[0]
    agg[k][0] += v
    agg[k][1] += 1
tot = sum(a[0] for a in agg.values())
print(f"Kernels in step: {len(half)}; sum of kernel time {tot / 1e9:.3f} s.\n")
print("| kernel | time (s) | share | launches |")
print("|---|---|---|---|")
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    if t / tot < 0.001:
        continue
    print(f"| {k} | {t / 1e9:.4f} | {100 * t / tot:.1f}% | {c} |")
