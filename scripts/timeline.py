"""GPU timeline of one C4 MLE step (CUPTI via torch.profiler): kernel busy
time vs wall time, and the largest idle gaps with their neighbouring kernels.

usage: python scripts/timeline.py [log2n] [out.json]
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
y = np.random.default_rng(1).standard_normal(n)
B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
X = np.zeros_like(B)
torch.zeros(1, device="cuda")
H.mle_evaluate(o, tau, 40, 7, y, B, X)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    ll, s, f, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
busy = sum(e["dur"] for e in k)
wall = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
print(f"stages {t} sum {t.sum():.3f}s")
print(f"events {len(k)} busy {busy/1e6:.3f}s wall {wall/1e6:.3f}s idle {(wall-busy)/1e6:.3f}s")
gaps = []
for a, b in zip(k, k[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 0:
        gaps.append((g, a["name"][:60], b["name"][:60]))
gaps.sort(reverse=True)
print("gap histogram (us): >1000:", sum(1 for g in gaps if g[0] > 1000), " 100-1000:",
      sum(1 for g in gaps if 100 < g[0] <= 1000), " 10-100:", sum(1 for g in gaps if 10 < g[0] <= 100),
      " <=10:", sum(1 for g in gaps if g[0] <= 10))
print("total gap time by size: >1000us %.3fs, 100-1000 %.3fs, <=100 %.3fs" % (
    sum(g[0] for g in gaps if g[0] > 1000) / 1e6, sum(g[0] for g in gaps if 100 < g[0] <= 1000) / 1e6,
    sum(g[0] for g in gaps if g[0] <= 100) / 1e6))
for g in gaps[:25]:
    print(f"{g[0]:10.0f} us  after {g[1]}  before {g[2]}")
