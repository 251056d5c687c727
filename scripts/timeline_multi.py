"""Timeline of several consecutive C4 MLE steps: per-step kernel busy time,
idle time, and per-kernel totals for the fastest and slowest step."""
import collections
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
out = "gpurun_out/timeline_multi.json"
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
y = np.random.default_rng(1).standard_normal(n)
B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
X = np.zeros_like(B)
torch.zeros(1, device="cuda")
H.mle_evaluate(o, tau, 40, 7, y, B, X)
marks = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for i in range(steps):
        with torch.profiler.record_function(f"step{i}"):
            ll, s, f, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
        print(f"step {i} stages {np.round(t, 3)} sum {t.sum():.3f}", flush=True)
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
cpu_steps = sorted([e for e in ev if e.get("name", "").startswith("step") and e.get("ph") == "X" and e.get("cat") == "user_annotation"], key=lambda e: e["ts"])
print("cpu step spans", [(e["name"], round(e["dur"] / 1e6, 3)) for e in cpu_steps])
# split kernels into steps by the largest gaps (steps are separated by host sync)
per = collections.defaultdict(list)
for e in k:
    for i, s in enumerate(cpu_steps):
        if s["ts"] <= e["ts"] <= s["ts"] + s["dur"] + 1e5:
            per[i].append(e)
            break
res = []
for i in sorted(per):
    kk = per[i]
    busy = sum(e["dur"] for e in kk)
    wall = kk[-1]["ts"] + kk[-1]["dur"] - kk[0]["ts"]
    agg = collections.defaultdict(float)
    for e in kk:
        agg[e["name"].replace("hg::(anonymous namespace)::", "").split("(")[0]] += e["dur"]
    res.append((i, busy, wall, agg))
    print(f"step {i}: kernels {len(kk)} busy {busy/1e6:.3f}s wall {wall/1e6:.3f}s idle {(wall-busy)/1e6:.3f}s")
lo = min(res, key=lambda r: r[2])
hi = max(res, key=lambda r: r[2])
print(f"fastest step {lo[0]} vs slowest {hi[0]} per-kernel delta (ms):")
names = set(lo[3]) | set(hi[3])
for nm in sorted(names, key=lambda m: -(hi[3].get(m, 0) - lo[3].get(m, 0)))[:15]:
    print(f"  {nm:45s} {lo[3].get(nm,0)/1e3:9.1f} {hi[3].get(nm,0)/1e3:9.1f}")
# biggest gaps in slowest step
kk = per[hi[0]]
gaps = sorted(((b["ts"] - a["ts"] - a["dur"], a["name"][:50], b["name"][:50]) for a, b in zip(kk, kk[1:])), reverse=True)
for g in gaps[:10]:
    print(f"  gap {g[0]:9.0f}us after {g[1]} before {g[2]}")
