"""Per-iteration time of the C4 model vs n (acceptance.cpp:270-331 analogue):
n = 2^14..2^20, Matern 5/2, leaf 128, k = 40; prints a markdown table and the
log-log slope over the upper half of the range."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

rows = []
for lg in range(14, 21):
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    tau = H.tree_depth(n, 128, 256)
    o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
    y = np.random.default_rng(1).standard_normal(n)
    B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
    X = np.zeros_like(B)
    H.mle_evaluate(o, tau, 40, 7, y, B, X)
    ts = []
    for _ in range(3):
        _, _, _, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
        ts.append(float(np.sum(t)))
    rows.append((lg, n, tau, min(ts)))
    print(f"n=2^{lg} tau={tau} {min(ts):.4f} s", flush=True)
print("\n| n | tau | s / iteration | per-point us | t / (n log2^2 n) x 1e9 |\n|---|---|---|---|---|")
for lg, n, tau, t in rows:
    print(f"| 2^{lg} | {tau} | {t:.4f} | {t / n * 1e6:.3f} | {t / (n * lg * lg) * 1e9:.3f} |")
lg = np.array([r[0] for r in rows], float)
t = np.array([r[3] for r in rows])
sl = np.polyfit(lg[3:] * np.log(2), np.log(t[3:]), 1)[0]
print(f"\nlog-log slope over n = 2^17..2^20: {sl:.3f} (reference acceptance window [0.9, 1.4])")
