"""Stage times of consecutive C4 MLE steps (variance check)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
y = np.random.default_rng(1).standard_normal(n)
B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
X = np.zeros_like(B)
for i in range(steps):
    w0 = time.perf_counter()
    ll, s, f, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
    print(f"step {i} wall {time.perf_counter() - w0:.3f}s stages {np.round(t, 3)} sum {t.sum():.3f}", flush=True)
