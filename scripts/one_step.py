"""One warm-up MLE step + one measured step at C4 settings (for ncu launch lists)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
y = np.random.default_rng(1).standard_normal(n)
B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
X = np.zeros_like(B)
ctx = H.context()
H.mle_evaluate(o, tau, 40, 7, y, B, X)
l0 = ctx.launches
ll, s, f, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
print(f"warmup launches {l0} step launches {ctx.launches - l0} stages {t} total {t.sum():.3f}", flush=True)
