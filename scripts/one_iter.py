"""One C4-shaped MLE iteration at n = 2^lg (default 18) after a warm-up — a
small driver for ncu captures of individual kernels (-k regex -c 1)."""
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 18
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
y = np.random.default_rng(1).standard_normal(n)
B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
X = np.zeros_like(B)
tau = H.tree_depth(n, 128, 256)
for _ in range(2):
    ll, s, f, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
print(ll, t)
