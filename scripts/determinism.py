"""Are repeated C4 evaluations bitwise identical (decisions, loglik, score)?"""
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
ref = None
for i in range(4):
    br = H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
    dec = br.decisions()
    ll, s, f, t = H.mle_evaluate(o, tau, 40, 7, y, B, X)
    cur = (dec, ll, s.copy(), f.copy())
    if ref is None:
        ref = cur
        print("decisions", dec.size, "sum", dec.sum(), "ll", ll)
    else:
        print(i, "decisions equal", np.array_equal(dec, ref[0]), "ndiff", int((dec != ref[0]).sum()) if dec.size == ref[0].size else "size",
              "ll equal", ll == ref[1], ll - ref[1], "score equal", np.array_equal(s, ref[2]), "fisher equal", np.array_equal(f, ref[3]))
