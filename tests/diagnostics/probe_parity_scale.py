"""GPU vs CPU oracle, one MLE iteration at C4 settings for growing n."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H
O.set_solve_association(True)
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    tau = H.tree_depth(n, 128, 256)
    y = np.random.default_rng(1).standard_normal(n)
    g = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
    llg, sg, fg, tg = H.mle_iteration(g, tau, 40, 7, y)
    print(f"n=2^{lg} GPU  ll={llg:.12e} s={sg} f={fg.ravel()}", flush=True)
    if lg <= 18:
        t0 = time.time()
        o = O.CovOracle.matern(x, 5, 1.0, 0.05, 1e-6, True)
        llo, so, fo, to = O.mle_iteration(o, tau, 40, 7, y, 2)
        print(f"n=2^{lg} CPU  ll={llo:.12e} s={so} f={fo.ravel()}  ({time.time()-t0:.1f}s)", flush=True)
