"""Smallest nugget (in units of Var(u)) that keeps the weak HODLR of the 2D SPDE
covariance factorizable, and its accuracy vs the spectral truth."""
import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import models as M
from paper_2303_10102_b200 import hodlrgp as H

for N, leaf, k in [(32, 64, 24), (256, 256, 42)]:
    th = (1.0, 0.05, 4.0)
    var = M.spde2d_variance(N, *th)
    order, tree = H.grid_kd_order(N, leaf)
    for rel in [1e-3, 1e-2, 1e-1, 1.0, 10.0]:
        o = H.Spde2dOracle(N, *th, order=order, nugget=rel * var)
        h = H.build_hodlr(o, tree, k, 7)
        try:
            f = H.factorize(h, H.LEFT)
            ld = f.logdet()
            ex = M.spde2d_exact(N, *th, nugget=rel * var)["logdet"]
            print(f"N={N} k={k} nugget={rel:g} Var: logdet {ld:.6e} exact {ex:.6e} rel {abs(ld - ex) / abs(ex):.2e}", flush=True)
        except Exception as e:
            print(f"N={N} k={k} nugget={rel:g} Var: {e}", flush=True)
