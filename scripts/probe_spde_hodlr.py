"""Weak-admissibility HODLR accuracy for the 2D SPDE covariance (C3-like)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import models as M
from paper_2303_10102_b200 import hodlrgp as H

for N, leaf, k in [(32, 64, 24), (32, 64, 48), (128, 256, 42), (256, 256, 42)]:
    th = (1.0, 0.05, 4.0)
    var = M.spde2d_variance(N, *th)
    order, tree = H.grid_kd_order(N, leaf)
    o = H.Spde2dOracle(N, *th, order=order, nugget=0.0)
    h = H.build_hodlr(o, tree, k, 7)
    v = np.random.default_rng(0).standard_normal(N * N)
    kv = o.apply(v)[:, 0]
    hv = h.matvec(v)
    lam = M.spde2d_spectra(N, *th, 0.0)[0]
    print(f"N={N} leaf={leaf} k={k}: ||(H-K)v||/||Kv|| = {np.linalg.norm(hv - kv) / np.linalg.norm(kv):.2e}; "
          f"lam_max/Var(u) = {lam.max() / var:.1f}; lam_min/Var = {lam.min() / var:.2e}", flush=True)
