"""Where does F_sigma-sigma's spread at the C4 settings come from?
F with the built dK/dsigma2 (D0) vs F with D0' = H - eta I formed exactly from
H's own panels (same off-diagonal factors, leaves minus eta), plus the
consistency ||(D0 - (H - eta I)) v|| / ||v||.
Usage: python scripts/diag_fss.py 17 20
"""
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H

SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    y = np.random.default_rng(1).standard_normal(n)
    tau = H.tree_depth(n, 128, 256)
    g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
    br = H.build_hodlr_with_derivatives(g, H.ClusterTree(n, tau), K, SEED)
    p = br.h.export_panels()
    off = sum(2 * n * r for r in p["R"])
    flat = p["flat"].copy()
    m = n >> tau
    nl = 1 << tau
    for b in range(nl):  # uniform leaves here
        base = off + b * m * m
        flat[base: base + m * m: m + 1] -= NUG
    p2 = dict(p)
    p2["flat"] = flat
    D0p = H.HodlrMatrix.from_panels(p2)
    V = np.asfortranarray(np.random.default_rng(9).standard_normal((n, 2)))
    e = np.linalg.norm(br.deriv[0].matvec(V) - D0p.matvec(V), axis=0) / np.linalg.norm(V, axis=0)
    fl = H.factorize(br.h, H.LEFT)
    f = H.fisher_information(fl, br.deriv)
    f2 = H.fisher_information(fl, [D0p, br.deriv[1]])
    s, s2 = H.score(fl, br.deriv, y), H.score(fl, [D0p, br.deriv[1]], y)
    print(f"n=2^{lg}: ||(D0-(H-eta I))v||/||v|| {e}  F_ss built D0 {f[0,0]:.6g}  exact H-eta I {f2[0,0]:.6g} "
          f"(n/2 {n/2:.0f}); F_sl {f[0,1]:.6g} / {f2[0,1]:.6g}; score_s {s[0]:.8g} / {s2[0]:.8g}", flush=True)
