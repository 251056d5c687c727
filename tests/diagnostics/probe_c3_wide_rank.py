"""C3 (256^2 SPDE grid) in the weak HODLR format at sketch widths up to the
k = 128 limit and nuggets far below the 10 Var(u) default: iteration time and
agreement of loglik / score / Fisher with the exact spectral values
(oracle/models.spde2d_exact). usage: python tests/diagnostics/probe_c3_wide_rank.py"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np

from oracle import models as M
from paper_2303_10102_b200 import hodlrgp as H

N, leaf = 256, 256
th = (1.0, 0.05, 4.0)
order, tree = H.grid_kd_order(N, leaf)
var = M.spde2d_variance(N, *th)
n = N * N


def nrm(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


for k, rel in ((42, 10.0), (42, 1.0), (96, 1e-1), (128, 1e-1), (128, 1e-2), (128, 1e-3), (128, 1e-4)):
    nug = rel * var
    o = H.Spde2dOracle(N, *th, order=order, nugget=nug)
    lam = M.spde2d_spectra(N, *th, nug)[0]
    z = np.fft.fft2(np.random.default_rng(2).standard_normal((N, N)))
    y = np.real(np.fft.ifft2(np.sqrt(lam) * z)).ravel()[order]
    ex = M.spde2d_exact(N, *th, y=y, order=order, nugget=nug)
    try:
        H.mle_iteration(o, tree.tau, k, 7, y)
        ll, s, f, t = H.mle_iteration(o, tree.tau, k, 7, y)
        out = dict(k=k, nugget_over_var=rel, seconds=float(np.sum(t)), stages=[round(float(v), 4) for v in t],
                   loglik_rel=abs(ll - ex["loglik"]) / abs(ex["loglik"]), score_rel=nrm(s, ex["score"]),
                   fisher_rel=nrm(f, ex["fisher"]))
    except Exception as e:  # NotPositiveDefinite: the approximation error exceeds the nugget
        out = dict(k=k, nugget_over_var=rel, error=f"{type(e).__name__}: {e}"[:160])
    print(json.dumps(out), flush=True)
