"""C1 MLE glue on identical inputs (oracle-built H, dK/dtheta imported to the
device) in each product association, against the unmodified restated oracle,
the oracle in the solve association, and the reference itself (oracle/_ref).
Also the spread of the oracle itself across thread counts (summation order).
Usage: python tests/diagnostics/probe_glue_modes.py
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np

from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H

n, leaf, k = 4096, 64, 24
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = O.tree_depth(n, leaf, 2 * leaf)
oo = O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, False)
K = oo.apply(np.eye(n))
y = np.linalg.cholesky(K) @ O.randn(n, 1, 1)[:, 0]
ob = O.Build(oo, tau, k, 0, True, p=2)
oh, od = ob.h(), [ob.deriv(0), ob.deriv(1)]
of = O.factorize(oh, 1)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


res = {}
for assoc in (False, True):
    O.set_solve_association(assoc)
    for th in (1, 16):
        C.CDLL("libgomp.so.1").omp_set_num_threads(th)
        res[f"oracle/{'solve' if assoc else 'ref'}/t{th}"] = (O.score(of, od, y), O.fisher_information(of, od, cache=True),
                                                             O.fisher_information(of, od, cache=False))
O.set_solve_association(False)
dh, dd = H.HodlrMatrix.from_panels(oh.export_panels()), [H.HodlrMatrix.from_panels(d.export_panels()) for d in od]
ctx = H.context()
for a in (H.ASSOC_SOLVE, H.ASSOC_REFERENCE):
    ctx.set_option(H.OPT_PRODUCT_ASSOCIATION, a)
    df = H.factorize(dh, H.LEFT)
    f = H.fisher_information(df, dd)
    res[f"device/{'solve' if a == 0 else 'ref'}"] = (H.score(df, dd, y), f, f)
ctx.set_option(H.OPT_PRODUCT_ASSOCIATION, H.ASSOC_SOLVE)
for kk, (s, f, fu) in res.items():
    print(f"{kk:22s} s {np.array2string(np.asarray(s), precision=14)} F {np.array2string(np.asarray(f).ravel(), precision=14)}")
for base in ("oracle/ref/t1", "oracle/solve/t1"):
    for kk in res:
        if kk != base:
            print(f"vs {base:16s} {kk:22s} score {rel(res[kk][0], res[base][0]):.2e} fisher {rel(res[kk][1], res[base][1]):.2e} "
                  f"fisher(uncached) {rel(res[kk][2], res[base][2]):.2e}")
