"""Parity modes on config C1 (n = 4096) and its n = 512 cut: the device path in
each (association, compression) mode against the reference itself (oracle/_ref),
the restated oracle in both associations, and the dense truth.
Usage: python tests/diagnostics/probe_parity_modes.py [n]
"""
import sys

sys.path.insert(0, ".")
import numpy as np

from oracle import pyoracle as O
from oracle import pyref as R
from paper_2303_10102_b200 import hodlrgp as H

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
x = np.sort(np.random.default_rng(0).uniform(size=n))
y = np.random.default_rng(1).standard_normal(n)
tau = O.tree_depth(n, 64, 128)
args = (3, 1.0, 0.2, 1e-4)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


res = {}
res["ref"] = R.mle_iteration(R.CovOracle.matern(x, *args, True), tau, 24, 0, y, 2)[:3]
for assoc in (False, True):
    O.set_solve_association(assoc)
    res[f"restated/{'solve' if assoc else 'ref'}"] = O.mle_iteration(O.CovOracle.matern(x, *args, True), tau, 24, 0,
                                                                     y, 2)[:3]
O.set_solve_association(False)
ctx = H.context()
for a in (H.ASSOC_SOLVE, H.ASSOC_REFERENCE):
    for c in (H.COMPRESS_PIVOTED_QR, H.COMPRESS_JACOBI_SVD):
        ctx.set_option(H.OPT_PRODUCT_ASSOCIATION, a)
        ctx.set_option(H.OPT_COMPRESSION, c)
        ctx.set_option(H.OPT_Q2_BASIS, H.Q2_REFERENCE if a == H.ASSOC_REFERENCE else H.Q2_REORTHOGONALIZED)
        res[f"device/{'solve' if a == 0 else 'ref'}/{'qr' if c == 0 else 'svd'}"] = H.mle_iteration(
            H.MaternOracle(x, *args, True), tau, 24, 0, y)[:3]
ctx.set_option(H.OPT_PRODUCT_ASSOCIATION, H.ASSOC_SOLVE)
ctx.set_option(H.OPT_COMPRESSION, H.COMPRESS_PIVOTED_QR)
ctx.set_option(H.OPT_Q2_BASIS, H.Q2_REORTHOGONALIZED)
ll, s, f = H.dense_exact(H.MaternOracle(x, *args, False), y)[:3] if n <= 8192 else (None, None, None)
if ll is not None:
    res["dense"] = (ll, s, f)
for k, (ll, s, f) in res.items():
    print(f"{k:22s} ll {ll:.15e} s {np.array2string(np.asarray(s), precision=12)} F {np.array2string(np.asarray(f).ravel(), precision=12)}")
print()
for base in ("ref", "restated/solve", "dense"):
    if base not in res:
        continue
    for k in res:
        if k == base:
            continue
        print(f"vs {base:15s} {k:22s} ll {rel(res[k][0], res[base][0]):.2e} score {rel(res[k][1], res[base][1]):.2e} "
              f"fisher {rel(res[k][2], res[base][2]):.2e}")
