"""Which GPU build stage costs derivative accuracy at large n (C4 settings)?
Per-level errors of D0/D1 and the GPU Fisher for build variants:
  default  — scan oracle with masked peel applies, pivoted-QR recompression,
             q2 re-orthogonalised against q
  q2ref    — q2 as the reference forms it (HG_Q2_REFERENCE)
  svd      — HG_COMPRESS_JACOBI_SVD recompression
  unmasked — the same scan oracle behind a callback (no masked applies)
  cpu      — the restated CPU oracle's build (n <= --cpu)
Usage: python scripts/diag_levels2.py 17 18 [--cpu=17]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import numpy as np

from diag_levels import report  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2303_10102_b200 import hodlrgp as H  # noqa: E402

O.set_solve_association(True)
SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
args = [int(a) for a in sys.argv[1:] if not a.startswith("--")]
cpu_max = 0
for a in sys.argv[1:]:
    if a.startswith("--cpu="):
        cpu_max = int(a.split("=")[1])

APPLY = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p)


def unmasked(base):
    L = H.lib()

    def cb(user, j, V, ldv, s, Y, ldy, stream):
        return L.hg_oracle_apply(base.ctx.ptr, base.ptr, j, V, ldv, s, Y, ldy, H.DEVICE)

    fn = APPLY(cb)
    o = C.c_void_p()
    H._check(L.hg_oracle_callback(base.ctx.ptr, base.n, base.p, C.cast(fn, C.c_void_p), None, C.byref(o)))
    view = H.CovarianceOracle(o, base.ctx, base.n, base.p)
    view._keep = (fn, base)
    return view


def fisher(h, d, y):
    fl = H.factorize(h, H.LEFT)
    return H.score(fl, d, y), H.fisher_information(fl, d)


for lg in args:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    y = np.random.default_rng(1).standard_normal(n)
    tau = H.tree_depth(n, 128, 256)
    print(f"===== n = 2^{lg} tau = {tau}", flush=True)
    g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
    ctx = H.context()
    for name in ("default", "q2ref", "svd", "unmasked"):
        ctx.set_option(H.OPT_COMPRESSION, H.COMPRESS_JACOBI_SVD if name == "svd" else H.COMPRESS_PIVOTED_QR)
        ctx.set_option(H.OPT_Q2_BASIS, H.Q2_REFERENCE if name == "q2ref" else H.Q2_REORTHOGONALIZED)
        orc = unmasked(g) if name == "unmasked" else g
        br = H.build_hodlr_with_derivatives(orc, H.ClusterTree(n, tau), K, SEED)
        gp = [br.h.export_panels()] + [d.export_panels() for d in br.deriv]
        report(name, gp, lambda W, j: g.apply(W, j), n, tau)
        s, f = fisher(br.h, br.deriv, y)
        print(f"{name} score {s} F {f.ravel()}  F_ss/(n/2) {f[0, 0] / (n / 2):.5f}", flush=True)
    ctx.set_option(H.OPT_COMPRESSION, H.COMPRESS_PIVOTED_QR)
    ctx.set_option(H.OPT_Q2_BASIS, H.Q2_REORTHOGONALIZED)
    if lg <= cpu_max:
        o = O.CovOracle.matern(x, 5, SIG2, ELL, NUG, True)
        bo = O.Build(o, tau, K, SEED, True, 2)
        cp = [bo.h().export_panels(), bo.deriv(0).export_panels(), bo.deriv(1).export_panels()]
        report("cpu", cp, lambda W, j: g.apply(W, j), n, tau)
