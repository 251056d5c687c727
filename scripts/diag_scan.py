"""Is the GPU Matérn scan the source of the fine-level derivative error at C4?

(1) Accuracy of the forward applies on a fine-level block: W supported on the
    right child of node j at level l; rows of the left child compared between
    the GPU scan, the CPU scan (oracle/matern1d.hpp) and the dense GPU kernel,
    relative to the block product's norm, for K, dK/dsigma2, dK/dell; plus the
    identity dK/dsigma2 W = K W off the diagonal (sigma2 = 1).
(2) GPU build driven by the CPU scan through a host callback (device <-> host
    copies), per-level errors against the GPU scan, and its Fisher.
Usage: python scripts/diag_scan.py 17
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import numpy as np

from diag_levels import ranges, report  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2303_10102_b200 import hodlrgp as H  # noqa: E402

SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 17
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
y = np.random.default_rng(1).standard_normal(n)
tau = H.tree_depth(n, 128, 256)
lv = ranges(n, tau)
gs = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
gd = H.MaternOracle(x, 5, SIG2, ELL, NUG, False)
cs = O.CovOracle.matern(x, 5, SIG2, ELL, NUG, True)
rng = np.random.default_rng(5)
print(f"===== n = 2^{lg} tau = {tau}", flush=True)
for l in (tau - 3, tau - 1, tau):
    nodes = 2 ** (l - 1)
    js = sorted(set(np.linspace(0, nodes - 1, 8).astype(int).tolist()))
    W = np.zeros((n, len(js)), order="F")
    for t, j in enumerate(js):
        lo, hi = lv[l][2 * j + 1]
        W[lo:hi, t] = rng.standard_normal(hi - lo)
    res = {}
    for which in (-1, 0, 1):
        a, b, c = gs.apply(W, which), cs.apply(W, which), gd.apply(W, which)
        es, ec = 0.0, 0.0
        for t, j in enumerate(js):
            lo, hi = lv[l][2 * j]
            ex = c[lo:hi, t]
            es = max(es, np.linalg.norm(a[lo:hi, t] - ex) / np.linalg.norm(ex))
            ec = max(ec, np.linalg.norm(b[lo:hi, t] - ex) / np.linalg.norm(ex))
        res[which] = (es, ec)
        if which == -1:
            K0s, K0c, K0d = a, b, c
        if which == 0:
            i0 = [np.linalg.norm((a - K0s)[lv[l][2 * j][0]:lv[l][2 * j][1], t]) /
                  np.linalg.norm(K0s[lv[l][2 * j][0]:lv[l][2 * j][1], t]) for t, j in enumerate(js)]
            i1 = [np.linalg.norm((b - K0c)[lv[l][2 * j][0]:lv[l][2 * j][1], t]) /
                  np.linalg.norm(K0c[lv[l][2 * j][0]:lv[l][2 * j][1], t]) for t, j in enumerate(js)]
    print(f"level {l}: block-row error vs dense  K gpu-scan {res[-1][0]:.1e} cpu-scan {res[-1][1]:.1e} | "
          f"dK/ds2 {res[0][0]:.1e} {res[0][1]:.1e} | dK/dl {res[1][0]:.1e} {res[1][1]:.1e} | "
          f"dK/ds2 - K: gpu {max(i0):.1e} cpu {max(i1):.1e}", flush=True)

# (2) GPU build from the CPU scan through a host callback.
APPLY = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p)


def _cudart():
    H.lib()
    for line in open("/proc/self/maps"):
        if "libcudart.so" in line:
            return C.CDLL(line.split()[-1])
    raise RuntimeError("libcudart not loaded")


CUDART = _cudart()
CUDART.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]


def cpu_cb(user, j, V, ldv, s, Y, ldy, stream):
    CUDART.cudaDeviceSynchronize()
    hv = np.empty((s, ldv))
    CUDART.cudaMemcpy(hv.ctypes.data, V, 8 * s * ldv, 2)
    ho = np.ascontiguousarray(cs.apply(np.asfortranarray(hv[:, :n].T), j).T)
    for c in range(s):
        CUDART.cudaMemcpy(Y + 8 * c * ldy, ho[c].ctypes.data, 8 * n, 1)
    return 0


fn = APPLY(cpu_cb)
o = C.c_void_p()
H._check(H.lib().hg_oracle_callback(gs.ctx.ptr, n, 2, C.cast(fn, C.c_void_p), None, C.byref(o)))
cbo = H.CovarianceOracle(o, gs.ctx, n, 2)
for name, orc in (("gpu-scan", gs), ("cpu-scan-cb", cbo)):
    br = H.build_hodlr_with_derivatives(orc, H.ClusterTree(n, tau), K, SEED)
    report(name, [br.h.export_panels()] + [d.export_panels() for d in br.deriv], lambda W, j: gd.apply(W, j), n, tau)
    fl = H.factorize(br.h, H.LEFT)
    s, f = H.score(fl, br.deriv, y), H.fisher_information(fl, br.deriv)
    print(f"{name} score {s} F {f.ravel()}  F_ss/(n/2) {f[0, 0] / (n / 2):.5f}", flush=True)
