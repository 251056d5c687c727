"""Per-level representation error of the built HODLRs (C4 settings): for each
level l and a few nodes j, || (D_l,j - K_j[cl, cr]) v || / || K_j[cl, cr] v || with v
supported on the right child only, plus the leaves, for H and each derivative.
Exact block products come from the forward model applied to vectors supported
on one child. Usage: python scripts/diag_levels.py 16 18 [--cpu]
"""
import sys

sys.path.insert(0, ".")
import numpy as np

from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H

SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
args = [int(a) for a in sys.argv[1:] if not a.startswith("--")]
use_cpu = "--cpu" in sys.argv
O.set_solve_association(True)


def ranges(n, tau):
    lv = [[(0, n)]]
    for d in range(1, tau + 1):
        nxt = []
        for lo, hi in lv[-1]:
            left = (hi - lo + 1) // 2
            nxt += [(lo, lo + left), (lo + left, hi)]
        lv.append(nxt)
    return lv


def block_apply(p, lv, l, j, v):
    """upper(l, j) of an exported HODLR applied to v (right-child rows)."""
    n = p["n"]
    off = 0
    for ll in range(1, l):
        off += 2 * n * p["R"][ll - 1]
    R = p["R"][l - 1]
    U = p["flat"][off: off + n * R].reshape(R, n).T
    V = p["flat"][off + n * R: off + 2 * n * R].reshape(R, n).T
    (cl_lo, cl_hi), (cr_lo, cr_hi) = lv[l][2 * j], lv[l][2 * j + 1]
    return U[cl_lo:cl_hi] @ (V[cr_lo:cr_hi].T @ v)


def report(tag, panels, apply_fn, n, tau, nodes_per_level=6):
    lv = ranges(n, tau)
    rng = np.random.default_rng(11)
    for which, p in enumerate(panels):
        name = "H" if which == 0 else f"D{which - 1}"
        j_oracle = -1 if which == 0 else which - 1
        line = []
        for l in range(1, tau + 1):
            nn = 2 ** (l - 1)
            js = sorted(set(np.linspace(0, nn - 1, min(nn, nodes_per_level)).astype(int).tolist()))
            W = np.zeros((n, len(js)), order="F")
            for t, j in enumerate(js):
                lo, hi = lv[l][2 * j + 1]
                W[lo:hi, t] = rng.standard_normal(hi - lo)
            KW = apply_fn(W, j_oracle)
            err = 0.0
            for t, j in enumerate(js):
                lo, hi = lv[l][2 * j + 1]
                cl_lo, cl_hi = lv[l][2 * j]
                exact = KW[cl_lo:cl_hi, t]
                got = block_apply(p, lv, l, j, W[lo:hi, t])
                err = max(err, np.linalg.norm(got - exact) / max(np.linalg.norm(exact), 1e-300))
            line.append(f"{err:.1e}")
        print(f"{tag} {name} per-level rel err: {' '.join(line)}  ranks {p['R']}", flush=True)


for lg in args:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    tau = H.tree_depth(n, 128, 256)
    print(f"===== n = 2^{lg} tau = {tau}", flush=True)
    g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
    br = H.build_hodlr_with_derivatives(g, H.ClusterTree(n, tau), K, SEED)
    gp = [br.h.export_panels()] + [d.export_panels() for d in br.deriv]
    report("GPU", gp, lambda W, j: g.apply(W, j), n, tau)
    if use_cpu and lg <= 16:
        o = O.CovOracle.matern(x, 5, SIG2, ELL, NUG, True)
        bo = O.Build(o, tau, K, SEED, True, 2)
        cp = [bo.h().export_panels(), bo.deriv(0).export_panels(), bo.deriv(1).export_panels()]
        report("CPU", cp, lambda W, j: o.apply(W, j), n, tau)
        dg = br.decisions()
        dc = bo.decisions()
        m = min(len(dg), len(dc))
        diff = np.nonzero(np.any(dg[:m] != dc[:m], axis=1))[0]
        print(f"decisions differ at {len(diff)} of {m} nodes; first: {[(int(i), dg[i].tolist(), dc[i].tolist()) for i in diff[:6]]}")
