"""TEST INFRASTRUCTURE ONLY (never imported by the product path).

Restatement of the strong-admissibility block-cluster tree of
paper_2303_10102_b200/csrc/hstrong.cu (hs_plan) in numpy, used by
tests/test_hstrong_plan.py to check the C ABI's block counts. The format is
not in the reference (weak HODLR only), so this restates
the standard eta-admissibility rule, not reference code:
  (t, s) admissible  <=>  dist(t, s) > 0, min(|t|, |s|) > k and
                          min(diam t, diam s) <= eta * dist(t, s),
diam = diagonal of the node's grid-index bounding box, dist = distance between
the two boxes on the torus of side nside.
"""
import numpy as np


def _tree_ranges(n, tau):
    """cluster_tree.cpp:10-22: uniform bisection, left child ceil(len/2)."""
    levels = [[(0, n)]]
    for _ in range(tau):
        nxt = []
        for lo, hi in levels[-1]:
            mid = lo + (hi - lo + 1) // 2
            nxt += [(lo, mid), (mid, hi)]
        levels.append(nxt)
    return levels


def _gap(a0, a1, b0, b1, N):
    return min(max(0, b0 + sh - a1, a0 - (b1 + sh)) for sh in (-N, 0, N))


def plan(order, nside, tau, eta, k):
    order = np.asarray(order, dtype=np.int64)
    n = nside * nside
    gx, gy = order % nside, order // nside
    levels = _tree_ranges(n, tau)
    boxes = [[(gx[lo:hi].min(), gx[lo:hi].max(), gy[lo:hi].min(), gy[lo:hi].max()) for lo, hi in lv] for lv in levels]

    def adm(d, t, s):
        a, b = boxes[d][t], boxes[d][s]
        dist = np.hypot(_gap(a[0], a[1], b[0], b[1], nside), _gap(a[2], a[3], b[2], b[3], nside))
        da, db = np.hypot(a[1] - a[0], a[3] - a[2]), np.hypot(b[1] - b[0], b[3] - b[2])
        mt = levels[d][t][1] - levels[d][t][0]
        ms = levels[d][s][1] - levels[d][s][0]
        return dist > 0 and min(mt, ms) > k and min(da, db) <= eta * dist

    lr, dn = [], []
    stack = [(0, 0, 0)]
    while stack:
        d, t, s = stack.pop()
        if t != s and adm(d, t, s):
            lr.append((d, t, s))
        elif d == tau:
            dn.append((t, s))
        elif t == s:
            stack += [(d + 1, 2 * t, 2 * t), (d + 1, 2 * t, 2 * t + 1), (d + 1, 2 * t + 1, 2 * t + 1)]
        else:
            stack += [(d + 1, 2 * t + a, 2 * s + b) for a in (0, 1) for b in (0, 1)]
    size = lambda d, t: levels[d][t][1] - levels[d][t][0]
    le = sum(size(d, t) * size(d, s) for d, t, s in lr)
    de = sum(size(tau, t) * size(tau, s) for t, s in dn)
    st = sum((size(d, t) + size(d, s)) * k for d, t, s in lr) + sum(
        size(tau, t) * size(tau, s) * (1 if t == s else 2) for t, s in dn)  # off-diagonal dense: D and D^T
    return {"n_lowrank": len(lr), "n_dense": len(dn), "lowrank_entries": le, "dense_entries": de,
            "stored_doubles": st}
