import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H
n, leaf, k = 1 << 15, 64, 16
x = np.sort(np.random.default_rng(3).uniform(size=n))
tau = O.tree_depth(n, leaf, 2 * leaf)
ob = O.Build(O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, True), tau, k, 0, False)
db = H.build_hodlr_with_derivatives(H.MaternOracle(x, 3, 1.0, 0.2, 1e-4, True), H.ClusterTree(n, tau), k, 0)
print("decisions equal:", np.array_equal(ob.decisions()[:, 0], db.decisions()[:, 0]), ob.decisions()[:8, 0])
p0, p1 = ob.h().export_panels(), db.h.export_panels()
lv = O.tree_ranges(n, tau)
off = 0
for l in range(1, tau + 1):
    R = p0["R"][l - 1]
    U0 = p0["flat"][off:off + n * R].reshape((n, R), order="F"); U1 = p1["flat"][off:off + n * R].reshape((n, R), order="F")
    off += 2 * n * R
    for j in range(min(2 ** (l - 1), 2)):
        (a, b), (c, d) = lv[l][2 * j], lv[l][2 * j + 1]
        dl = np.abs(U0[a:b] - U1[a:b]).max(axis=0)
        print(f"l={l} node={j} rows={b-a} left col maxdiff: {np.array2string(dl, precision=1, max_line_width=200)}")
