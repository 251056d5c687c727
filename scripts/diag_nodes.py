"""Node-level view of one bad level (C4 settings): D_j block error per node for
the GPU and the CPU builds next to each build's decisions (numeric rank, w2,
rw per param). Usage: python scripts/diag_nodes.py 18 8
"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import numpy as np

from diag_levels import block_apply, ranges  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2303_10102_b200 import hodlrgp as H  # noqa: E402

SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
lg, lev = int(sys.argv[1]), int(sys.argv[2])
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
lv = ranges(n, tau)
g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
br = H.build_hodlr_with_derivatives(g, H.ClusterTree(n, tau), K, SEED)
gp = [d.export_panels() for d in br.deriv]
o = O.CovOracle.matern(x, 5, SIG2, ELL, NUG, True)
bo = O.Build(o, tau, K, SEED, True, 2)
cp = [bo.deriv(0).export_panels(), bo.deriv(1).export_panels()]
nodes = 2 ** (lev - 1)
first = 2 ** (lev - 1) - 1  # decision rows are level-major
dg, dc = br.decisions(), bo.decisions()
rng = np.random.default_rng(3)
W = np.zeros((n, nodes), order="F")
for j in range(nodes):
    lo, hi = lv[lev][2 * j + 1]
    W[lo:hi, j] = rng.standard_normal(hi - lo)
for q in range(2):
    KW = g.apply(W, q)
    rows = []
    for j in range(nodes):
        lo, hi = lv[lev][2 * j + 1]
        cl0, cl1 = lv[lev][2 * j]
        ex = KW[cl0:cl1, j]
        eg = np.linalg.norm(block_apply(gp[q], lv, lev, j, W[lo:hi, j]) - ex) / np.linalg.norm(ex)
        ec = np.linalg.norm(block_apply(cp[q], lv, lev, j, W[lo:hi, j]) - ex) / np.linalg.norm(ex)
        rows.append((eg, ec, j))
    rows.sort(reverse=True)
    print(f"D{q} level {lev}: worst GPU nodes (err_gpu, err_cpu, node, dec_gpu [nr,w2,rw0,rw1], dec_cpu)")
    for eg, ec, j in rows[:12]:
        print(f"  {eg:.2e} {ec:.2e} node {j:4d} gpu {dg[first + j].tolist()} cpu {dc[first + j].tolist()}")
    print(f"  median gpu {np.median([r[0] for r in rows]):.2e} cpu {np.median([r[1] for r in rows]):.2e}")
diff = np.nonzero(np.any(dg != dc, axis=1))[0]
print(f"decisions differ at {len(diff)} of {len(dg)} nodes; by level:",
      np.bincount(np.floor(np.log2(diff + 1)).astype(int) + 1, minlength=tau + 1)[1:].tolist())
