import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import models as M
from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H

m, leaf, k = 256, 32, 16
th = (1.0, 0.1, 2.0)
K, dK = M.cokriging_dense(m, *th)
n = 2 * m
tau = O.tree_depth(n, leaf, 2 * leaf)
ob = O.Build(O.CovOracle.dense(K, dK), tau, k, 0, True, p=3)
db = H.build_hodlr_with_derivatives(H.DenseMatrixOracle(K, dK), H.ClusterTree(n, tau), k, 0)
d0, d1 = ob.decisions(), db.decisions()
print("decisions", d0.shape, d1.shape, "rows differing", int((d0 != d1).any(axis=1).sum()))
for i in np.where((d0 != d1).any(axis=1))[0][:10]:
    print(i, d0[i], d1[i])
a0, a1 = ob.h().densify(), db.h.densify()
print("H diff", np.linalg.norm(a1 - a0) / np.linalg.norm(a0))
for j in range(3):
    e0, e1 = ob.deriv(j).densify(), db.deriv[j].densify()
    print("D", j, np.linalg.norm(e1 - e0) / np.linalg.norm(e0))
