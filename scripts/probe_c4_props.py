"""Size-independent properties of the C4 path at n = 2^20 (probe for the tests)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << lg
tau = H.tree_depth(n, 128, 256)
x = np.sort(np.random.default_rng(0).uniform(size=n))
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
t0 = time.time()
br = H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
h = br.h
d = br.deriv
print("build", time.time() - t0)
rng = np.random.default_rng(5)
X = np.asfortranarray(rng.standard_normal((n, 2)))
y1 = h.matvec(X[:, 0]); y2 = h.matvec(X[:, 1]); y12 = h.matvec(2 * X[:, 0] - 3 * X[:, 1])
print("linearity rel", np.linalg.norm(y12 - (2 * y1 - 3 * y2)) / np.linalg.norm(y12))
Y = h.matvec(X)
print("batch vs single rel", np.linalg.norm(Y[:, 0] - y1) / np.linalg.norm(y1), np.array_equal(Y[:, 0], y1))
fr = H.factorize(h, H.RIGHT)
b = rng.standard_normal(n)
xs = fr.solve(b)
r = h.matvec(xs) - b
print("solve residual rel", np.linalg.norm(r) / np.linalg.norm(b))
fl = H.factorize(h, H.LEFT)
print("logdet R/L", fr.logdet(), fl.logdet(), fr.logdet() - fl.logdet())
t0 = time.time()
tr = H.trace_solve(fl, h)
print("tr(H^-1 H) - n", tr - n, (tr - n) / n, time.time() - t0)
for j in range(2):
    t1 = H.trace_solve(fl, d[j])
    pj = H.solve_multiply(fl, d[j])
    t2 = H.trace_product_rep(pj)
    print("trace_solve vs trace_product_rep", j, t1, t2, (t1 - t2) / abs(t2))
# quadratic form identity: y^T K^-1 K_j K^-1 y via solves
yv = np.random.default_rng(1).standard_normal(n)
a = fl.solve(yv)
for j in range(2):
    q1 = a @ d[j].matvec(a)
    print("quad", j, q1)
# determinism
ll1 = H.mle_evaluate(o, tau, 40, 7, yv, np.zeros((n, 0), order="F"), np.zeros((n, 0), order="F"))
ll2 = H.mle_evaluate(o, tau, 40, 7, yv, np.zeros((n, 0), order="F"), np.zeros((n, 0), order="F"))
print("determinism", ll1[0] == ll2[0], np.array_equal(ll1[1], ll2[1]), np.array_equal(ll1[2], ll2[2]))
print("score", ll1[1], "quad/2 - tr/2", [0.5 * (a @ d[j].matvec(a)) - 0.5 * H.trace_solve(fl, d[j]) for j in range(2)])
