import sys; sys.path.insert(0, ".")
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
Hd = oh.densify(); Dd = [d.densify() for d in od]
print("H sym err", np.linalg.norm(Hd - Hd.T) / np.linalg.norm(Hd), "cond", np.linalg.cond(Hd))
of = O.factorize(oh, 1)
dh, dd = H.HodlrMatrix.from_panels(oh.export_panels()), [H.HodlrMatrix.from_panels(d.export_panels()) for d in od]
df = H.factorize(dh, H.LEFT)
w_o, w_g = of.solve(y), df.solve(y)
w_t = np.linalg.solve(Hd, y)
print("solve rel err oracle", np.linalg.norm(w_o - w_t) / np.linalg.norm(w_t), "gpu", np.linalg.norm(w_g - w_t) / np.linalg.norm(w_t))
for j in range(2):
    t_true = np.trace(np.linalg.solve(Hd, Dd[j]))
    t_o = O.trace_solve(of, od[j]); t_g = H.trace_solve(df, dd[j])
    q_t = w_t @ Dd[j] @ w_t; q_o = w_o @ od[j].matvec(w_o); q_g = w_g @ dd[j].matvec(w_g)
    print(f"j={j} trace true {t_true:.12e} oracle {t_o:.12e} gpu {t_g:.12e} | quad true {q_t:.12e} oracle {q_o:.12e} gpu {q_g:.12e}")
    print("   rank info", od[j].info()[3])
print("scores oracle", O.score(of, od, y), "gpu", H.score(df, dd, y))
print("leaf kinds gpu", np.unique(df.leaf_llt()[:64], return_counts=True))
