import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H
n, leaf, k = 4096, 64, 24
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = O.tree_depth(n, leaf, 2 * leaf)
oo = O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, False)
ob = O.Build(oo, tau, k, 0, True, p=2)
oh, od = ob.h(), [ob.deriv(0), ob.deriv(1)]
Hd = oh.densify()
for lo, hi in O.tree_ranges(n, tau)[tau]:
    B = Hd[lo:hi, lo:hi]; Hd[lo:hi, lo:hi] = np.tril(B) + np.tril(B, -1).T
M = [np.linalg.solve(Hd, d.densify()) for d in od]
Ft = np.array([[0.5 * np.sum(M[i] * M[j].T) for j in range(2)] for i in range(2)])
of = O.factorize(oh, 1)
f_ref = O.fisher_information(of, od, cache=True)
O.set_solve_association(True)
f_sol = O.fisher_information(of, od, cache=True)
O.set_solve_association(False)
df = H.factorize(H.HodlrMatrix.from_panels(oh.export_panels()), 1)
f_gpu = H.fisher_information(df, [H.HodlrMatrix.from_panels(d.export_panels()) for d in od])
np.set_printoptions(precision=15)
for name, F in (("truth", Ft), ("oracle-ref", f_ref), ("oracle-solve", f_sol), ("gpu", f_gpu)):
    print(name, F.ravel(), "rel vs truth", np.max(np.abs(F - Ft) / np.abs(Ft)))
