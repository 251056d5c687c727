import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import pyoracle as O
n, leaf, k = 1024, 64, 16
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = O.tree_depth(n, leaf, 2 * leaf)
oo = O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-2, False)
ob = O.Build(oo, tau, k, 0, True, p=2)
oh, od = ob.h(), ob.deriv(0)
def sym_leaves(h):
    A = h.densify(); lv = O.tree_ranges(n, tau)[tau]
    for lo, hi in lv:
        B = A[lo:hi, lo:hi]; A[lo:hi, lo:hi] = np.tril(B) + np.tril(B, -1).T
    return A
def check(name, ha, hb):
    f = O.factorize(ha, 1)
    P = O.solve_multiply(f, hb).densify()
    T = np.linalg.solve(sym_leaves(ha), hb.densify())
    print(f"{name}: rel err {np.linalg.norm(P-T)/np.linalg.norm(T):.2e}  cond {np.linalg.cond(ha.densify()):.1e}")
rs = O.Hodlr.random_spd(n, tau, 4, 3); rsym = O.Hodlr.random_symmetric(n, tau, 4, 4)
check("spd x sym", rs, rsym)
check("Hbuild x sym", oh, rsym)
check("spd x Dbuild", rs, od)
check("Hbuild x Dbuild", oh, od)
print("H ranks", oh.info()[3], "D ranks", od.info()[3])
from paper_2303_10102_b200 import hodlrgp as H
def gcheck(name, ha, hb):
    dha, dhb = H.HodlrMatrix.from_panels(ha.export_panels()), H.HodlrMatrix.from_panels(hb.export_panels())
    f = H.factorize(dha, 1)
    P = H.solve_multiply(f, dhb).densify()
    T = np.linalg.solve(sym_leaves(ha), hb.densify())
    Po = O.solve_multiply(O.factorize(ha, 1), hb).densify()
    print(f"GPU {name}: rel err {np.linalg.norm(P-T)/np.linalg.norm(T):.2e}; gpu vs oracle {np.linalg.norm(P-Po)/np.linalg.norm(T):.2e}; traces gpu {np.trace(P):.14e} oracle {np.trace(Po):.14e} true {np.trace(T):.14e}")
gcheck("Hbuild x sym", oh, rsym)
gcheck("Hbuild x Dbuild", oh, od)
