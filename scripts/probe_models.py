"""Diagnostics for the C2/C3 model MLE parity (device vs CPU oracle vs dense truth)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import models as M
from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H


def dense_truth(K, dKs, y):
    n = len(y)
    L = np.linalg.cholesky(K)
    Ki = np.linalg.inv(K)
    a = Ki @ y
    ll = -0.5 * n * np.log(2 * np.pi) - np.sum(np.log(np.diag(L))) - 0.5 * y @ a
    s = np.array([-0.5 * np.trace(Ki @ d) + 0.5 * a @ d @ a for d in dKs])
    f = np.array([[0.5 * np.trace(Ki @ di @ Ki @ dj) for dj in dKs] for di in dKs])
    return ll, s, f


def run(name, odev, K, dKs, tau, k, y):
    oo = O.CovOracle.dense(K, dKs)
    try:
        O.set_solve_association(True)
        ll0, s0, f0, _ = O.mle_iteration(oo, tau, k, 0, y, len(dKs))
    except Exception as e:
        print(name, "CPU oracle failed:", e)
        ll0 = s0 = f0 = None
    finally:
        O.set_solve_association(False)
    try:
        ll1, s1, f1, _ = H.mle_iteration(odev, tau, k, 0, y)
    except Exception as e:
        print(name, "GPU failed:", e)
        ll1 = s1 = f1 = None
    llt, st, ft = dense_truth(K, dKs, y)
    print(name, "cond(K) %.2e" % np.linalg.cond(K))
    print(" ll  cpu", ll0, "gpu", ll1, "dense", llt)
    print(" s   cpu", s0, "\n     gpu", s1, "\n     dense", st)
    print(" f   cpu", None if f0 is None else f0.ravel(), "\n     gpu", None if f1 is None else f1.ravel(), "\n     dense", ft.ravel())


m, leaf, k = 256, 32, 16
th = (1.0, 0.1, 2.0)
K, dK = M.cokriging_dense(m, *th)
n = 2 * m
tau = O.tree_depth(n, leaf, 2 * leaf)
y = np.linalg.cholesky(K) @ O.randn(n, 1, 1)[:, 0]
run("C2 small", H.CoKrigingOracle(m, *th), K, dK, tau, k, y)

N, leaf, k = 32, 64, 20
th = (1.0, 0.05, 4.0)
order, tree = H.grid_kd_order(N, leaf)
K, dK = M.spde2d_dense(N, *th, order)
n = N * N
y = np.linalg.cholesky(K) @ O.randn(n, 1, 2)[:, 0]
run("SPDE small", H.Spde2dOracle(N, *th, order=order), K, dK, tree.tau, k, y)
