"""Dense FP64 truth of one C4-settings MLE iteration (Matérn 5/2, sigma2 = 1,
ell = 0.05, nugget 1e-6) on the GPU, memory-lean enough for n = 2^16 on one
B200 (peak three n x n matrices, 103 GB): torch Cholesky, L^-1 D L^-T per
derivative, score and Fisher from those, next to the device HODLR iteration.
Usage: python scripts/dense_c4.py 16
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2303_10102_b200 import hodlrgp as H

SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
y = np.random.default_rng(1).standard_normal(n)
dev = "cuda" if torch.cuda.is_available() else "cpu"
xt = torch.tensor(x, dtype=torch.float64, device=dev)
c = np.sqrt(5.0) / ELL


def rows_of(which, r0, r1):
    """Rows r0:r1 of K (which -1), dK/dsigma2 (0) or dK/dell (1)."""
    a = (xt[r0:r1, None] - xt[None, :]).abs_().mul_(c)
    e = torch.exp(-a)
    if which <= 0:
        out = (1 + a + a * a / 3) * e * SIG2
        if which == -1:
            out[torch.arange(r1 - r0, device=dev), torch.arange(r0, r1, device=dev)] += NUG
        return out
    return SIG2 * a * a * (1 + a) / 3 * e / ELL


B = min(4096, n)
t0 = time.time()
Km = torch.empty((n, n), dtype=torch.float64, device=dev)
for r0 in range(0, n, B):
    Km[r0:r0 + B] = rows_of(-1, r0, r0 + B)
L = torch.linalg.cholesky(Km)  # lower, zeros above
del Km
torch.cuda.empty_cache()
ld = 2 * torch.log(L.diagonal()).sum().item()
yt = torch.tensor(y, dtype=torch.float64, device=dev)[:, None]
w = torch.cholesky_solve(yt, L)
ll = -0.5 * n * np.log(2 * np.pi) - 0.5 * ld - 0.5 * (yt * w).sum().item()
LT = L.mT


def whiten(which, X):
    """X <- L^-1 D L^-T for D = dK/dtheta_which (symmetric): column blocks of
    L^-1 D from D's rows (D[:, c] = D[c, :]^T), then row blocks times L^-T in
    place (row block r of X L^-T depends on row block r of X only).
    Returns (tr(L^-1 D L^-T), w^T D w)."""
    quad = 0.0
    for c0 in range(0, n, B):
        Dr = rows_of(which, c0, c0 + B)  # = D[:, c0:c0+B]^T
        quad += (w[c0:c0 + B] * (Dr @ w)).sum().item()
        X[:, c0:c0 + B] = torch.linalg.solve_triangular(L, Dr.T.contiguous(), upper=False)
        del Dr
    tr = 0.0
    for r0 in range(0, n, B):
        X[r0:r0 + B] = torch.linalg.solve_triangular(LT, X[r0:r0 + B].contiguous(), upper=True, left=False)
        tr += X[r0:r0 + B, r0:r0 + B].diagonal().sum().item()
    return tr, quad


M0 = torch.empty((n, n), dtype=torch.float64, device=dev)
tr0, q0 = whiten(0, M0)
M1 = torch.empty((n, n), dtype=torch.float64, device=dev)
tr1, q1 = whiten(1, M1)
sc = [-0.5 * tr0 + 0.5 * q0, -0.5 * tr1 + 0.5 * q1]
Ms = (M0, M1)
F = np.array([[0.5 * sum((Ms[i][r0:r0 + B] * Ms[j][r0:r0 + B]).sum().item() for r0 in range(0, n, B))
               for j in range(2)] for i in range(2)])
dense_s = time.time() - t0
del Ms, M0, M1, L, LT
torch.cuda.empty_cache()
print(f"n = 2^{lg}: dense ({dense_s:.1f}s) ll {ll:.12e} score {np.array2string(np.array(sc), precision=10)} "
      f"F {np.array2string(F.ravel(), precision=10)}  F_ss/(n/2) {F[0, 0] / (n / 2):.5f}", flush=True)
if dev == "cpu":
    sys.exit(0)
tau = H.tree_depth(n, 128, 256)
g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
ll1, s1, f1, _ = H.mle_iteration(g, tau, K, SEED, y)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


print(f"n = 2^{lg}: device ll {ll1:.12e} score {np.array2string(np.asarray(s1), precision=10)} "
      f"F {np.array2string(np.asarray(f1).ravel(), precision=10)}", flush=True)
print(f"relative to dense: ll {rel(ll1, ll):.2e} score {rel(s1, sc)} F {rel(f1, F).ravel()}", flush=True)
