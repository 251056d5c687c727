"""C4 numerics, second pass: dense truth vs GPU vs CPU restatement.

For n = 2^lg at the C4 settings:
  * dense truth (n <= 2^15; torch FP64 Cholesky on the GPU): loglik, score, Fisher;
  * GPU build + GPU pipeline;
  * with --cpu: CPU-built HODLRs (solve association) through both pipelines.
Usage: python scripts/diag_c4b.py 13 14 15 16 18 [--cpu=18]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H

O.set_solve_association(True)
O.set_q2_reorthogonalize(True)  # the device defaults
SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
args = [int(a) for a in sys.argv[1:] if not a.startswith("--")]
cpu_max = 0
for a in sys.argv[1:]:
    if a.startswith("--cpu="):
        cpu_max = int(a.split("=")[1])


def dense_truth(x, y):
    dev = "cuda"
    xt = torch.tensor(x, dtype=torch.float64, device=dev)
    d = (xt[:, None] - xt[None, :]).abs_()
    a = d.mul_(np.sqrt(5.0) / ELL)
    e = torch.exp(-a)
    C = SIG2 * (1 + a + a * a / 3) * e          # dK/dsigma2 = C (sigma2 = 1)
    Cl = SIG2 * a * a * (1 + a) / 3 * e / ELL     # dK/dell
    del a, e, d
    Kd = C.clone()
    Kd.diagonal().add_(NUG)
    L = torch.linalg.cholesky(Kd)
    del Kd
    ld = 2 * torch.log(L.diagonal()).sum().item()
    yt = torch.tensor(y, dtype=torch.float64, device=dev)[:, None]
    w = torch.cholesky_solve(yt, L)
    n = len(x)
    ll = -0.5 * n * np.log(2 * np.pi) - 0.5 * ld - 0.5 * (yt * w).sum().item()
    Ms = []
    sc = []
    for D in (C, Cl):
        M = torch.linalg.solve_triangular(L, D, upper=False)
        M = torch.linalg.solve_triangular(L, M.T, upper=False)  # L^-1 D L^-T (symmetric)
        Ms.append(M)
        sc.append(-0.5 * M.diagonal().sum().item() + 0.5 * (w * (D @ w)).sum().item())
        del D
    F = np.array([[0.5 * (Ms[i] * Ms[j]).sum().item() for j in range(2)] for i in range(2)])
    return ll, np.array(sc), F


def gpu_pipeline(h, d, y):
    fl = H.factorize(h, H.LEFT)
    return H.log_likelihood(fl, y), H.score(fl, d, y), H.fisher_information(fl, d)


def cpu_pipeline(h, d, y):
    fl = O.factorize(h, O.Factor.LEFT)
    return O.log_likelihood(fl, y), O.score(fl, d, y), O.fisher_information(fl, d, cache=True)


def show(tag, r, n, t=None):
    ll, s, f = r
    extra = f" ({t:.1f}s)" if t is not None else ""
    print(f"  {tag:10s} ll {ll:.12e} score {np.array2string(np.asarray(s), precision=10)} "
          f"F {np.array2string(np.asarray(f).ravel(), precision=10)}  F_ss/(n/2) {f[0][0] / (n / 2):.5f}{extra}",
          flush=True)


for lg in args:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    y = np.random.default_rng(1).standard_normal(n)
    tau = H.tree_depth(n, 128, 256)
    print(f"===== n = 2^{lg} tau = {tau}", flush=True)
    if lg <= 15:
        t0 = time.time()
        tr = dense_truth(x, y)
        torch.cuda.empty_cache()
        show("dense", tr, n, time.time() - t0)
    g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
    br = H.build_hodlr_with_derivatives(g, H.ClusterTree(n, tau), K, SEED)
    show("gpuH/gpu", gpu_pipeline(br.h, br.deriv, y), n)
    if lg <= cpu_max:
        t0 = time.time()
        o = O.CovOracle.matern(x, 5, SIG2, ELL, NUG, True)
        bo = O.Build(o, tau, K, SEED, True, 2)
        hc, dc = bo.h(), [bo.deriv(0), bo.deriv(1)]
        print(f"  CPU build {time.time() - t0:.1f}s", flush=True)
        dd = [H.HodlrMatrix.from_panels(m.export_panels()) for m in [hc] + dc]
        show("cpuH/gpu", gpu_pipeline(dd[0], dd[1:], y), n)
        t0 = time.time()
        show("cpuH/cpu", cpu_pipeline(hc, dc, y), n, time.time() - t0)
