"""C4 numerics diagnosis (VERDICT r1 "Next" #1): GPU vs CPU oracle stage by stage.

For n = 2^lg at the C4 settings (Matérn 5/2, sigma2 = 1, ell = 0.05, nugget 1e-6,
leaf 128, k = 40, sketch seed 7) this prints, for each n:
  * the forward models: GPU scan apply vs CPU scan apply vs direct kernel rows;
  * the built HODLRs: ||(H - K) V|| / ||V|| for GPU-built and CPU-built H and D_j;
  * a 2x2 cross table: {GPU-built, CPU-built} H x {GPU, CPU} downstream
    (factorize, logdet, tr(K^-1 K_j), Fisher) so the stage that drifts is named;
  * lambda_min(H) by inverse power iteration on each factorization;
  * the bound F_ss <= n / (2 sigma^4).
Usage: python scripts/diag_c4.py 14 16 18 [--cpu-max 18]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from oracle import pyoracle as O
from paper_2303_10102_b200 import hodlrgp as H

# The reference association (product_rep.cpp:74-78) is unstable at these
# condition numbers (Fisher_ss < 0 at 2^13); compare in the device association.
O.set_solve_association(True)

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cpu_max = 18
for a in sys.argv[1:]:
    if a.startswith("--cpu-max="):
        cpu_max = int(a.split("=")[1])
SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7


def kernel_rows(x, rows, V):
    """Direct Matérn 5/2 rows of K times V (plus nugget): the independent truth."""
    out = np.zeros((len(rows), V.shape[1]))
    for t, i in enumerate(rows):
        a = np.sqrt(5.0) * np.abs(x - x[i]) / ELL
        kr = SIG2 * (1 + a + a * a / 3) * np.exp(-a)
        kr[i] += NUG
        out[t] = kr @ V
    return out


def inv_power(f, n, it=30, seed=3):
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(it):
        w = f.solve(v)
        lam = np.linalg.norm(w)
        v = w / lam
    return 1.0 / lam


def pipeline(mod, h, d, y, lhs_is_gpu):
    t0 = time.time()
    if lhs_is_gpu:
        fl = H.factorize(h, H.LEFT)
        ld = fl.logdet()
        ll = H.log_likelihood(fl, y)
        sc = H.score(fl, d, y)
        tr = [H.trace_solve(fl, dj) for dj in d]
        fi = H.fisher_information(fl, d)
    else:
        fl = O.factorize(h, O.Factor.LEFT)
        ld = fl.logdet()
        ll = O.log_likelihood(fl, y)
        sc = O.score(fl, d, y)
        tr = [O.trace_solve(fl, dj) for dj in d]
        fi = O.fisher_information(fl, d, cache=True)
    lmin = inv_power(fl, len(y))
    return dict(ld=ld, ll=ll, sc=sc, tr=np.array(tr), fi=fi, lmin=lmin, t=time.time() - t0)


for lg in [int(a) for a in args]:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    y = np.random.default_rng(1).standard_normal(n)
    tau = H.tree_depth(n, 128, 256)
    print(f"===== n = 2^{lg}  tau = {tau}  bound F_ss <= n/2 = {n / 2:.6g}", flush=True)
    g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
    V = np.asfortranarray(np.random.default_rng(9).standard_normal((n, 4)))
    rows = np.random.default_rng(4).choice(n, 64, replace=False)
    KV_rows = kernel_rows(x, rows, V)
    gv = g.apply(V)
    print(f"GPU scan apply vs direct rows: {np.linalg.norm(gv[rows] - KV_rows) / np.linalg.norm(KV_rows):.3e}")
    do_cpu = lg <= cpu_max
    if do_cpu:
        o = O.CovOracle.matern(x, 5, SIG2, ELL, NUG, True)
        ov = o.apply(V)
        print(f"CPU scan apply vs direct rows: {np.linalg.norm(ov[rows] - KV_rows) / np.linalg.norm(KV_rows):.3e}"
              f"   GPU vs CPU apply: {np.linalg.norm(gv - ov) / np.linalg.norm(ov):.3e}")
    t0 = time.time()
    br = H.build_hodlr_with_derivatives(g, H.ClusterTree(n, tau), K, SEED)
    hg, dg = br.h, br.deriv
    print(f"GPU build {time.time() - t0:.2f}s  R = {hg.info()}", flush=True)
    nrm = np.linalg.norm(V)
    HgV = hg.matvec(V)
    print(f"GPU H: ||(H-K)V||/||V|| = {np.linalg.norm(HgV - gv) / nrm:.3e}  (nugget {NUG:g}),"
          f" rows vs direct {np.linalg.norm(HgV[rows] - KV_rows) / np.linalg.norm(KV_rows):.3e}")
    for j in range(2):
        gdv = g.apply(V, j)
        print(f"GPU D{j}: ||(D-Kj)V||/||KjV|| = {np.linalg.norm(dg[j].matvec(V) - gdv) / np.linalg.norm(gdv):.3e}")
    gp = [hg.export_panels()] + [dj.export_panels() for dj in dg]
    res = {}
    res["gpuH/gpu"] = pipeline(H, hg, dg, y, True)
    if do_cpu:
        t0 = time.time()
        bo = O.Build(o, tau, K, SEED, True, 2)
        hc, dc = bo.h(), [bo.deriv(0), bo.deriv(1)]
        print(f"CPU build {time.time() - t0:.2f}s  R = {hc.info()[3]}", flush=True)
        HcV = hc.matvec(V)
        print(f"CPU H: ||(H-K)V||/||V|| = {np.linalg.norm(HcV - ov) / nrm:.3e}; ||Hgpu V - Hcpu V||/||V|| ="
              f" {np.linalg.norm(HgV - HcV) / nrm:.3e}")
        for j in range(2):
            odv = o.apply(V, j)
            print(f"CPU D{j}: ||(D-Kj)V||/||KjV|| = {np.linalg.norm(dc[j].matvec(V) - odv) / np.linalg.norm(odv):.3e}")
        dg_h = [O.Hodlr.import_panels(p) for p in gp]
        cp = [hc.export_panels()] + [dj.export_panels() for dj in dc]
        dc_d = [H.HodlrMatrix.from_panels(p) for p in cp]
        res["gpuH/cpu"] = pipeline(O, dg_h[0], dg_h[1:], y, False)
        res["cpuH/gpu"] = pipeline(H, dc_d[0], dc_d[1:], y, True)
        res["cpuH/cpu"] = pipeline(O, hc, dc, y, False)
    for key, r in res.items():
        f = r["fi"]
        print(f"{key:9s} logdet {r['ld']:.12e} ll {r['ll']:.12e} tr {r['tr']} score {r['sc']}\n"
              f"          fisher {f.ravel()}  F_ss/(n/2) = {f[0, 0] / (n / 2):.4f}  lmin(H) = {r['lmin']:.4e}"
              f"  ({r['t']:.1f}s)", flush=True)
