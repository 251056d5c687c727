"""Strong-admissibility H-matrix (eta = 1) of the C3/C5 SPDE covariance vs the
weak HODLR at the same rank: accuracy against the exact FFT apply, storage,
build and matvec times on one GPU.

usage: python scripts/probe_hstrong.py [small|c3|c5 ...]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2303_10102_b200 import hodlrgp as H

TH = {"small": (64, 64, 24, 0.05), "c3": (256, 256, 42, 0.05), "c5": (512, 256, 64, 0.03)}


def norm2_est(apply_err, n, its=25, seed=5):
    """Power iteration for ||E||_2 of the symmetric error operator E."""
    v = torch.randn(1, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(seed)).T
    lam = 0.0
    for _ in range(its):
        v = (v / torch.linalg.norm(v)).T.contiguous().T  # column-major n x 1
        w = apply_err(v)
        lam = float(torch.linalg.norm(w))
        v = w
    return lam


def ev_time(f, reps=3):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(torch.cuda.current_stream())
        f()
        b.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return min(ts)


def run(name, power_iters=0):
    if H._ctx is None:  # one stream for torch and the library (torch's default is the legacy NULL stream)
        torch.cuda.set_stream(torch.cuda.Stream())
        H._ctx = H.Context(0, torch.cuda.current_stream().cuda_stream)
    N, leaf, k, ell = TH[name]
    n = N * N
    var = H.spde2d_variance(N, 1.0, ell, 4.0)
    nug = 1e-8 * var
    order, tree = H.grid_kd_order(N, leaf)
    o = H.Spde2dOracle(N, 1.0, ell, 4.0, order=order, nugget=nug)
    plan = H.hstrong_plan(order, N, tree.tau, 1.0, k)
    H.HStrongMatrix(o, order, N, tree.tau, k, 1.0, -1, power_iters, 7)  # warm-up (allocator, module load)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hs = H.HStrongMatrix(o, order, N, tree.tau, k, 1.0, -1, power_iters, 7)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    H.prof_enable(True)
    H.HStrongMatrix(o, order, N, tree.tau, k, 1.0, -1, power_iters, 7)
    prof = {c: v for c, v in H.prof_read(True).items() if v["launches"]}
    H.prof_enable(False)
    g = torch.Generator().manual_seed(3)
    V = torch.randn(8, n, generator=g, dtype=torch.float64).cuda().T  # column-major n x 8
    KV = o.apply(V)
    HV = hs.matvec(V)
    err_s = float(torch.linalg.norm(HV - KV) / torch.linalg.norm(KV))
    hw = H.build_hodlr(o, tree, k, 7)
    WV = hw.matvec(V)
    err_w = float(torch.linalg.norm(WV - KV) / torch.linalg.norm(KV))
    e2s = norm2_est(lambda v: hs.matvec(v) - o.apply(v), n)
    e2w = norm2_est(lambda v: hw.matvec(v) - o.apply(v), n)
    k2 = norm2_est(lambda v: o.apply(v), n)
    out = dict(config=name, n=n, tau=tree.tau, k=k, power_iters=power_iters, plan=plan, blocks=hs.blocks,
               build_s=t_build, build_prof=prof, rel_err_strong=err_s, rel_err_weak=err_w, nugget_over_var=1e-8,
               var_u=var, norm2_K_over_var=k2 / var, norm2_err_strong_over_var=e2s / var,
               norm2_err_weak_over_var=e2w / var)
    for s in (1, 64):
        X = torch.randn(s, n, dtype=torch.float64, device="cuda").T
        out[f"matvec_s{s}_ms"] = 1e3 * ev_time(lambda: hs.matvec(X))
        out[f"matvec_s{s}_GBps"] = hs.blocks["bytes"] / (out[f"matvec_s{s}_ms"] / 1e3) / 1e9
    if n <= 4096:
        K = o.apply(np.eye(n))
        Hd = hs.matvec(np.eye(n))
        out["dense_rel_err_strong"] = float(np.linalg.norm(Hd - K) / np.linalg.norm(K))
        out["dense_asym"] = float(np.linalg.norm(Hd - Hd.T) / np.linalg.norm(Hd))
        Wd = hw.densify()
        out["dense_rel_err_weak"] = float(np.linalg.norm(Wd - K) / np.linalg.norm(K))
        ev = np.linalg.eigvalsh(0.5 * (Hd + Hd.T))
        out["lambda_min_strong_over_var"] = float(ev[0] / var)
        out["lambda_min_weak_over_var"] = float(np.linalg.eigvalsh(0.5 * (Wd + Wd.T))[0] / var)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["small", "c3"]:
        nm, _, q = a.partition(":")
        run(nm, int(q) if q else 0)
