"""MLE-iteration time of every BASELINE.json config on one GPU (secondary lines;
bench.py's headline is C4). Each config: 1 warm-up + `steps` timed iterations
of hg_mle_evaluate (build with derivatives, factorize, logdet, loglik, score,
Fisher), device-event timed. Synthetic inputs as in DESIGN.md §5; y is a
seeded N(0, I) draw (timing does not depend on it).

usage: python scripts/bench_configs.py [steps] [configs...]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2303_10102_b200 import hodlrgp as H


def c1():
    n = 4096
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    return dict(name="C1", oracle=H.MaternOracle(x, 3, 1.0, 0.2, 1e-4, True), n=n,
                tau=H.tree_depth(n, 64, 128), k=24, seed=0, p=2)


def c2():
    m = 16384
    n = 2 * m
    return dict(name="C2", oracle=H.CoKrigingOracle(m, 1.0, 0.1, 2.0), n=n, tau=H.tree_depth(n, 128, 256), k=32,
                seed=7, p=3)


def spde(name, N, ell, k):
    order, tree = H.grid_kd_order(N, 256)
    return dict(name=name, oracle=H.Spde2dOracle(N, 1.0, ell, 4.0, order=order), n=N * N, tau=tree.tau, k=k,
                seed=7, p=3)


CONFIGS = {"C1": c1, "C2": c2, "C3": lambda: spde("C3", 256, 0.05, 42), "C5": lambda: spde("C5", 512, 0.03, 64)}


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    names = sys.argv[2:] or list(CONFIGS)
    torch.zeros(1, device="cuda")
    for nm in names:
        cfg = CONFIGS[nm]()
        n = cfg["n"]
        y = np.random.default_rng(1).standard_normal(n)
        empty = np.zeros((n, 0), order="F")
        w0 = time.perf_counter()
        ll, s, f, t = H.mle_evaluate(cfg["oracle"], cfg["tau"], cfg["k"], cfg["seed"], y, empty, empty)
        first = time.perf_counter() - w0
        ts = []
        for _ in range(steps):
            ll, s, f, t = H.mle_evaluate(cfg["oracle"], cfg["tau"], cfg["k"], cfg["seed"], y, empty, empty)
            ts.append(float(t.sum()))
        print(json.dumps({"config": nm, "n": n, "tau": cfg["tau"], "k": cfg["k"], "p": cfg["p"],
                          "s_per_iteration": min(ts), "median_s": float(np.median(ts)), "first_call_s": first,
                          "stages_s": [round(float(v), 4) for v in t], "loglik": ll,
                          "score": [float(v) for v in s], "fisher_diag": [float(v) for v in np.diag(f)]}),
              flush=True)




def profile(nm):
    """Per-kernel-class ledger of one iteration of config nm (after a warm-up)."""
    cfg = CONFIGS[nm]()
    n = cfg["n"]
    y = np.random.default_rng(1).standard_normal(n)
    empty = np.zeros((n, 0), order="F")
    H.mle_evaluate(cfg["oracle"], cfg["tau"], cfg["k"], cfg["seed"], y, empty, empty)
    H.prof_enable(True)
    H.prof_read(reset=True)
    H.mle_evaluate(cfg["oracle"], cfg["tau"], cfg["k"], cfg["seed"], y, empty, empty)
    p = H.prof_read(reset=True)
    H.prof_enable(False)
    print(nm, {k: round(v["ms"], 1) for k, v in p.items() if v["launches"]}, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "profile":
        for nm in sys.argv[2:]:
            profile(nm)
    else:
        main()
