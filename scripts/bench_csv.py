"""The reference CLI's bench report (tools/hodlr_gp.cpp:378-477, cmd_bench) on
the device path: `OUT/bench.csv` with header `n,k,metric,value,repeat` and the
same metric names, values in 17 significant digits (io.cpp fmt17).

Stage times are wall-clock around each public-API call with the context
synchronized on both sides (the reference's now_seconds brackets). The
reference's OpenMP comparison rows become `eval_seconds_parallel` (one device
evaluation: factorize + loglik + score + Fisher); `eval_seconds_serial` has no
device meaning and is not written. Model: 1-D Matérn on sorted U[0,1] points
(seeded), data y ~ N(0, I) (the timings do not depend on y).

usage: python scripts/bench_csv.py OUT [--sizes 4096 65536] [--repeats 3]
           [--nu2 3] [--sigma2 1] [--ell 0.2] [--nugget 1e-4] [--rank 24]
           [--leaf-min 64] [--leaf-max 128] [--sketch-seed 0]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H


def fmt17(v):
    return "%.17g" % v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--sizes", type=int, nargs="+", default=[4096])
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--nu2", type=int, default=3)
    ap.add_argument("--sigma2", type=float, default=1.0)
    ap.add_argument("--ell", type=float, default=0.2)
    ap.add_argument("--nugget", type=float, default=1e-4)
    ap.add_argument("--rank", type=int, default=24)
    ap.add_argument("--leaf-min", type=int, default=64)
    ap.add_argument("--leaf-max", type=int, default=128)
    ap.add_argument("--sketch-seed", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    if not a.sizes:
        raise SystemExit("bench.sizes must be non-empty")
    os.makedirs(a.out, exist_ok=True)
    ctx = H.context()
    rows = ["n,k,metric,value,repeat"]

    def row(n, metric, value, rep):
        rows.append(f"{n},{a.rank},{metric},{fmt17(float(value))},{rep}")

    def timed(f):
        ctx.synchronize()
        t0 = time.perf_counter()
        r = f()
        ctx.synchronize()
        return r, time.perf_counter() - t0

    for n in a.sizes:
        x = np.sort(np.random.default_rng(0).uniform(size=n))
        o = H.MaternOracle(x, a.nu2, a.sigma2, a.ell, a.nugget, True)
        tree = H.ClusterTree(n, H.tree_depth(n, a.leaf_min, a.leaf_max))
        for rep in range(a.repeats):
            y = np.random.default_rng(a.seed + rep).standard_normal(n)
            o.reset_counters()
            h, t = timed(lambda: H.build_hodlr(o, tree, a.rank, a.sketch_seed))
            row(n, "build_seconds", t, rep)
            row(n, "build_apply_columns", o.apply_columns(), rep)
            row(n, "build_apply_columns_expected", 2 * a.rank * tree.tau + tree.max_leaf_size(), rep)
            o.reset_counters()
            built, t = timed(lambda: H.build_hodlr_with_derivatives(o, tree, a.rank, a.sketch_seed))
            row(n, "build_deriv_seconds", t, rep)
            row(n, "deriv_apply_columns", o.apply_columns(), rep)
            row(n, "deriv_derivative_columns", o.derivative_columns(), rep)
            hd, dd = built.h, built.deriv
            fac, t = timed(lambda: H.factorize(hd, H.LEFT))
            row(n, "factorize_seconds", t, rep)
            _, t = timed(lambda: H.log_likelihood(fac, y))
            row(n, "loglik_seconds", t, rep)
            _, t = timed(lambda: H.score(fac, dd, y))
            row(n, "score_seconds", t, rep)
            _, t = timed(lambda: H.fisher_information(fac, dd))
            row(n, "fisher_seconds", t, rep)

            def evaluate():
                f2 = H.factorize(h, H.LEFT)
                v = H.log_likelihood(f2, y)
                return v + float(np.sum(H.score(f2, dd, y))) + float(np.sum(H.fisher_information(f2, dd)))

            _, t = timed(evaluate)
            row(n, "eval_seconds_parallel", t, rep)
    with open(os.path.join(a.out, "bench.csv"), "w") as f:
        f.write("\n".join(rows) + "\n")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
