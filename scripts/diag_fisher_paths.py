"""C4 settings at n = 2^lg: the Fisher matrix through fisher_information
(shared-Gram correction pairs) vs per-pair trace_pair on the same reps, for
builds with the derivative compression at each level (default) and at the
end (reference order); dense truth for n <= 2^15.
Usage: python scripts/diag_fisher_paths.py 15 17
"""
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H

SIG2, ELL, NUG, K, SEED = 1.0, 0.05, 1e-6, 40, 7
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    tau = H.tree_depth(n, 128, 256)
    g = H.MaternOracle(x, 5, SIG2, ELL, NUG, True)
    ctx = H.context()
    for at in (H.COMPRESS_AT_LEVEL, H.COMPRESS_AT_END):
        ctx.set_option(H.OPT_COMPRESS_AT, at)
        br = H.build_hodlr_with_derivatives(g, H.ClusterTree(n, tau), K, SEED)
        fl = H.factorize(br.h, H.LEFT)
        f_new = H.fisher_information(fl, br.deriv)
        reps = [H.solve_multiply(fl, d) for d in br.deriv]
        f_old = np.array([[0.5 * H.trace_pair(reps[i], reps[j]) for j in range(2)] for i in range(2)])
        tag = "level" if at == H.COMPRESS_AT_LEVEL else "end"
        print(f"n=2^{lg} compress-at-{tag}: shared {f_new.ravel()}  per-pair {f_old.ravel()}", flush=True)
    ctx.set_option(H.OPT_COMPRESS_AT, H.COMPRESS_AT_LEVEL)
