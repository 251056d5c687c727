"""Full-size iterations at sketch widths above the configs' (robustness of the k <= 128 path):
C4 settings at k = 96 and C5 settings at k = 128. Prints stage times and the results."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H


def run(name, oracle, n, tau, k):
    y = np.random.default_rng(1).standard_normal(n)
    empty = np.zeros((n, 0), order="F")
    H.mle_evaluate(oracle, tau, k, 7, y, empty, empty)
    ll, s, f, t = H.mle_evaluate(oracle, tau, k, 7, y, empty, empty)
    print(json.dumps(dict(config=name, n=n, tau=tau, k=k, seconds=float(np.sum(t)), stages=[round(float(v), 3) for v in t],
                          loglik=ll, score=[float(v) for v in s], fisher_diag=[float(v) for v in np.diag(f)],
                          finite=bool(np.isfinite(ll) and np.all(np.isfinite(s)) and np.all(np.isfinite(f))))),
          flush=True)


which = sys.argv[1:] or ["c4", "c5"]
if "c4" in which:
    n = 1 << 20
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    run("C4 settings", H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True), n, H.tree_depth(n, 128, 256), 96)
if "c5" in which:
    N = 512
    order, tree = H.grid_kd_order(N, 256)
    run("C5 settings", H.Spde2dOracle(N, 1.0, 0.03, 4.0, order=order), N * N, tree.tau, 128)
