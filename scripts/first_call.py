"""Time of the first C4-size MLE evaluation (SketchPlan generation + upload included) vs a warm one."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
y = np.random.default_rng(1).standard_normal(n)
B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 4)))
X = np.zeros_like(B)
H.context().synchronize() if hasattr(H.context(), "synchronize") else None
t0 = time.perf_counter()
H.sketch_sampler(n, tau, 40, 7, 1)
t1 = time.perf_counter()
H.mle_evaluate(o, tau, 40, 7, y, B, X)
t2 = time.perf_counter()
H.mle_evaluate(o, tau, 40, 7, y, B, X)
t3 = time.perf_counter()
print(f"n=2^{lg}: plan (reference host stream) {t1 - t0:.2f} s, first evaluation {t2 - t1:.2f} s, warm {t3 - t2:.2f} s", flush=True)
ctx = H.context()
ctx.set_option(H.OPT_SKETCH_RNG, H.SKETCH_RNG_DEVICE)
t0 = time.perf_counter()
H.sketch_sampler(n, tau, 40, 7, 1)
t1 = time.perf_counter()
print(f"plan (device generator) {t1 - t0:.3f} s", flush=True)
