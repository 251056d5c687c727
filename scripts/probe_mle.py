"""Probe one MLE iteration (C4 settings) at growing n: stage times, memory."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H
import ctypes as C
for lg in [int(a) for a in sys.argv[1:]] or [14, 16, 18, 20]:
    n = 1 << lg
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    tau = H.tree_depth(n, 128, 256)
    o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
    y = np.random.default_rng(1).standard_normal(n)
    t0 = time.time()
    ll, s, f, t = H.mle_iteration(o, tau, 40, 7, y)   # includes plan generation (host RNG)
    t1 = time.time()
    ll, s, f, t = H.mle_iteration(o, tau, 40, 7, y)
    t2 = time.time()
    free, total = C.c_size_t(), C.c_size_t()
    C.CDLL("libcudart.so").cudaMemGetInfo(C.byref(free), C.byref(total)) if False else None
    print(f"n=2^{lg} tau={tau} first {t1-t0:.2f}s second {t2-t1:.2f}s stages(build,fact,ll,score,fisher)={np.round(t,4)} ll={ll:.10e} score={s} fisher={f.ravel()} launches={H.context().launches}", flush=True)
