"""Quick H-matvec timing probe at C4 scale (n=2^20, leaf 128, k=40, s=64/1)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2303_10102_b200 import hodlrgp as H

n, tau, k = 1 << 20, 13, 40
torch.cuda.init()
stream = torch.cuda.current_stream()
ctx = H.Context(0, C.c_void_p(stream.cuda_stream))
t0 = time.time()
h = H.HodlrMatrix.random_spd(H.ClusterTree(n, tau), k, 7, ctx=ctx)
ctx.synchronize()
print("random_spd host gen", time.time() - t0, flush=True)
for s in [int(a) for a in sys.argv[1:]] or (64, 4, 2, 1):
    X = torch.randn(s, n, dtype=torch.float64, device="cuda").T
    Y = torch.empty(s, n, dtype=torch.float64, device="cuda").T
    for _ in range(3):
        H._check(H.lib().hg_hodlr_matvec(ctx.ptr, h.ptr, X.data_ptr(), n, s, Y.data_ptr(), n, H.DEVICE))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    ev0.record(stream)
    for _ in range(reps):
        H._check(H.lib().hg_hodlr_matvec(ctx.ptr, h.ptr, X.data_ptr(), n, s, Y.data_ptr(), n, H.DEVICE))
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    b = 8 * n * (128 + k * tau) + 16 * n * s
    f = 2 * n * s * (128 + 2 * k * tau)
    print(f"s={s}: {ms:.3f} ms  {b/ms/1e6:.1f} GB/s  {f/ms/1e9:.2f} TFLOP/s", flush=True)
