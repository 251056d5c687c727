"""Per-class / per-shape device time of the C4 build with derivatives alone."""
import os
import sys

os.environ["HG_PROF_DETAIL"] = "1"
sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

n = 1 << 20
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
H.prof_enable(True)
H.prof_read(reset=True)
H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
p = H.prof_read(reset=True)
H.prof_enable(False)
tot = 0
for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        tot += v["ms"]
        print(f"{k:12s} {v['ms']:9.1f} ms {v['launches']:6d}")
print("total profiled", tot)
