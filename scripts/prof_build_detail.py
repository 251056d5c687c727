"""Per-shape kernel breakdown of the C4 build only (HG_PROF_DETAIL=1)."""
import os
import sys

os.environ["HG_PROF_DETAIL"] = "1"
sys.path.insert(0, ".")
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << lg
x = np.sort(np.random.default_rng(0).uniform(size=n))
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
H.prof_enable(True)
H.prof_read(reset=True)
H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
p = H.prof_read(reset=True)
H.prof_enable(False)
for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        print(f"{k:12s} {v['ms']:9.1f} ms {v['launches']:6d}")
