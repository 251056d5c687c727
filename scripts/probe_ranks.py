"""Per-level rank capacities R_l of H and dK/dtheta_j at C4 (n = 2^20)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2303_10102_b200 import hodlrgp as H

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << lg
tau = H.tree_depth(n, 128, 256)
x = np.sort(np.random.default_rng(0).uniform(size=n))
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
br = H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
print("H ", br.h.info()[3])
for j, d in enumerate(br.deriv):
    print(f"D{j}", d.info()[2], d.info()[3])
