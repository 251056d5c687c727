"""Per-shape kernel breakdown of one stage of the C4 iteration (HG_PROF_DETAIL=1):
stage in {factorize, score, fisher}. Usage: python scripts/prof_stage_detail.py score"""
import os
import sys

os.environ["HG_PROF_DETAIL"] = "1"
sys.path.insert(0, ".")
import numpy as np

from paper_2303_10102_b200 import hodlrgp as H

stage = sys.argv[1] if len(sys.argv) > 1 else "score"
n = 1 << 20
x = np.sort(np.random.default_rng(0).uniform(size=n))
y = np.random.default_rng(1).standard_normal(n)
tau = H.tree_depth(n, 128, 256)
o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
br = H.build_hodlr_with_derivatives(o, H.ClusterTree(n, tau), 40, 7)
fl = H.factorize(br.h, H.LEFT)


def run():
    if stage == "factorize":
        H.factorize(br.h, H.LEFT)
    elif stage == "score":
        H.score(fl, br.deriv, y)
    else:
        H.fisher_information(fl, br.deriv)


run()
H.prof_enable(True)
H.prof_read(reset=True)
run()
p = H.prof_read(reset=True)
H.prof_enable(False)
for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        print(f"{k:12s} {v['ms']:9.1f} ms {v['launches']:6d}")
