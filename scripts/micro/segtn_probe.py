"""Time seg_tn-like shapes through the library (trace_pair pair terms dominate)."""
import sys, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2303_10102_b200 import hodlrgp as H
n = 1 << 20
ctx = H.context()
L = H.lib()
H.prof_enable(True)
# Fisher-sized ProductReps via random HODLRs (k=40 -> corrections 80 wide)
t = H.ClusterTree(n, 13)
a = H.HodlrMatrix.random_spd(t, 40, 1)
b = H.HodlrMatrix.random_symmetric(t, 40, 2)
f = H.factorize(a, H.LEFT)
H.prof_read(True)
p = H.solve_multiply(f, b)
pr1 = H.prof_read(True)
v = H.trace_pair(p, p)
pr2 = H.prof_read(True)
for name, pr in (("solve_multiply", pr1), ("trace_pair", pr2)):
    print(name, {k: (round(x["ms"], 1), round(x["flops"] / max(x["ms"], 1e-9) / 1e9, 2), x["launches"]) for k, x in pr.items() if x["launches"]})
