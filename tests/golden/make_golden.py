"""Generate the committed golden fixtures (run here, on CPU; not at test time).

    python tests/golden/make_golden.py

The reference ships no golden vectors; these are made by the
CPU restatement in oracle/ and stored in the reference's own debug-serializer
layout (io.cpp:171-233: JSON manifest + row-major little-endian float64
sidecars), as SURVEY.md §8c asks:

* spd50_sym / spd50_asym — the matrices of test_io.cpp:92-107:
  HodlrMatrix::random_spd(ClusterTree(50, 2), 3, 4), then make_asymmetric()
  with lower(1, 0).left doubled.
* c1s_h, c1s_d0, c1s_d1 — config C1's model (Matérn 3/2, sigma^2 = 1,
  ell = 0.2, nugget 1e-4, k = 24, sketch seed 0) at n = 512 (leaf 64,
  tau = 3): the built H and dH/dsigma^2, dH/dell. Points c1s_x.bin and the
  data vector c1s_y.bin (seed-1 normals coloured by the dense Cholesky
  factor) are sidecars too, so the GPU tests need no host RNG.
* c1 — config C1 in full (n = 4096): points and data as sidecars; the
  results (log-likelihood, score, Fisher, per-block rank decisions) live in
  golden.json only (its HODLR panels would be ~20 MB).

golden.json holds the scalar results, each computed by the oracle in both
product associations (`reference` = product_rep.cpp's, `solve` = the one the
device path uses; DESIGN.md §4 explains why they differ at C1's condition
number).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as O  # noqa: E402
from oracle import serial as S  # noqa: E402


def c1_model(n):
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    oo = O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, False)
    K = oo.apply(np.eye(n))
    y = np.linalg.cholesky(K) @ O.randn(n, 1, 1)[:, 0]
    return x, y, oo


def results(oo, tau, k, y):
    out = {}
    for tag, on in (("reference", False), ("solve", True)):
        try:
            O.set_solve_association(on)
            ll, s, f, _ = O.mle_iteration(oo, tau, k, 0, y, 2)
        finally:
            O.set_solve_association(False)
        out[tag] = {"loglik": ll, "score": s.tolist(), "fisher": f.tolist()}
    return out


def main():
    g = {"generator": "tests/golden/make_golden.py", "format": "io.cpp:171-233 debug serializer"}

    h = O.Hodlr.random_spd(50, 2, 3, 4)
    S.write_hodlr_debug(HERE, "spd50_sym", h.export_panels())
    b = O.randn(50, 1, 7)[:, 0]
    f = O.factorize(h, 1)
    g["spd50_sym"] = {"n": 50, "depth": 2, "k": 3, "seed": 4, "trace": h.trace(),
                      "logdet": f.logdet(), "solve_rhs": "randn(50, 1, seed 7)",
                      "solve": f.solve(b).tolist()}
    p = h.export_panels()
    a = O.Hodlr.import_panels(p)
    a.make_asymmetric()
    q = a.export_panels()
    # lower(1, 0).left: U_1 rows of the right child, its first rank_lo columns
    n, R1 = q["n"], q["R"][0]
    U1 = q["flat"][:n * R1].reshape(R1, n).T
    lo, hi = S.tree_ranges(n, 2)[1][1]
    U1[lo:hi, :int(q["ranks_lo"][0])] *= 2.0
    S.write_hodlr_debug(HERE, "spd50_asym", q)
    g["spd50_asym"] = {"from": "spd50_sym", "edit": "make_asymmetric; lower(1,0).left *= 2",
                       "trace": O.Hodlr.import_panels(q).trace()}

    n, leaf, k = 512, 64, 24
    tau = O.tree_depth(n, leaf, 2 * leaf)
    x, y, oo = c1_model(n)
    S.write_sidecar(os.path.join(HERE, "c1s_x.bin"), x)
    S.write_sidecar(os.path.join(HERE, "c1s_y.bin"), y)
    bd = O.Build(oo, tau, k, 0, True, p=2)
    for nm, m in (("c1s_h", bd.h()), ("c1s_d0", bd.deriv(0)), ("c1s_d1", bd.deriv(1))):
        S.write_hodlr_debug(HERE, nm, m.export_panels())
    fh = O.factorize(bd.h(), 1)
    g["c1s"] = {"n": n, "depth": tau, "k": k, "seed": 0, "nu2": 3, "sigma2": 1.0, "ell": 0.2, "nugget": 1e-4,
                "logdet": fh.logdet(), "decisions": bd.decisions().tolist(), **results(oo, tau, k, y)}

    n = 4096
    tau = O.tree_depth(n, leaf, 2 * leaf)
    x, y, oo = c1_model(n)
    S.write_sidecar(os.path.join(HERE, "c1_x.bin"), x)
    S.write_sidecar(os.path.join(HERE, "c1_y.bin"), y)
    bd = O.Build(oo, tau, k, 0, True, p=2)
    g["c1"] = {"n": n, "depth": tau, "k": k, "seed": 0, "nu2": 3, "sigma2": 1.0, "ell": 0.2, "nugget": 1e-4,
               "logdet": O.factorize(bd.h(), 1).logdet(), "decisions": bd.decisions().tolist(),
               **results(oo, tau, k, y)}

    with open(os.path.join(HERE, "golden.json"), "w") as fp:
        fp.write(json.dumps(g, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
