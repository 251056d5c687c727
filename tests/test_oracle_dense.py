"""CPU: the numpy restatements of dense_exact and accuracy_metrics
(oracle/fit.py) pinned on the reference's own cases (test_mle.cpp:153-186)
and on independent identities. Test infrastructure for test_gpu_dense.py."""
import numpy as np
import pytest

from oracle import fit as F
from oracle import pyoracle as O


def test_accuracy_metrics_reference_cases():  # test_mle.cpp:172-186
    s = np.array([1.0, 2.0])
    fi = np.array([[2.0, 0.3], [0.3, 1.0]])
    m = F.accuracy_metrics(-10.0, s, fi, -10.0, s, fi)
    assert m["eps_L"] == m["eps_S"] == m["eps_I"] == m["eta_g"] == 0.0
    assert m["eta_I"] == pytest.approx(0.0, abs=1e-12)
    assert F.accuracy_metrics(-10.0, s, fi, -10.1, s, fi)["eps_L"] == pytest.approx(0.01, rel=1e-9)


def test_dense_exact_against_factorized_oracle():  # test_mle.cpp:153-170
    n = 72
    x = np.sort(np.random.default_rng(7).uniform(size=n))
    o = O.CovOracle.matern(x, 3, 0.8, 1.1, 1e-3, False)
    K, dK = o.apply(np.eye(n)), [o.apply(np.eye(n), 0), o.apply(np.eye(n), 1)]
    y = O.randn(n, 1, 9)[:, 0]
    ll, s, f = F.dense_exact(K, dK, y)
    h = O.Hodlr.from_dense(2, K)
    d = [O.Hodlr.from_dense(2, a) for a in dK]
    fac = O.factorize(h, 1)
    assert ll == pytest.approx(O.log_likelihood(fac, y), rel=1e-9)
    assert np.linalg.norm(s - O.score(fac, d, y)) <= 1e-8 * (1 + np.linalg.norm(s))
    assert np.linalg.norm(f - O.fisher_information(fac, d)) <= 1e-8 * np.linalg.norm(f)
    # the score formula through an independent solve path
    w = np.linalg.solve(K, y)
    assert s[0] == pytest.approx(-0.5 * np.trace(np.linalg.solve(K, dK[0])) + 0.5 * w @ dK[0] @ w, rel=1e-9)
