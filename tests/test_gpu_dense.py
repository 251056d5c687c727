"""GPU: the exact dense evaluation (dense_exact, mle.cpp:345-380), fit_mle's
dense path (FitOptions::dense, mle.cpp:128-175) and accuracy_metrics
(mle.cpp:382-403) against their numpy restatements in oracle/fit.py, and the
reference's own test cases for them (test_mle.cpp:153-186)."""
import numpy as np
import pytest

from oracle import fit as F
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    return hodlrgp


def matern(x, nu2, s2, ell, nug):
    o = O.CovOracle.matern(x, nu2, s2, ell, nug, False)
    n = len(x)
    return o.apply(np.eye(n)), [o.apply(np.eye(n), 0), o.apply(np.eye(n), 1)]


def test_dense_exact_matches_restatement(H):
    n = 1024
    x = np.sort(np.random.default_rng(3).uniform(size=n))
    K, dK = matern(x, 3, 1.3, 0.15, 1e-4)
    y = np.linalg.cholesky(K) @ O.randn(n, 1, 5)[:, 0] + 0.3
    ybar = np.full(n, 0.25)
    ll0, s0, f0 = F.dense_exact(K, dK, y - ybar)
    ll1, s1, f1 = H.dense_exact(H.MaternOracle(x, 3, 1.3, 0.15, 1e-4, False), y, ybar)
    assert ll1 == pytest.approx(ll0, rel=1e-11)
    assert np.allclose(s1, s0, rtol=1e-8, atol=1e-8 * np.abs(s0).max())
    assert np.allclose(f1, f0, rtol=1e-10)
    # the same on a DenseMatrixOracle (p = 2)
    o = H.DenseMatrixOracle(K, dK)
    ll2, s2, f2 = H.dense_exact(o, y, ybar)
    assert ll2 == pytest.approx(ll0, rel=1e-12) and np.allclose(f2, f0, rtol=1e-10)
    assert o.counters() == (n, 2 * n)  # apply(I) and apply_derivative(j, I)


def test_dense_exact_agrees_with_factorized_evaluation(H):  # test_mle.cpp:153-170
    """The dense evaluation vs the HODLR pipeline on the same oracle (C1 model,
    n = 2048): identical up to the HODLR approximation."""
    n = 2048
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    K, _ = matern(x, 3, 1.0, 0.2, 1e-4)
    y = np.linalg.cholesky(K) @ O.randn(n, 1, 1)[:, 0]
    o = H.MaternOracle(x, 3, 1.0, 0.2, 1e-4, True)
    ll0, s0, f0 = H.dense_exact(o, y)
    ll1, s1, f1, _ = H.mle_iteration(o, O.tree_depth(n, 64, 128), 24, 0, y)
    assert ll1 == pytest.approx(ll0, rel=1e-9)
    assert np.linalg.norm(s1 - s0) <= 1e-6 * (1.0 + np.linalg.norm(s0))
    assert np.linalg.norm(f1 - f0) <= 1e-6 * np.linalg.norm(f0)
    m = H.accuracy_metrics(ll0, s0, f0, ll1, s1, f1)
    assert m["eps_L"] < 1e-9 and m["eps_I"] < 1e-6 and m["eta_g"] < 1e-3


def test_dense_exact_guards(H):
    x = np.sort(np.random.default_rng(1).uniform(size=(1 << 13) + 1))
    with pytest.raises(OverflowError, match="dense guard"):
        H.dense_exact(H.MaternOracle(x, 3, 1.0, 0.2, 1e-4, True), np.zeros(len(x)))
    a = -np.eye(64)
    with pytest.raises(H.NotPositiveDefinite):
        H.dense_exact(H.DenseMatrixOracle(a, [np.eye(64)]), np.ones(64))


def test_accuracy_metrics(H):  # test_mle.cpp:172-186
    s = np.array([1.0, 2.0])
    fi = np.array([[2.0, 0.3], [0.3, 1.0]])
    m = H.accuracy_metrics(-10.0, s, fi, -10.0, s, fi)
    assert m["eps_L"] == 0.0 and m["eps_S"] == 0.0 and m["eps_I"] == 0.0 and m["eta_g"] == 0.0
    assert m["eta_I"] == pytest.approx(0.0, abs=1e-12)
    m2 = H.accuracy_metrics(-10.0, s, fi, -10.1, s, fi)
    assert m2["eps_L"] == pytest.approx(0.01, rel=1e-9)
    g = np.random.default_rng(2)
    a = g.standard_normal((3, 3))
    fe = a @ a.T + 3 * np.eye(3)
    fa = fe + 0.05 * g.standard_normal((3, 3))
    se, sa = g.standard_normal(3), g.standard_normal(3)
    got, want = H.accuracy_metrics(-5.0, se, fe, -5.2, sa, fa), F.accuracy_metrics(-5.0, se, fe, -5.2, sa, fa)
    for key in want:
        assert got[key] == pytest.approx(want[key], rel=1e-12), key
    with pytest.raises(ValueError, match="not SPD"):
        H.accuracy_metrics(-5.0, se, -fe, -5.2, sa, fa)


def test_fit_mle_dense_matches_restatement(H):
    """FitOptions::dense on the device vs oracle/fit.py over numpy dense
    evaluators: same BFGS trajectory (loglik 1e-10 per common iterate; the
    relative stopping rule may fire an iterate or two apart once the steps
    reach rounding level, so the optima agree to the rule's own resolution:
    theta_hat 1e-5, Fisher at theta_hat 1e-4)."""
    n = 400
    x = np.sort(np.random.default_rng(4).uniform(size=n))
    K, _ = matern(x, 3, 1.0, 0.2, 1e-4)
    y = np.linalg.cholesky(K) @ O.randn(n, 1, 3)[:, 0]
    theta0 = np.array([1.5, 0.1])
    cpu = F.fit_mle(*F.dense_evaluators(lambda th: matern(x, 3, th[0], th[1], 1e-4), y), theta0,
                    [F.POSITIVE, F.POSITIVE])
    dev = H.fit_mle(H.MaternOracle(x, 3, 1.5, 0.1, 1e-4, False), H.ClusterTree(n, 0), 0, 0, y, theta0, dense=True)
    assert dev["status"] == cpu["status"], (dev["status"], cpu["status"])
    m = min(len(dev["loglik_trace"]), len(cpu["loglik_trace"]))
    assert m >= 3 and abs(len(dev["loglik_trace"]) - len(cpu["loglik_trace"])) <= 3
    ll0, ll1 = np.array(cpu["loglik_trace"][:m]), dev["loglik_trace"][:m]
    assert np.max(np.abs(ll1 - ll0) / np.abs(ll0)) <= 1e-10
    assert np.max(np.abs(dev["theta_hat"] - cpu["theta_hat"]) / cpu["theta_hat"]) <= 1e-5
    assert np.linalg.norm(dev["fisher"] - cpu["fisher"]) <= 1e-4 * np.linalg.norm(cpu["fisher"])
    # the Fisher matrix at the device optimum is the dense exact one there
    ll, s, f = F.dense_exact(*matern(x, 3, dev["theta_hat"][0], dev["theta_hat"][1], 1e-4), y)
    assert np.linalg.norm(dev["fisher"] - f) <= 1e-9 * np.linalg.norm(f)
    assert dev["apply_columns"] > 0 and dev["apply_columns"] % n == 0


def test_fit_dense_vs_hodlr(H):
    """The paper's accuracy claim on a C1-like problem: the HODLR fit lands on
    the dense optimum (theta_hat within 1e-4 relative, far inside the CI)."""
    n = 2048
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    K, _ = matern(x, 3, 1.0, 0.2, 1e-4)
    y = np.linalg.cholesky(K) @ O.randn(n, 1, 1)[:, 0]
    theta0 = np.array([1.5, 0.1])
    tree = H.ClusterTree(n, O.tree_depth(n, 64, 128))
    d = H.fit_mle(H.MaternOracle(x, 3, 1.5, 0.1, 1e-4, True), tree, 24, 0, y, theta0, dense=True)
    h = H.fit_mle(H.MaternOracle(x, 3, 1.5, 0.1, 1e-4, True), tree, 24, 0, y, theta0)
    assert d["converged"] and h["converged"]
    assert np.max(np.abs(h["theta_hat"] - d["theta_hat"]) / d["theta_hat"]) <= 1e-4
    assert np.all(d["ci"][:, 0] < h["theta_hat"]) and np.all(h["theta_hat"] < d["ci"][:, 1])
