"""Size-independent parity properties at BASELINE.json's full C4 size
(n = 2^20, Matern 5/2, leaf 128, k = 40, seed 7).

The CPU oracle does not finish at this size within a test's budget (one
iteration at 2^17 takes ~5 min on 16 host cores), so the device path is
checked here through identities that hold for any exact execution of the
reference algorithm, through hard bounds on the score and Fisher entries,
and through agreement with the oracle and the dense truth at the C4 settings
on n = 2^14 (profiles/r2_c4_parity.md has the scan up to 2^17 and 2^20):

* H-matvec is linear, and a batched apply equals column-by-column applies
  bit for bit (deterministic kernels);
* the Woodbury solve is backward stable: ||H x - b|| <= c eps ||H|| ||x||;
* Right and Left factorizations give the same log-determinant;
* tr(H^-1 H) = n through the product representation (solve_multiply + traces);
* score_j = 1/2 y^T K^-1 K_j K^-1 y - 1/2 tr(K^-1 K_j) (mle.cpp:32-41) with the
  quadratic form from explicit solves/matvecs and the trace from trace_solve;
* two evaluations of the whole MLE iteration are bitwise identical.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 1 << 20
K_RANK, SEED = 40, 7


@pytest.fixture(scope="module")
def c4():
    from paper_2303_10102_b200 import hodlrgp as H

    tau = H.tree_depth(N, 128, 256)
    x = np.sort(np.random.default_rng(0).uniform(size=N))
    o = H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True)
    br = H.build_hodlr_with_derivatives(o, H.ClusterTree(N, tau), K_RANK, SEED)
    return H, o, tau, br.h, br.deriv


def test_c4_matvec_linear_and_batch_consistent(c4):
    H, _, _, h, _ = c4
    X = np.asfortranarray(np.random.default_rng(5).standard_normal((N, 2)))
    y1, y2 = h.matvec(X[:, 0]), h.matvec(X[:, 1])
    y12 = h.matvec(2.0 * X[:, 0] - 3.0 * X[:, 1])
    assert np.linalg.norm(y12 - (2.0 * y1 - 3.0 * y2)) <= 1e-13 * np.linalg.norm(y12)
    Y = h.matvec(X)
    assert np.array_equal(Y[:, 0], y1) and np.array_equal(Y[:, 1], y2)


def test_c4_solve_backward_stable(c4):
    H, _, _, h, _ = c4
    rng = np.random.default_rng(6)
    v = rng.standard_normal(N)
    for _ in range(8):  # ||H||_2 estimate by power iteration
        v = h.matvec(v)
        v /= np.linalg.norm(v)
    hnorm = np.linalg.norm(h.matvec(v))
    f = H.factorize(h, H.RIGHT)
    b = rng.standard_normal(N)
    x = f.solve(b)
    r = h.matvec(x) - b
    eta = np.linalg.norm(r) / (hnorm * np.linalg.norm(x) + np.linalg.norm(b))
    assert eta <= 1e-12, eta


def test_c4_logdet_orientation_independent(c4):
    H, _, _, h, _ = c4
    a = H.factorize(h, H.RIGHT).logdet()
    b = H.factorize(h, H.LEFT).logdet()
    assert abs(a - b) <= 1e-12 * abs(a)


def test_c4_trace_of_identity_product(c4):
    H, _, _, h, _ = c4
    tr = H.trace_solve(H.factorize(h, H.LEFT), h)
    assert abs(tr - N) <= 1e-8 * N, tr - N


def test_c4_score_identity_and_determinism(c4):
    H, o, tau, h, d = c4
    y = np.random.default_rng(1).standard_normal(N)
    empty = np.zeros((N, 0), order="F")
    ll1, s1, f1, _ = H.mle_evaluate(o, tau, K_RANK, SEED, y, empty, empty)
    ll2, s2, f2, _ = H.mle_evaluate(o, tau, K_RANK, SEED, y, empty, empty)
    assert ll1 == ll2 and np.array_equal(s1, s2) and np.array_equal(f1, f2)
    assert np.array_equal(f1, f1.T)
    fl = H.factorize(h, H.LEFT)
    a = fl.solve(y)
    for j in range(2):
        ref = 0.5 * (a @ d[j].matvec(a)) - 0.5 * H.trace_solve(fl, d[j])
        assert abs(s1[j] - ref) <= 1e-9 * abs(ref), (j, s1[j], ref)


def test_c4_fisher_and_score_bounds(c4):
    """With K = sigma^2 C + eta I and dK/dsigma^2 = C (eta not differentiated):
    F_ss = 1/2 sum (l/(l+eta))^2 in [0, n/(2 sigma^4)] and score_s2 >=
    -n/(2 sigma^2) (the quadratic term is a PSD form). The derivative block
    errors of the reference's q2 basis broke both at n = 2^20 (F_ss = 1.04e6,
    score_s2 = -5.7e8). F_ss is a few hundred left after cancelling traces of
    size n/2 at cond(K) ~ 1e11: even with dK/dsigma^2 replaced by exactly
    H - eta I the pipeline's F_ss lands anywhere in about +-0.7% of n/2
    (profiles/r2_c4_parity.md §6), so the bound is asserted to 1% of n/2; the
    score bound holds with a margin of 1e2."""
    H, o, tau, h, d = c4
    y = np.random.default_rng(1).standard_normal(N)
    fl = H.factorize(h, H.LEFT)
    s, f = H.score(fl, d, y), H.fisher_information(fl, d)
    assert -0.01 * N / 2 <= f[0, 0] <= 1.01 * N / 2, f
    assert s[0] >= -N / 2, s
    assert f[1, 1] >= 0.0, f


def test_c4_sigma2_derivative_consistent_with_h(c4):
    """sigma^2 = 1: dK/dsigma^2 = K - eta I exactly, so the derivative HODLR
    must agree with H - eta I far below the nugget (eta = 1e-6), or every
    sigma^2 quantity inherits the difference amplified by ||K^-1|| = 1/eta.
    Also the HODLR approximation error itself, against the exact (scan)
    forward model, stays far below the nugget."""
    H, o, tau, h, d = c4
    V = np.asfortranarray(np.random.default_rng(9).standard_normal((N, 4)))
    HV, DV, KV = h.matvec(V), d[0].matvec(V), o.apply(V)
    nv = np.linalg.norm(V, axis=0)
    e_d = np.linalg.norm(DV - (HV - 1e-6 * V), axis=0) / nv
    e_h = np.linalg.norm(HV - KV, axis=0) / nv
    assert e_d.max() <= 1e-8 and e_h.max() <= 1e-8, (e_d, e_h)


def test_c4_settings_agree_with_oracle_and_dense_at_2_14():
    """The C4 settings at n = 2^14 (the largest size the CPU oracle runs in
    seconds): device iteration against the restated oracle in the device's
    modes (solve association, q2 re-orthogonalised) and the dense FP64 truth.
    F_ss = n/2 - (cancelling traces of size n/2), so its tolerance is
    absolute in units of n/2 (1e-4); loglik 2e-9 (y^T K^-1 y ~ 1e10 carries
    the HODLR approximation at cond(K) ~ 1e10: the oracle's own loglik is
    8e-10 from the dense truth); score 1e-6; F_sl, F_ll 1e-4 relative."""
    import torch

    from oracle import pyoracle as O
    from paper_2303_10102_b200 import hodlrgp as H

    n = 1 << 14
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    y = np.random.default_rng(1).standard_normal(n)
    tau = H.tree_depth(n, 128, 256)
    ll1, s1, f1, _ = H.mle_iteration(H.MaternOracle(x, 5, 1.0, 0.05, 1e-6, True), tau, K_RANK, SEED, y)
    O.device_defaults(True)
    try:
        ll0, s0, f0, _ = O.mle_iteration(O.CovOracle.matern(x, 5, 1.0, 0.05, 1e-6, True), tau, K_RANK, SEED, y, 2)
    finally:
        O.device_defaults(False)
    # dense truth (torch FP64 on the GPU)
    xt = torch.tensor(x, dtype=torch.float64, device="cuda")
    a = (xt[:, None] - xt[None, :]).abs_().mul_(np.sqrt(5.0) / 0.05)
    e = torch.exp(-a)
    D = [(1 + a + a * a / 3) * e, a * a * (1 + a) / 3 * e / 0.05]
    del a, e
    Kd = D[0].clone()
    Kd.diagonal().add_(1e-6)
    L = torch.linalg.cholesky(Kd)
    del Kd
    yt = torch.tensor(y, dtype=torch.float64, device="cuda")[:, None]
    w = torch.cholesky_solve(yt, L)
    ll2 = (-0.5 * n * np.log(2 * np.pi) - torch.log(L.diagonal()).sum() - 0.5 * (yt * w).sum()).item()
    M = [torch.linalg.solve_triangular(L, torch.linalg.solve_triangular(L, Dj, upper=False).mT, upper=False)
         for Dj in D]
    s2 = np.array([(-0.5 * M[j].diagonal().sum() + 0.5 * (w * (D[j] @ w)).sum()).item() for j in range(2)])
    f2 = np.array([[0.5 * (M[i] * M[j]).sum().item() for j in range(2)] for i in range(2)])
    for ref in ((ll0, s0, f0), (ll2, s2, f2)):
        assert abs(ll1 - ref[0]) <= 2e-9 * abs(ref[0]), (ll1, ref[0])
        assert np.all(np.abs(s1 - ref[1]) <= 1e-6 * np.abs(ref[1])), (s1, ref[1])
        assert abs(f1[0, 0] - ref[2][0, 0]) <= 1e-4 * n / 2, (f1, ref[2])
        assert np.all(np.abs(f1 - ref[2])[1:, :].ravel() <= 1e-4 * np.abs(ref[2])[1:, :].ravel()), (f1, ref[2])
