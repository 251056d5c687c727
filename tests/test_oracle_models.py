"""CPU restatement of the configs' forward models (oracle/models.py): the
restatement's internal consistency, no GPU."""
import numpy as np
import pytest

from oracle import models as M


def test_cokriging_dense_is_spd_and_derivatives_match_fd():
    m, th = 24, (1.0, 0.1, 2.0)
    K, dK = M.cokriging_dense(m, *th)
    assert np.allclose(K, K.T) and np.linalg.eigvalsh(K).min() > 0
    for j in range(3):
        e = 1e-6 * th[j]
        tp, tm = list(th), list(th)
        tp[j] += e
        tm[j] -= e
        fd = (M.cokriging_dense(m, *tp)[0] - M.cokriging_dense(m, *tm)[0]) / (2 * e)
        assert np.linalg.norm(fd - dK[j]) <= 1e-6 * np.linalg.norm(dK[j])


def test_cokriging_blocks_follow_the_fd_operator():
    m, th = 16, (1.0, 0.1, 2.0)
    K, _ = M.cokriging_dense(m, *th, nugget=0.0)
    h = 1.0 / (m + 1)
    A = (np.diag(np.full(m, 2.0)) - np.diag(np.ones(m - 1), 1) - np.diag(np.ones(m - 1), -1)) / h**2 + 4.0 * np.eye(m)
    # cov(A u, f) = cov(f, f): A K_uf = K_ff
    assert np.allclose(A @ K[0::2, 1::2], K[1::2, 1::2], atol=1e-10)


@pytest.mark.parametrize("N", [8, 16])
def test_spde2d_dense_spectral_consistency(N):
    th = (1.0, 0.05, 4.0)
    order = np.random.default_rng(N).permutation(N * N)
    K, dK = M.spde2d_dense(N, *th, order)
    assert np.allclose(K, K.T)
    ex = M.spde2d_exact(N, *th, order=order)
    assert np.linalg.slogdet(K)[1] == pytest.approx(ex["logdet"], rel=1e-10)
    Ki = np.linalg.inv(K)
    F = np.array([[0.5 * np.trace(Ki @ a @ Ki @ b) for b in dK] for a in dK])
    assert np.linalg.norm(F - ex["fisher"]) <= 1e-8 * np.linalg.norm(ex["fisher"])
    # derivatives against finite differences of the spectrum
    for j in range(3):
        e = 1e-6 * th[j]
        tp, tm = list(th), list(th)
        tp[j] += e
        tm[j] -= e
        nug = 10.0 * M.spde2d_variance(N, *th)
        fd = (M.spde2d_dense(N, *tp, order, nugget=nug)[0] - M.spde2d_dense(N, *tm, order, nugget=nug)[0]) / (2 * e)
        assert np.linalg.norm(fd - dK[j]) <= 1e-5 * np.linalg.norm(dK[j])


def test_spde2d_variance_is_the_diagonal():
    N, th = 16, (1.3, 0.07, 3.0)
    K, _ = M.spde2d_dense(N, *th, nugget=0.0)
    assert np.allclose(np.diag(K), M.spde2d_variance(N, *th))
