"""Sketching entry points of the drop-in boundary (sketch.hpp:17-66) on the
device vs the CPU oracle: SketchPlan sampler bytes (bit-exact),
randomized_range (pivot order, numeric rank identical; q, r 1e-12) and diff_qr
(1e-10), including rank-deficient blocks (completion) and the TSQR path."""
import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    return hodlrgp


@pytest.mark.parametrize("n,tau,k,seed", [(1000, 4, 12, 3), (4096, 6, 24, 0)])
def test_sketch_sampler_bit_exact(H, n, tau, k, seed):
    for level in range(tau + 1):
        a = H.sketch_sampler(n, tau, k, seed, level)
        b = O.sketch_sampler(n, tau, k, seed, level)
        assert np.array_equal(a, b), level


def _blocks():
    g = np.random.default_rng(11)
    full = g.standard_normal((300, 24))
    low = g.standard_normal((300, 5)) @ g.standard_normal((5, 24))  # numeric rank 5 -> completion
    tall = g.standard_normal((5000, 40)) * np.logspace(0, -6, 40)   # TSQR chunks, graded columns
    wide = g.standard_normal((2100, 64))                             # blocked-QR chunks
    # widths above 64, one block: the thread-block-cluster pivoted QR (qr_cluster.cuh), resident and
    # as the root of a TSQR tree, graded columns and a numerically rank-deficient block
    c96 = g.standard_normal((700, 96)) * np.logspace(0, -5, 96)
    c128 = g.standard_normal((6000, 128)) * np.logspace(0, -4, 128)
    clow = g.standard_normal((900, 7)) @ g.standard_normal((7, 80))
    return [full, low, tall, wide, c96, c128, clow]


@pytest.mark.parametrize("i", range(7))
def test_randomized_range_matches_oracle(H, i):
    y = _blocks()[i]
    k = y.shape[1]
    q1, r1, p1, nr1 = H.randomized_range(y, k)
    q0, r0, p0, nr0 = O.randomized_range(y, k)
    # pivots past the numeric rank are decided on noise (any platform may differ)
    assert nr1 == nr0 and np.array_equal(p1[:nr0], p0[:nr0])
    assert np.linalg.norm(q1.T @ q1 - np.eye(k)) <= 1e-12 * k
    assert np.linalg.norm(r1[:nr0, :nr0] - r0[:nr0, :nr0]) <= 1e-12 * np.linalg.norm(r0)
    # q r reproduces the permuted block (test_sketch.cpp:53-66)
    assert np.linalg.norm(q1 @ r1 - y[:, p1]) <= 1e-12 * np.linalg.norm(y)
    # the numerically significant part of the basis agrees
    assert np.linalg.norm(q1[:, :nr0] - q0[:, :nr0]) <= 1e-10 * np.sqrt(nr0)
    assert np.all(np.diag(r1) >= 0)


def test_diff_qr_matches_oracle(H):
    g = np.random.default_rng(5)
    b = g.standard_normal((500, 16))
    db = g.standard_normal((500, 16))
    q, r, _, _ = O.randomized_range(b, 16)
    out1 = H.diff_qr(db, q, r)
    out0 = O.diff_qr(db, q, r)
    for a, c in zip(out1[:3], out0[:3]):
        assert np.linalg.norm(a - c) <= 1e-10 * np.linalg.norm(c)
    assert out1[3] == out0[3]
    # ill-conditioned flag
    r2 = r.copy()
    r2[-1, -1] = 1e-13 * r2[0, 0]
    assert H.diff_qr(db, q, r2)[3] and O.diff_qr(db, q, r2)[3]
