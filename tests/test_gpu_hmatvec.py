"""GPU parity of the streaming narrow-block H-matvec (csrc/hmatvec.cu, s <= 4)
against the CPU oracle's HodlrMatrix::matvec (hodlr_matrix.cpp:198-226) and
against the wide-block path (s >= 5) on the same matrices.

Covers the path's own structure: one- and two-tier partial folds (children
wider than 32 leaves), 2 rows per thread (leaves > 128), ranks above one
register block and past the path's 256 limit (fallback), asymmetric storage,
sub-matvecs (levels d+1..tau), bitwise column independence and run-to-run
determinism.
"""
import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    return hodlrgp


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,tau,k", [(65536, 9, 8), (2000, 3, 12), (3001, 4, 70), (4096, 3, 300), (5, 2, 1),
                                     (1 << 14, 7, 40), (256, 1, 6), (512, 2, 10), (1000, 3, 9)])
def test_narrow_matches_oracle_and_wide(H, n, tau, k):
    oh = O.Hodlr.random_spd(n, tau, k, 11)
    dh = H.HodlrMatrix.from_panels(oh.export_panels())
    X = O.randn(n, 5, 12)
    wide = dh.matvec(X)  # s = 5: tensor-core path
    ref = oh.matvec(X)
    assert rel(wide, ref) <= 1e-13
    for s in (1, 2, 3, 4):
        y = dh.matvec(np.asfortranarray(X[:, :s]))
        assert rel(y, ref[:, :s]) <= 1e-13, s
        assert rel(y, wide[:, :s]) <= 1e-13, s


def test_narrow_columns_bitwise_and_deterministic(H):
    n, tau = 1 << 15, 8
    oh = O.Hodlr.random_spd(n, tau, 24, 3)
    dh = H.HodlrMatrix.from_panels(oh.export_panels())
    X = O.randn(n, 4, 4)
    Y4 = dh.matvec(X)
    for c in range(4):
        assert np.array_equal(dh.matvec(X[:, c]), Y4[:, c])
    Y2 = dh.matvec(np.asfortranarray(X[:, 1:3]))
    assert np.array_equal(Y2, Y4[:, 1:3])
    for _ in range(3):
        assert np.array_equal(dh.matvec(X), Y4)


def test_narrow_asymmetric_and_sub_matvec(H):
    n, tau = 512, 3
    a = O.randn(n, n, 21)
    a = a @ a.T / n + np.eye(n)
    oh = O.Hodlr.from_dense(tau, a, False)
    dh = H.HodlrMatrix.from_panels(oh.export_panels())
    dense = oh.densify()
    for s in (1, 3):
        x = O.randn(n, s, 30 + s)
        assert rel(dh.matvec(x), dense @ x) <= 1e-12
    for d in range(tau + 1):
        lv = O.tree_ranges(n, tau)[d]
        node = (1 << d) - 1
        lo, hi = lv[node]
        xs = O.randn(hi - lo, 2, 40 + d)
        sub = dense[lo:hi, lo:hi]
        assert rel(dh.sub_matvec(d, node, xs), sub @ xs) <= 1e-12
