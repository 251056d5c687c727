"""GPU parity: HODLR container, matvec family and traces vs the CPU oracle.

Inputs are generated once by the oracle (identical bytes) and imported into
the device library through the C ABI. Tolerances follow the reference tests
(test_hodlr_matrix.cpp) and north_star (1e-9 traces).
"""
import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    return hodlrgp


def to_dev(H, oh):
    return H.HodlrMatrix.from_panels(oh.export_panels())


@pytest.mark.parametrize("n,tau,k", [(61, 3, 5), (77, 2, 4), (256, 3, 4), (4096, 6, 24), (1000, 4, 16)])
def test_roundtrip_and_matvec(H, n, tau, k):
    oh = O.Hodlr.random_spd(n, tau, k, 7)
    dh = to_dev(H, oh)
    p0, p1 = oh.export_panels(), dh.export_panels()
    assert np.array_equal(p0["flat"], p1["flat"])
    x = O.randn(n, 7, 3)
    y0, y1 = oh.matvec(x), dh.matvec(x)
    assert np.linalg.norm(y1 - y0) <= 1e-13 * np.linalg.norm(y0)
    v = x[:, 0]
    assert np.linalg.norm(dh.matvec(v) - oh.matvec(v)) <= 1e-13 * np.linalg.norm(oh.matvec(v))


def test_matvec_asymmetric_dense(H):
    a = O.randn(64, 64, 5)
    oh = O.Hodlr.from_dense(3, a, False)
    dh = to_dev(H, oh)
    x = O.randn(64, 3, 8)
    assert np.linalg.norm(dh.matvec(x) - a @ x) <= 1e-11 * np.linalg.norm(a @ x)
    for d in range(4):
        lv = O.tree_ranges(64, 3)[d]
        for node in range(2 ** d):
            lo, hi = lv[node]
            xs = O.randn(hi - lo, 3, 100 + d)
            sub = a[lo:hi, lo:hi]
            assert np.linalg.norm(dh.sub_matvec(d, node, xs) - sub @ xs) <= 1e-11 * np.linalg.norm(xs)
            assert np.linalg.norm(dh.sub_matvec(d, node, xs, True) - sub.T @ xs) <= 1e-11 * np.linalg.norm(xs)


def test_random_spd_matches_oracle(H):
    t = H.ClusterTree(144, 3)
    dh = H.HodlrMatrix.random_spd(t, 5, 2)
    oh = O.Hodlr.random_spd(144, 3, 5, 2)
    a0, a1 = oh.densify(), dh.densify()
    assert np.linalg.norm(a1 - a0) <= 1e-14 * np.linalg.norm(a0)


@pytest.mark.parametrize("n,tau,k", [(80, 3, 4), (2048, 5, 16)])
def test_trace_and_trace_product(H, n, tau, k):
    oa = O.Hodlr.random_spd(n, tau, k, 21)
    ob = O.Hodlr.random_symmetric(n, tau, k, 22)
    da, db = to_dev(H, oa), to_dev(H, ob)
    assert da.trace() == pytest.approx(oa.trace(), rel=1e-13)
    t0 = O.trace_product(oa, ob)
    assert H.trace_product(da, db) == pytest.approx(t0, rel=1e-12)
    oa.make_asymmetric()
    da2 = to_dev(H, oa)
    assert H.trace_product(da2, db) == pytest.approx(t0, rel=1e-12)
