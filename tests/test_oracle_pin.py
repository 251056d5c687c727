"""Pin the parity oracle against the reference's own hot-path test suite.

The reference ships no golden vectors; its tests are dense
cross-checks at small n. Each test below restates one reference test case
(cited file:line) with the same inputs and tolerance, checked with numpy's
dense LAPACK — independent of the oracle's own kernels. Inputs the reference
draws with Eigen::MatrixXd::Random (std::rand) are replaced by seeded
mt19937_64 draws (SURVEY.md §4 porting note).
"""
import numpy as np
import pytest

from oracle import pyoracle as O

R = "/root/reference/proj/tests/"


def random_sym(n, seed):
    a = O.randn(n, n, seed)
    return 0.5 * (a + a.T)


# ------------------------------------------------ test_cluster_tree.cpp
def test_uniform_tree_partitions():  # test_cluster_tree.cpp:12-23
    lv = O.tree_ranges(100, 3)
    for d in range(4):
        assert len(lv[d]) == 2 ** d
        assert lv[d][0][0] == 0 and lv[d][-1][1] == 100
        for j in range(1, len(lv[d])):
            assert lv[d][j][0] == lv[d][j - 1][1]


def test_left_child_ceiling():  # test_cluster_tree.cpp:25-29
    lv = O.tree_ranges(11, 1)
    assert lv[1][0][1] - lv[1][0][0] == 6 and lv[1][1][1] - lv[1][1][0] == 5


def test_depth_rule():  # test_cluster_tree.cpp:31-37 (known-answer values)
    assert O.tree_depth(100, 32, 128) == 0
    assert O.tree_depth(1024, 128, 256) == 3
    assert O.tree_depth(512, 32, 64) == 4
    assert O.tree_depth(8192, 32, 64) == 8
    assert O.tree_depth(130, 64, 128) == 1


def test_kd_permutation_inverse():  # test_cluster_tree.cpp:39-60
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, size=(37, 2))
    perm, inv, tau = O.kd_ordering(pts, 4, 8)
    assert sorted(perm.tolist()) == list(range(37))
    assert all(inv[perm[i]] == i for i in range(37))


def test_kd_longest_axis():  # test_cluster_tree.cpp:62-74
    pts = np.array([[10.0 * i, float(i % 2)] for i in range(8)])
    perm, inv, tau = O.kd_ordering(pts, 2, 4)
    assert tau >= 1
    left = O.tree_ranges(8, tau)[1][0]
    for r in range(*left):
        assert pts[inv[r], 0] < 40.0


def test_kd_leaf_min():  # test_cluster_tree.cpp:76-83
    rng = np.random.default_rng(9)
    pts = rng.uniform(0, 1, size=(129, 1))
    perm, inv, tau = O.kd_ordering(pts, 16, 32)
    for lo, hi in O.tree_ranges(129, tau)[tau]:
        assert hi - lo >= 16


def test_kd_1d_sorted_is_identity():  # 1D sorted inputs (C1, C4) keep their order
    x = np.sort(np.random.default_rng(0).uniform(size=(256, 1)), axis=0)
    perm, inv, tau = O.kd_ordering(x, 32, 64)
    assert (perm == np.arange(256)).all()


# ------------------------------------------------ test_hodlr_matrix.cpp
def test_from_dense_roundtrip_sym():  # :24-29
    a = random_sym(70, 1)
    h = O.Hodlr.from_dense(3, a, True)
    assert np.linalg.norm(h.densify() - a) <= 1e-12 * np.linalg.norm(a)


def test_from_dense_roundtrip_asym():  # :31-40
    a = O.randn(64, 64, 2)
    h = O.Hodlr.from_dense(2, a, False)
    assert np.linalg.norm(h.densify() - a) <= 1e-12 * np.linalg.norm(a)


def test_matvec_dense():  # :42-50
    a = random_sym(61, 3)
    h = O.Hodlr.from_dense(3, a, True)
    x = random_sym(61, 4)[:, :5]
    assert np.linalg.norm(h.matvec(x) - a @ x) <= 1e-11 * np.linalg.norm(a @ x)
    v = x[:, 0]
    assert np.linalg.norm(h.matvec(v) - a @ v) <= 1e-11 * np.linalg.norm(a @ v)


def test_sub_matvec():  # :52-70
    a = O.randn(64, 64, 5)
    h = O.Hodlr.from_dense(3, a, False)
    lv = O.tree_ranges(64, 3)
    for d in range(4):
        for node in range(2 ** d):
            lo, hi = lv[d][node]
            sub = a[lo:hi, lo:hi]
            x = random_sym(hi - lo, 100 + d)[:, :3]
            assert np.linalg.norm(h.sub_matvec(d, node, x) - sub @ x) <= 1e-11 * np.linalg.norm(x)
            assert np.linalg.norm(h.sub_matvec(d, node, x, True) - sub.T @ x) <= 1e-11 * np.linalg.norm(x)


def test_random_spd():  # :72-79
    a = O.Hodlr.random_spd(96, 3, 5, 11).densify()
    assert np.linalg.norm(a - a.T) <= 1e-13 * np.linalg.norm(a)
    np.linalg.cholesky(a)


def test_symmetric_lower_is_transpose():  # :81-91
    h = O.Hodlr.random_spd(32, 2, 3, 7)
    before = h.densify()
    h.make_asymmetric()
    assert np.linalg.norm(h.densify() - before) <= 1e-14 * np.linalg.norm(before)


def test_trace_and_trace_product():  # :93-106
    ha = O.Hodlr.random_spd(80, 3, 4, 21)
    hb = O.Hodlr.random_symmetric(80, 3, 4, 22)
    a, b = ha.densify(), hb.densify()
    assert ha.trace() == pytest.approx(np.trace(a), rel=1e-12)
    assert O.trace_product(ha, hb) == pytest.approx(np.trace(a @ b), rel=1e-10)
    ha.make_asymmetric()
    assert O.trace_product(ha, hb) == pytest.approx(np.trace(a @ b), rel=1e-10)


def test_ragged_leaves():  # :108-114
    a = random_sym(77, 31)
    h = O.Hodlr.from_dense(2, a, True)
    v = np.linspace(-1, 1, 77)
    assert np.linalg.norm(h.matvec(v) - a @ v) <= 1e-11 * np.linalg.norm(a @ v)


def test_panel_export_import_roundtrip():
    h = O.Hodlr.random_spd(144, 3, 5, 2)
    h2 = O.Hodlr.import_panels(h.export_panels())
    assert np.array_equal(h.densify(), h2.densify())
    h.make_asymmetric()
    h3 = O.Hodlr.import_panels(h.export_panels())
    assert np.array_equal(h.densify(), h3.densify())


# ------------------------------------------------ test_factorization.cpp
def test_right_solve():  # :10-18
    h = O.Hodlr.random_spd(128, 3, 4, 1)
    a = h.densify()
    f = O.factorize(h, O.Factor.RIGHT)
    b = O.randn(128, 4, 901)
    x = f.solve(b)
    assert np.linalg.norm(a @ x - b) <= 1e-9 * np.linalg.norm(b)


def test_left_solve_ragged():  # :20-28
    h = O.Hodlr.random_spd(144, 3, 5, 2)
    a = h.densify()
    f = O.factorize(h, O.Factor.LEFT)
    b = O.randn(144, 1, 902)[:, 0]
    x = f.solve(b)
    assert np.linalg.norm(a @ x - b) <= 1e-9 * np.linalg.norm(b)


def test_logdet_both_orientations():  # :30-41
    h = O.Hodlr.random_spd(100, 2, 3, 3)
    exact = np.linalg.slogdet(h.densify())[1]
    for orient in (O.Factor.RIGHT, O.Factor.LEFT):
        assert O.factorize(h, orient).logdet() == pytest.approx(exact, rel=1e-10)


def test_logdet_rejects_negative_det():  # :76-83
    a = np.eye(32)
    a[0, 0] = -1.0
    h = O.Hodlr.from_dense(1, a, True)
    f = O.factorize(h)
    with pytest.raises(O.NotPositiveDefinite):
        f.logdet()


def test_depth0_dense():  # :85-96
    g = O.randn(20, 20, 903)
    a = g @ g.T + 20 * np.eye(20)
    h = O.Hodlr.from_dense(0, a, True)
    f = O.factorize(h)
    b = O.randn(20, 1, 904)[:, 0]
    assert np.linalg.norm(a @ f.solve(b) - b) <= 1e-10 * np.linalg.norm(b)
    assert f.logdet() == pytest.approx(np.linalg.slogdet(a)[1], rel=1e-11)


# ------------------------------------------------ test_sketch.cpp
def test_plan_pattern():  # :24-51
    lv = O.tree_ranges(64, 2)
    for l in (1, 2):
        s = O.sketch_sampler(64, 2, 3, 99, l)
        assert s.shape == (64, 3)
        for j in range(2 ** (l - 1)):
            (a, b), (c, d) = lv[l][2 * j], lv[l][2 * j + 1]
            assert np.linalg.norm(s[a:b]) == 0.0
            assert np.linalg.norm(s[c:d]) > 0.0
    leaf = O.sketch_sampler(64, 2, 3, 99, 0)
    for lo, hi in lv[2]:
        assert np.array_equal(leaf[lo:hi, : hi - lo], np.eye(hi - lo))
    assert np.array_equal(O.sketch_sampler(64, 2, 3, 99, 1), O.sketch_sampler(64, 2, 3, 99, 1))


def test_randomized_range():  # :53-66
    y = O.randn(40, 6, 1)
    q, r, perm, nr = O.randomized_range(y, 6)
    assert nr == 6
    assert np.linalg.norm(q.T @ q - np.eye(6)) <= 1e-12
    yp = y[:, perm]
    assert np.linalg.norm(q @ r - yp) <= 1e-12 * np.linalg.norm(y)
    assert (np.diag(r) >= 0).all() and np.array_equal(np.tril(r, -1), np.zeros((6, 6)))
    # pivoting: first pivot is the largest-norm column (ColPivHouseholderQR)
    assert perm[0] == int(np.argmax(np.linalg.norm(y, axis=0)))


def test_randomized_range_completion():  # :68-77
    basis = O.randn(30, 2, 2)
    y = basis @ O.randn(2, 5, 3)
    q, r, perm, nr = O.randomized_range(y, 5)
    assert nr == 2
    assert np.linalg.norm(q.T @ q - np.eye(5)) <= 1e-10
    assert np.linalg.norm(q @ (q.T @ y) - y) <= 1e-10 * np.linalg.norm(y)


def test_diff_qr():  # :79-115
    b = O.randn(25, 5, 4)
    db = O.randn(25, 5, 5)
    q, r, perm, nr = O.randomized_range(b, 5)
    bp, dbp = b[:, perm], db[:, perm]
    dq, dqs, dr, ill = O.diff_qr(dbp, q, r)
    assert not ill
    assert np.linalg.norm(dq @ r + q @ dr - dbp) <= 1e-11 * np.linalg.norm(dbp)
    s = q.T @ dq
    assert np.linalg.norm(s + s.T) <= 1e-11
    assert np.array_equal(np.tril(dr, -1), np.zeros((5, 5)))
    h = 1e-6

    def qr_fixed(m):
        qq, rr = np.linalg.qr(m)
        sg = np.sign(np.diag(rr))
        return qq * sg, rr * sg[:, None]

    qp, rp = qr_fixed(bp + h * dbp)
    qm, rm = qr_fixed(bp - h * dbp)
    assert np.linalg.norm(dq - (qp - qm) / (2 * h)) <= 1e-5 * np.linalg.norm(dq)
    assert np.linalg.norm(dr - (rp - rm) / (2 * h)) <= 1e-5 * np.linalg.norm(dr)


def test_diff_qr_ill_conditioned():  # :117-124
    b = O.randn(20, 4, 6)
    q, r, perm, nr = O.randomized_range(b, 4)
    r = r.copy()
    r[3, 3] = r[0, 0] * 1e-14
    assert O.diff_qr(O.randn(20, 4, 7), q, r)[3]


def test_peeling_exact_and_budget():  # :126-138
    src = O.Hodlr.random_spd(256, 3, 4, 10)
    a = src.densify()
    orc = O.CovOracle.dense(a)
    orc.counters(reset=True)
    b = O.Build(orc, 3, 4, 123, False)
    assert np.linalg.norm(b.h().densify() - a) <= 1e-11 * np.linalg.norm(a)
    assert orc.counters()[0] == 2 * 4 * 3 + 32


def test_peeling_smooth_kernel():  # :140-156
    n = 128
    x = np.linspace(0, 1, n)
    a = np.exp(-((x[:, None] - x[None, :]) ** 2) / (2 * 0.3 * 0.3)) + 1e-6 * np.eye(n)
    b = O.Build(O.CovOracle.dense(a), 2, 16, 5, False)
    assert np.linalg.norm(b.h().densify() - a) <= 1e-9 * np.linalg.norm(a)


def test_derivative_build_leaves_value_bitwise():  # :158-176
    kv = O.Hodlr.random_spd(192, 2, 5, 20)
    d0 = O.Hodlr.random_symmetric(192, 2, 5, 21)
    orc = O.CovOracle.dense(kv.densify(), [d0.densify()])
    plain = O.Build(orc, 2, 5, 42, False).h().export_panels()
    both = O.Build(orc, 2, 5, 42, True, p=1).h().export_panels()
    assert np.array_equal(plain["flat"], both["flat"])


def _compatible_derivative(kv, seed):
    """test_sketch.cpp:184-208: block derivatives x v^T + u z^T on the value factors."""
    p = kv.export_panels()
    n, tau = p["n"], p["tau"]
    lv = O.tree_ranges(n, tau)
    rng_state = np.random.default_rng(seed)
    d = np.zeros((n, n))
    off = 0
    for l in range(1, tau + 1):
        Rl = p["R"][l - 1]
        U = p["flat"][off: off + n * Rl].reshape((n, Rl), order="F")
        off += 2 * n * Rl
        for j in range(2 ** (l - 1)):
            (a, b), (c, e) = lv[l][2 * j], lv[l][2 * j + 1]
            left, right = U[a:b], U[c:e]
            x = rng_state.standard_normal(left.shape)
            z = rng_state.standard_normal(right.shape)
            blk = x @ right.T + left @ z.T
            d[a:b, c:e] = blk
            d[c:e, a:b] = blk.T
    for lo, hi in lv[tau]:
        m = rng_state.standard_normal((hi - lo, hi - lo))
        d[lo:hi, lo:hi] = 0.5 * (m + m.T)
    return d


def test_derivative_build_exact_recovery():  # :212-233
    kv = O.Hodlr.random_spd(256, 3, 4, 30)
    kd1 = _compatible_derivative(kv, 31)
    kd2 = _compatible_derivative(kv, 32)
    orc = O.CovOracle.dense(kv.densify(), [kd1, kd2])
    b = O.Build(orc, 3, 4, 77, True, p=2)
    kvd = kv.densify()
    assert np.linalg.norm(b.h().densify() - kvd) <= 1e-11 * np.linalg.norm(kvd)
    assert np.linalg.norm(b.deriv(0).densify() - kd1) <= 1e-10 * np.linalg.norm(kd1)
    assert np.linalg.norm(b.deriv(1).densify() - kd2) <= 1e-10 * np.linalg.norm(kd2)
    r10 = b.deriv(0).export_panels()["ranks_up"][0]
    assert 8 <= r10 <= 16


# ------------------------------------------------ test_product_rep.cpp
def test_multiply_exact():  # :10-22
    ha = O.Hodlr.random_spd(160, 3, 4, 1)
    hb = O.Hodlr.random_symmetric(160, 3, 4, 2)
    a, b = ha.densify(), hb.densify()
    p = O.multiply(O.factorize(ha, O.Factor.RIGHT), hb)
    assert np.linalg.norm(p.densify() - a @ b) <= 1e-10 * np.linalg.norm(a @ b)


def test_solve_multiply_exact_ragged():  # :24-33
    ha = O.Hodlr.random_spd(176, 3, 5, 3)
    hb = O.Hodlr.random_symmetric(176, 3, 5, 4)
    a, b = ha.densify(), hb.densify()
    p = O.solve_multiply(O.factorize(ha, O.Factor.LEFT), hb)
    exact = np.linalg.solve(a, b)
    assert np.linalg.norm(p.densify() - exact) <= 1e-9 * np.linalg.norm(exact)


def test_orientation_errors():  # :35-43
    ha = O.Hodlr.random_spd(64, 2, 3, 5)
    hb = O.Hodlr.random_symmetric(64, 2, 3, 6)
    with pytest.raises(ValueError):
        O.multiply(O.factorize(ha, O.Factor.LEFT), hb)
    with pytest.raises(ValueError):
        O.solve_multiply(O.factorize(ha, O.Factor.RIGHT), hb)


def test_trace_product_rep():  # :45-53
    ha = O.Hodlr.random_spd(128, 2, 4, 7)
    hb = O.Hodlr.random_symmetric(128, 2, 4, 8)
    a, b = ha.densify(), hb.densify()
    p = O.multiply(O.factorize(ha, O.Factor.RIGHT), hb)
    assert O.trace_product_rep(p) == pytest.approx(np.trace(a @ b), rel=1e-10)


def test_trace_solve():  # :55-64
    ha = O.Hodlr.random_spd(192, 3, 4, 9)
    hb = O.Hodlr.random_symmetric(192, 3, 4, 10)
    exact = np.trace(np.linalg.solve(ha.densify(), hb.densify()))
    assert O.trace_solve(O.factorize(ha, O.Factor.LEFT), hb) == pytest.approx(exact, rel=1e-10)


def test_trace_quad():  # :66-79
    ha = O.Hodlr.random_spd(160, 3, 4, 11)
    hb = O.Hodlr.random_symmetric(160, 3, 4, 12)
    hc = O.Hodlr.random_spd(160, 3, 4, 13)
    hd = O.Hodlr.random_symmetric(160, 3, 4, 14)
    exact = np.trace(np.linalg.solve(ha.densify(), hb.densify()) @ np.linalg.solve(hc.densify(), hd.densify()))
    fa, fc = O.factorize(ha, O.Factor.LEFT), O.factorize(hc, O.Factor.LEFT)
    assert O.trace_quad(fa, hb, fc, hd) == pytest.approx(exact, rel=1e-9)


def test_trace_quad_depth0():  # :81-91
    g = O.randn(24, 24, 905)
    a = g @ g.T + 24 * np.eye(24)
    b = random_sym(24, 906)
    ha, hb = O.Hodlr.from_dense(0, a), O.Hodlr.from_dense(0, b)
    m = np.linalg.solve(a, b)
    fa = O.factorize(ha, O.Factor.LEFT)
    assert O.trace_quad(fa, hb, fa, hb) == pytest.approx(np.trace(m @ m), rel=1e-10)


def test_acceptance_c1_sample():  # acceptance.cpp:54-80 (first 3 of 50 quadruples)
    n, k = 512, 8
    tau = O.tree_depth(n, 64, 128)
    for rep in range(3):
        s = 100 + 4 * rep
        ha = O.Hodlr.random_spd(n, tau, k, s)
        hb = O.Hodlr.random_symmetric(n, tau, k, s + 1)
        hc = O.Hodlr.random_spd(n, tau, k, s + 2)
        hd = O.Hodlr.random_symmetric(n, tau, k, s + 3)
        aib = np.linalg.solve(ha.densify(), hb.densify())
        fa, fc = O.factorize(ha, O.Factor.LEFT), O.factorize(hc, O.Factor.LEFT)
        ts = O.trace_solve(fa, hb)
        tq = O.trace_quad(fa, hb, fc, hd)
        assert abs(ts - np.trace(aib)) <= 1e-8 * abs(np.trace(aib))
        tq_exact = np.trace(aib @ np.linalg.solve(hc.densify(), hd.densify()))
        assert abs(tq - tq_exact) <= 1e-8 * abs(tq_exact)


# ------------------------------------------------ test_mle.cpp
def _family(n, seed):
    """test_mle.cpp:17-47 two-parameter dense SPD family (numpy RNG stand-in)."""
    g = np.random.default_rng(seed)

    def rnd(shift):
        m = g.standard_normal((n, n))
        s = m @ m.T / n
        return s + shift * np.eye(n)

    return rnd(4.0), rnd(1.0), rnd(1.0)


def test_mle_glue_dense():  # test_mle.cpp:53-84
    k0, d0, d1 = _family(96, 1)
    t = (0.7, 1.3)
    kk = k0 + t[0] * d0 + t[1] * d1
    h = O.Hodlr.from_dense(2, kk)
    der = [O.Hodlr.from_dense(2, d0), O.Hodlr.from_dense(2, d1)]
    f = O.factorize(h, O.Factor.LEFT)
    y = O.randn(96, 1, 907)[:, 0]
    sign, ld = np.linalg.slogdet(kk)
    w = np.linalg.solve(kk, y)
    ll = -0.5 * 96 * np.log(2 * np.pi) - 0.5 * ld - 0.5 * y @ w
    assert O.log_likelihood(f, y) == pytest.approx(ll, rel=1e-10)
    kinv = np.linalg.inv(kk)
    s = O.score(f, der, y)
    for j, dj in enumerate((d0, d1)):
        assert s[j] == pytest.approx(-0.5 * np.trace(kinv @ dj) + 0.5 * w @ dj @ w, rel=1e-9)
    fi = O.fisher_information(f, der)
    m0, m1 = kinv @ d0, kinv @ d1
    assert fi[0, 0] == pytest.approx(0.5 * np.trace(m0 @ m0), rel=1e-9)
    assert fi[0, 1] == pytest.approx(0.5 * np.trace(m0 @ m1), rel=1e-9)
    assert fi[1, 0] == fi[0, 1]
    assert fi[1, 1] == pytest.approx(0.5 * np.trace(m1 @ m1), rel=1e-9)
    fic = O.fisher_information(f, der, cache=True)
    assert np.array_equal(fi, fic)


def test_hutchinson_trace():  # test_mle.cpp:119-133
    ha, hb = O.Hodlr.random_spd(256, 3, 4, 5), O.Hodlr.random_spd(256, 3, 4, 6)
    f = O.factorize(ha, O.Factor.LEFT)
    exact = O.trace_solve(f, hb)
    e, se = O.hutchinson_trace(f, hb, 400, 17)
    assert se > 0.0 and abs(e - exact) <= 4.0 * se
    e4, se4 = O.hutchinson_trace(f, hb, 1600, 17)
    assert se4 <= 0.6 * se
    assert O.hutchinson_trace(f, hb, 400, 17) == (e, se)
    with pytest.raises(ValueError):
        O.hutchinson_trace(f, hb, 1, 17)


def test_mle_nonzero_mean():  # test_mle.cpp:107-118
    k0, d0, d1 = _family(64, 3)
    kk = k0 + d0 + d1
    f = O.factorize(O.Hodlr.from_dense(2, kk), O.Factor.LEFT)
    y = O.randn(64, 1, 908)[:, 0]
    mu = np.full(64, 0.37)
    r = y - mu
    ll = -0.5 * 64 * np.log(2 * np.pi) - 0.5 * np.linalg.slogdet(kk)[1] - 0.5 * r @ np.linalg.solve(kk, r)
    assert O.log_likelihood(f, y, mu) == pytest.approx(ll, rel=1e-10)


# ------------------------------------------------ Matérn forward models
@pytest.mark.parametrize("nu2", [1, 3, 5])
def test_matern_scan_equals_dense(nu2):
    x = np.sort(np.random.default_rng(0).uniform(size=300))
    v = O.randn(300, 4, 5)
    for which in (-1, 0, 1):
        a = O.CovOracle.matern(x, nu2, 1.3, 0.2, 1e-4, False).apply(v, which)
        b = O.CovOracle.matern(x, nu2, 1.3, 0.2, 1e-4, True).apply(v, which)
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)


@pytest.mark.parametrize("nu2", [1, 3, 5])
def test_matern_derivatives_fd(nu2):
    x = np.sort(np.random.default_rng(1).uniform(size=64))
    v = O.randn(64, 2, 6)
    s2, ell, h = 1.3, 0.2, 1e-6
    d_s = (O.CovOracle.matern(x, nu2, s2 + h, ell, 0, False).apply(v)
           - O.CovOracle.matern(x, nu2, s2 - h, ell, 0, False).apply(v)) / (2 * h)
    d_l = (O.CovOracle.matern(x, nu2, s2, ell + h, 0, False).apply(v)
           - O.CovOracle.matern(x, nu2, s2, ell - h, 0, False).apply(v)) / (2 * h)
    o = O.CovOracle.matern(x, nu2, s2, ell, 0, False)
    assert np.linalg.norm(o.apply(v, 0) - d_s) <= 1e-7 * np.linalg.norm(d_s)
    assert np.linalg.norm(o.apply(v, 1) - d_l) <= 1e-6 * np.linalg.norm(d_l)
