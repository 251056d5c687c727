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


def test_device_sketch_rng(H):
    """HG_OPT_SKETCH_RNG = HG_SKETCH_RNG_DEVICE: counter-based Gaussian samplers generated on
    the device with the reference's sparsity pattern (sketch.cpp:12-24: N(0,1) on right-child
    rows, zero on left-child rows); not the reference's bytes. The build stays exact."""
    n, tau, k = 4096, 4, 24
    ctx = H.context()
    ctx.set_option(H.OPT_SKETCH_RNG, H.SKETCH_RNG_DEVICE)
    try:
        tree = H.ClusterTree(n, tau)
        for level in (1, 3, tau):
            a = H.sketch_sampler(n, tau, k, 5, level)
            assert np.array_equal(a, H.sketch_sampler(n, tau, k, 5, level))       # deterministic
            assert not np.array_equal(a, H.sketch_sampler(n, tau, k, 6, level))  # seeded
            assert not np.array_equal(a, O.sketch_sampler(n, tau, k, 5, level))  # not the host stream
            right = np.zeros(n, bool)
            for j, (lo, hi) in enumerate(tree.level(level)):
                right[lo:hi] = j & 1
            assert np.all(a[~right] == 0.0)
            g = a[right]
            assert abs(g.mean()) < 0.02 and abs(g.std() - 1.0) < 0.02 and abs((g ** 4).mean() - 3.0) < 0.2
            # neighbouring rows / columns uncorrelated (>= 2047 x 23 pairs: sigma <= 0.005)
            assert abs(np.corrcoef(g[:-1].ravel(), g[1:].ravel())[0, 1]) < 0.025
            assert abs(np.corrcoef(g[:, :-1].ravel(), g[:, 1:].ravel())[0, 1]) < 0.025
        assert np.array_equal(H.sketch_sampler(n, tau, k, 5, 0), O.sketch_sampler(n, tau, k, 5, 0))  # identity stacks
        x = np.sort(np.random.default_rng(0).uniform(size=n))
        o = H.MaternOracle(x, 3, 1.0, 0.2, 1e-4, False)
        K = o.apply(np.eye(n))
        br = H.build_hodlr_with_derivatives(o, tree, k, 5)
        assert np.linalg.norm(br.h.densify() - K) <= 1e-9 * np.linalg.norm(K)
        y = np.linalg.cholesky(K) @ O.randn(n, 1, 1)[:, 0]
        ll1, s1, f1, _ = H.mle_iteration(o, tau, k, 5, y)
    finally:
        ctx.set_option(H.OPT_SKETCH_RNG, H.SKETCH_RNG_REFERENCE)
    ll0, s0, f0, _ = H.mle_iteration(o, tau, k, 5, y)
    assert ll1 == pytest.approx(ll0, rel=1e-8)
    assert np.allclose(s1, s0, rtol=1e-5, atol=1e-6 * np.abs(s0).max()) and np.allclose(f1, f0, rtol=1e-5)


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


def test_cluster_qr_bitwise_equals_single_cta(H, tmp_path):
    """The thread-block-cluster pivoted QR (qr_cluster.cuh) performs the same operations in the
    same order as the one-CTA kernel: with HG_QR_CLUSTER=0 (read once per process, hence the
    subprocess) the range finder returns bitwise the same q, r, pivots and numeric rank
    whenever only the pivoted kernel is swapped."""
    import os
    import subprocess
    import sys

    mats = {f"m{i}": y for i, y in enumerate(_blocks()[4:])}
    g = np.random.default_rng(3)
    mats["m3"] = g.standard_normal((400, 128)) * np.logspace(0, -9, 128)
    mats["m4"] = g.standard_normal((180, 100))
    np.savez(tmp_path / "in.npz", **mats)
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.')\n"
        "from paper_2303_10102_b200 import hodlrgp as H\n"
        f"d = np.load(r'{tmp_path / 'in.npz'}'); out = {{}}\n"
        "for k in d.files:\n"
        "    q, r, p, nr = H.randomized_range(d[k], d[k].shape[1])\n"
        "    out[k + '_q'], out[k + '_r'], out[k + '_p'], out[k + '_n'] = q, r, p, np.array(nr)\n"
        f"np.savez(r'{tmp_path / 'out.npz'}', **out)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, env=dict(os.environ, HG_QR_CLUSTER="0"))
    ref = np.load(tmp_path / "out.npz")
    for k, y in mats.items():
        q, r, p, nr = H.randomized_range(y, y.shape[1])
        assert nr == int(ref[k + "_n"]) and np.array_equal(p[:nr], ref[k + "_p"][:nr]), k
        if y.shape[1] < 128 or y.shape[0] <= 4 * y.shape[1]:
            assert np.array_equal(r, ref[k + "_r"]) and np.array_equal(q, ref[k + "_q"]), k
        else:
            # TSQR chunks of >= 128 columns: the unpivoted cluster kernel replaces the blocked
            # compact-WY kernel (same reflectors in exact arithmetic, another summation order)
            assert np.linalg.norm(r - ref[k + "_r"]) <= 1e-12 * np.linalg.norm(r), k
            assert np.linalg.norm(q[:, :nr] - ref[k + "_q"][:, :nr]) <= 1e-10 * np.sqrt(nr), k
