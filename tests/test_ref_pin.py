"""Pin the parity oracle to the reference ITSELF (CPU only).

oracle/_ref/libhodlrgp_ref.so is /root/reference/proj/src/*.cpp compiled
unmodified against the restated Eigen-API shim (oracle/eigen_shim, recipe
oracle/ref.mk); oracle/_ref/ref_unit_tests is the reference's own doctest
suites (proj/tests/test_{cluster_tree,hodlr_matrix,sketch,factorization,
product_rep,mle}.cpp, unmodified) linked against it. These tests check
  1. the reference's own 45 test cases pass on that build (pins the shim), and
  2. the restated oracle (oracle/hodlr.cpp, used where the reference exposes
     no hook: decision logs, the solve association) equals the reference:
     bit-exact on trees, KD order, sketch plans, test fixtures, logdet and
     traces of the fixtures; 1e-13 on built HODLRs; the C1 iteration within the
     reference association's own roundoff spread.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref as R

HERE = os.path.dirname(os.path.abspath(__file__))
REF_TESTS = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_unit_tests")

pytestmark = pytest.mark.skipif(not R.available() and not os.path.isdir("/root/reference"),
                                reason="oracle/_ref not built and /root/reference absent")


def _ensure_built():
    if not R.available() or not os.path.exists(REF_TESTS):
        R.build()


def test_reference_unit_suites_pass_on_the_shim_build():
    _ensure_built()
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    last = r.stdout.strip().splitlines()[-1]
    assert last.startswith("test cases: 45 | 45 passed | 0 failed"), last


def test_library_is_the_reference():
    _ensure_built()
    assert R.IS_REFERENCE and not O.IS_REFERENCE
    assert R.lib().or_is_reference() == 1


@pytest.mark.parametrize("n,lmin,lmax", [(100, 32, 128), (1024, 128, 256), (4096, 64, 128), (1 << 20, 128, 256),
                                         (130, 64, 128), (77, 8, 16)])
def test_tree_bitwise(n, lmin, lmax):
    tau = R.tree_depth(n, lmin, lmax)
    assert O.tree_depth(n, lmin, lmax) == tau
    if n <= 1 << 16:
        assert R.tree_ranges(n, tau) == O.tree_ranges(n, tau)


@pytest.mark.parametrize("d", [1, 2])
def test_kd_ordering_bitwise(d):
    pts = np.random.default_rng(3).uniform(-1, 1, size=(777, d))
    a, b = R.kd_ordering(pts, 16, 32), O.kd_ordering(pts, 16, 32)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


@pytest.mark.parametrize("n,tau,k,seed", [(64, 2, 3, 99), (1000, 3, 8, 7), (4096, 6, 24, 0)])
def test_sketch_plan_bitwise(n, tau, k, seed):
    for l in range(0, tau + 1):
        assert np.array_equal(R.sketch_sampler(n, tau, k, seed, l), O.sketch_sampler(n, tau, k, seed, l))


@pytest.mark.parametrize("n,tau,k,seed", [(512, 3, 8, 100), (300, 3, 5, 9), (176, 3, 5, 3)])
def test_fixtures_factor_and_traces_bitwise(n, tau, k, seed):
    ar, br = R.Hodlr.random_spd(n, tau, k, seed), R.Hodlr.random_symmetric(n, tau, k, seed + 1)
    ao, bo = O.Hodlr.random_spd(n, tau, k, seed), O.Hodlr.random_symmetric(n, tau, k, seed + 1)
    assert np.array_equal(ar.densify(), ao.densify()) and np.array_equal(br.densify(), bo.densify())
    fr, fo = R.factorize(ar, 1), O.factorize(ao, 1)
    assert fr.logdet() == fo.logdet()
    assert R.trace_solve(fr, br) == O.trace_solve(fo, bo)
    assert R.trace_quad(fr, br, fr, br) == O.trace_quad(fo, bo, fo, bo)
    x = O.randn(n, 3, 5)
    assert np.array_equal(fr.solve(x), fo.solve(x))


def test_hutchinson_trace_bitwise():  # mle.cpp:56-75 (same libstdc++ Rademacher stream, same solves)
    ar, br = R.Hodlr.random_spd(256, 3, 4, 5), R.Hodlr.random_spd(256, 3, 4, 6)
    ao, bo = O.Hodlr.random_spd(256, 3, 4, 5), O.Hodlr.random_spd(256, 3, 4, 6)
    er, sr = R.hutchinson_trace(R.factorize(ar, 1), br, 400, 17)
    eo, so = O.hutchinson_trace(O.factorize(ao, 1), bo, 400, 17)
    assert er == eo and sr == pytest.approx(so, rel=1e-10)


@pytest.mark.parametrize("scan", [False, True])
def test_build_matches_reference(scan):
    n = 512
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    br = R.Build(R.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, scan), 3, 24, 0, True, 2)
    bo = O.Build(O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, scan), 3, 24, 0, True, 2)
    for a, b in [(br.h(), bo.h()), (br.deriv(0), bo.deriv(0)), (br.deriv(1), bo.deriv(1))]:
        assert a.info()[3] == b.info()[3]  # per-level ranks
        da, db = a.densify(), b.densify()
        assert np.linalg.norm(da - db) <= 1e-13 * np.linalg.norm(da)


def test_c1_iteration_matches_reference():
    """Config C1 in full through the reference and the restatement (reference
    association in both). loglik agrees to 1e-10; score and Fisher only to the
    reference association's own roundoff spread (~1e-4 at C1's cond(K) ~ 1e7,
    DESIGN.md §4): two executions of the same algorithm, differing only in
    the dense kernels' summation order."""
    n = 4096
    x = np.sort(np.random.default_rng(0).uniform(size=n))
    y = np.random.default_rng(1).standard_normal(n)
    tau = O.tree_depth(n, 64, 128)
    llr, sr, fr, _ = R.mle_iteration(R.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, True), tau, 24, 0, y, 2)
    llo, so, fo, _ = O.mle_iteration(O.CovOracle.matern(x, 3, 1.0, 0.2, 1e-4, True), tau, 24, 0, y, 2)
    assert abs(llr - llo) <= 1e-10 * abs(llr)
    assert np.allclose(so, sr, rtol=1e-6, atol=0)
    assert np.allclose(fo, fr, rtol=1e-4, atol=0)
