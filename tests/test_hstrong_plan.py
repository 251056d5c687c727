"""Strong-admissibility block-cluster tree, host side, no GPU:
the C ABI's plan (csrc/hstrong.cu hs_plan) against the numpy restatement of
the eta-admissibility rule (oracle/hstrong.py), and the structural invariants
every eta-admissible partition of the grid must satisfy."""
import numpy as np
import pytest

from oracle import hstrong as R


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    hodlrgp.lib()
    return hodlrgp


@pytest.mark.parametrize("nside,leaf,k,eta", [(16, 16, 8, 1.0), (32, 32, 12, 1.0), (64, 64, 24, 1.0),
                                              (64, 64, 24, 0.5), (64, 64, 24, 2.0), (32, 64, 24, 1.0)])
def test_plan_matches_restatement(H, nside, leaf, k, eta):
    order, tree = H.grid_kd_order(nside, leaf)
    got = H.hstrong_plan(order, nside, tree.tau, eta, k)
    assert got == R.plan(order, nside, tree.tau, eta, k)


@pytest.mark.parametrize("nside,leaf,k", [(64, 64, 24), (256, 256, 42)])
def test_plan_covers_the_matrix_once(H, nside, leaf, k):
    """Upper-triangle blocks (t <= s, off-diagonal counted twice, diagonal
    leaves once) tile the n x n matrix exactly."""
    order, tree = H.grid_kd_order(nside, leaf)
    p = H.hstrong_plan(order, nside, tree.tau, 1.0, k)
    n = nside * nside
    nleaves = 2 ** tree.tau
    diag = nleaves * (n // nleaves) ** 2
    assert 2 * p["lowrank_entries"] + 2 * (p["dense_entries"] - diag) + diag == n * n


def test_plan_eta_monotone(H):
    """A larger eta admits more pairs: fewer dense entries."""
    order, tree = H.grid_kd_order(64, 64)
    de = [H.hstrong_plan(order, 64, tree.tau, eta, 24)["dense_entries"] for eta in (0.5, 1.0, 2.0, 4.0)]
    assert de == sorted(de, reverse=True) and de[0] > de[-1]


def test_plan_rejects_bad_input(H):
    order, tree = H.grid_kd_order(16, 16)
    dup = np.array(order, dtype=np.int64)
    dup[1] = dup[0]
    with pytest.raises(ValueError):
        H.hstrong_plan(dup, 16, tree.tau, 1.0, 8)  # not a permutation
    with pytest.raises(ValueError):
        H.hstrong_plan(order, 16, tree.tau, 0.0, 8)
    with pytest.raises(ValueError):
        H.hstrong_plan(order, 16, tree.tau, 1.0, 65)
