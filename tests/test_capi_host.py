"""CPU-only checks of the product library (no GPU calls).

- every entry point declared in include/hodlrgp_b200.h is exported by the
  built library (the drop-in boundary);
- the host-side cluster-tree logic behind the C ABI is bit-exact with the
  reference (tree_depth known answers, test_cluster_tree.cpp:31-37) and with
  the oracle (ranges, KD ordering).
"""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hodlrgp_b200.h")


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    hodlrgp.lib()
    return hodlrgp


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["hg_factorize", "hg_factor_solve", "hg_factor_logdet", "hg_hodlr_matvec", "hg_trace_quad",
              "hg_solve_multiply", "hg_build", "hg_mle_iteration", "hg_fisher_information"]:
        assert s in syms


def test_library_exports_every_declared_symbol(H):
    lib = H.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only(H):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", H.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_tree_depth_known_answers(H):  # test_cluster_tree.cpp:31-37
    assert H.tree_depth(100, 32, 128) == 0
    assert H.tree_depth(1024, 128, 256) == 3
    assert H.tree_depth(512, 32, 64) == 4
    assert H.tree_depth(8192, 32, 64) == 8
    assert H.tree_depth(130, 64, 128) == 1
    assert H.tree_depth(1 << 20, 128, 256) == 13  # C4
    assert H.tree_depth(4096, 64, 128) == 6  # C1


@pytest.mark.parametrize("n,tau", [(100, 3), (11, 1), (77, 2), (4096, 6), (1 << 20, 13), (12345, 7)])
def test_tree_ranges_bit_exact(H, n, tau):
    t = H.ClusterTree(n, tau)
    ref = O.tree_ranges(n, tau)
    for d in range(tau + 1):
        assert t.level(d) == ref[d]


@pytest.mark.parametrize("n,d,lmin,lmax,seed", [(37, 2, 4, 8, 3), (129, 1, 16, 32, 9), (5000, 2, 64, 128, 1)])
def test_kd_ordering_bit_exact(H, n, d, lmin, lmax, seed):
    pts = np.random.default_rng(seed).uniform(-1, 1, size=(n, d))
    perm, inv, tree = H.build_kd_ordering(pts, lmin, lmax)
    p0, i0, tau0 = O.kd_ordering(pts, lmin, lmax)
    assert np.array_equal(perm, p0) and np.array_equal(inv, i0) and tree.tau == tau0


def test_invalid_arguments_map_to_exceptions(H):
    with pytest.raises(ValueError):
        H.build_kd_ordering(np.zeros((0, 2)), 4, 8)
    with pytest.raises(ValueError):
        H.build_kd_ordering(np.zeros((10, 3)), 4, 8)
