"""C++ drop-in (include/hodlrgp_b200.hpp): reference-style caller code,
compiled with g++ against the header, runs on the GPU and agrees with the
Python binding and the reference itself (oracle/_ref) on config C1."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _build():
    subprocess.run(["make", "-s", "-C", CPP], check=True)


def test_dropin_header_compiles_and_links():
    """CPU: the header compiles against the C ABI and links the product .so."""
    _build()
    out = subprocess.run(["nm", "-u", os.path.join(CPP, "test_dropin")], capture_output=True, text=True).stdout
    assert "hg_build" in out and "hg_fisher_information" in out and "hg_oracle_permuted" in out


@pytest.mark.gpu
def test_dropin_runs_c1_on_the_gpu():
    _build()
    r = subprocess.run([os.path.join(CPP, "test_dropin")], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["failures"] == 0
    from paper_2303_10102_b200 import hodlrgp as H

    x = np.fromfile(os.path.join(ROOT, "tests", "golden", "c1_x.bin"), dtype="<f8")
    y = np.fromfile(os.path.join(ROOT, "tests", "golden", "c1_y.bin"), dtype="<f8")
    tau = H.tree_depth(4096, 64, 128)
    ll, s, f, _ = H.mle_iteration(H.MaternOracle(x, 3, 1.0, 0.2, 1e-4, True), tau, 24, 0, y)
    # same library, same inputs, same call sequence: bitwise
    assert got["loglik"] == ll
    assert got["score"] == s.tolist()
    assert got["fisher"] == f.ravel(order="F").tolist()
    # the reference's oracle-column budget (sketch.hpp:69-71 plus the p k tau
    # applies of the differentiated pass, sketch.cpp:275-277)
    assert got["apply_columns"] == 2 * 24 * tau + 64 + 2 * 24 * tau
