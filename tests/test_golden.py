"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py) pinned
against the CPU oracle, and the oracle's restatement of the debug serializer
(io.cpp:78-101, :171-275) checked on them. CPU only."""
import filecmp
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import serial as S

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(G, "golden.json")))


def sidecar(name):
    raw = open(os.path.join(G, name), "rb").read()
    return np.frombuffer(raw, dtype="<f8").astype(np.float64)


def load(name):
    return O.Hodlr.import_panels(S.read_hodlr_debug(G, name))


def test_spd50_fixture_is_random_spd_bitwise():  # test_io.cpp:94
    p = O.Hodlr.random_spd(50, 2, 3, 4).export_panels()
    q = S.read_hodlr_debug(G, "spd50_sym")
    assert q["sym"] and q["n"] == 50 and q["tau"] == 2
    assert list(q["ranks_up"]) == list(p["ranks_up"])
    assert np.array_equal(load("spd50_sym").densify(), O.Hodlr.import_panels(p).densify())


def test_spd50_results():
    g = GOLD["spd50_sym"]
    h = load("spd50_sym")
    f = O.factorize(h, 1)
    assert h.trace() == g["trace"]
    assert f.logdet() == g["logdet"]
    assert np.array_equal(f.solve(O.randn(50, 1, 7)[:, 0]), np.array(g["solve"]))


def test_spd50_asym_differs_only_in_lower_block():  # test_io.cpp:100-106
    a, s = load("spd50_asym"), load("spd50_sym")
    assert not a.info()[2]
    da, ds = a.densify(), s.densify()
    lv = S.tree_ranges(50, 2)[1]
    (l0, l1), (r0, r1) = lv[0], lv[1]
    d = da - ds
    assert np.array_equal(d[l0:l1, :], np.zeros_like(d[l0:l1, :]))
    assert np.array_equal(d[r0:r1, r0:r1], np.zeros((r1 - r0, r1 - r0)))
    assert np.array_equal(d[r0:r1, l0:l1], ds[r0:r1, l0:l1])  # the lower block doubled
    assert a.trace() == GOLD["spd50_asym"]["trace"]


def test_sidecars_are_row_major_little_endian():  # io.cpp:78-87
    h = load("c1s_h").densify()
    man = json.load(open(os.path.join(G, "c1s_h.json")))
    for e in man["leaves"]:
        lo, hi = e["rows"]
        m = hi - lo
        assert np.array_equal(sidecar(e["file"]).reshape(m, m), h[lo:hi, lo:hi])
    for lev in man["upper"]:
        for e in lev["blocks"]:
            (r0, r1), (c0, c1), r = e["rows"], e["cols"], e["rank"]
            left = sidecar(e["left"]).reshape(r1 - r0, r)
            right = sidecar(e["right"]).reshape(c1 - c0, r)
            assert np.allclose(left @ right.T, h[r0:r1, c0:c1], rtol=0, atol=1e-15)


def test_manifest_schema():  # io.cpp:176-232
    man = json.load(open(os.path.join(G, "spd50_asym.json")))
    assert sorted(man) == ["depth", "leaves", "lower", "n", "symmetric", "upper"]
    assert [lev["level"] for lev in man["upper"]] == [1, 2]
    e = man["lower"][1]["blocks"][1]
    assert sorted(e) == ["cols", "left", "node", "rank", "right", "rows"]
    assert e["left"] == "spd50_asym_lo_l2_n1_left.bin" and e["node"] == 1
    lv = S.tree_ranges(50, 2)[2]
    assert e["rows"] == list(lv[3]) and e["cols"] == list(lv[2])  # lower: rows = right child
    assert "lower" not in json.load(open(os.path.join(G, "spd50_sym.json")))


@pytest.mark.parametrize("name", ["spd50_sym", "spd50_asym", "c1s_h", "c1s_d1"])
def test_oracle_serializer_roundtrip_byte_identical(tmp_path, name):
    p = S.read_hodlr_debug(G, name)
    S.write_hodlr_debug(str(tmp_path), name, p)
    files = [f for f in os.listdir(G) if f.startswith(name + "_") or f == name + ".json"]
    assert sorted(os.listdir(tmp_path)) == sorted(files)
    match, mismatch, errors = filecmp.cmpfiles(G, str(tmp_path), files, shallow=False)
    assert not mismatch and not errors


def test_serializer_errors(tmp_path):
    p = O.Hodlr.random_spd(50, 2, 3, 4).export_panels()
    S.write_hodlr_debug(str(tmp_path), "t", p)
    with pytest.raises(S.SerialError, match="cannot open manifest"):
        S.read_hodlr_debug(str(tmp_path), "missing")
    f = tmp_path / "t_leaf2.bin"
    f.write_bytes(f.read_bytes()[:-8])
    with pytest.raises(S.SerialError, match="truncated sidecar"):
        S.read_hodlr_debug(str(tmp_path), "t")
    f.write_bytes(b"\0" * (13 * 13 * 8 + 16))  # trailing bytes are ignored (io.cpp:89-101)
    S.read_hodlr_debug(str(tmp_path), "t")


def test_c1s_fixture_is_the_oracle_build():
    """The committed n = 512 build equals the oracle's on the stored points;
    per-block decisions bit-exact, densified H and dH/dtheta to 1e-13."""
    g = GOLD["c1s"]
    x = sidecar("c1s_x.bin")
    oo = O.CovOracle.matern(x, g["nu2"], g["sigma2"], g["ell"], g["nugget"], False)
    bd = O.Build(oo, g["depth"], g["k"], g["seed"], True, p=2)
    assert bd.decisions().tolist() == g["decisions"]
    for nm, m in (("c1s_h", bd.h()), ("c1s_d0", bd.deriv(0)), ("c1s_d1", bd.deriv(1))):
        a, b = load(nm).densify(), m.densify()
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)
    # and the HODLR approximates the dense covariance (acceptance criterion 1)
    K = oo.apply(np.eye(len(x)))
    assert np.linalg.norm(load("c1s_h").densify() - K) <= 1e-10 * np.linalg.norm(K)


def test_c1s_results():
    g = GOLD["c1s"]
    y = sidecar("c1s_y.bin")
    h, d = load("c1s_h"), [load("c1s_d0"), load("c1s_d1")]
    f = O.factorize(h, 1)
    assert f.logdet() == pytest.approx(g["logdet"], rel=1e-13)
    for tag, on in (("reference", False), ("solve", True)):
        try:
            O.set_solve_association(on)
            ll = O.log_likelihood(f, y)
            s = O.score(f, d, y)
            fi = O.fisher_information(f, d, cache=True)
        finally:
            O.set_solve_association(False)
        assert ll == pytest.approx(g[tag]["loglik"], rel=1e-12)
        assert np.allclose(s, g[tag]["score"], rtol=1e-11, atol=0)
        assert np.allclose(fi, g[tag]["fisher"], rtol=1e-11, atol=0)
