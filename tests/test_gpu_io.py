"""GPU: the device library's debug serializer (hg_write_hodlr_debug /
hg_read_hodlr_debug, io.cpp:171-275) against the committed golden fixtures
(tests/golden/, io.cpp layout), and the hot path run on those fixtures
against their golden results."""
import filecmp
import json
import os

import numpy as np
import pytest

from oracle import serial as S

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(G, "golden.json")))
NAMES = ["spd50_sym", "spd50_asym", "c1s_h", "c1s_d0", "c1s_d1"]


@pytest.fixture(scope="module")
def H():
    from paper_2303_10102_b200 import hodlrgp

    return hodlrgp


def sidecar(name):
    return np.frombuffer(open(os.path.join(G, name), "rb").read(), dtype="<f8").astype(np.float64)


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def test_roundtrip_sym_and_asym(H, tmp_path):  # test_io.cpp:92-107 on the device
    h = H.HodlrMatrix.random_spd(H.ClusterTree(50, 2), 3, 4)
    H.write_hodlr_debug(str(tmp_path), "sym", h)
    back = H.read_hodlr_debug(str(tmp_path), "sym")
    assert back.info()[2]
    assert np.linalg.norm(back.densify() - h.densify()) == 0.0
    p = h.export_panels()
    p["sym"] = False
    n, R1 = p["n"], p["R"][0]
    nu = n * R1
    U1 = p["flat"][:nu].reshape(R1, n).T.copy()
    V1 = U1.copy()
    lo, hi = S.tree_ranges(n, 2)[1][1]
    U1[lo:hi, :] *= 2.0  # lower(1, 0).left *= 2
    p["flat"] = np.concatenate([U1.T.ravel(), V1.T.ravel(), p["flat"][2 * nu:]])
    p["ranks_lo"] = p["ranks_up"].copy()
    a = H.HodlrMatrix.from_panels(p)
    H.write_hodlr_debug(str(tmp_path), "asym", a)
    back2 = H.read_hodlr_debug(str(tmp_path), "asym")
    assert not back2.info()[2]
    assert np.linalg.norm(back2.densify() - a.densify()) == 0.0


@pytest.mark.parametrize("name", NAMES)
def test_read_golden_bitwise(H, name):
    d = H.read_hodlr_debug(G, name).export_panels()
    o = S.read_hodlr_debug(G, name)
    assert d["sym"] == o["sym"] and list(d["R"]) == list(o["R"])
    assert list(d["ranks_up"]) == list(o["ranks_up"])
    if not o["sym"]:
        assert list(d["ranks_lo"]) == list(o["ranks_lo"])
    assert np.array_equal(d["flat"], o["flat"])


@pytest.mark.parametrize("name", NAMES)
def test_write_byte_identical(H, name, tmp_path):
    """Device write of a fixture reproduces every file byte for byte (the
    manifest in the reference's nlohmann dump(2) form)."""
    h = H.read_hodlr_debug(G, name)
    H.write_hodlr_debug(str(tmp_path / "sub" / "dir"), name, h)  # creates directories
    out = str(tmp_path / "sub" / "dir")
    files = [f for f in os.listdir(G) if f.startswith(name + "_") or f == name + ".json"]
    assert sorted(os.listdir(out)) == sorted(files)
    match, mismatch, errors = filecmp.cmpfiles(G, out, files, shallow=False)
    assert not mismatch and not errors, mismatch


def test_errors(H, tmp_path):
    h = H.read_hodlr_debug(G, "spd50_sym")
    H.write_hodlr_debug(str(tmp_path), "t", h)
    with pytest.raises(H.SerializationError, match="cannot open manifest"):
        H.read_hodlr_debug(str(tmp_path), "nope")
    leaf = tmp_path / "t_leaf1.bin"
    full = leaf.read_bytes()
    leaf.write_bytes(full[:-1])
    with pytest.raises(H.SerializationError, match="truncated sidecar"):
        H.read_hodlr_debug(str(tmp_path), "t")
    leaf.write_bytes(full + b"\1" * 24)  # trailing bytes ignored (io.cpp:89-101)
    assert np.array_equal(H.read_hodlr_debug(str(tmp_path), "t").densify(), h.densify())
    (tmp_path / "t_u_l1_n0_right.bin").unlink()
    with pytest.raises(H.SerializationError, match="cannot open"):
        H.read_hodlr_debug(str(tmp_path), "t")
    man = json.load(open(tmp_path / "t.json"))
    man["upper"][0]["blocks"][0]["rows"] = [0, 24]
    (tmp_path / "u.json").write_text(json.dumps(man))
    with pytest.raises(ValueError, match="cluster tree"):
        H.read_hodlr_debug(str(tmp_path), "u")
    (tmp_path / "v.json").write_text('{"n": 50, "depth": 2, ')
    with pytest.raises(H.SerializationError, match="malformed manifest"):
        H.read_hodlr_debug(str(tmp_path), "v")


def test_spd50_results(H):
    g = GOLD["spd50_sym"]
    h = H.read_hodlr_debug(G, "spd50_sym")
    f = H.factorize(h, H.LEFT)
    assert f.logdet() == pytest.approx(g["logdet"], rel=1e-12)
    b = np.asarray(g["solve"])
    x = f.solve(h.matvec(b))
    assert np.linalg.norm(x - b) <= 1e-12 * np.linalg.norm(b)


def test_c1s_hot_path_on_fixtures(H):
    """Factorization, log-likelihood, score and Fisher on the committed
    n = 512 C1 fixtures; golden values of the solve association (DESIGN.md
    §4): loglik and logdet 1e-9, score 1e-9, Fisher 1e-7."""
    g = GOLD["c1s"]
    y = sidecar("c1s_y.bin")
    h = H.read_hodlr_debug(G, "c1s_h")
    d = [H.read_hodlr_debug(G, "c1s_d0"), H.read_hodlr_debug(G, "c1s_d1")]
    f = H.factorize(h, H.LEFT)
    assert f.logdet() == pytest.approx(g["logdet"], rel=1e-9)
    assert H.log_likelihood(f, y) == pytest.approx(g["solve"]["loglik"], rel=1e-9)
    assert _rel(H.score(f, d, y), g["solve"]["score"]) <= 1e-9
    assert _rel(H.fisher_information(f, d), g["solve"]["fisher"]) <= 1e-7


def test_c1s_device_build_matches_fixture(H, tmp_path):
    """The device build on the stored points: identical per-block decisions,
    densified H and dH/dtheta within 1e-10 / 1e-9 of the fixtures, and its
    own serialization reads back bit-exactly."""
    g = GOLD["c1s"]
    x = sidecar("c1s_x.bin")
    do = H.MaternOracle(x, g["nu2"], g["sigma2"], g["ell"], g["nugget"], False)
    br = H.build_hodlr_with_derivatives(do, H.ClusterTree(g["n"], g["depth"]), g["k"], g["seed"])
    assert br.decisions().tolist() == g["decisions"]
    for nm, m, tol in (("c1s_h", br.h, 1e-10), ("c1s_d0", br.deriv[0], 1e-9), ("c1s_d1", br.deriv[1], 1e-9)):
        ref = H.read_hodlr_debug(G, nm).densify()
        assert np.linalg.norm(m.densify() - ref) <= tol * np.linalg.norm(ref)
        H.write_hodlr_debug(str(tmp_path), nm, m)
        man_d = json.load(open(tmp_path / (nm + ".json")))
        man_g = json.load(open(os.path.join(G, nm + ".json")))
        assert man_d == man_g  # same ranks, ranges and sidecar names
        back = H.read_hodlr_debug(str(tmp_path), nm)
        assert np.array_equal(back.export_panels()["flat"], m.export_panels()["flat"])


def test_c1_full_against_golden(H):
    """Config C1 at full size (n = 4096) through the device MLE iteration on
    the committed points and data: loglik 1e-9, score and Fisher 1e-7 against
    the oracle's solve-association values. Per-block rank decisions: at most
    one of the 63 may differ (a singular value at the truncation threshold
    is decided by rounding; same allowance as test_gpu_build_mle.py)."""
    g = GOLD["c1"]
    x, y = sidecar("c1_x.bin"), sidecar("c1_y.bin")
    do = H.MaternOracle(x, g["nu2"], g["sigma2"], g["ell"], g["nugget"], False)
    ll, s, fi, _ = H.mle_iteration(do, g["depth"], g["k"], g["seed"], y)
    assert ll == pytest.approx(g["solve"]["loglik"], rel=1e-9)
    assert _rel(s, g["solve"]["score"]) <= 1e-7 and _rel(fi, g["solve"]["fisher"]) <= 1e-7
    br = H.build_hodlr_with_derivatives(do, H.ClusterTree(g["n"], g["depth"]), g["k"], g["seed"])
    dec, ref = br.decisions(), np.asarray(g["decisions"])
    assert dec.shape == ref.shape and int((dec != ref).any(axis=1).sum()) <= 1


def test_bench_csv_schema(tmp_path):  # tools/hodlr_gp.cpp:378-477
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, os.path.join(root, "scripts", "bench_csv.py"), str(tmp_path), "--sizes", "1024",
                    "--repeats", "2"], check=True, capture_output=True)
    lines = open(tmp_path / "bench.csv").read().splitlines()
    assert lines[0] == "n,k,metric,value,repeat"
    rows = [r.split(",") for r in lines[1:]]
    metrics = [r[2] for r in rows if r[4] == "0"]
    assert metrics == ["build_seconds", "build_apply_columns", "build_apply_columns_expected", "build_deriv_seconds",
                       "deriv_apply_columns", "deriv_derivative_columns", "factorize_seconds", "loglik_seconds",
                       "score_seconds", "fisher_seconds", "eval_seconds_parallel"]
    val = {r[2]: float(r[3]) for r in rows if r[4] == "1"}
    assert val["build_apply_columns"] == val["build_apply_columns_expected"]  # 2 k tau + b
    assert all(r[0] == "1024" and r[1] == "24" for r in rows)
