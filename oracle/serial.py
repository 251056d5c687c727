"""CPU restatement of the reference HODLR debug serializer — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module (see oracle/__init__.py). It restates, over the panel exchange
dict of pyoracle.Hodlr.export_panels (oracle/capi.cpp or_hodlr_export):

* write_hodlr_debug — reference io.cpp:171-233: manifest `dir/name.json`
  (nlohmann dump(2): two-space indent, sorted keys) holding n, depth,
  symmetric, "upper" (and "lower" when not symmetric) as per-level lists of
  blocks {node, rows, cols, rank, left, right}, and "leaves" {index, rows,
  file}; sidecar names `name_u_l<l>_n<j>_{left,right}.bin` ("lo" for the
  lower triangle) and `name_leaf<b>.bin`.
* read_hodlr_debug — io.cpp:235-275 (blocks missing from the manifest stay
  empty, as HodlrMatrix::zero leaves them).
* sidecars — io.cpp:78-101: row-major little-endian float64; a short file is
  an error ("truncated sidecar"), trailing bytes are ignored.
"""
import json
import os

import numpy as np


class SerialError(RuntimeError):
    pass


def tree_ranges(n, tau):
    """cluster_tree.cpp:10-22 (left child takes the ceiling half)."""
    lv = [[(0, n)]]
    for _ in range(tau):
        nxt = []
        for lo, hi in lv[-1]:
            mid = lo + (hi - lo + 1) // 2
            nxt += [(lo, mid), (mid, hi)]
        lv.append(nxt)
    return lv


def _panels_at(p):
    """Per-level (U_l, V_l) views (n x R_l, column-major) and leaf offsets."""
    n, tau = p["n"], p["tau"]
    flat = np.asarray(p["flat"], dtype=np.float64)
    out, off = [], 0
    for l in range(1, tau + 1):
        r = int(p["R"][l - 1])
        u = flat[off:off + n * r].reshape(r, n).T
        v = flat[off + n * r:off + 2 * n * r].reshape(r, n).T
        out.append((u, v))
        off += 2 * n * r
    return out, off


def blocks(p):
    """The reference's per-block view of a panel dict: yields
    (tag, level, node, rows, cols, left, right) in manifest order."""
    n, tau = p["n"], p["tau"]
    lv = tree_ranges(n, tau)
    pan, _ = _panels_at(p)
    tags = [("u", True)] + ([] if p["sym"] else [("lo", False)])
    for tag, upper in tags:
        idx = 0
        for l in range(1, tau + 1):
            u, v = pan[l - 1]
            for j in range(2 ** (l - 1)):
                a, b = lv[l][2 * j], lv[l][2 * j + 1]
                rows, cols = (a, b) if upper else (b, a)
                r = int((p["ranks_up"] if upper else p["ranks_lo"])[idx])
                idx += 1
                yield (tag, l, j, rows, cols, u[rows[0]:rows[1], :r], v[cols[0]:cols[1], :r])


def leaves(p):
    n, tau = p["n"], p["tau"]
    _, off = _panels_at(p)
    flat = np.asarray(p["flat"], dtype=np.float64)
    for b, (lo, hi) in enumerate(tree_ranges(n, tau)[tau]):
        m = hi - lo
        yield b, (lo, hi), flat[off:off + m * m].reshape(m, m).T
        off += m * m


def write_sidecar(path, a):
    with open(path, "wb") as f:
        f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def read_sidecar(path, rows, cols):
    try:
        with open(path, "rb") as f:
            raw = f.read(8 * rows * cols)
    except OSError as e:
        raise SerialError(f"cannot open {path}") from e
    if len(raw) < 8 * rows * cols:
        raise SerialError(f"{path}: truncated sidecar")
    return np.frombuffer(raw, dtype="<f8").reshape(rows, cols).astype(np.float64)


def write_hodlr_debug(dir, name, p):
    """io.cpp:171-233"""
    os.makedirs(dir, exist_ok=True)
    man = {"n": int(p["n"]), "depth": int(p["tau"]), "symmetric": bool(p["sym"])}
    tris = {}
    for tag, l, j, rows, cols, left, right in blocks(p):
        key = "upper" if tag == "u" else "lower"
        levels = tris.setdefault(key, [])
        if len(levels) < l:
            levels.append({"level": l, "blocks": []})
        base = f"{name}_{tag}_l{l}_n{j}"
        write_sidecar(os.path.join(dir, base + "_left.bin"), left)
        write_sidecar(os.path.join(dir, base + "_right.bin"), right)
        levels[l - 1]["blocks"].append({"node": j, "rows": list(rows), "cols": list(cols),
                                        "rank": int(left.shape[1]), "left": base + "_left.bin",
                                        "right": base + "_right.bin"})
    man["upper"] = tris.get("upper", [])
    if not p["sym"]:
        man["lower"] = tris.get("lower", [])
    man["leaves"] = []
    for b, rows, a in leaves(p):
        file = f"{name}_leaf{b}.bin"
        write_sidecar(os.path.join(dir, file), a)
        man["leaves"].append({"index": b, "rows": list(rows), "file": file})
    with open(os.path.join(dir, name + ".json"), "w") as f:
        f.write(json.dumps(man, indent=2, sort_keys=True) + "\n")


def read_hodlr_debug(dir, name):
    """io.cpp:235-275 -> panel exchange dict (import with
    pyoracle.Hodlr.import_panels)."""
    path = os.path.join(dir, name + ".json")
    try:
        with open(path) as f:
            man = json.load(f)
    except OSError as e:
        raise SerialError(f"cannot open manifest in {dir}") from e
    n, tau, sym = int(man["n"]), int(man["depth"]), bool(man["symmetric"])
    lv = tree_ranges(n, tau)
    nn = max(2 ** tau - 1, 0)
    ru, rl = np.zeros(nn, dtype=np.int32), np.zeros(nn, dtype=np.int32)
    got = []
    for key, upper in [("upper", True)] + ([] if sym else [("lower", False)]):
        for lev in man[key]:
            l = int(lev["level"])
            for e in lev["blocks"]:
                j = int(e["node"])
                a, b = lv[l][2 * j], lv[l][2 * j + 1]
                rows, cols = (a, b) if upper else (b, a)
                if tuple(e["rows"]) != rows or tuple(e["cols"]) != cols:
                    raise ValueError(f"{path}: block ranges do not match the cluster tree")
                r = int(e["rank"])
                (ru if upper else rl)[2 ** (l - 1) - 1 + j] = r
                left = read_sidecar(os.path.join(dir, e["left"]), rows[1] - rows[0], r)
                right = read_sidecar(os.path.join(dir, e["right"]), cols[1] - cols[0], r)
                got.append((l, upper, rows, cols, left, right))
    if sym:
        rl = ru.copy()
    R = [0] * tau
    for l in range(1, tau + 1):
        sl = slice(2 ** (l - 1) - 1, 2 ** l - 1)
        R[l - 1] = int(max(ru[sl].max(initial=0), rl[sl].max(initial=0)))
    U = [np.zeros((n, r)) for r in R]
    V = [np.zeros((n, r)) for r in R]
    for l, upper, rows, cols, left, right in got:
        r = left.shape[1]
        U[l - 1][rows[0]:rows[1], :r] = left
        (U if sym else V)[l - 1][cols[0]:cols[1], :r] = right
    parts = []
    for l in range(tau):
        parts += [U[l].T.ravel(), (U[l] if sym else V[l]).T.ravel()]
    lvs = {}
    for e in man["leaves"]:
        b = int(e["index"])
        lo, hi = lv[tau][b]
        if tuple(e["rows"]) != (lo, hi):
            raise ValueError(f"{path}: leaf ranges do not match the cluster tree")
        lvs[b] = read_sidecar(os.path.join(dir, e["file"]), hi - lo, hi - lo)
    for b, (lo, hi) in enumerate(lv[tau]):
        parts.append(lvs.get(b, np.zeros((hi - lo, hi - lo))).T.ravel())
    flat = np.concatenate(parts) if parts else np.zeros(0)
    return dict(n=n, tau=tau, sym=sym, R=R, flat=flat, ranks_up=ru, ranks_lo=rl)
