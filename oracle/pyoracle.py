"""TEST INFRASTRUCTURE ONLY — ctypes view of the parity oracle (oracle/_build/liboracle.so).

The oracle is the CPU restatement of the reference hot path (see oracle/oracle.hpp).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this
module, and only as the checker / CPU baseline — never as the measured product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# Loaded as oracle.pyref_impl (oracle/pyref.py) this module binds the REFERENCE
# itself (oracle/_ref/libhodlrgp_ref.so: /root/reference/proj/src compiled
# unmodified against oracle/eigen_shim, same or_* ABI); otherwise the restated
# oracle (oracle/_build/liboracle.so).
IS_REFERENCE = __name__.endswith("pyref_impl")
LIB_PATH = os.path.join(_HERE, "_ref", "libhodlrgp_ref.so") if IS_REFERENCE else os.path.join(
    _HERE, "_build", "liboracle.so")

i64 = C.c_int64
u64 = C.c_uint64
dbl = C.c_double
vp = C.c_void_p
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
lp = C.POINTER(C.c_int64)

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE] + (["-f", "ref.mk"] if IS_REFERENCE else []), check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        sig = {
            "or_last_error": (C.c_char_p, []),
            "or_enable_blas": (C.c_int, [C.c_char_p, C.c_int]),
            "or_blas_backend": (C.c_char_p, []),
            "or_set_solve_association": (None, [C.c_int]),
            "or_set_q2_reorthogonalize": (None, [C.c_int]),
            "or_set_compress_at_level": (None, [C.c_int]),
            "or_tree_depth": (C.c_int, [i64, i64, i64]),
            "or_tree_ranges": (C.c_int, [i64, C.c_int, lp]),
            "or_kd_ordering": (C.c_int, [i64, C.c_int, dp, i64, i64, lp, lp, ip]),
            "or_hodlr_random": (vp, [i64, C.c_int, i64, u64, C.c_int]),
            "or_hodlr_from_dense": (vp, [i64, C.c_int, dp, C.c_int]),
            "or_hodlr_identity": (vp, [i64, C.c_int]),
            "or_hodlr_free": (None, [vp]),
            "or_hodlr_copy": (vp, [vp]),
            "or_hodlr_info": (C.c_int, [vp, lp, ip, ip, ip]),
            "or_hodlr_export": (C.c_int, [vp, dp, ip, ip]),
            "or_hodlr_import": (vp, [i64, C.c_int, C.c_int, ip, dp, ip, ip]),
            "or_hodlr_densify": (C.c_int, [vp, dp]),
            "or_hodlr_matvec": (C.c_int, [vp, dp, i64, dp]),
            "or_hodlr_sub_matvec": (C.c_int, [vp, C.c_int, i64, dp, i64, i64, C.c_int, dp]),
            "or_hodlr_trace": (dbl, [vp]),
            "or_trace_product": (C.c_int, [vp, vp, dp]),
            "or_hodlr_make_asymmetric": (None, [vp]),
            "or_factorize": (vp, [vp, C.c_int]),
            "or_factor_free": (None, [vp]),
            "or_factor_solve": (C.c_int, [vp, dp, i64, dp]),
            "or_factor_logdet": (C.c_int, [vp, dp]),
            "or_factor_leaf_llt": (C.c_int, [vp, ip]),
            "or_solve_multiply": (vp, [vp, vp]),
            "or_multiply": (vp, [vp, vp]),
            "or_prodrep_free": (None, [vp]),
            "or_prodrep_densify": (C.c_int, [vp, dp]),
            "or_trace_product_rep": (dbl, [vp]),
            "or_trace_pair": (dbl, [vp, vp]),
            "or_trace_solve": (C.c_int, [vp, vp, dp]),
            "or_hutchinson_trace": (C.c_int, [vp, vp, C.c_int, u64, dp]),
            "or_trace_quad": (C.c_int, [vp, vp, vp, vp, dp]),
            "or_sketch_sampler": (C.c_int, [i64, C.c_int, i64, u64, C.c_int, dp]),
            "or_randomized_range": (C.c_int, [dp, i64, i64, dp, dp, ip, lp]),
            "or_diff_qr": (C.c_int, [dp, dp, dp, i64, i64, dp, dp, dp, ip]),
            "or_oracle_dense": (vp, [i64, dp, C.c_int, dp]),
            "or_oracle_matern": (vp, [i64, dp, C.c_int, dbl, dbl, dbl, C.c_int]),
            "or_oracle_free": (None, [vp]),
            "or_oracle_apply": (C.c_int, [vp, C.c_int, dp, i64, dp]),
            "or_oracle_counters": (C.c_int, [vp, C.POINTER(u64), C.POINTER(u64), C.c_int]),
            "or_build": (vp, [vp, C.c_int, i64, u64, C.c_int]),
            "or_build_free": (None, [vp]),
            "or_build_h": (vp, [vp]),
            "or_build_deriv": (vp, [vp, C.c_int]),
            "or_build_num_warnings": (C.c_int, [vp]),
            "or_build_decisions": (C.c_int, [vp, C.c_int, lp]),
            "or_log_likelihood": (C.c_int, [vp, dp, dp, dp]),
            "or_score": (C.c_int, [vp, C.POINTER(vp), C.c_int, dp, dp, dp]),
            "or_fisher": (C.c_int, [vp, C.POINTER(vp), C.c_int, C.c_int, dp]),
            "or_mle_iteration": (C.c_int, [vp, C.c_int, i64, u64, dp, C.c_int, dp, dp, dp, dp]),
            "or_randn": (None, [i64, i64, u64, dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class NotPositiveDefinite(OracleError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    if rc == 1:
        raise NotPositiveDefinite(rc, msg)
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise OverflowError(msg)
    raise OracleError(rc, msg)


def _d(a):
    return a.ctypes.data_as(dp)


def _f(a):
    """Fortran-ordered float64 copy."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def set_solve_association(on):
    """Diagnostic: product association of the device path (see oracle.hpp)."""
    lib().or_set_solve_association(int(on))


def set_q2_reorthogonalize(on):
    """Diagnostic: the device's default q2 basis (HG_Q2_REORTHOGONALIZED, see oracle.hpp)."""
    lib().or_set_q2_reorthogonalize(int(on))


def set_compress_at_level(on):
    """Diagnostic: the device's default HG_COMPRESS_AT_LEVEL (see oracle.hpp)."""
    lib().or_set_compress_at_level(int(on))


def device_defaults(on):
    """Every oracle switch set to the device's default numerical modes (on) or
    back to the reference (off)."""
    set_solve_association(on)
    set_q2_reorthogonalize(on)
    set_compress_at_level(on)


def randn(r, c, seed):
    out = np.zeros((r, c), order="F")
    lib().or_randn(r, c, seed, _d(out))
    return out


def tree_depth(n, lmin, lmax):
    return lib().or_tree_depth(n, lmin, lmax)


def tree_ranges(n, tau):
    cnt = 2 ** (tau + 1) - 1
    out = np.zeros(2 * cnt, dtype=np.int64)
    _check(lib().or_tree_ranges(n, tau, out.ctypes.data_as(lp)))
    res, o = [], 0
    for d in range(tau + 1):
        lv = []
        for _ in range(2 ** d):
            lv.append((int(out[o]), int(out[o + 1])))
            o += 2
        res.append(lv)
    return res


def kd_ordering(coords, lmin, lmax):
    c = _f(coords)
    n, d = c.shape
    perm = np.zeros(n, dtype=np.int64)
    inv = np.zeros(n, dtype=np.int64)
    tau = C.c_int()
    _check(lib().or_kd_ordering(n, d, _d(c), lmin, lmax, perm.ctypes.data_as(lp),
                                inv.ctypes.data_as(lp), C.byref(tau)))
    return perm, inv, tau.value


class Hodlr:
    def __init__(self, ptr):
        if not ptr:
            _check(9)
        self.ptr = ptr

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.or_hodlr_free(self.ptr)
            self.ptr = None

    @staticmethod
    def random_spd(n, tau, k, seed):
        return Hodlr(lib().or_hodlr_random(n, tau, k, seed, 1))

    @staticmethod
    def random_symmetric(n, tau, k, seed):
        return Hodlr(lib().or_hodlr_random(n, tau, k, seed, 0))

    @staticmethod
    def identity(n, tau):
        return Hodlr(lib().or_hodlr_identity(n, tau))

    @staticmethod
    def from_dense(tau, a, symmetric=True):
        a = _f(a)
        p = lib().or_hodlr_from_dense(a.shape[0], tau, _d(a), int(symmetric))
        if not p:
            _check(2)
        return Hodlr(p)

    def copy(self):
        return Hodlr(lib().or_hodlr_copy(self.ptr))

    def info(self):
        n = C.c_int64()
        tau = C.c_int()
        sym = C.c_int()
        lib().or_hodlr_info(self.ptr, C.byref(n), C.byref(tau), C.byref(sym), None)
        R = np.zeros(max(tau.value, 1), dtype=np.int32)
        lib().or_hodlr_info(self.ptr, C.byref(n), C.byref(tau), C.byref(sym), R.ctypes.data_as(ip))
        return n.value, tau.value, bool(sym.value), [int(x) for x in R[: tau.value]]

    @property
    def n(self):
        return self.info()[0]

    def export_panels(self):
        """Panel exchange format (see oracle/capi.cpp): returns dict."""
        n, tau, sym, R = self.info()
        ranges = tree_ranges(n, tau)
        leaf_sizes = [hi - lo for lo, hi in ranges[tau]]
        total = sum(2 * n * r for r in R) + sum(m * m for m in leaf_sizes)
        flat = np.zeros(total)
        nn = max(2 ** tau - 1, 1)
        ru = np.zeros(nn, dtype=np.int32)
        rl = np.zeros(nn, dtype=np.int32)
        _check(lib().or_hodlr_export(self.ptr, _d(flat), ru.ctypes.data_as(ip), rl.ctypes.data_as(ip)))
        return dict(n=n, tau=tau, sym=sym, R=R, flat=flat, ranks_up=ru[: 2 ** tau - 1],
                    ranks_lo=rl[: 2 ** tau - 1])

    @staticmethod
    def import_panels(p):
        R = np.asarray(p["R"] if len(p["R"]) else [0], dtype=np.int32)
        ru = np.asarray(p["ranks_up"] if len(p["ranks_up"]) else [0], dtype=np.int32)
        rl = np.asarray(p["ranks_lo"] if len(p["ranks_lo"]) else [0], dtype=np.int32)
        flat = np.ascontiguousarray(p["flat"], dtype=np.float64)
        ptr = lib().or_hodlr_import(p["n"], p["tau"], int(p["sym"]), R.ctypes.data_as(ip), _d(flat),
                                    ru.ctypes.data_as(ip), rl.ctypes.data_as(ip))
        if not ptr:
            _check(2)
        return Hodlr(ptr)

    def densify(self):
        n = self.n
        out = np.zeros((n, n), order="F")
        _check(lib().or_hodlr_densify(self.ptr, _d(out)))
        return out

    def matvec(self, x):
        x = _f(x)
        vec = x.ndim == 1
        if vec:
            x = x.reshape(-1, 1, order="F")
        y = np.zeros_like(x, order="F")
        _check(lib().or_hodlr_matvec(self.ptr, _d(x), x.shape[1], _d(y)))
        return y[:, 0] if vec else y

    def sub_matvec(self, d, node, x, transpose=False):
        x = _f(x)
        y = np.zeros_like(x, order="F")
        _check(lib().or_hodlr_sub_matvec(self.ptr, d, node, _d(x), x.shape[0], x.shape[1], int(transpose), _d(y)))
        return y

    def trace(self):
        return lib().or_hodlr_trace(self.ptr)

    def make_asymmetric(self):
        lib().or_hodlr_make_asymmetric(self.ptr)


def trace_product(a, b):
    out = C.c_double()
    _check(lib().or_trace_product(a.ptr, b.ptr, C.byref(out)))
    return out.value


class Factor:
    RIGHT, LEFT = 0, 1

    def __init__(self, h, orient):
        self.ptr = lib().or_factorize(h.ptr, orient)
        if not self.ptr:
            _check(9)
        self.n = h.n

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.or_factor_free(self.ptr)
            self.ptr = None

    def solve(self, b):
        b = _f(b)
        vec = b.ndim == 1
        if vec:
            b = b.reshape(-1, 1, order="F")
        x = np.zeros_like(b, order="F")
        _check(lib().or_factor_solve(self.ptr, _d(b), b.shape[1], _d(x)))
        return x[:, 0] if vec else x

    def logdet(self):
        out = C.c_double()
        _check(lib().or_factor_logdet(self.ptr, C.byref(out)))
        return out.value


def factorize(h, orient=Factor.RIGHT):
    return Factor(h, orient)


class ProductRep:
    def __init__(self, ptr, n):
        if not ptr:
            _check(2)
        self.ptr = ptr
        self.n = n

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.or_prodrep_free(self.ptr)
            self.ptr = None

    def densify(self):
        out = np.zeros((self.n, self.n), order="F")
        _check(lib().or_prodrep_densify(self.ptr, _d(out)))
        return out


def solve_multiply(f, b):
    p = lib().or_solve_multiply(f.ptr, b.ptr)
    if not p:
        _check(2)
    return ProductRep(p, f.n)


def multiply(f, b):
    p = lib().or_multiply(f.ptr, b.ptr)
    if not p:
        _check(2)
    return ProductRep(p, f.n)


def trace_product_rep(p):
    return lib().or_trace_product_rep(p.ptr)


def trace_pair(p, q):
    return lib().or_trace_pair(p.ptr, q.ptr)


def trace_solve(f, b):
    out = C.c_double()
    _check(lib().or_trace_solve(f.ptr, b.ptr, C.byref(out)))
    return out.value


def hutchinson_trace(f, b, n_samples, seed):
    """mle.cpp:56-75 -> (estimate, std_error)."""
    out = (C.c_double * 2)()
    _check(lib().or_hutchinson_trace(f.ptr, b.ptr, n_samples, seed, out))
    return out[0], out[1]


def trace_quad(fa, b, fc, d):
    out = C.c_double()
    _check(lib().or_trace_quad(fa.ptr, b.ptr, fc.ptr, d.ptr, C.byref(out)))
    return out.value


def sketch_sampler(n, tau, k, seed, level):
    """level 0 = leaf sampler (n x max_leaf_size)."""
    if level == 0:
        rngs = tree_ranges(n, tau)[tau]
        cols = max(hi - lo for lo, hi in rngs)
    else:
        cols = k
    out = np.zeros((n, cols), order="F")
    _check(lib().or_sketch_sampler(n, tau, k, seed, level, _d(out)))
    return out


def randomized_range(y, k):
    y = _f(y)
    m = y.shape[0]
    q = np.zeros((m, k), order="F")
    r = np.zeros((k, k), order="F")
    perm = np.zeros(k, dtype=np.int32)
    nr = C.c_int64()
    _check(lib().or_randomized_range(_d(y), m, k, _d(q), _d(r), perm.ctypes.data_as(ip), C.byref(nr)))
    return q, r, perm, nr.value


def diff_qr(db, q, r):
    db, q, r = _f(db), _f(q), _f(r)
    m, k = q.shape
    dq = np.zeros((m, k), order="F")
    dqs = np.zeros((m, k), order="F")
    dr = np.zeros((k, k), order="F")
    ill = C.c_int()
    _check(lib().or_diff_qr(_d(db), _d(q), _d(r), m, k, _d(dq), _d(dqs), _d(dr), C.byref(ill)))
    return dq, dqs, dr, bool(ill.value)


class CovOracle:
    def __init__(self, ptr, n):
        if not ptr:
            _check(2)
        self.ptr = ptr
        self.n = n

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.or_oracle_free(self.ptr)
            self.ptr = None

    @staticmethod
    def dense(k, dks=()):
        k = _f(k)
        n = k.shape[0]
        p = len(dks)
        buf = np.concatenate([_f(d).ravel(order="F") for d in dks]) if p else np.zeros(1)
        keep = (k, buf)
        o = CovOracle(lib().or_oracle_dense(n, _d(k), p, _d(buf)), n)
        o._keep = keep
        return o

    @staticmethod
    def matern(x, nu2, sigma2, ell, nugget, scan):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return CovOracle(lib().or_oracle_matern(len(x), _d(x), nu2, sigma2, ell, nugget, int(scan)), len(x))

    def apply(self, v, which=-1):
        v = _f(v)
        y = np.zeros_like(v, order="F")
        _check(lib().or_oracle_apply(self.ptr, which, _d(v), v.shape[1], _d(y)))
        return y

    def counters(self, reset=False):
        a = C.c_uint64()
        d = C.c_uint64()
        lib().or_oracle_counters(self.ptr, C.byref(a), C.byref(d), int(reset))
        return a.value, d.value


class Build:
    def __init__(self, oracle, tau, k, seed, with_deriv, p=0):
        self.ptr = lib().or_build(oracle.ptr, tau, k, seed, int(with_deriv))
        if not self.ptr:
            _check(2)
        self.p = p
        self.tau = tau

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.or_build_free(self.ptr)
            self.ptr = None

    def h(self):
        return Hodlr(lib().or_build_h(self.ptr))

    def deriv(self, j):
        return Hodlr(lib().or_build_deriv(self.ptr, j))

    def num_warnings(self):
        return lib().or_build_num_warnings(self.ptr)

    def decisions(self):
        cnt = 2 ** self.tau - 1
        out = np.zeros((max(cnt, 1), 2 + self.p), dtype=np.int64)
        k = lib().or_build_decisions(self.ptr, self.p, out.ctypes.data_as(lp))
        return out[:k]


def _vec(y):
    return np.ascontiguousarray(y, dtype=np.float64)


def log_likelihood(f, y, ybar=None):
    y = _vec(y)
    out = C.c_double()
    yb = _vec(ybar) if ybar is not None else None
    _check(lib().or_log_likelihood(f.ptr, _d(y), _d(yb) if yb is not None else None, C.byref(out)))
    return out.value


def score(f, derivs, y, ybar=None):
    y = _vec(y)
    p = len(derivs)
    arr = (vp * p)(*[d.ptr for d in derivs])
    out = np.zeros(p)
    yb = _vec(ybar) if ybar is not None else None
    _check(lib().or_score(f.ptr, arr, p, _d(y), _d(yb) if yb is not None else None, _d(out)))
    return out


def fisher_information(f, derivs, cache=False):
    p = len(derivs)
    arr = (vp * p)(*[d.ptr for d in derivs])
    out = np.zeros((p, p), order="F")
    _check(lib().or_fisher(f.ptr, arr, p, int(cache), _d(out)))
    return out


def mle_iteration(oracle, tau, k, seed, y, p, cache=True):
    y = _vec(y)
    ll = C.c_double()
    s = np.zeros(p)
    fi = np.zeros((p, p), order="F")
    t = np.zeros(5)
    _check(lib().or_mle_iteration(oracle.ptr, tau, k, seed, _d(y), int(cache), C.byref(ll), _d(s), _d(fi), _d(t)))
    return ll.value, s, fi, t
