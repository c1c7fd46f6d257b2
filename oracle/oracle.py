"""TEST INFRASTRUCTURE ONLY — ctypes binding of the fp64 CPU check oracle
(oracle/renyi_oracle.cpp). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
(paper_2205_07426_b200) never does.

Parity status: pinned by the reference's own analytic known-answer tests
(tests/test_oracle_kats.py); the reference itself is unbuildable here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "librenyi_oracle.so"

_D = C.POINTER(C.c_double)
_I64 = C.c_int64


class CParams(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("method", C.c_int), ("s", C.c_int), ("m", C.c_int),
        ("epsilon", C.c_double), ("delta", C.c_double), ("seed", C.c_uint64),
        ("power_max_iters", C.c_int), ("power_tol", C.c_double), ("power_seed", C.c_uint64),
        ("power_rank_floor", C.c_double), ("has_bounds", C.c_int), ("bu", C.c_double), ("bv", C.c_double),
        ("probe_kind", C.c_int), ("s_q", C.c_int), ("s_g", C.c_int),
    ]


class COut(C.Structure):
    _fields_ = [
        ("entropy", C.c_double), ("trace", C.c_double), ("low", C.c_double), ("residual", C.c_double),
        ("method", C.c_int), ("s", C.c_int), ("m", C.c_int), ("queries", C.c_int), ("rank", C.c_int),
        ("exact", C.c_int), ("deterministic", C.c_int), ("has_bounds", C.c_int),
        ("bu", C.c_double), ("bv", C.c_double), ("kappa", C.c_double),
        ("iterations_used", C.c_int), ("v_converged", C.c_int), ("u_converged", C.c_int),
        ("rank_deficient", C.c_int),
    ]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None
MUL_FN = C.CFUNCTYPE(C.c_int, C.c_int64, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double))
KINDS = {"int": 0, "int_power": 0, "taylor": 1, "chebyshev": 2}
METHODS = {"exact": 0, "int": 1, "taylor": 2, "chebyshev": 3, "auto": 4}
PROBES = {"gaussian": 0, "rademacher": 1}


def build() -> Path:
    """Compiles the oracle (make, g++ -O3 -fopenmp) if needed."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


NATIVE = HERE / "_build" / "librenyi_oracle_native.so"


def lib():
    """The portable build; ORACLE_NATIVE=1 selects the -march=native build of the same source
    (tests/golden/gen_fullsize.py, one-off fixture generation on this container)."""
    global _lib
    if _lib is None:
        path = LIB
        if os.environ.get("ORACLE_NATIVE") == "1":
            subprocess.run(["make", "-s", "-C", str(HERE), "native"], check=True)
            path = NATIVE
        elif not LIB.exists():
            build()
        h = C.CDLL(str(path))
        h.oracle_last_error.restype = C.c_char_p
        for name in ("oracle_mix64", "oracle_derive_key", "oracle_hash_name"):
            getattr(h, name).restype = C.c_uint64
        h.oracle_mix64.argtypes = [C.c_uint64]
        _PD = C.POINTER(C.c_double)
        for name in ("oracle_rank_features", "oracle_select_features"):
            getattr(h, name).argtypes = [_PD, C.c_int64, C.c_int64, C.POINTER(C.c_char_p), C.c_int64,
                                         C.POINTER(C.c_char_p), C.c_double, C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                         _PD]
        h.oracle_derive_key.argtypes = [C.c_uint64, C.c_uint64]
        h.oracle_hash_name.argtypes = [C.c_char_p]
        h.oracle_taylor_tail_constant.restype = C.c_double
        h.oracle_taylor_tail_constant.argtypes = [C.c_double, C.c_int]
        h.oracle_safeguard.restype = C.c_double
        h.oracle_safeguard.argtypes = [C.c_double, C.c_double]
        h.oracle_expected_queries.restype = C.c_long
        h.oracle_expected_queries.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, C.c_int]
        h.oracle_slab_sample.restype = C.c_double
        h.oracle_slab_sample.argtypes = [_D, _I64, _I64, C.c_double, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int]
        h.oracle_probe_panel.argtypes = [_I64, C.c_int, C.c_uint64, C.c_char_p, C.c_int, _D]
        h.oracle_stream_gaussian.argtypes = [C.c_uint64, _I64, _D]
        h.oracle_mixture_samples.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, _D]
        h.oracle_gaussian_gram.argtypes = [_D, _I64, _I64, C.c_double, _D]
        h.oracle_build_kernel.argtypes = [_D, _I64, _I64, C.c_double, _D]
        h.oracle_hadamard_joint_n.argtypes = [C.POINTER(_D), C.c_int, _I64, _D]
        h.oracle_polynomial_gram.argtypes = [_D, _I64, _I64, C.c_int, C.c_double, _D]
        h.oracle_build_kernel_polynomial.argtypes = [_D, _I64, _I64, C.c_int, C.c_double, _D]
        h.oracle_hadamard_joint.argtypes = [_D, _I64, _D, _I64, _D]
        h.oracle_matvec.argtypes = [_D, _I64, _D, _D]
        h.oracle_matmul_panel.argtypes = [_D, _I64, _D, C.c_int, _D]
        h.oracle_apply_panel.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, _D, _I64, _D,
                                         C.c_int, _D]
        h.oracle_scalar_value.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, C.c_double, _D]
        h.oracle_spec_coeffs.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, _D, _D]
        h.oracle_binomial_coeffs.argtypes = [C.c_double, C.c_int, _D]
        h.oracle_chebyshev_coeffs.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, _D]
        h.oracle_power_method.argtypes = [_D, _I64, C.c_int, C.c_double, C.c_uint64, _D, C.POINTER(C.c_int),
                                          C.POINTER(C.c_int)]
        h.oracle_estimate_bounds.argtypes = [_D, _I64, C.c_int, C.c_double, C.c_uint64, C.c_double,
                                             C.POINTER(COut)]
        h.oracle_colpiv_rank.argtypes = [_D, _I64, C.c_int, C.c_double, C.POINTER(C.c_int), _D]
        h.oracle_hutchpp.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, _D, _I64, C.c_int,
                                     C.c_int, C.c_uint64, C.c_int, _D, _D, C.POINTER(COut)]
        h.oracle_estimate.argtypes = [_D, _I64, C.POINTER(CParams), C.POINTER(COut)]
        h.oracle_eigvals.argtypes = [_D, _I64, _D]
        h.oracle_cb_estimate.argtypes = [_I64, MUL_FN, C.POINTER(CParams), C.POINTER(COut)]
        h.oracle_cb_matfun_traces.argtypes = [_I64, MUL_FN, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                              _D, C.c_int, _D]
        h.oracle_kernel_block.argtypes = [_D, _I64, _I64, _D, _D, C.c_double, C.c_double, C.c_double, C.c_int, _D]
        h.oracle_kernel_block_rows.argtypes = [_D, _D, _I64, _I64, _I64, _D, _D, C.c_double, C.c_double, C.c_double,
                                               C.c_int, _D]
        _MF = [_D, _I64, _I64, C.c_double, _D, _I64, C.c_double]
        h.oracle_mf_matmul.argtypes = _MF + [_D, C.c_int, _D]
        h.oracle_mf_estimate.argtypes = _MF + [C.POINTER(CParams), C.POINTER(COut)]
        h.oracle_mf_matfun_traces.argtypes = _MF + [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, _D,
                                                    C.c_int, _D]
        h.oracle_entropy_from_trace.argtypes = [C.c_double, C.c_double, _D]
        h.oracle_select_params.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                           _I64, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        h.oracle_mu_bound.argtypes = [C.c_double, C.c_double, C.c_double, _I64, _D, _D, _D]
        h.oracle_csv_parse.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        h.oracle_csv_shape.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        h.oracle_csv_features.argtypes = [C.c_void_p, _D]
        h.oracle_csv_string.restype = C.c_int64
        h.oracle_csv_string.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_char_p, C.c_int64]
        h.oracle_csv_free.argtypes = [C.c_void_p]
        h.oracle_threads.restype = C.c_int
        h.oracle_set_threads.argtypes = [C.c_int]
        h.oracle_set_merge_panels.argtypes = [C.c_int]
        _lib = h
    return _lib


def _chk(code: int):
    if code != 0:
        raise OracleError(code, lib().oracle_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _u64(x: int) -> int:
    return x & (2**64 - 1)


# ---- rng ----
def mix64(x): return int(lib().oracle_mix64(_u64(x)))
def derive_key(s, t): return int(lib().oracle_derive_key(_u64(s), _u64(t)))
def hash_name(s: str): return int(lib().oracle_hash_name(s.encode()))


def probe_panel(n, cols, seed, label, kind="gaussian"):
    out = np.empty((n, cols), order="F")
    _chk(lib().oracle_probe_panel(n, cols, _u64(seed), label.encode(), PROBES[kind], _p(out)))
    return out


gaussian_panel = probe_panel


def stream_gaussian(key, count):
    out = np.empty(count)
    _chk(lib().oracle_stream_gaussian(_u64(key), count, _p(out)))
    return out


def fill_gaussian(key, rows, cols):
    """RandomStream(key).fill_gaussian(Matrix(rows, cols)) — column-wise (rng.cpp:60-64)."""
    return stream_gaussian(key, rows * cols).reshape((rows, cols), order="F")


def mixture_samples(n, d, seed, center=1.0):
    out = np.empty((n, d), order="F")
    _chk(lib().oracle_mixture_samples(n, d, _u64(seed), center, _p(out)))
    return out


# ---- ops / kernel ----
def gaussian_gram(x, sigma):
    x = _f(x)
    out = np.empty((x.shape[0], x.shape[0]), order="F")
    _chk(lib().oracle_gaussian_gram(_p(x), x.shape[0], x.shape[1], sigma, _p(out)))
    return out


def build_kernel(x, sigma):
    x = _f(x)
    out = np.empty((x.shape[0], x.shape[0]), order="F")
    _chk(lib().oracle_build_kernel(_p(x), x.shape[0], x.shape[1], sigma, _p(out)))
    return out


def hadamard_joint_n(mats):
    """hadamard_joint over any number of kernels (kernel.cpp:74-101, canonical FNV content order)."""
    ms = [_f(m) for m in mats]
    n = ms[0].shape[0]
    arr = (_D * len(ms))(*[_p(m) for m in ms])
    out = np.empty((n, n), order="F")
    _chk(lib().oracle_hadamard_joint_n(arr, len(ms), n, _p(out)))
    return out


def polynomial_gram(x, degree, offset):
    x = _f(x)
    out = np.empty((x.shape[0], x.shape[0]), order="F")
    _chk(lib().oracle_polynomial_gram(_p(x), x.shape[0], x.shape[1], int(degree), float(offset), _p(out)))
    return out


def build_kernel_polynomial(x, degree, offset):
    """build_kernel(X, PolynomialKernel{degree, offset}) (kernel.cpp:35-72, ops.cpp:22-28)."""
    x = _f(x)
    out = np.empty((x.shape[0], x.shape[0]), order="F")
    _chk(lib().oracle_build_kernel_polynomial(_p(x), x.shape[0], x.shape[1], int(degree), float(offset), _p(out)))
    return out


def hadamard_joint(a, b):
    a, b = _f(a), _f(b)
    out = np.empty_like(a, order="F")
    _chk(lib().oracle_hadamard_joint(_p(a), a.shape[0], _p(b), b.shape[0], _p(out)))
    return out


def matvec(a, x):
    a = _f(a)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(a.shape[0])
    _chk(lib().oracle_matvec(_p(a), a.shape[0], _p(x), _p(y)))
    return y


def matmul_panel(a, x):
    a, x = _f(a), _f(x)
    y = np.empty((a.shape[0], x.shape[1]), order="F")
    _chk(lib().oracle_matmul_panel(_p(a), a.shape[0], _p(x), x.shape[1], _p(y)))
    return y


# ---- poly ----
@dataclass
class Spec:
    kind: str
    alpha: float
    m: int = 0
    u: float = 0.0
    v: float = 1.0

    def args(self):
        return (KINDS[self.kind], float(self.alpha), int(self.m), float(self.u), float(self.v))


def apply_panel(spec: Spec, a, x):
    a, x = _f(a), _f(x)
    if x.ndim == 1:
        x = x.reshape(-1, 1, order="F")
    y = np.empty_like(x, order="F")
    _chk(lib().oracle_apply_panel(*spec.args(), _p(a), a.shape[0], _p(x), x.shape[1], _p(y)))
    return y


def scalar_value(spec: Spec, lam):
    out = C.c_double()
    _chk(lib().oracle_scalar_value(*spec.args(), lam, C.byref(out)))
    return out.value


def spec_coeffs(spec: Spec):
    n = max(spec.m, 0) + 1
    c = np.empty(n)
    sv = C.c_double()
    _chk(lib().oracle_spec_coeffs(*spec.args(), _p(c), C.byref(sv)))
    return c, sv.value


def binomial_coeffs(alpha, m):
    out = np.empty(m + 1)
    _chk(lib().oracle_binomial_coeffs(alpha, m, _p(out)))
    return out


def chebyshev_coeffs(alpha, m, u, v):
    out = np.empty(m + 1)
    _chk(lib().oracle_chebyshev_coeffs(alpha, m, u, v, _p(out)))
    return out


def taylor_tail_constant(alpha, k_max=10000):
    return lib().oracle_taylor_tail_constant(alpha, k_max)


def safeguard(u, v):
    return lib().oracle_safeguard(u, v)


def expected_queries(spec: Spec, s):
    return int(lib().oracle_expected_queries(*spec.args(), s))


# ---- spectrum ----
def power_method(a, max_iters=100, tol=1e-6, seed=0):
    a = _f(a)
    r, it, cv = C.c_double(), C.c_int(), C.c_int()
    _chk(lib().oracle_power_method(_p(a), a.shape[0], max_iters, tol, _u64(seed), C.byref(r), C.byref(it),
                                   C.byref(cv)))
    return r.value, it.value, bool(cv.value)


def estimate_bounds(a, max_iters=100, tol=1e-6, seed=0, rank_floor=1e-12):
    a = _f(a)
    o = COut()
    _chk(lib().oracle_estimate_bounds(_p(a), a.shape[0], max_iters, tol, _u64(seed), rank_floor, C.byref(o)))
    return dict(u=o.bu, v=o.bv, kappa=o.kappa, iterations_used=o.iterations_used, v_converged=bool(o.v_converged),
                u_converged=bool(o.u_converged), rank_deficient=bool(o.rank_deficient))


def colpiv_rank(y, threshold=1e-12, want_q=False):
    y = _f(y)
    r = C.c_int()
    q = np.empty(y.shape, order="F") if want_q else None
    _chk(lib().oracle_colpiv_rank(_p(y), y.shape[0], y.shape[1], threshold, C.byref(r),
                                  _p(q) if want_q else None))
    return (r.value, q[:, :r.value]) if want_q else r.value


# ---- hutchpp / entropy ----
def _out(o: COut):
    return dict(entropy=o.entropy, value=o.trace, trace=o.trace, low_rank_part=o.low, residual_part=o.residual,
                method=o.method, s=o.s, m=o.m, queries_used=o.queries, sketch_rank=o.rank, exact=bool(o.exact),
                deterministic=bool(o.deterministic), has_bounds=bool(o.has_bounds), u=o.bu, v=o.bv,
                kappa=o.kappa, iterations_used=o.iterations_used)


def hutchpp(spec: Spec, a, s_q, s_g, seed=0, probe_kind="gaussian", sketch=None, probes=None):
    a = _f(a)
    S = _f(sketch) if sketch is not None else None
    G = _f(probes) if probes is not None else None
    o = COut()
    _chk(lib().oracle_hutchpp(*spec.args(), _p(a), a.shape[0], s_q, s_g, _u64(seed), PROBES[probe_kind],
                              _p(S) if S is not None else None, _p(G) if G is not None else None, C.byref(o)))
    return _out(o)


def estimate(a, alpha=2.0, method="auto", s=0, m=0, epsilon=1e-2, delta=1e-2, seed=0, bounds=None,
             probe_kind="gaussian", s_q=None, s_g=None, power_max_iters=100, power_tol=1e-6):
    a = _f(a)
    p = CParams(alpha, METHODS[method], s, m, epsilon, delta, _u64(seed), power_max_iters, power_tol, 0, 1e-12,
                1 if bounds is not None else 0, bounds[0] if bounds else 0.0, bounds[1] if bounds else 1.0,
                PROBES[probe_kind], -1 if s_q is None else s_q, -1 if s_g is None else s_g)
    o = COut()
    _chk(lib().oracle_estimate(_p(a), a.shape[0], C.byref(p), C.byref(o)))
    return _out(o)


def _params(alpha=2.0, method="auto", s=0, m=0, epsilon=1e-2, delta=1e-2, seed=0, bounds=None,
            probe_kind="gaussian", s_q=None, s_g=None, power_max_iters=100, power_tol=1e-6):
    return CParams(alpha, METHODS[method], s, m, epsilon, delta, _u64(seed), power_max_iters, power_tol, 0, 1e-12,
                   1 if bounds is not None else 0, bounds[0] if bounds else 0.0, bounds[1] if bounds else 1.0,
                   PROBES[probe_kind], -1 if s_q is None else s_q, -1 if s_g is None else s_g)


def _cstrs(items):
    if items is None:
        return None
    arr = (C.c_char_p * len(items))()
    arr[:] = [str(v).encode() for v in items]
    return arr


def rank_features(x, labels, sigma, k, names=None, **params):
    """rank_features (features.cpp:95-123) -> (columns, scores) of the top k."""
    x = _f(x)
    cols = (C.c_int * k)()
    scores = np.empty(k)
    prm = _params(**params)
    _chk(lib().oracle_rank_features(_p(x), x.shape[0], x.shape[1], _cstrs(labels), len(labels or []), _cstrs(names),
                                    float(sigma),
                                    C.cast(C.byref(prm), C.c_void_p), k, cols, _p(scores)))
    return list(cols), scores


def select_features(x, labels, sigma, k, names=None, **params):
    """select_features (features.cpp:125-162) -> (columns in pick order, objective after each pick)."""
    x = _f(x)
    cols = (C.c_int * k)()
    obj = np.empty(k)
    prm = _params(**params)
    _chk(lib().oracle_select_features(_p(x), x.shape[0], x.shape[1], _cstrs(labels), len(labels or []),
                                      _cstrs(names), float(sigma),
                                      C.cast(C.byref(prm), C.c_void_p), k, cols, _p(obj)))
    return list(cols), obj


def eigvals(a):
    a = _f(a)
    out = np.empty(a.shape[0])
    _chk(lib().oracle_eigvals(_p(a), a.shape[0], _p(out)))
    return out


def entropy_from_trace(trace, alpha):
    out = C.c_double()
    _chk(lib().oracle_entropy_from_trace(trace, alpha, C.byref(out)))
    return out.value


def entropy_exact(a, alpha):
    return estimate(a, alpha=alpha, method="exact")["entropy"]


def select_params(alpha, epsilon, delta, u, v, kappa, n, method):
    s, m = C.c_int(), C.c_int()
    _chk(lib().oracle_select_params(alpha, epsilon, delta, u, v, kappa, n, METHODS[method], C.byref(s), C.byref(m)))
    return s.value, m.value


def mu_bound(u, v, alpha, n):
    mu, lo, hi = C.c_double(), C.c_double(), C.c_double()
    _chk(lib().oracle_mu_bound(u, v, alpha, n, C.byref(mu), C.byref(lo), C.byref(hi)))
    return mu.value, lo.value, hi.value


def mutual_information(a, b, **params):
    """measures.cpp:36-46 with per-term seeds."""
    seed = params.pop("seed", 0)
    j = hadamard_joint(a, b)
    sv = estimate(a, seed=derive_key(seed, hash_name("term:vars")), **params)["entropy"]
    st = estimate(b, seed=derive_key(seed, hash_name("term:target")), **params)["entropy"]
    sj = estimate(j, seed=derive_key(seed, hash_name("term:joint")), **params)["entropy"]
    return dict(value=sv + st - sj, vars_entropy=sv, target_entropy=st, joint_entropy=sj)


def threads():
    return lib().oracle_threads()


def set_threads(t):
    lib().oracle_set_threads(t)


def slab_sample_seconds(x, sigma, r0, h, sketch_cols, passes, cols_q, cols_w):
    """Seconds for rows [r0, r0+h) of one estimate: Gram rows + sketch pass + `passes` (Q, W) passes."""
    x = _f(x)
    return lib().oracle_slab_sample(_p(x), x.shape[0], x.shape[1], sigma, r0, h, sketch_cols, passes, cols_q, cols_w)


def load_csv(text, label_column=None, source=None):
    """load_csv (proj/src/csv.cpp:63-115) restated over a buffer with glibc std::strtod.
    Returns dict(n, d, features (n x d), names, labels) or raises OracleError(10, message)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    _chk(lib().oracle_csv_parse(data, len(data), label_column.encode() if label_column else None,
                                source.encode() if source else None, C.byref(h)))
    try:
        n, d, hl = C.c_int64(), C.c_int64(), C.c_int()
        lib().oracle_csv_shape(h, C.byref(n), C.byref(d), C.byref(hl))
        x = np.empty((n.value, d.value), dtype=np.float64, order="F")
        if x.size:
            lib().oracle_csv_features(h, x.ctypes.data_as(_D))

        def strings(which, count):
            out = []
            for i in range(count):
                size = lib().oracle_csv_string(h, which, i, None, 0)
                buf = C.create_string_buffer(max(size, 1))
                lib().oracle_csv_string(h, which, i, buf, size)
                out.append(buf.raw[:size].decode("utf-8", errors="surrogateescape"))
            return out

        return dict(n=n.value, d=d.value, features=x, names=strings(0, d.value),
                    labels=strings(1, n.value) if hl.value else [])
    finally:
        lib().oracle_csv_free(h)


# ---- matrix-free (kernel entries recomputed from the samples; full-size fixtures) ----
def _mf_args(x, sigma, y=None, sigma_y=None):
    x = _f(x)
    yy = _f(y) if y is not None else None
    keep = (x, yy)
    args = (_p(x), x.shape[0], x.shape[1], float(sigma), _p(yy) if yy is not None else None,
            yy.shape[1] if yy is not None else 0, float(sigma_y or 0.0))
    return keep, args


def mf_matmul(x, sigma, v, y=None, sigma_y=None):
    """A·V with A = build_kernel(X, sigma) (or the joint n·A∘B of X, Y), never stored."""
    keep, args = _mf_args(x, sigma, y, sigma_y)
    v = _f(v)
    out = np.empty((x.shape[0], v.shape[1]), order="F")
    _chk(lib().oracle_mf_matmul(*args, _p(v), v.shape[1], _p(out)))
    return out


def mf_estimate(x, sigma, y=None, sigma_y=None, **params):
    """estimate(build_kernel(X, sigma) [∘ joint with Y], params) without storing A."""
    keep, args = _mf_args(x, sigma, y, sigma_y)
    p = _params(**params)
    o = COut()
    _chk(lib().oracle_mf_estimate(*args, C.byref(p), C.byref(o)))
    return _out(o)


def mf_matfun_traces(spec: Spec, x, sigma, probes, y=None, sigma_y=None):
    keep, args = _mf_args(x, sigma, y, sigma_y)
    q = _f(probes)
    out = np.empty(q.shape[1])
    _chk(lib().oracle_mf_matfun_traces(*args, *spec.args(), _p(q), q.shape[1], _p(out)))
    return out


def mf_mutual_information(x, sigma_x, y, sigma_y, **params):
    """measures.cpp:36-46 (per-term seeds) over the three kernels, none stored."""
    seed = params.pop("seed", 0)
    tv = mf_estimate(x, sigma_x, seed=derive_key(seed, hash_name("term:vars")), **params)
    tt = mf_estimate(y, sigma_y, seed=derive_key(seed, hash_name("term:target")), **params)
    tj = mf_estimate(x, sigma_x, y, sigma_y, seed=derive_key(seed, hash_name("term:joint")), **params)
    return dict(value=tv["entropy"] + tt["entropy"] - tj["entropy"], vars_entropy=tv["entropy"],
                target_entropy=tt["entropy"], joint_entropy=tj["entropy"], terms=dict(vars=tv, target=tt, joint=tj))


class KernelBlocksOp:
    """y = A x for A = build_kernel(X, sigma) (or the joint n·A∘B with Y) in square blocks,
    never stored: feature dots by BLAS (X_I X_J^T), entries by oracle_kernel_block (the
    reference's d2/clamp/exp/normalisation arithmetic), both triangles from one block, products
    by BLAS. The estimator itself is the restated C++ one (oracle_cb_*), called back through
    ctypes. Differs from GaussOp (bit-exact entries) only in BLAS summation order (~1e-15, checked
    in tests/test_oracle_fullsize.py)."""

    def __init__(self, x, sigma, y=None, sigma_y=None, block=4096):
        self.n = x.shape[0]
        self.block = block
        self.inv_n = 1.0 / self.n
        self.feats = []
        for z, sg in ((x, sigma), (y, sigma_y)):
            if z is None:
                continue
            z = np.ascontiguousarray(z, dtype=np.float64)
            sq = np.zeros(self.n)
            for k in range(z.shape[1]):  # rowwise sum of squares in feature order (ops.cpp:41)
                sq += z[:, k] * z[:, k]
            self.feats.append((z, sq, 1.0 / (2.0 * sg * sg)))
        self.calls = 0
        self._fn = MUL_FN(self._cb)

    def kernel_block(self, i0, i1, j0, j1):
        out = np.empty((i1 - i0, j1 - j0))
        for f, (z, sq, inv2) in enumerate(self.feats):
            sqi, sqj = np.ascontiguousarray(sq[i0:i1]), np.ascontiguousarray(sq[j0:j1])
            if z.shape[1] <= 64:  # few features: dots in feature order in C (BLAS is slow at small K)
                zi, zjt = np.ascontiguousarray(z[i0:i1]), np.ascontiguousarray(z[j0:j1].T)
                lib().oracle_kernel_block_rows(_p(zi), _p(zjt), i1 - i0, j1 - j0, z.shape[1], _p(sqi), _p(sqj),
                                               inv2, self.inv_n, float(self.n), 1 if f else 0, _p(out))
                continue
            dot = np.ascontiguousarray(z[i0:i1] @ z[j0:j1].T)
            lib().oracle_kernel_block(_p(dot), i1 - i0, j1 - j0, _p(sqi), _p(sqj), inv2, self.inv_n,
                                      float(self.n), 1 if f else 0, _p(out))
        if i0 == j0:
            np.fill_diagonal(out, self.inv_n)
        return out

    def mul(self, v):
        n, b = self.n, self.block
        y = np.zeros_like(v)
        for i0 in range(0, n, b):
            i1 = min(n, i0 + b)
            for j0 in range(i0, n, b):
                j1 = min(n, j0 + b)
                k = self.kernel_block(i0, i1, j0, j1)
                y[i0:i1] += k @ v[j0:j1]
                if j0 != i0:
                    y[j0:j1] += k.T @ v[i0:i1]
        return y

    def _cb(self, n, c, x, out):
        try:
            v = np.ctypeslib.as_array(x, shape=(c, n)).T  # column-major n x c
            y = self.mul(np.ascontiguousarray(v))
            np.ctypeslib.as_array(out, shape=(c, n))[...] = y.T
            self.calls += 1
            return 0
        except Exception:  # reported as a failed callback by the C++ side
            import traceback

            traceback.print_exc()
            return 1

    def estimate(self, **params):
        p = _params(**params)
        o = COut()
        _chk(lib().oracle_cb_estimate(self.n, self._fn, C.byref(p), C.byref(o)))
        return _out(o)

    def matfun_traces(self, spec: Spec, probes):
        q = _f(probes)
        out = np.empty(q.shape[1])
        _chk(lib().oracle_cb_matfun_traces(self.n, self._fn, *spec.args(), _p(q), q.shape[1], _p(out)))
        return out


def blocks_mutual_information(x, sigma_x, y, sigma_y, block=4096, **params):
    """measures.cpp:36-46 (per-term seeds) over KernelBlocksOp operators."""
    seed = params.pop("seed", 0)
    tv = KernelBlocksOp(x, sigma_x, block=block).estimate(seed=derive_key(seed, hash_name("term:vars")), **params)
    tt = KernelBlocksOp(y, sigma_y, block=block).estimate(seed=derive_key(seed, hash_name("term:target")), **params)
    tj = KernelBlocksOp(x, sigma_x, y, sigma_y, block=block).estimate(seed=derive_key(seed, hash_name("term:joint")),
                                                                      **params)
    return dict(value=tv["entropy"] + tt["entropy"] - tj["entropy"], vars_entropy=tv["entropy"],
                target_entropy=tt["entropy"], joint_entropy=tj["entropy"], terms=dict(vars=tv, target=tt, joint=tj))


def set_merge_panels(on: bool):
    """Hutch++ applies f(A) to [Q, W - Q(Q^T W)] in one apply_panel instead of two (the same
    per-column recurrences, half the operator passes). Off by default (the reference's
    structure); on only for the one-off full-size fixtures."""
    lib().oracle_set_merge_panels(1 if on else 0)


class _Lockstep:
    """Runs several callback estimators in threads whose operator calls are served together:
    each call posts its panel and waits until every active estimator has posted one, then one
    sweep over the kernel blocks serves all of them (shared block evaluations)."""

    def __init__(self, serve):
        import threading

        self.serve = serve  # serve({term: v}) -> {term: y}
        self.cv = threading.Condition()
        self.active = set()
        self.pending = {}
        self.results = {}
        self.gen = 0
        self.error = None

    def _run_if_ready(self):
        if self.pending and set(self.pending) >= self.active:
            reqs, self.pending = self.pending, {}
            try:
                self.results = self.serve(reqs)
            except Exception as e:  # surfaced to every waiting estimator
                self.error = e
                self.results = {}
            self.gen += 1
            self.cv.notify_all()

    def fn(self, term):
        def cb(n, c, x, out):
            try:
                v = np.ascontiguousarray(np.ctypeslib.as_array(x, shape=(c, n)).T)
                with self.cv:
                    self.pending[term] = v
                    g = self.gen
                    self._run_if_ready()
                    while self.gen == g:
                        self.cv.wait()
                    if self.error is not None:
                        return 1
                    y = self.results.pop(term)
                np.ctypeslib.as_array(out, shape=(c, n))[...] = y.T
                return 0
            except Exception:
                import traceback

                traceback.print_exc()
                return 1

        return MUL_FN(cb)

    def run(self, n, jobs):
        """jobs: {term: params dict} -> {term: estimate dict}"""
        import threading

        out, errs, fns = {}, {}, {t: self.fn(t) for t in jobs}
        self.active = set(jobs)

        def work(term):
            try:
                p = _params(**jobs[term])
                o = COut()
                _chk(lib().oracle_cb_estimate(n, fns[term], C.byref(p), C.byref(o)))
                out[term] = _out(o)
            except Exception as e:
                errs[term] = e
            finally:
                with self.cv:
                    self.active.discard(term)
                    self._run_if_ready()

        ths = [threading.Thread(target=work, args=(t,)) for t in jobs]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if errs:
            raise next(iter(errs.values()))
        return out


def lockstep_mutual_information(x, sigma_x, y, sigma_y, block=4096, **params):
    """measures.cpp:36-46 (per-term seeds) like blocks_mutual_information, with the three terms'
    operator passes served together: one evaluation of the A and B blocks per sweep gives the
    vars, target and joint (n·A∘B, hadamard_scaled's scale·(a·b)) blocks. Same estimator, same
    blocks as KernelBlocksOp; only the scheduling differs."""
    seed = params.pop("seed", 0)
    ox = KernelBlocksOp(x, sigma_x, block=block)
    oy = KernelBlocksOp(y, sigma_y, block=block)
    n = ox.n
    scale = float(n)

    def serve(reqs):
        ys = {t: np.zeros_like(v) for t, v in reqs.items()}
        for i0 in range(0, n, block):
            i1 = min(n, i0 + block)
            for j0 in range(i0, n, block):
                j1 = min(n, j0 + block)
                ka = ox.kernel_block(i0, i1, j0, j1) if ("vars" in reqs or "joint" in reqs) else None
                kb = oy.kernel_block(i0, i1, j0, j1) if ("target" in reqs or "joint" in reqs) else None
                blocks = {"vars": ka, "target": kb}
                if "joint" in reqs:
                    kj = scale * (ka * kb)
                    if i0 == j0:
                        np.fill_diagonal(kj, 1.0 / n)
                    blocks["joint"] = kj
                for t, v in reqs.items():
                    k = blocks[t]
                    ys[t][i0:i1] += k @ v[j0:j1]
                    if j0 != i0:
                        ys[t][j0:j1] += k.T @ v[i0:i1]
        return ys

    terms = {"vars": "term:vars", "target": "term:target", "joint": "term:joint"}
    jobs = {t: dict(params, seed=derive_key(seed, hash_name(lbl))) for t, lbl in terms.items()}
    est = _Lockstep(serve).run(n, jobs)
    tv, tt, tj = est["vars"], est["target"], est["joint"]
    return dict(value=tv["entropy"] + tt["entropy"] - tj["entropy"], vars_entropy=tv["entropy"],
                target_entropy=tt["entropy"], joint_entropy=tj["entropy"], terms=est)
