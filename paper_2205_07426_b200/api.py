"""Python mirror of the reference C++ API (proj/include/renyi/*.hpp) over the
C ABI of librenyi_b200.so. Names, argument meaning and error behaviour follow
the reference so parity tests read like its own doctest suites; the arrays are
numpy (host, column-major semantics of Eigen's MatrixXd: shape (rows, cols)).

Every compute call runs on the B200 through the C ABI. The only exception is
entropy_exact, which the reference itself uses as an O(n^3) check oracle
(proj/src/entropy.cpp:71-90): it runs torch.linalg.eigvalsh on the CUDA device.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import RenyiError, check

F64 = 0
F32 = 1
MF = 2  # matrix-free: bf16 samples, kernel entries recomputed per pass, A never stored
PRECISIONS = {"fp64": F64, "f64": F64, "float64": F64, F64: F64, "fp32": F32, "f32": F32, "float32": F32, F32: F32,
              "mf": MF, "matrix_free": MF, "bf16_mf": MF, MF: MF}

METHODS = {"exact": 0, "int": 1, "int_power": 1, "taylor": 2, "chebyshev": 3, "auto": 4}
METHOD_NAMES = {0: "exact", 1: "int", 2: "taylor", 3: "chebyshev", 4: "auto"}
PROBES = {"gaussian": 0, "rademacher": 1}


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _colmajor(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------- context
class Context:
    """One device context (stream, scratch, tuning). Not shared across threads."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(L.lib().renyi_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def set_tuning(self, grid: int = 0, kc: int = 16) -> None:
        check(L.lib().renyi_ctx_set_tuning(self._h, grid, kc))

    def set_matrix_free_chunk(self, jblocks: int = 4) -> None:
        """Matrix-free product: j-blocks of 128 samples accumulated in TMEM between fp32 drains."""
        check(L.lib().renyi_ctx_set_matrix_free_chunk(self._h, jblocks))

    def set_operand_mode(self, mode: str = "split") -> None:
        """'split' (default; V as fp16 hi+lo, 3 MMAs), 'fast' (V hi only, 2 MMAs) or 'auto' (split
        where vectors are returned, fast for trace-only passes)."""
        check(L.lib().renyi_ctx_set_operand_mode(self._h, {"split": 0, "fast": 1, "auto": 2}[mode]))

    def set_fused_mi(self, on: bool = True) -> None:
        """Mutual information over fp32 kernels: one pass over A and B serves all three terms (the
        joint kernel n·A∘B is formed on the fly, never stored); False: three separate estimates."""
        check(L.lib().renyi_ctx_set_fused_mi(self._h, 1 if on else 0))

    def set_feature_grouping(self, on: bool = True) -> None:
        """rank_features / select_features over fp32 kernels: score each step's candidates as grouped
        stacks (default) or one at a time (the reference's loop)."""
        check(L.lib().renyi_ctx_set_feature_grouping(self._h, 1 if on else 0))

    def set_probe_source(self, source: str = "device") -> None:
        """Seeded Gaussian probes: "device" (default; CUDA log/sin/cos, <= 2 ulp per draw from the
        reference's glibc draws) or "host" (the reference's own arithmetic on the host threads: bitwise
        the reference's probes, copied to the device; overlapped with the kernel builds for mutual
        information)."""
        codes = {"device": 0, "host": 1}
        if source not in codes:
            raise ValueError(f"probe source must be one of {sorted(codes)}")
        check(L.lib().renyi_ctx_set_probe_source(self._h, codes[source]))

    def sync(self) -> None:
        check(L.lib().renyi_ctx_sync(self._h))

    def profile(self, enable: bool) -> None:
        check(L.lib().renyi_ctx_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """(launches, device ms, algorithmic bytes, flops) of block products since profile(True)."""
        n = C.c_int()
        ms, b, f = C.c_double(), C.c_double(), C.c_double()
        check(L.lib().renyi_ctx_profile_read(self._h, C.byref(n), C.byref(ms), C.byref(b), C.byref(f)))
        return n.value, ms.value, b.value, f.value

    def io_bytes(self):
        h, d = C.c_longlong(), C.c_longlong()
        check(L.lib().renyi_ctx_io_bytes(self._h, C.byref(h), C.byref(d)))
        return h.value, d.value

    def timer_begin(self) -> None:
        check(L.lib().renyi_ctx_timer_begin(self._h))

    def timer_end(self) -> float:
        ms = C.c_double()
        check(L.lib().renyi_ctx_timer_end(self._h, C.byref(ms)))
        return ms.value

    def init_nccl(self, rank: int, world: int, unique_id: bytes) -> None:
        """Join an NCCL group (one process per GPU); unique_id from nccl_unique_id() on rank 0."""
        if len(unique_id) != 128:
            raise RenyiError(1, "NCCL unique id must be 128 bytes")
        check(L.lib().renyi_ctx_init_nccl(self._h, rank, world, unique_id))

    def join_local_group(self, group: "LocalGroup", rank: int) -> None:
        check(L.lib().renyi_ctx_join_local_group(self._h, group.handle, rank))

    def rank_world(self):
        r, w = C.c_int(), C.c_int()
        check(L.lib().renyi_ctx_rank(self._h, C.byref(r), C.byref(w)))
        return r.value, w.value

    def launch_count(self) -> int:
        n = C.c_long()
        check(L.lib().renyi_ctx_launch_count(self._h, C.byref(n)))
        return n.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().renyi_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """Ranks as threads of this process (host-driven collectives), e.g. to validate the sharded path."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(L.lib().renyi_local_group_create(world, C.byref(h)))
        self._h = h
        self.world = world

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                L.lib().renyi_local_group_destroy(self._h)
                self._h = None
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(L.lib().renyi_nccl_unique_id(buf))
    return buf.raw


def shard_rows(n: int, world: int, rank: int):
    """(row0, rows, rows_per_rank) of this rank's row block of A."""
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    check(L.lib().renyi_shard_rows(n, world, rank, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def release_cached_memory() -> None:
    """Returns the engine's cached device blocks to the driver."""
    check(L.lib().renyi_release_cached_memory())


_default = threading.local()


def default_context() -> Context:
    ctx = getattr(_default, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _default.ctx = ctx
    return ctx


# ---------------------------------------------------------------- kernels (kernel.hpp)
@dataclass
class GaussianKernel:
    sigma: float = 1.0


@dataclass
class PolynomialKernel:  # proj/include/renyi/kernel.hpp:16-19
    degree: int = 2
    offset: float = 1.0


class NormalizedKernel:
    """Device-resident trace-one kernel matrix (proj/include/renyi/kernel.hpp:27-42)."""

    def __init__(self, handle, ctx: Context, precision: int):
        self._h = handle
        self.ctx = ctx
        self.precision = precision

    @classmethod
    def from_matrix(cls, a, precision="fp64", ctx: Optional[Context] = None) -> "NormalizedKernel":
        ctx = ctx or default_context()
        a = _colmajor(a)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise RenyiError(4, "NormalizedKernel needs a square matrix")
        h = C.c_void_p()
        check(L.lib().renyi_kernel_from_matrix(ctx.handle, _dptr(a), a.shape[0], PRECISIONS[precision], C.byref(h)))
        return cls(h, ctx, PRECISIONS[precision])

    def size(self) -> int:
        n = C.c_int64()
        check(L.lib().renyi_kernel_size(self._h, C.byref(n)))
        return n.value

    def matrix(self) -> np.ndarray:
        n = self.size()
        out = np.empty((n, n), dtype=np.float64, order="F")
        check(L.lib().renyi_kernel_download(self.ctx.handle, self._h, _dptr(out)))
        return out

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                L.lib().renyi_kernel_destroy(self._h)
                self._h = None
        except Exception:
            pass


def build_kernel(samples, spec: GaussianKernel, precision="fp64", ctx: Optional[Context] = None) -> NormalizedKernel:
    """build_kernel (proj/src/kernel.cpp:35-72); samples: (n, d) rows = samples."""
    ctx = ctx or default_context()
    x = _colmajor(samples)
    if x.ndim != 2:
        raise RenyiError(1, "samples must be a 2-D array")
    h = C.c_void_p()
    n, d = x.shape
    if isinstance(spec, PolynomialKernel):
        check(L.lib().renyi_kernel_build_polynomial(ctx.handle, _dptr(x), n, d, max(n, 1), int(spec.degree),
                                                    float(spec.offset), PRECISIONS[precision], C.byref(h)))
        return NormalizedKernel(h, ctx, PRECISIONS[precision])
    if not isinstance(spec, GaussianKernel):
        raise RenyiError(1, "kernel spec must be GaussianKernel or PolynomialKernel")
    check(L.lib().renyi_kernel_build_gaussian(ctx.handle, _dptr(x), n, d, max(n, 1), spec.sigma,
                                              PRECISIONS[precision], C.byref(h)))
    return NormalizedKernel(h, ctx, PRECISIONS[precision])


def build_joint_kernel(x, sx: GaussianKernel, y, sy: GaussianKernel, precision="fp64",
                       ctx: Optional[Context] = None) -> NormalizedKernel:
    """hadamard_joint({build_kernel(x), build_kernel(y)}) fused from samples."""
    ctx = ctx or default_context()
    xa, ya = _colmajor(x), _colmajor(y)
    if xa.shape[0] != ya.shape[0]:
        raise RenyiError(4, "input and target sample counts differ")
    h = C.c_void_p()
    check(L.lib().renyi_kernel_build_gaussian_joint(ctx.handle, _dptr(xa), xa.shape[0], xa.shape[1], xa.shape[0],
                                                    sx.sigma, _dptr(ya), ya.shape[1], ya.shape[0], sy.sigma,
                                                    PRECISIONS[precision], C.byref(h)))
    return NormalizedKernel(h, ctx, PRECISIONS[precision])


def hadamard_joint(kernels: Sequence[NormalizedKernel]) -> NormalizedKernel:
    """hadamard_joint (proj/src/kernel.cpp:74-101)."""
    if len(kernels) < 2:
        raise RenyiError(1, "hadamard_joint needs at least 2 kernels")
    ctx = kernels[0].ctx
    arr = (C.c_void_p * len(kernels))(*[k.handle for k in kernels])
    h = C.c_void_p()
    check(L.lib().renyi_kernel_hadamard_joint_n(ctx.handle, arr, len(kernels), C.byref(h)))
    return NormalizedKernel(h, ctx, kernels[0].precision)


# ---------------------------------------------------------------- ops (ops.hpp)
class ops:  # namespace mirror of renyi::ops
    @staticmethod
    def matmul_panel(a: NormalizedKernel, x) -> np.ndarray:
        """Y = A X (proj/src/ops.cpp:98-107)."""
        xa = _colmajor(x)
        if xa.ndim == 1:
            xa = xa.reshape(-1, 1, order="F")
        n = a.size()
        if xa.shape[0] != n:
            raise RenyiError(4, f"matmul_panel: matrix is {n}x{n}, panel has {xa.shape[0]} rows")
        y = np.empty_like(xa, order="F")
        check(L.lib().renyi_matmul_panel(a.ctx.handle, a.handle, _dptr(xa), xa.shape[1], _dptr(y)))
        return y

    @staticmethod
    def matvec(a: NormalizedKernel, x) -> np.ndarray:
        """y = A x (proj/src/ops.cpp:73-85)."""
        return ops.matmul_panel(a, np.asarray(x, dtype=np.float64).reshape(-1, 1))[:, 0]

    @staticmethod
    def gaussian_gram(samples, sigma: float, ctx: Optional[Context] = None) -> np.ndarray:
        """K_ij = exp(-||x_i - x_j||^2 / (2 sigma^2)), unnormalised (proj/src/ops.cpp:9-20,39-47)."""
        ctx = ctx or default_context()
        x = _colmajor(samples)
        n, d = x.shape
        k = np.empty((n, n), order="F")
        check(L.lib().renyi_ops_gaussian_gram(ctx.handle, _dptr(x), n, d, max(n, 1), float(sigma), _dptr(k)))
        return k

    @staticmethod
    def polynomial_gram(samples, degree: int, offset: float, ctx: Optional[Context] = None) -> np.ndarray:
        """K_ij = (x_i . x_j + offset)^degree, unnormalised (proj/src/ops.cpp:22-28,58-64)."""
        ctx = ctx or default_context()
        x = _colmajor(samples)
        n, d = x.shape
        k = np.empty((n, n), order="F")
        check(L.lib().renyi_ops_polynomial_gram(ctx.handle, _dptr(x), n, d, max(n, 1), int(degree), float(offset),
                                                _dptr(k)))
        return k

    @staticmethod
    def hadamard_scaled(a, b, scale: float, ctx: Optional[Context] = None) -> np.ndarray:
        """C = scale * (A o B) elementwise (proj/src/ops.cpp:116-122)."""
        ctx = ctx or default_context()
        am, bm = _colmajor(a), _colmajor(b)
        if am.shape != bm.shape or am.ndim != 2:
            raise RenyiError(4, "hadamard_scaled: matrices must have the same 2-D shape")
        c = np.empty_like(am, order="F")
        check(L.lib().renyi_ops_hadamard_scaled(ctx.handle, _dptr(am), _dptr(bm), am.shape[0], am.shape[1],
                                                float(scale), _dptr(c)))
        return c


# ---------------------------------------------------------------- matrix functions (poly.hpp)
def binomial_coeffs(alpha: float, m: int) -> np.ndarray:
    out = np.empty(max(m + 1, 1))
    check(L.lib().renyi_binomial_coeffs(alpha, m, _dptr(out)))
    return out


def chebyshev_coeffs(alpha: float, m: int, u: float, v: float) -> np.ndarray:
    out = np.empty(max(m + 1, 1))
    check(L.lib().renyi_chebyshev_coeffs(alpha, m, u, v, _dptr(out)))
    return out


_SCALAR_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)


class RandomStream:
    """RandomStream (proj/include/renyi/rng.hpp:12-36): the reference's host stream, bit for bit."""

    def __init__(self, key: int = 0, _handle=None):
        self._h = _handle
        if self._h is None:
            self._h = C.c_void_p()
            check(L.lib().renyi_rng_create(int(key) & (2**64 - 1), C.byref(self._h)))

    def derive(self, tag: int) -> "RandomStream":
        h = C.c_void_p()
        check(L.lib().renyi_rng_derive(self._h, int(tag) & (2**64 - 1), C.byref(h)))
        return RandomStream(_handle=h)

    def key(self) -> int:
        return int(L.lib().renyi_rng_key(self._h))

    def next_u64(self) -> int:
        return int(L.lib().renyi_rng_next_u64(self._h))

    def next_uniform(self) -> float:
        return float(L.lib().renyi_rng_next_uniform(self._h))

    def next_gaussian(self) -> float:
        return float(L.lib().renyi_rng_next_gaussian(self._h))

    def fill_gaussian(self, rows: int, cols: int = 1) -> np.ndarray:
        """A rows x cols panel filled column-wise (rng.cpp:60-64)."""
        out = np.empty((rows, cols), order="F")
        check(L.lib().renyi_rng_fill_gaussian(self._h, rows, cols, _dptr(out)))
        return out

    def __del__(self):
        try:
            if self._h:
                L.lib().renyi_rng_destroy(self._h)
                self._h = None
        except Exception:
            pass


def chebyshev_node_coeffs(f, m: int, a: float, b: float) -> np.ndarray:
    """Chebyshev coefficients of f on [a, b] from the m + 1 first-kind nodes (proj/src/poly.cpp:18-40)."""
    out = np.empty(max(m + 1, 1))
    cb = _SCALAR_FN(lambda x, _user: float(f(x)))
    check(L.lib().renyi_chebyshev_node_coeffs(C.cast(cb, C.c_void_p), None, m, a, b, _dptr(out)))
    return out


def method_name(method) -> str:
    """method_name (proj/src/entropy.cpp:51-60)."""
    code = METHODS[method] if isinstance(method, str) else int(method)
    return L.lib().renyi_method_name(code).decode()


def chebyshev_safeguard(u: float, v: float) -> float:
    return L.lib().renyi_chebyshev_safeguard(u, v)


def taylor_tail_constant(alpha: float, k_max: int = 10000) -> float:
    return L.lib().renyi_taylor_tail_constant(alpha, k_max)


@dataclass
class MatrixFunctionSpec:
    kind: int
    alpha: float
    degree: int
    u: float = 0.0
    v: float = 1.0

    @staticmethod
    def int_power(alpha: int) -> "MatrixFunctionSpec":
        if alpha < 1:
            raise RenyiError(1, "int_power needs alpha >= 1")
        return MatrixFunctionSpec(0, float(alpha), int(alpha))

    @staticmethod
    def taylor(alpha: float, m: int, v: float) -> "MatrixFunctionSpec":
        s = MatrixFunctionSpec(1, float(alpha), int(m), 0.0, float(v))
        s._validate()
        return s

    @staticmethod
    def chebyshev(alpha: float, m: int, u: float, v: float) -> "MatrixFunctionSpec":
        s = MatrixFunctionSpec(2, float(alpha), int(m), float(u), float(v))
        s._validate()
        return s

    def _c(self) -> L.Matfun:
        return L.Matfun(self.kind, self.alpha, self.degree, self.u, self.v)

    def _validate(self) -> None:
        out = C.c_double()
        check(L.lib().renyi_matfun_scalar(C.byref(self._c()), 0.5, C.byref(out)))

    def query_cost(self) -> int:
        return self.degree

    @property
    def safe_v(self) -> float:
        return chebyshev_safeguard(self.u, self.v) if self.kind == 2 else self.v


def scalar_value(spec: MatrixFunctionSpec, lam: float) -> float:
    out = C.c_double()
    check(L.lib().renyi_matfun_scalar(C.byref(spec._c()), lam, C.byref(out)))
    return out.value


def apply_panel(spec: MatrixFunctionSpec, a: NormalizedKernel, x) -> np.ndarray:
    """p(A) X (proj/src/poly.cpp:158-164)."""
    xa = _colmajor(x)
    vec = xa.ndim == 1
    if vec:
        xa = xa.reshape(-1, 1, order="F")
    n = a.size()
    if xa.shape[0] != n:
        raise RenyiError(4, f"apply_panel: matrix is {n}x{n}, panel has {xa.shape[0]} rows")
    y = np.empty_like(xa, order="F")
    check(L.lib().renyi_apply_panel(a.ctx.handle, a.handle, C.byref(spec._c()), _dptr(xa), xa.shape[1], _dptr(y)))
    return y[:, 0] if vec else y


def apply(spec: MatrixFunctionSpec, a: NormalizedKernel, x) -> np.ndarray:
    """p(A) x (proj/src/poly.cpp:150-156)."""
    return apply_panel(spec, a, np.asarray(x, dtype=np.float64).reshape(-1))


def matfun_traces(spec: MatrixFunctionSpec, a: NormalizedKernel, x) -> np.ndarray:
    """Per-column x_j^T p(A) x_j, fused (no f(A)X vector is formed)."""
    xa = _colmajor(x)
    if xa.ndim == 1:
        xa = xa.reshape(-1, 1, order="F")
    out = np.empty(xa.shape[1])
    check(L.lib().renyi_matfun_traces(a.ctx.handle, a.handle, C.byref(spec._c()), _dptr(xa), xa.shape[1],
                                      _dptr(out)))
    return out


# ---------------------------------------------------------------- spectrum (spectrum.hpp)
@dataclass
class PowerOptions:
    max_iters: int = 100
    tol: float = 1e-6
    seed: int = 0
    rank_floor: float = 1e-12

    def _c(self) -> L.PowerOptionsC:
        return L.PowerOptionsC(self.max_iters, self.tol, self.seed & (2**64 - 1), self.rank_floor)


@dataclass
class SpectrumBounds:
    u: float = 0.0
    v: float = 1.0
    kappa: float = math.inf
    iterations_used: int = 0
    v_converged: bool = True
    u_converged: bool = True
    rank_deficient: bool = False

    def _c(self) -> L.SpectrumBoundsC:
        return L.SpectrumBoundsC(self.u, self.v, self.kappa, self.iterations_used, int(self.v_converged),
                                 int(self.u_converged), int(self.rank_deficient))

    @staticmethod
    def _from(c: L.SpectrumBoundsC) -> "SpectrumBounds":
        return SpectrumBounds(c.u, c.v, c.kappa, c.iterations_used, bool(c.v_converged), bool(c.u_converged),
                              bool(c.rank_deficient))


@dataclass
class PowerResult:
    rayleigh: float
    iterations: int
    converged: bool


def power_method(a: NormalizedKernel, opts: PowerOptions = PowerOptions(), shift: float = 0.0) -> PowerResult:
    out = L.PowerResultC()
    check(L.lib().renyi_power_method(a.ctx.handle, a.handle, C.byref(opts._c()), shift, C.byref(out)))
    return PowerResult(out.rayleigh, out.iterations, bool(out.converged))


def estimate_bounds(a: NormalizedKernel, opts: PowerOptions = PowerOptions()) -> SpectrumBounds:
    out = L.SpectrumBoundsC()
    check(L.lib().renyi_estimate_bounds(a.ctx.handle, a.handle, C.byref(opts._c()), C.byref(out)))
    return SpectrumBounds._from(out)


def estimate_v(a: NormalizedKernel, opts: PowerOptions = PowerOptions()) -> float:
    n = a.size()
    r = power_method(a, opts)
    return min(max(r.rayleigh * (1.0 + opts.tol), 1.0 / n), 1.0)


# ---------------------------------------------------------------- Hutch++ (hutchpp.hpp)
@dataclass
class SketchConfig:
    s: int = 8
    seed: int = 0
    s_q: Optional[int] = None  # explicit split (None: floor(s/4), s - 2 floor(s/4))
    s_g: Optional[int] = None
    probe_kind: str = "gaussian"
    sketch: Optional[np.ndarray] = None  # injected n x s_q probes
    probes: Optional[np.ndarray] = None  # injected n x s_g probes

    def split(self):
        if self.s_q is not None or self.s_g is not None:
            return int(self.s_q or 0), int(self.s_g or 0)
        return self.s // 4, self.s - 2 * (self.s // 4)


@dataclass
class TraceEstimate:
    value: float
    low_rank_part: float
    residual_part: float
    queries_used: int
    sketch_rank: int
    exact: bool


def hutchpp(f: MatrixFunctionSpec, a: NormalizedKernel, cfg: SketchConfig) -> TraceEstimate:
    """hutchpp (proj/src/hutchpp.cpp:69-115) with probe injection."""
    s_q, s_g = cfg.split()
    if cfg.s_q is None and cfg.s_g is None and cfg.s < 8:
        raise RenyiError(1, "hutchpp needs a query budget s >= 8")
    n = a.size()
    keep = []
    sk = L.Sketch(s_q, s_g, cfg.seed & (2**64 - 1), PROBES[cfg.probe_kind], None, None)
    if cfg.sketch is not None:
        m = _colmajor(cfg.sketch)
        if m.shape != (n, s_q):
            raise RenyiError(4, "sketch panel must be n x s_q")
        keep.append(m)
        sk.sketch = _dptr(m)
    if cfg.probes is not None:
        m = _colmajor(cfg.probes)
        if m.shape != (n, s_g):
            raise RenyiError(4, "probe panel must be n x s_g")
        keep.append(m)
        sk.probes = _dptr(m)
    out = L.TraceEstimateC()
    check(L.lib().renyi_hutchpp(a.ctx.handle, a.handle, C.byref(f._c()), C.byref(sk), C.byref(out)))
    return TraceEstimate(out.value, out.low_rank_part, out.residual_part, out.queries_used, out.sketch_rank,
                         bool(out.exact))


def expected_queries(f: MatrixFunctionSpec, cfg: SketchConfig) -> int:
    return int(L.lib().renyi_expected_queries(C.byref(f._c()), cfg.s))


def gaussian_panel(n: int, cols: int, seed: int, label: str, kind: str = "gaussian") -> np.ndarray:
    """detail::gaussian_panel (proj/src/hutchpp.cpp:13-22), reference RNG, host."""
    out = np.empty((n, cols), dtype=np.float64, order="F")
    check(L.lib().renyi_probe_panel(n, cols, seed & (2**64 - 1), label.encode(), PROBES[kind], _dptr(out)))
    return out


def mix64(x: int) -> int:
    return int(L.lib().renyi_mix64(x & (2**64 - 1)))


def derive_key(seed: int, tag: int) -> int:
    return int(L.lib().renyi_derive_key(seed & (2**64 - 1), tag & (2**64 - 1)))


def hash_name(name: str) -> int:
    return int(L.lib().renyi_hash_name(name.encode()))


# ---------------------------------------------------------------- estimators (entropy.hpp)
@dataclass
class EstimatorParams:
    alpha: float = 2.0
    method: str = "auto"
    s: int = 0
    m: int = 0
    epsilon: float = 1e-2
    delta: float = 1e-2
    seed: int = 0
    power: PowerOptions = field(default_factory=PowerOptions)
    bounds: Optional[SpectrumBounds] = None
    probe_kind: str = "gaussian"
    s_q: Optional[int] = None
    s_g: Optional[int] = None

    def _c(self) -> L.EstimatorParamsC:
        c = L.EstimatorParamsC()
        L.lib().renyi_default_params(C.byref(c))
        c.alpha = self.alpha
        c.method = METHODS[self.method] if isinstance(self.method, str) else int(self.method)
        c.s, c.m = self.s, self.m
        c.epsilon, c.delta = self.epsilon, self.delta
        c.seed = self.seed & (2**64 - 1)
        c.power = self.power._c()
        if self.bounds is not None:
            c.has_bounds = 1
            c.bounds = self.bounds._c()
        c.probe_kind = PROBES[self.probe_kind]
        c.s_q = -1 if self.s_q is None else self.s_q
        c.s_g = -1 if self.s_g is None else self.s_g
        return c


@dataclass
class EntropyEstimate:
    entropy: float
    trace_estimate: float
    method_used: str
    s_used: int
    m_used: int
    bounds_used: Optional[SpectrumBounds]
    elapsed: float
    deterministic: bool
    trace: Optional[TraceEstimate] = None

    @staticmethod
    def _from(c: L.EntropyEstimateC) -> "EntropyEstimate":
        t = c.trace
        return EntropyEstimate(c.entropy, c.trace_estimate, METHOD_NAMES.get(c.method_used, "?"), c.s_used,
                               c.m_used, SpectrumBounds._from(c.bounds_used) if c.has_bounds else None, c.elapsed,
                               bool(c.deterministic),
                               TraceEstimate(t.value, t.low_rank_part, t.residual_part, t.queries_used,
                                             t.sketch_rank, bool(t.exact)))


def estimate(a: NormalizedKernel, params: EstimatorParams) -> EntropyEstimate:
    """estimate (proj/src/entropy.cpp:201-275); method 'exact' runs entropy_exact."""
    if params.method == "exact":
        return entropy_exact(a, params.alpha)
    out = L.EntropyEstimateC()
    check(L.lib().renyi_estimate(a.ctx.handle, a.handle, C.byref(params._c()), C.byref(out)))
    return EntropyEstimate._from(out)


def estimate_trials(a: NormalizedKernel, params: EstimatorParams, trials: int) -> list:
    """K trials of estimate() with seeds derive_key(params.seed, t), bounds resolved once (the
    measure_cell protocol, proj/src/simulate.cpp:19-51); all trials' probes share the passes over A."""
    if params.method == "exact":
        raise RenyiError(1, "method=exact has no trials")
    out = (L.EntropyEstimateC * max(int(trials), 1))()
    check(L.lib().renyi_estimate_trials(a.ctx.handle, a.handle, C.byref(params._c()), int(trials), out))
    return [EntropyEstimate._from(out[t]) for t in range(int(trials))]


@dataclass
class MreCell:
    alpha: float
    s: int
    m: int
    method: str
    mre: float
    sd: float
    mean_elapsed: float
    trials: int
    oracle_elapsed: float = 0.0


def measure_cell(a: NormalizedKernel, exact_entropy: float, params: EstimatorParams, trials: int) -> MreCell:
    """measure_cell (proj/src/simulate.cpp:19-72): MRE / SD of K batched trials against exact_entropy."""
    out = L.MreCellC()
    check(L.lib().renyi_measure_cell(a.ctx.handle, a.handle, float(exact_entropy), C.byref(params._c()),
                                     int(trials), C.byref(out)))
    return MreCell(out.alpha, out.s, out.m, METHOD_NAMES.get(out.method, "?"), out.mre, out.sd, out.mean_elapsed,
                   out.trials)


def mixture_samples(n: int, d: int, seed: int, center: float = 1.0) -> np.ndarray:
    """(1/2) N(-center, I_d) + (1/2) N(+center, I_d) from the reference stream (proj/src/simulate.cpp:9-17)."""
    out = np.empty((n, d), order="F")
    check(L.lib().renyi_mixture_samples(int(n), int(d), seed & (2**64 - 1), float(center), _dptr(out)))
    return out


@dataclass
class SimulationSpec:
    """proj/include/renyi/simulate.hpp:13-25."""
    n: int = 1000
    d: int = 10
    center: float = 1.0
    sigma: float = 1.0
    alphas: Sequence[float] = (2.0,)
    s_list: Sequence[int] = (64,)
    m_list: Sequence[int] = (0,)
    trials: int = 100
    seed: int = 0
    method: str = "auto"
    precision: str = "fp64"


def run_simulation(spec: SimulationSpec, ctx: Optional["Context"] = None) -> list:
    """run_simulation (proj/src/simulate.cpp:74-104): mixture samples, one kernel, the exact entropy
    per alpha (eigendecomposition on the GPU), then measure_cell for every (alpha, s, m)."""
    if spec.trials < 1:
        raise RenyiError(1, "K must be >= 1")
    if spec.n < 16:
        raise RenyiError(1, "simulation needs n >= 16")
    x = mixture_samples(spec.n, spec.d, spec.seed, spec.center)
    k = build_kernel(x, GaussianKernel(spec.sigma), spec.precision, ctx=ctx)
    cells = []
    for alpha in spec.alphas:
        oracle = entropy_exact(k, alpha)
        for s in spec.s_list:
            for m in spec.m_list:
                p = EstimatorParams(alpha=alpha, method=spec.method, s=s, m=m, seed=spec.seed)
                try:
                    cell = measure_cell(k, oracle.entropy, p, spec.trials)
                except RenyiError as e:
                    raise RenyiError(e.status, f"cell alpha={alpha} s={s} m={m}: {e}") from None
                cell.oracle_elapsed = oracle.elapsed
                cells.append(cell)
    return cells


# ---------------------------------------------------------------- feature tools (features.hpp)
@dataclass
class RankingResult:
    names: list
    columns: list
    scores: list
    elapsed: list


@dataclass
class SelectionResult:
    names: list
    columns: list
    objective: list
    elapsed: list


def _cstrs(items):
    arr = (C.c_char_p * max(len(items), 1))()
    arr[:len(items)] = [str(v).encode() for v in items]
    return arr


def _feature_names(d, names):
    return [names[j] if names is not None and j < len(names) else f"feature_{j}" for j in range(d)]


def one_hot_labels(labels) -> np.ndarray:
    """one_hot_labels (proj/src/features.cpp:83-93): distinct labels in sorted order."""
    classes = {c: i for i, c in enumerate(sorted(set(labels)))}
    out = np.zeros((len(labels), len(classes)))
    for i, l in enumerate(labels):
        out[i, classes[l]] = 1.0
    return out


def _exact_score_fn(ctx, label_k, params, step_seed, precision):
    """The reference's scorer with method=exact (entropy_exact on the device matrices)."""
    h_y = entropy_exact(label_k, params.alpha).entropy

    def score(feats):
        h_f = entropy_exact(feats, params.alpha).entropy
        return h_f + h_y - entropy_exact(hadamard_joint([feats, label_k]), params.alpha).entropy

    return score


def rank_features(x, labels, spec: GaussianKernel, params: EstimatorParams, k: int, names=None,
                  precision="fp64", ctx: Optional[Context] = None) -> RankingResult:
    """rank_features (proj/src/features.cpp:95-123): top k features by I_alpha(X_j; Y), ties by column."""
    ctx = ctx or default_context()
    xa = _colmajor(x)
    n, d = xa.shape
    fnames = _feature_names(d, names)
    if params.method == "exact":  # eigendecomposition check path (entropy_exact on the device)
        _validate_features(n, d, labels, k)
        score = _exact_score_fn(ctx, build_kernel(one_hot_labels(labels), spec, precision, ctx), params, 0, precision)
        scores, elapsed = [], []
        for j in range(d):
            t0 = time.time()
            scores.append(score(build_kernel(xa[:, j:j + 1], spec, precision, ctx)))
            elapsed.append(time.time() - t0)
        order = sorted(range(d), key=lambda j: (-scores[j], j))[:k]
        return RankingResult([fnames[j] for j in order], order, [scores[j] for j in order], elapsed)
    cols = (C.c_int * k)()
    scores = np.empty(k)
    elapsed = np.empty(d)
    check(L.lib().renyi_rank_features(ctx.handle, _dptr(xa), n, d, n, _cstrs(list(labels)), len(labels),
                                      _cstrs(fnames), spec.sigma, C.byref(params._c()), PRECISIONS[precision], k,
                                      cols, _dptr(scores), _dptr(elapsed)))
    order = list(cols)
    return RankingResult([fnames[j] for j in order], order, list(scores), list(elapsed))


def select_features(x, labels, spec: GaussianKernel, params: EstimatorParams, k: int, names=None,
                    precision="fp64", ctx: Optional[Context] = None) -> SelectionResult:
    """select_features (proj/src/features.cpp:125-162): greedy forward selection over Hadamard joints."""
    ctx = ctx or default_context()
    xa = _colmajor(x)
    n, d = xa.shape
    fnames = _feature_names(d, names)
    if params.method == "exact":
        _validate_features(n, d, labels, k)
        label_k = build_kernel(one_hot_labels(labels), spec, precision, ctx)
        kernels = [build_kernel(xa[:, j:j + 1], spec, precision, ctx) for j in range(d)]
        score = _exact_score_fn(ctx, label_k, params, 0, precision)
        taken, selected, res = set(), None, SelectionResult([], [], [], [])
        for step in range(k):
            t0 = time.time()
            best, best_score, best_joint = -1, 0.0, None
            for j in range(d):
                if j in taken:
                    continue
                cand = kernels[j] if step == 0 else hadamard_joint([selected, kernels[j]])
                sc = score(cand)
                if best < 0 or sc > best_score:
                    best, best_score, best_joint = j, sc, cand
            taken.add(best)
            selected = best_joint
            res.names.append(fnames[best])
            res.columns.append(best)
            res.objective.append(best_score)
            res.elapsed.append(time.time() - t0)
        return res
    cols = (C.c_int * k)()
    obj = np.empty(k)
    elapsed = np.empty(k)
    check(L.lib().renyi_select_features(ctx.handle, _dptr(xa), n, d, n, _cstrs(list(labels)), len(labels),
                                        _cstrs(fnames), spec.sigma, C.byref(params._c()), PRECISIONS[precision], k,
                                        cols, _dptr(obj), _dptr(elapsed)))
    order = list(cols)
    return SelectionResult([fnames[j] for j in order], order, list(obj), list(elapsed))


def _validate_features(n, d, labels, k):  # features.cpp:18-26
    if not labels:
        raise RenyiError(1, "dataset has no label column")
    if len(labels) != n:
        raise RenyiError(4, "label count does not match sample count")
    if k < 1 or k > d:
        raise RenyiError(1, f"k must be in [1, d]; got k={k} with d={d}")


def entropy_int(a: NormalizedKernel, alpha: int, s: int, seed: int) -> EntropyEstimate:
    out = L.EntropyEstimateC()
    check(L.lib().renyi_entropy_int(a.ctx.handle, a.handle, int(alpha), s, seed & (2**64 - 1), C.byref(out)))
    return EntropyEstimate._from(out)


def entropy_taylor(a: NormalizedKernel, alpha: float, s: int, m: int, v: float, seed: int) -> EntropyEstimate:
    out = L.EntropyEstimateC()
    check(L.lib().renyi_entropy_taylor(a.ctx.handle, a.handle, alpha, s, m, v, seed & (2**64 - 1), C.byref(out)))
    return EntropyEstimate._from(out)


def entropy_chebyshev(a: NormalizedKernel, alpha: float, s: int, m: int, u: float, v: float,
                      seed: int) -> EntropyEstimate:
    out = L.EntropyEstimateC()
    check(L.lib().renyi_entropy_chebyshev(a.ctx.handle, a.handle, alpha, s, m, u, v, seed & (2**64 - 1),
                                          C.byref(out)))
    return EntropyEstimate._from(out)


def entropy_from_trace(trace: float, alpha: float) -> float:
    out = C.c_double()
    check(L.lib().renyi_entropy_from_trace(trace, alpha, C.byref(out)))
    return out.value


def entropy_exact(a: NormalizedKernel, alpha: float) -> EntropyEstimate:
    """O(n^3) check oracle (proj/src/entropy.cpp:71-90) on the device via torch.linalg.eigvalsh."""
    import time

    import torch

    if a.size() > 20000:
        raise RenyiError(1, "entropy_exact is guarded at n <= 20000")
    entropy_from_trace(1.0, alpha)  # validate alpha
    t0 = time.perf_counter()
    dev = torch.device("cuda", a.ctx.device)
    lam = torch.linalg.eigvalsh(torch.from_numpy(np.ascontiguousarray(a.matrix())).to(dev))
    lam = lam.clamp(0.0, 1.0)
    lam = lam[lam > 0]
    trace = float(torch.sum(lam ** alpha).item())
    return EntropyEstimate(entropy_from_trace(trace, alpha), trace, "exact", 0, 0, None,
                           time.perf_counter() - t0, True, None)


@dataclass
class SelectedParams:
    s: int
    m: int


def select_params(alpha, epsilon, delta, bounds: SpectrumBounds, n: int, method: str) -> SelectedParams:
    s, m = C.c_int(), C.c_int()
    check(L.lib().renyi_select_params(alpha, epsilon, delta, C.byref(bounds._c()), n, METHODS[method], C.byref(s),
                                      C.byref(m)))
    return SelectedParams(s.value, m.value)


@dataclass
class MuBound:
    u: float
    v: float
    alpha: float
    n: int
    mu: float
    lower: float
    upper: float


def mu_bound(u: float, v: float, alpha: float, n: int) -> MuBound:
    mu, lo, hi = C.c_double(), C.c_double(), C.c_double()
    check(L.lib().renyi_mu_bound(u, v, alpha, n, C.byref(mu), C.byref(lo), C.byref(hi)))
    return MuBound(u, v, alpha, n, mu.value, lo.value, hi.value)


# ---------------------------------------------------------------- measures (measures.hpp)
@dataclass
class MutualInformation:
    value: float
    vars_entropy: float
    target_entropy: float
    joint_entropy: float


def _with_seed(params: EstimatorParams, term: str) -> EstimatorParams:
    from dataclasses import replace

    return replace(params, seed=derive_key(params.seed, hash_name(term)))


def _joint(vars_: Sequence[NormalizedKernel]) -> NormalizedKernel:
    if len(vars_) == 0:
        raise RenyiError(1, "empty variable set")
    return vars_[0] if len(vars_) == 1 else hadamard_joint(list(vars_))


def joint_entropy(vars_: Sequence[NormalizedKernel], params: EstimatorParams) -> EntropyEstimate:
    """joint_entropy (proj/src/measures.cpp:23-25)."""
    return estimate(_joint(vars_), params)


def conditional_entropy(vars_: Sequence[NormalizedKernel], given: NormalizedKernel,
                        params: EstimatorParams) -> float:
    """conditional_entropy (proj/src/measures.cpp:27-34)."""
    allk = hadamard_joint([_joint(vars_), given])
    return (estimate(allk, _with_seed(params, "term:joint")).entropy
            - estimate(given, _with_seed(params, "term:given")).entropy)


def mutual_information(vars_: Sequence[NormalizedKernel], target: NormalizedKernel,
                       params: EstimatorParams) -> MutualInformation:
    """mutual_information (proj/src/measures.cpp:36-46)."""
    vj = _joint(vars_)
    if params.method != "exact":
        out = L.MiEstimateC()
        check(L.lib().renyi_mutual_information(vj.ctx.handle, vj.handle, target.handle, C.byref(params._c()),
                                               C.byref(out)))
        return MutualInformation(out.value, out.vars_entropy, out.target_entropy, out.joint_entropy)
    allk = hadamard_joint([vj, target])
    sv = estimate(vj, _with_seed(params, "term:vars")).entropy
    st = estimate(target, _with_seed(params, "term:target")).entropy
    sj = estimate(allk, _with_seed(params, "term:joint")).entropy
    return MutualInformation(sv + st - sj, sv, st, sj)


def mutual_information_samples(x, sx: GaussianKernel, y, sy: GaussianKernel, params: EstimatorParams,
                               precision="fp32", ctx: Optional[Context] = None) -> MutualInformation:
    """MI from host samples (the bench path): fp32 kernels with bounds / integer alpha run the fused
    pass (A and B resident, the joint formed on the fly), otherwise one n x n matrix at a time."""
    ctx = ctx or default_context()
    xa, ya = _colmajor(x), _colmajor(y)
    out = L.MiEstimateC()
    check(L.lib().renyi_mutual_information_samples(ctx.handle, _dptr(xa), xa.shape[0], xa.shape[1], xa.shape[0],
                                                   sx.sigma, _dptr(ya), ya.shape[1], ya.shape[0], sy.sigma,
                                                   C.byref(params._c()), PRECISIONS[precision], C.byref(out)))
    return MutualInformation(out.value, out.vars_entropy, out.target_entropy, out.joint_entropy)


def mutual_information_samples_dev(d_x: int, n: int, dx: int, ldx: int, sx: GaussianKernel, d_y: int, dy: int,
                                   ldy: int, sy: GaussianKernel, params: EstimatorParams, precision="fp32",
                                   ctx: Optional[Context] = None) -> MutualInformation:
    """MI from device-resident column-major samples (raw device pointers, e.g. torch data_ptr())."""
    ctx = ctx or default_context()
    out = L.MiEstimateC()
    check(L.lib().renyi_mutual_information_samples_dev(ctx.handle, C.c_void_p(d_x), n, dx, ldx, sx.sigma,
                                                       C.c_void_p(d_y), dy, ldy, sy.sigma, C.byref(params._c()),
                                                       PRECISIONS[precision], C.byref(out)))
    return MutualInformation(out.value, out.vars_entropy, out.target_entropy, out.joint_entropy)


def entropy_dev(d_x: int, n: int, d: int, ldx: int, sigma: float, params: EstimatorParams, precision="fp32",
                ctx: Optional[Context] = None) -> EntropyEstimate:
    """North-star composition from device-resident column-major samples."""
    ctx = ctx or default_context()
    out = L.EntropyEstimateC()
    check(L.lib().renyi_entropy_dev(ctx.handle, C.c_void_p(d_x), n, d, ldx, sigma, C.byref(params._c()),
                                    PRECISIONS[precision], C.byref(out)))
    return EntropyEstimate._from(out)


def build_kernel_dev(d_x: int, n: int, d: int, ldx: int, spec: GaussianKernel, precision="fp32",
                     ctx: Optional[Context] = None) -> NormalizedKernel:
    ctx = ctx or default_context()
    h = C.c_void_p()
    if isinstance(spec, PolynomialKernel):
        check(L.lib().renyi_kernel_build_polynomial_dev(ctx.handle, C.c_void_p(d_x), n, d, ldx, int(spec.degree),
                                                        float(spec.offset), PRECISIONS[precision], C.byref(h)))
        return NormalizedKernel(h, ctx, PRECISIONS[precision])
    check(L.lib().renyi_kernel_build_gaussian_dev(ctx.handle, C.c_void_p(d_x), n, d, ldx, spec.sigma, None, 0, 0,
                                                  1.0, PRECISIONS[precision], C.byref(h)))
    return NormalizedKernel(h, ctx, PRECISIONS[precision])


def entropy(x, sigma: float, params: EstimatorParams, precision="fp32",
            ctx: Optional[Context] = None) -> EntropyEstimate:
    """North-star composition build_kernel(X, sigma) + estimate (cmd_entropy, renyi_cli.cpp:144-154)."""
    ctx = ctx or default_context()
    xa = _colmajor(x)
    out = L.EntropyEstimateC()
    check(L.lib().renyi_entropy(ctx.handle, _dptr(xa), xa.shape[0], xa.shape[1], xa.shape[0], sigma,
                                C.byref(params._c()), PRECISIONS[precision], C.byref(out)))
    return EntropyEstimate._from(out)


class Dataset:
    """renyi::Dataset (proj/include/renyi/features.hpp:12-19) with the n x d features resident on the
    device; names / labels are host strings. Built by load_csv / parse_csv."""

    def __init__(self, handle, ctx: Context):
        self._h = handle
        self.ctx = ctx
        n, d, hl = C.c_int64(), C.c_int64(), C.c_int()
        check(L.lib().renyi_dataset_shape(handle, C.byref(n), C.byref(d), C.byref(hl)))
        self.n, self.d = n.value, d.value
        lib = L.lib()
        self.names = [lib.renyi_dataset_name(handle, j).decode("utf-8", errors="surrogateescape")
                      for j in range(self.d)]
        self.labels = ([lib.renyi_dataset_label(handle, i).decode("utf-8", errors="surrogateescape")
                        for i in range(self.n)] if hl.value else [])

    @property
    def features(self) -> np.ndarray:
        """n x d fp64 copy of the device-resident features (column-major)."""
        out = np.empty((self.n, self.d), dtype=np.float64, order="F")
        if out.size:
            check(L.lib().renyi_dataset_features(self.ctx.handle, self._h, _dptr(out), max(self.n, 1)))
        return out

    def kernel(self, spec: GaussianKernel, precision="fp64", columns=None) -> NormalizedKernel:
        """build_kernel(features[:, columns], spec) straight from the device copy."""
        h = C.c_void_p()
        if columns is None:
            cols, nc = None, 0
        else:
            arr = (C.c_int64 * len(columns))(*[int(c) for c in columns])
            cols, nc = arr, len(columns)
        check(L.lib().renyi_kernel_build_gaussian_dataset(self.ctx.handle, self._h, cols, nc, spec.sigma,
                                                          PRECISIONS[precision], C.byref(h)))
        return NormalizedKernel(h, self.ctx, PRECISIONS[precision])

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                L.lib().renyi_dataset_destroy(h)
            except Exception:
                pass


def load_csv(path, label_column: Optional[str] = None, ctx: Optional[Context] = None) -> Dataset:
    """load_csv (proj/src/csv.cpp:63-115): the file is parsed on the device."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    check(L.lib().renyi_csv_load(ctx.handle, str(path).encode(), label_column.encode() if label_column else None,
                                 C.byref(h)))
    return Dataset(h, ctx)


def parse_csv(text, label_column: Optional[str] = None, source: Optional[str] = None,
              ctx: Optional[Context] = None) -> Dataset:
    """load_csv over an in-memory CSV (bytes or str); `source` names it in error messages."""
    ctx = ctx or default_context()
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    check(L.lib().renyi_csv_parse(ctx.handle, data, len(data), label_column.encode() if label_column else None,
                                  source.encode() if source else None, C.byref(h)))
    return Dataset(h, ctx)
