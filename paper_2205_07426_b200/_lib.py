"""ctypes binding of librenyi_b200.so (include/renyi_b200.h).

Loading fails loudly when the in-tree library is missing: there is no CPU
fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# RB_LIB_VARIANT=<name> loads librenyi_b200_<name>.so (same-box A/B experiments built with
# RB_LIB_VARIANT and RB_EXTRA_NVCC_FLAGS, see build.py); unset: the product library
_VARIANT = os.environ.get("RB_LIB_VARIANT", "")
LIB_PATH = Path(__file__).resolve().parent / (f"librenyi_b200_{_VARIANT}.so" if _VARIANT else "librenyi_b200.so")

# errc kinds (proj/include/renyi/common.hpp:14-25) + 1, then device/runtime kinds
STATUS_NAMES = {
    0: "ok",
    1: "invalid_argument",
    2: "zero_diagonal",
    3: "non_finite",
    4: "size_mismatch",
    5: "domain_error",
    6: "rank_collapse",
    7: "non_positive_trace",
    8: "alpha_is_one",
    9: "degenerate_bounds",
    10: "parse_error",
    20: "cuda_error",
    21: "nccl_error",
    22: "out_of_memory",
    23: "no_device",
    24: "internal",
}
USAGE_KINDS = {"invalid_argument", "size_mismatch", "domain_error", "parse_error", "alpha_is_one"}


class RenyiError(RuntimeError):
    """Mirror of renyi::error: `kind` is the errc name, is_usage() splits CLI exit 2 / 3."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status_{status}")

    def is_usage(self) -> bool:
        return self.kind in USAGE_KINDS


class Matfun(C.Structure):
    _fields_ = [("kind", C.c_int), ("alpha", C.c_double), ("degree", C.c_int), ("u", C.c_double), ("v", C.c_double)]


class Sketch(C.Structure):
    _fields_ = [
        ("s_q", C.c_int),
        ("s_g", C.c_int),
        ("seed", C.c_uint64),
        ("probe_kind", C.c_int),
        ("sketch", C.POINTER(C.c_double)),
        ("probes", C.POINTER(C.c_double)),
    ]


class TraceEstimateC(C.Structure):
    _fields_ = [
        ("value", C.c_double),
        ("low_rank_part", C.c_double),
        ("residual_part", C.c_double),
        ("queries_used", C.c_int),
        ("sketch_rank", C.c_int),
        ("exact", C.c_int),
    ]


class PowerOptionsC(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("tol", C.c_double), ("seed", C.c_uint64), ("rank_floor", C.c_double)]


class SpectrumBoundsC(C.Structure):
    _fields_ = [
        ("u", C.c_double),
        ("v", C.c_double),
        ("kappa", C.c_double),
        ("iterations_used", C.c_int),
        ("v_converged", C.c_int),
        ("u_converged", C.c_int),
        ("rank_deficient", C.c_int),
    ]


class PowerResultC(C.Structure):
    _fields_ = [("rayleigh", C.c_double), ("iterations", C.c_int), ("converged", C.c_int)]


class EstimatorParamsC(C.Structure):
    _fields_ = [
        ("alpha", C.c_double),
        ("method", C.c_int),
        ("s", C.c_int),
        ("m", C.c_int),
        ("epsilon", C.c_double),
        ("delta", C.c_double),
        ("seed", C.c_uint64),
        ("power", PowerOptionsC),
        ("has_bounds", C.c_int),
        ("bounds", SpectrumBoundsC),
        ("probe_kind", C.c_int),
        ("s_q", C.c_int),
        ("s_g", C.c_int),
    ]


class MreCellC(C.Structure):
    _fields_ = [
        ("alpha", C.c_double),
        ("s", C.c_int),
        ("m", C.c_int),
        ("method", C.c_int),
        ("mre", C.c_double),
        ("sd", C.c_double),
        ("mean_elapsed", C.c_double),
        ("trials", C.c_int),
    ]


class EntropyEstimateC(C.Structure):
    _fields_ = [
        ("entropy", C.c_double),
        ("trace_estimate", C.c_double),
        ("method_used", C.c_int),
        ("s_used", C.c_int),
        ("m_used", C.c_int),
        ("has_bounds", C.c_int),
        ("bounds_used", SpectrumBoundsC),
        ("elapsed", C.c_double),
        ("deterministic", C.c_int),
        ("trace", TraceEstimateC),
    ]


class MiEstimateC(C.Structure):
    _fields_ = [
        ("value", C.c_double),
        ("vars_entropy", C.c_double),
        ("target_entropy", C.c_double),
        ("joint_entropy", C.c_double),
    ]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.c_int64

# name -> (restype, argtypes); the set of exported symbols include/renyi_b200.h declares
SIGNATURES = {
    "renyi_last_error": (C.c_char_p, []),
    "renyi_status_is_usage": (C.c_int, [C.c_int]),
    "renyi_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "renyi_ctx_destroy": (C.c_int, [_P]),
    "renyi_ctx_set_tuning": (C.c_int, [_P, C.c_int, C.c_int]),
    "renyi_ctx_set_operand_mode": (C.c_int, [_P, C.c_int]),
    "renyi_ctx_set_fused_mi": (C.c_int, [_P, C.c_int]),
    "renyi_ctx_set_feature_grouping": (C.c_int, [_P, C.c_int]),
    "renyi_ctx_set_probe_source": (C.c_int, [_P, C.c_int]),
    "renyi_ctx_set_matrix_free_chunk": (C.c_int, [_P, C.c_int]),
    "renyi_ctx_sync": (C.c_int, [_P]),
    "renyi_release_cached_memory": (C.c_int, []),
    "renyi_ctx_profile": (C.c_int, [_P, C.c_int]),
    "renyi_ctx_profile_read": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
    "renyi_ctx_io_bytes": (C.c_int, [_P, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "renyi_ctx_timer_begin": (C.c_int, [_P]),
    "renyi_ctx_timer_end": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "renyi_ctx_launch_count": (C.c_int, [_P, C.POINTER(C.c_long)]),
    "renyi_shard_rows": (C.c_int, [_I64, C.c_int, C.c_int, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)]),
    "renyi_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "renyi_ctx_init_nccl": (C.c_int, [_P, C.c_int, C.c_int, C.c_char_p]),
    "renyi_local_group_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "renyi_local_group_destroy": (C.c_int, [_P]),
    "renyi_ctx_join_local_group": (C.c_int, [_P, _P, C.c_int]),
    "renyi_ctx_rank": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "renyi_kernel_build_gaussian": (C.c_int, [_P, _D, _I64, _I64, _I64, C.c_double, C.c_int, C.POINTER(_P)]),
    "renyi_kernel_hadamard_joint_n": (C.c_int, [_P, C.POINTER(_P), C.c_int, C.POINTER(_P)]),
    "renyi_ops_gaussian_gram": (C.c_int, [_P, _D, _I64, _I64, _I64, C.c_double, _D]),
    "renyi_ops_polynomial_gram": (C.c_int, [_P, _D, _I64, _I64, _I64, C.c_int, C.c_double, _D]),
    "renyi_ops_hadamard_scaled": (C.c_int, [_P, _D, _D, _I64, _I64, C.c_double, _D]),
    "renyi_kernel_build_polynomial": (C.c_int, [_P, _D, _I64, _I64, _I64, C.c_int, C.c_double, C.c_int,
                                                C.POINTER(_P)]),
    "renyi_kernel_build_polynomial_dev": (C.c_int, [_P, C.c_void_p, _I64, _I64, _I64, C.c_int, C.c_double, C.c_int,
                                                    C.POINTER(_P)]),
    "renyi_csv_load": (C.c_int, [_P, C.c_char_p, C.c_char_p, C.POINTER(_P)]),
    "renyi_csv_parse": (C.c_int, [_P, C.c_char_p, _I64, C.c_char_p, C.c_char_p, C.POINTER(_P)]),
    "renyi_dataset_shape": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(C.c_int)]),
    "renyi_dataset_features": (C.c_int, [_P, _P, _D, _I64]),
    "renyi_dataset_name": (C.c_char_p, [_P, _I64]),
    "renyi_dataset_label": (C.c_char_p, [_P, _I64]),
    "renyi_kernel_build_gaussian_dataset": (C.c_int, [_P, _P, C.POINTER(_I64), _I64, C.c_double, C.c_int,
                                                      C.POINTER(_P)]),
    "renyi_dataset_destroy": (C.c_int, [_P]),
    "renyi_kernel_build_gaussian_joint": (
        C.c_int,
        [_P, _D, _I64, _I64, _I64, C.c_double, _D, _I64, _I64, C.c_double, C.c_int, C.POINTER(_P)],
    ),
    "renyi_kernel_build_gaussian_dev": (
        C.c_int,
        [_P, C.c_void_p, _I64, _I64, _I64, C.c_double, C.c_void_p, _I64, _I64, C.c_double, C.c_int, C.POINTER(_P)],
    ),
    "renyi_kernel_from_matrix": (C.c_int, [_P, _D, _I64, C.c_int, C.POINTER(_P)]),
    "renyi_kernel_hadamard_joint": (C.c_int, [_P, _P, _P, C.POINTER(_P)]),
    "renyi_kernel_size": (C.c_int, [_P, C.POINTER(_I64)]),
    "renyi_kernel_download": (C.c_int, [_P, _P, _D]),
    "renyi_kernel_destroy": (C.c_int, [_P]),
    "renyi_matmul_panel": (C.c_int, [_P, _P, _D, C.c_int, _D]),
    "renyi_matvec": (C.c_int, [_P, _P, _D, _D]),
    "renyi_apply_panel": (C.c_int, [_P, _P, C.POINTER(Matfun), _D, C.c_int, _D]),
    "renyi_matfun_traces": (C.c_int, [_P, _P, C.POINTER(Matfun), _D, C.c_int, _D]),
    "renyi_power_method": (C.c_int, [_P, _P, C.POINTER(PowerOptionsC), C.c_double, C.POINTER(PowerResultC)]),
    "renyi_estimate_bounds": (C.c_int, [_P, _P, C.POINTER(PowerOptionsC), C.POINTER(SpectrumBoundsC)]),
    "renyi_hutchpp": (C.c_int, [_P, _P, C.POINTER(Matfun), C.POINTER(Sketch), C.POINTER(TraceEstimateC)]),
    "renyi_estimate": (C.c_int, [_P, _P, C.POINTER(EstimatorParamsC), C.POINTER(EntropyEstimateC)]),
    "renyi_estimate_trials": (C.c_int, [_P, _P, C.POINTER(EstimatorParamsC), C.c_int, C.POINTER(EntropyEstimateC)]),
    "renyi_measure_cell": (C.c_int, [_P, _P, C.c_double, C.POINTER(EstimatorParamsC), C.c_int, C.POINTER(MreCellC)]),
    "renyi_mixture_samples": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_double, C.POINTER(C.c_double)]),
    "renyi_rank_features": (C.c_int, [_P, C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_int64,
                                      C.POINTER(C.c_char_p), C.c_int64, C.POINTER(C.c_char_p), C.c_double,
                                      C.POINTER(EstimatorParamsC), C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "renyi_select_features": (C.c_int, [_P, C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_char_p), C.c_int64, C.POINTER(C.c_char_p), C.c_double,
                                        C.POINTER(EstimatorParamsC), C.c_int, C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "renyi_entropy_int": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_uint64, C.POINTER(EntropyEstimateC)]),
    "renyi_entropy_taylor": (
        C.c_int,
        [_P, _P, C.c_double, C.c_int, C.c_int, C.c_double, C.c_uint64, C.POINTER(EntropyEstimateC)],
    ),
    "renyi_entropy_chebyshev": (
        C.c_int,
        [_P, _P, C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64, C.POINTER(EntropyEstimateC)],
    ),
    "renyi_mutual_information": (C.c_int, [_P, _P, _P, C.POINTER(EstimatorParamsC), C.POINTER(MiEstimateC)]),
    "renyi_mutual_information_samples": (
        C.c_int,
        [_P, _D, _I64, _I64, _I64, C.c_double, _D, _I64, _I64, C.c_double, C.POINTER(EstimatorParamsC), C.c_int,
         C.POINTER(MiEstimateC)],
    ),
    "renyi_mutual_information_samples_dev": (
        C.c_int,
        [_P, C.c_void_p, _I64, _I64, _I64, C.c_double, C.c_void_p, _I64, _I64, C.c_double,
         C.POINTER(EstimatorParamsC), C.c_int, C.POINTER(MiEstimateC)],
    ),
    "renyi_entropy_dev": (
        C.c_int,
        [_P, C.c_void_p, _I64, _I64, _I64, C.c_double, C.POINTER(EstimatorParamsC), C.c_int,
         C.POINTER(EntropyEstimateC)],
    ),
    "renyi_entropy": (
        C.c_int,
        [_P, _D, _I64, _I64, _I64, C.c_double, C.POINTER(EstimatorParamsC), C.c_int, C.POINTER(EntropyEstimateC)],
    ),
    "renyi_default_params": (None, [C.POINTER(EstimatorParamsC)]),
    "renyi_default_power_options": (None, [C.POINTER(PowerOptionsC)]),
    "renyi_mix64": (C.c_uint64, [C.c_uint64]),
    "renyi_derive_key": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "renyi_hash_name": (C.c_uint64, [C.c_char_p]),
    "renyi_probe_panel": (C.c_int, [_I64, C.c_int, C.c_uint64, C.c_char_p, C.c_int, _D]),
    "renyi_binomial_coeffs": (C.c_int, [C.c_double, C.c_int, _D]),
    "renyi_chebyshev_coeffs": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, _D]),
    "renyi_rng_create": (C.c_int, [C.c_uint64, C.POINTER(_P)]),
    "renyi_rng_destroy": (C.c_int, [_P]),
    "renyi_rng_derive": (C.c_int, [_P, C.c_uint64, C.POINTER(_P)]),
    "renyi_rng_key": (C.c_uint64, [_P]),
    "renyi_rng_next_u64": (C.c_uint64, [_P]),
    "renyi_rng_next_uniform": (C.c_double, [_P]),
    "renyi_rng_next_gaussian": (C.c_double, [_P]),
    "renyi_rng_fill_gaussian": (C.c_int, [_P, _I64, _I64, _D]),
    "renyi_chebyshev_node_coeffs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double, _D]),
    "renyi_method_name": (C.c_char_p, [C.c_int]),
    "renyi_chebyshev_safeguard": (C.c_double, [C.c_double, C.c_double]),
    "renyi_taylor_tail_constant": (C.c_double, [C.c_double, C.c_int]),
    "renyi_matfun_scalar": (C.c_int, [C.POINTER(Matfun), C.c_double, _D]),
    "renyi_expected_queries": (C.c_long, [C.POINTER(Matfun), C.c_int]),
    "renyi_select_params": (
        C.c_int,
        [C.c_double, C.c_double, C.c_double, C.POINTER(SpectrumBoundsC), _I64, C.c_int, C.POINTER(C.c_int),
         C.POINTER(C.c_int)],
    ),
    "renyi_mu_bound": (C.c_int, [C.c_double, C.c_double, C.c_double, _I64, _D, _D, _D]),
    "renyi_entropy_from_trace": (C.c_int, [C.c_double, C.c_double, _D]),
}

_lib = None


def lib():
    """Loads the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RenyiError(24, f"{LIB_PATH} is missing: run paper_2205_07426_b200.build (no CPU fallback exists)")
        h = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().renyi_last_error().decode(errors="replace")
        raise RenyiError(status, msg)
