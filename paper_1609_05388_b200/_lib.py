"""ctypes binding of libadg.so (include/adg.h).

The product path has no fallback: if the library is missing or no sm_100
device is visible, every call raises.  (The CPU oracle under oracle/ is test
infrastructure and is never imported from this package.)
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# ADG_LIB: another build of the same library (the checked build, tests only)
LIB_PATH = os.environ.get("ADG_LIB") or os.path.join(HERE, "libadg.so")

ADG_OK, ADG_EINVAL, ADG_ENUMERIC, ADG_EIO, ADG_ECUDA, ADG_ENOMEM, ADG_ENCCL = range(7)
ADG_SUM_U64, ADG_SUM_F64, ADG_MAX_F32, ADG_MAX_U64 = range(4)
ADG_F64, ADG_F32, ADG_BF16 = 0, 1, 2
ENGINES = {"auto": 0, "exact": 1, "screen": 2, "screen_exact_hist": 3}


class AdgError(RuntimeError):
    """Base class of errors raised through the C ABI."""


class InvalidArgument(AdgError, ValueError):
    """std::invalid_argument in the reference."""


class NumericError(AdgError, ArithmeticError):
    """adagio::NumericError (proj/include/adagio/errors.hpp:16)."""


class IoError(AdgError, OSError):
    """adagio::IoError (proj/include/adagio/errors.hpp:10)."""


class CudaError(AdgError):
    """Device / CUDA failure (no reference analogue)."""


class CollectiveError(AdgError):
    """A collective of the multi-GPU exchange failed (ADG_ENCCL)."""


_ERRS = {ADG_EINVAL: InvalidArgument, ADG_ENUMERIC: NumericError, ADG_EIO: IoError,
         ADG_ECUDA: CudaError, ADG_ENOMEM: CudaError, ADG_ENCCL: CollectiveError}


class Report(ctypes.Structure):
    _fields_ = [("max_distortion", ctypes.c_double), ("mean_distortion", ctypes.c_double),
                ("n_pairs_evaluated", ctypes.c_uint64),
                ("n_zero_distance_pairs", ctypes.c_uint64),
                ("argmax_i", ctypes.c_uint64), ("argmax_j", ctypes.c_uint64),
                ("hist_bins", ctypes.c_int32), ("sampled", ctypes.c_int32),
                ("hist_max", ctypes.c_double), ("sample_seed", ctypes.c_uint64),
                ("engine", ctypes.c_int32), ("candidate_rows", ctypes.c_int32),
                ("screen_error_bound", ctypes.c_double), ("edge_pairs", ctypes.c_uint64)]


class PairSamplingC(ctypes.Structure):
    _fields_ = [("all_pairs", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("m", ctypes.c_uint64), ("seed", ctypes.c_uint64)]


class Partials(ctypes.Structure):
    _fields_ = [("hist", ctypes.c_void_p), ("tile_sums", ctypes.c_void_p),
                ("row_max", ctypes.c_void_p), ("row_bound", ctypes.c_void_p),
                ("near_pairs", ctypes.c_void_p), ("near_count", ctypes.c_void_p),
                ("num_tiles", ctypes.c_int64), ("near_capacity", ctypes.c_int64),
                ("n", ctypes.c_int64), ("hist_bins", ctypes.c_int32),
                ("tile_slots", ctypes.c_int32)]


class SweepRowC(ctypes.Structure):
    """include/adg.h adg_sweep_row (proj/include/adagio/sweep.hpp:19-28)."""
    _fields_ = [("method", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("target_dim", ctypes.c_int64), ("seed", ctypes.c_uint64),
                ("max_distortion", ctypes.c_double), ("fit_seconds", ctypes.c_double),
                ("eval_seconds", ctypes.c_double)]


class MinDimC(ctypes.Structure):
    """include/adg.h adg_min_dim_result (proj/include/adagio/sweep.hpp:38-43)."""
    _fields_ = [("target_dim", ctypes.c_int64), ("achieved_distortion", ctypes.c_double),
                ("achieved", ctypes.c_int32), ("monotone", ctypes.c_int32),
                ("probes", ctypes.c_int32), ("probes_refined", ctypes.c_int32)]


class KnnEdgeC(ctypes.Structure):
    """include/adg.h adg_knn_edge (proj/include/adagio/downstream.hpp:15-19)."""
    _fields_ = [("u", ctypes.c_int32), ("v", ctypes.c_int32), ("weight", ctypes.c_double)]


ALL_REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_int32, ctypes.c_void_p)
ALL_GATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_int64, ctypes.c_void_p)


class Collectives(ctypes.Structure):
    """include/adg.h adg_collectives."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("user", ctypes.c_void_p),
                ("all_reduce", ALL_REDUCE_FN), ("all_gather", ALL_GATHER_FN)]


# every symbol include/adg.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "adg_abi_version", "adg_last_error", "adg_ctx_create", "adg_ctx_destroy",
    "adg_ctx_set_stream", "adg_ctx_synchronize", "adg_derive_seed", "adg_sample_jl",
    "adg_jl_dimension", "adg_center", "adg_exact_top_svd", "adg_randomized_top_svd",
    "adg_fit_with_split", "adg_fit", "adg_transform_all", "adg_evaluate", "adg_distort_model",
    "adg_max_distortion",
    "adg_pair_distortion", "adg_report_to_json", "adg_histogram_csv", "adg_eval_plan_create",
    "adg_eval_plan_partials", "adg_eval_plan_reset", "adg_eval_plan_run",
    "adg_eval_plan_finalize", "adg_eval_plan_destroy", "adg_method_name", "adg_method_from_name",
    "adg_tradeoff", "adg_min_dim_for_distortion", "adg_sweep_csv", "adg_knn_query",
    "adg_majority_classify", "adg_build_knn_graph", "adg_last_screen_kernel_ms",
    "adg_kernel_launch_count", "adg_last_knn_engine", "adg_transform_plan_create",
    "adg_transform_plan_run", "adg_transform_plan_destroy", "adg_column_sums", "adg_gram",
    "adg_fit_from_gram", "adg_eval_plan_exchange", "adg_eval_plan_set_engine",
    "adg_eval_plan_shard", "adg_evaluate_multi", "adg_nccl_unique_id", "adg_comm_nccl_create",
    "adg_comm_nccl_create_all", "adg_comm_nccl_destroy",
    "adg_last_screen_orig_passes", "adg_eval_plan_refresh",
]

_lib = None
_lock = threading.Lock()


def load():
    """Load libadg.so (building it first if absent and nvcc is present)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import build as _build
            _build.build()
        L = ctypes.CDLL(LIB_PATH)
        P, i64, u64, i32, dbl = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
                                 ctypes.c_double)
        st = ctypes.c_int
        sig = {
            "adg_abi_version": (i32, []),
            "adg_last_error": (ctypes.c_char_p, []),
            "adg_ctx_create": (st, [i32, ctypes.POINTER(P)]),
            "adg_ctx_destroy": (st, [P]),
            "adg_ctx_set_stream": (st, [P, P]),
            "adg_ctx_synchronize": (st, [P]),
            "adg_derive_seed": (u64, [u64, ctypes.c_char_p]),
            "adg_sample_jl": (st, [P, i64, i64, u64, P]),
            "adg_jl_dimension": (st, [i64, dbl, dbl, ctypes.POINTER(i64)]),
            "adg_center": (st, [P, P, i32, i64, i64, P, P]),
            "adg_exact_top_svd": (st, [P, P, i32, i64, i64, i64, P, P, i64]),
            "adg_randomized_top_svd": (st, [P, P, i32, i64, i64, i64, i64, i32, u64, P, P]),
            "adg_fit_with_split": (st, [P, P, i32, i64, i64, i64, i64, i32, u64, P, P, P]),
            "adg_fit": (st, [P, P, i32, i64, i64, i64, i32, u64, P, P, P]),
            "adg_column_sums": (st, [P, P, i32, i64, i64, P]),
            "adg_last_screen_orig_passes": (i32, [P]),
            "adg_eval_plan_refresh": (st, [P]),
            "adg_eval_plan_exchange": (st, [P, ctypes.POINTER(Collectives)]),
            "adg_eval_plan_set_engine": (st, [P, i32]),
            "adg_eval_plan_shard": (st, [P, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
            "adg_evaluate_multi": (st, [i32, P, P, i32, i64, i64, P, i32, i64, i64,
                                        ctypes.POINTER(PairSamplingC), i32, dbl, i32,
                                        ctypes.POINTER(Report), P]),
            "adg_nccl_unique_id": (st, [P]),
            "adg_comm_nccl_create": (st, [P, i32, i32, P, ctypes.POINTER(Collectives)]),
            "adg_comm_nccl_create_all": (st, [i32, P, ctypes.POINTER(Collectives)]),
            "adg_comm_nccl_destroy": (st, [ctypes.POINTER(Collectives)]),
            "adg_gram": (st, [P, P, i32, i64, i64, P, i32, P]),
            "adg_fit_from_gram": (st, [P, P, i64, i64, i64, i64, i32, u64, P, P]),
            "adg_transform_all": (st, [P, P, P, i64, P, i64, i64, P, i32, i64, P, i32]),
            "adg_evaluate": (st, [P, P, i32, i64, i64, P, i32, i64, i64,
                                  ctypes.POINTER(PairSamplingC), i32, dbl, u64, i32,
                                  ctypes.POINTER(Report), P]),
            "adg_distort_model": (st, [P, P, P, i64, P, i64, i64, P, i32, i64,
                                       ctypes.POINTER(PairSamplingC), i32, dbl, i32,
                                       ctypes.POINTER(Report), P, P, i32]),
            "adg_max_distortion": (st, [P, P, i32, i64, i64, P, i32, i64, ctypes.POINTER(dbl)]),
            "adg_pair_distortion": (st, [P, P, P, i64, P, P, i64, ctypes.POINTER(dbl)]),
            "adg_report_to_json": (ctypes.c_size_t, [ctypes.POINTER(Report), P, ctypes.c_char_p,
                                                     ctypes.c_size_t]),
            "adg_histogram_csv": (ctypes.c_size_t, [ctypes.POINTER(Report), P, ctypes.c_char_p,
                                                    ctypes.c_size_t]),
            "adg_eval_plan_create": (st, [P, P, i32, i64, i64, P, i32, i64, i32, dbl,
                                          ctypes.POINTER(P)]),
            "adg_eval_plan_partials": (st, [P, ctypes.POINTER(Partials)]),
            "adg_eval_plan_reset": (st, [P]),
            "adg_eval_plan_run": (st, [P, i64, i64]),
            "adg_eval_plan_finalize": (st, [P, ctypes.POINTER(Report), P]),
            "adg_eval_plan_destroy": (st, [P]),
            "adg_method_name": (ctypes.c_char_p, [i32]),
            "adg_method_from_name": (st, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32)]),
            "adg_tradeoff": (st, [P, P, i32, i64, i64, P, i64, P, i64, P, i64,
                                  ctypes.POINTER(PairSamplingC), P, i64, i64,
                                  ctypes.POINTER(SweepRowC), i64, ctypes.POINTER(i64)]),
            "adg_min_dim_for_distortion": (st, [P, P, i32, i64, i64, i32, dbl, u64, i64, i64,
                                                ctypes.POINTER(MinDimC)]),
            "adg_sweep_csv": (ctypes.c_size_t, [ctypes.POINTER(SweepRowC), i64, ctypes.c_char_p,
                                                ctypes.c_size_t]),
            "adg_knn_query": (st, [P, P, i32, i64, i64, P, i32, i64, i64, i32, P, P]),
            "adg_majority_classify": (st, [P, P, i32, i64, i64, P, i32, i64, i64, P, i32, u64,
                                           ctypes.POINTER(ctypes.c_int32)]),
            "adg_build_knn_graph": (st, [P, P, i32, i64, i64, i32, i32, ctypes.POINTER(KnnEdgeC),
                                         i64, ctypes.POINTER(i64)]),
            "adg_last_screen_kernel_ms": (dbl, [P]),
            "adg_kernel_launch_count": (u64, [P]),
            "adg_last_knn_engine": (i32, [P]),
            "adg_transform_plan_create": (st, [P, P, P, i64, P, i64, i64, i32, ctypes.POINTER(P)]),
            "adg_transform_plan_run": (st, [P, P, i32, i64, P, i32]),
            "adg_transform_plan_destroy": (st, [P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    if status != ADG_OK:
        msg = load().adg_last_error().decode(errors="replace")
        raise _ERRS.get(status, AdgError)(msg)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy

_tls = threading.local()


def context(device: int = 0):
    """Per-thread, per-device adg_ctx (created on first use)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        h = ctypes.c_void_p()
        check(load().adg_ctx_create(device, ctypes.byref(h)))
        ctxs[device] = h
    return ctxs[device]
