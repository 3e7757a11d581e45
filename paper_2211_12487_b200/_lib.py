"""ctypes binding of the C ABI in include/ttg.h (libttg.so, built in-tree).

There is no fallback: if the CUDA library is missing the import fails loudly
(build it with ``python -c 'import __graft_entry__ as g; g.build()'``).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TTG_LIB overrides the in-tree build (A/B timing of two builds on one box)
LIB_PATH = os.environ.get("TTG_LIB") or os.path.join(_HERE, "libttg.so")

MAX_CORES = 32


class Report(ctypes.Structure):
    """ttg_report (mirrors UpdateReport, tt_ice.hpp:10-20)."""

    _fields_ = [
        ("increment_index", ctypes.c_int64),
        ("obs_in_batch", ctypes.c_int64),
        ("obs_used", ctypes.c_int64),
        ("n_ranks", ctypes.c_int32),
        ("tolerance_clamped", ctypes.c_int32),
        ("ranks_before", ctypes.c_int64 * (MAX_CORES + 1)),
        ("ranks_after", ctypes.c_int64 * (MAX_CORES + 1)),
        ("eps_target", ctypes.c_double),
        ("batch_rel_error_estimate", ctypes.c_double),
        ("seconds", ctypes.c_double),
        ("guard_reorthogonalised", ctypes.c_int32),
        ("modes_updated", ctypes.c_int32),
        ("accurate_modes", ctypes.c_int32),
        ("raw_fallbacks", ctypes.c_int32),
        ("gram_only_unstable", ctypes.c_int32),
    ]


class Heuristics(ctypes.Structure):
    """ttg_heuristics (mirrors HeuristicConfig, tt_ice_star.hpp:14-20)."""

    _fields_ = [
        ("occupancy_threshold", ctypes.c_double),
        ("skip_enabled", ctypes.c_int32),
        ("subselect_enabled", ctypes.c_int32),
        ("skip_statistic", ctypes.c_int32),
        ("use_approx_tolerance", ctypes.c_int32),
    ]


# host-collective callbacks (ttg_host_allreduce_fn / ttg_host_allgather_fn)
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64)
HOST_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)

# (name, restype, argtypes) for every symbol of include/ttg.h
_P = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)
SIGNATURES = [
    ("ttg_heuristics_default", None, [ctypes.POINTER(Heuristics)]),
    ("ttg_ctx_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)]),
    ("ttg_nccl_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("ttg_ctx_create_dist", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_P)]),
    ("ttg_ctx_create_hostcoll", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, ctypes.POINTER(_P)]),
    ("ttg_ctx_destroy", None, [_P]),
    ("ttg_last_error", ctypes.c_char_p, [_P]),
    ("ttg_ctx_rank", ctypes.c_int, [_P]),
    ("ttg_ctx_world", ctypes.c_int, [_P]),
    ("ttg_ctx_stream", ctypes.c_void_p, [_P]),
    ("ttg_ctx_launch_count", ctypes.c_int64, [_P]),
    ("ttg_ctx_synchronize", ctypes.c_int, [_P]),
    ("ttg_ctx_wait_stream", ctypes.c_int, [_P, _P]),
    ("ttg_ctx_join_stream", ctypes.c_int, [_P, _P]),
    ("ttg_ctx_set_profiling", ctypes.c_int, [_P, ctypes.c_int]),
    ("ttg_ctx_reset_stats", None, [_P]),
    ("ttg_ctx_num_kernel_stats", ctypes.c_int, [_P]),
    ("ttg_ctx_kernel_stat", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, _I64P, _DP, _DP, _DP]),
    ("ttg_ctx_io_bytes", ctypes.c_int, [_P, _I64P, _I64P]),
    ("ttg_ctx_spec_stats", ctypes.c_int, [_P, _I64P, _I64P]),
    ("ttg_ctx_reserve", ctypes.c_int, [_P, ctypes.c_int64]),
    ("ttg_prefetch", ctypes.c_int, [_P, _DP, ctypes.c_int64]),
    ("ttg_tt_upload", ctypes.c_int, [_P, ctypes.c_int, _I64P, _I64P, _I64P, ctypes.POINTER(_DP), ctypes.c_int64,
                                     _I64P, ctypes.c_int64, ctypes.POINTER(_P)]),
    ("ttg_tt_destroy", None, [_P]),
    ("ttg_tt_num_cores", ctypes.c_int, [_P]),
    ("ttg_tt_shape", ctypes.c_int, [_P, _I64P, _I64P, _I64P, _I64P]),
    ("ttg_tt_bounds", ctypes.c_int, [_P, _I64P]),
    ("ttg_tt_download_core", ctypes.c_int, [_P, _P, ctypes.c_int, _DP]),
    ("ttg_bootstrap", ctypes.c_int, [_P, _DP, ctypes.c_int, _I64P, ctypes.c_int, ctypes.c_double, ctypes.POINTER(_P),
                                     ctypes.POINTER(Report)]),
    ("ttg_tt_ice_update", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, ctypes.c_double,
                                         ctypes.POINTER(Report)]),
    ("ttg_tt_ice_update_with_tolerances", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, _DP,
                                                         ctypes.c_int, ctypes.POINTER(Report)]),
    ("ttg_tt_ice_star_update", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, ctypes.c_double,
                                              ctypes.POINTER(Heuristics), ctypes.POINTER(Report)]),
    ("ttg_per_obs_errors", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, _DP]),
    ("ttg_project", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, _DP]),
    ("ttg_reconstruct", ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int64, _DP, ctypes.c_int]),
    # metrics (metrics.hpp), checkpoint (serialization.hpp), ingest (stream_io.hpp)
    ("ttg_compression_ratio", ctypes.c_int, [_P, _DP]),
    ("ttg_rre", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _DP,
                               ctypes.POINTER(ctypes.c_int)]),
    ("ttg_rpe", ctypes.c_int, [_P, _P, _DP, ctypes.c_int, _I64P, ctypes.c_int, _DP, ctypes.POINTER(ctypes.c_int)]),
    ("ttg_tt_measure_ortho_count", ctypes.c_int, [_P, _P, ctypes.c_double, _I64P]),
    ("ttg_tt_serialize", ctypes.c_int, [_P, _P, ctypes.c_void_p, ctypes.c_int64, _I64P]),
    ("ttg_tt_deserialize", ctypes.c_int, [_P, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(_P)]),
    ("ttg_tt_save_ttc", ctypes.c_int, [_P, _P, ctypes.c_char_p]),
    ("ttg_tt_load_ttc", ctypes.c_int, [_P, ctypes.c_char_p, ctypes.POINTER(_P)]),
    ("ttg_write_batch", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.c_int, _DP]),
    ("ttg_read_batch", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.POINTER(ctypes.c_int), _DP, ctypes.c_int64,
                                      _I64P]),
    ("ttg_stream_open", ctypes.c_int, [_P, ctypes.c_char_p, ctypes.POINTER(_P)]),
    ("ttg_stream_count", ctypes.c_int64, [_P]),
    ("ttg_stream_next", ctypes.c_int, [_P, ctypes.POINTER(_DP), _I64P, ctypes.POINTER(ctypes.c_int)]),
    ("ttg_stream_close", ctypes.c_int, [_P]),
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libttg.so once and bind every ABI symbol; raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: the CUDA library must be built (no CPU fallback exists)")
    # libttg.so needs libnccl.so.2.  torch bundles a newer NCCL under the same
    # soname, and libtorch_cuda fails to load against the older system copy, so
    # torch (the plumbing: device memory, streams) is loaded first; libttg's
    # dependency then binds to the NCCL already in the process.
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
