"""ctypes binding of oracle/_ref/libttref.so: the reference library itself
(/root/reference/proj/src/*.cpp, compiled unchanged against the Eigen-API
shim in oracle/eigen_shim by oracle/Makefile).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
only as the checker or the timed CPU baseline.

The functions mirror ``oracle/ttstream_oracle.py`` (same names, same
argument meaning, same exception classes) and return that module's
``TensorTrain`` / ``UpdateReport`` objects, so a test can swap one for the
other.  Tensors are numpy arrays in first-index-fastest (Fortran) order.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from oracle import ttstream_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libttref.so")

_MAX_RANKS = 64


class _Report(C.Structure):
    _fields_ = [
        ("increment_index", C.c_int64),
        ("obs_in_batch", C.c_int64),
        ("obs_used", C.c_int64),
        ("n_ranks", C.c_int32),
        ("tolerance_clamped", C.c_int32),
        ("ranks_before", C.c_int64 * _MAX_RANKS),
        ("ranks_after", C.c_int64 * _MAX_RANKS),
        ("eps_target", C.c_double),
        ("batch_rel_error_estimate", C.c_double),
        ("seconds", C.c_double),
        ("wall_seconds", C.c_double),
    ]


class _Heur(C.Structure):
    _fields_ = [
        ("occupancy_threshold", C.c_double),
        ("skip_enabled", C.c_int32),
        ("subselect_enabled", C.c_int32),
        ("skip_statistic", C.c_int32),
        ("use_approx_tolerance", C.c_int32),
    ]


_ERRORS = {
    1: O.DimensionError,
    2: O.NumericError,
    3: O.StateError,
    4: O.FormatError,
    5: O.IndexError_,
    6: O.ConfigError,
    7: O.ResourceError,
}

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        vp, dp, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.tref_last_error.restype = C.c_char_p
        L.tref_set_threads.argtypes = [C.c_int]
        L.tref_tt_free.argtypes = [vp]
        L.tref_tt_num_cores.argtypes = [vp]
        L.tref_tt_core_shape.argtypes = [vp, C.c_int, i64p]
        L.tref_tt_core_data.argtypes = [vp, C.c_int, dp]
        L.tref_tt_ortho_count.argtypes = [vp]
        L.tref_tt_ortho_count.restype = C.c_int64
        L.tref_tt_num_increments.argtypes = [vp]
        L.tref_tt_boundaries.argtypes = [vp, i64p]
        L.tref_tt_from_cores.argtypes = [C.c_int, i64p, i64p, i64p, C.POINTER(dp), C.c_int64, i64p, C.c_int,
                                         C.POINTER(vp)]
        L.tref_bootstrap.argtypes = [dp, i64p, C.c_int, C.c_double, C.POINTER(_Report), C.POINTER(vp)]
        L.tref_ice_update.argtypes = [vp, dp, i64p, C.c_int, C.c_double, C.POINTER(_Report), C.POINTER(vp)]
        L.tref_ice_update_with_tolerances.argtypes = [vp, dp, i64p, C.c_int, dp, C.c_int, C.POINTER(_Report),
                                                      C.POINTER(vp)]
        L.tref_star_update.argtypes = [vp, dp, i64p, C.c_int, C.c_double, C.POINTER(_Heur), C.POINTER(_Report),
                                       C.POINTER(vp)]
        L.tref_tt_svd.argtypes = [dp, i64p, C.c_int, C.c_double, C.POINTER(vp)]
        L.tref_svd_trunc.argtypes = [dp, C.c_int64, C.c_int64, C.c_double, dp, dp, dp, i64p, dp]
        L.tref_append_directions.argtypes = [dp, C.c_int64, C.c_int64, dp, C.c_int64, dp]
        L.tref_compute_residual.argtypes = [dp, C.c_int64, C.c_int64, dp, C.c_int64, dp]
        L.tref_pad_core.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, dp]
        L.tref_per_obs_errors.argtypes = [vp, dp, i64p, C.c_int, dp]
        L.tref_relaxed_tolerance.argtypes = [dp, i64p, C.c_int, dp, C.c_double, dp, C.POINTER(C.c_int32)]
        L.tref_relaxed_tolerance_approx.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, dp]
        L.tref_tt_project.argtypes = [vp, dp, i64p, C.c_int, dp]
        L.tref_tt_reconstruct.argtypes = [vp, C.c_int64, C.c_int64, dp]
        L.tref_rre.argtypes = [vp, dp, i64p, C.c_int, C.c_int64, C.c_int64, dp]
        L.tref_tt_norm.argtypes = [vp, dp]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenBLAS threads under the reference (it is single-threaded itself;
    SURVEY §8(d) asks for the 1-core figure)."""
    lib().tref_set_threads(int(n))


def _check(code: int) -> None:
    if code:
        msg = lib().tref_last_error().decode()
        raise _ERRORS.get(code, O.Error)(msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64(seq):
    arr = np.ascontiguousarray(np.asarray(seq, dtype=np.int64))
    return arr, arr.ctypes.data_as(C.POINTER(C.c_int64))


def _flat(y: np.ndarray) -> np.ndarray:
    """The tensor's buffer in first-index-fastest order (no copy when it already is)."""
    y = np.asarray(y, dtype=np.float64)
    return np.ravel(y, order="F") if not y.flags.f_contiguous else y.reshape(-1, order="F")


class RefTrain:
    """Owns one reference ``TensorTrain`` handle (tensor_train.hpp:51-124)."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.tref_tt_free(self.h)
            self.h = C.c_void_p(0)

    def to_oracle(self) -> O.TensorTrain:
        L = lib()
        cores = []
        shp = np.zeros(3, dtype=np.int64)
        for i in range(L.tref_tt_num_cores(self.h)):
            L.tref_tt_core_shape(self.h, i, shp.ctypes.data_as(C.POINTER(C.c_int64)))
            rl, n, rr = (int(v) for v in shp)
            buf = np.empty(rl * n * rr, dtype=np.float64)
            L.tref_tt_core_data(self.h, i, _dptr(buf))
            cores.append(O.TTCore(np.reshape(buf, (rl, n, rr), order="F")))
        nb = L.tref_tt_num_increments(self.h)
        b = np.zeros(nb, dtype=np.int64)
        L.tref_tt_boundaries(self.h, b.ctypes.data_as(C.POINTER(C.c_int64)))
        return O.TensorTrain(cores, int(L.tref_tt_ortho_count(self.h)), [int(v) for v in b])

    @staticmethod
    def from_oracle(tt: O.TensorTrain) -> "RefTrain":
        L = lib()
        rl, rla = _i64([c.r_left for c in tt.cores])
        nn, nna = _i64([c.n for c in tt.cores])
        rr, rra = _i64([c.r_right for c in tt.cores])
        bufs = [np.ascontiguousarray(np.ravel(c.data, order="F")) for c in tt.cores]
        ptrs = (C.POINTER(C.c_double) * len(bufs))(*[_dptr(b) for b in bufs])
        bd, bda = _i64(tt.batch_boundaries)
        out = C.c_void_p()
        _check(L.tref_tt_from_cores(len(bufs), rla, nna, rra, ptrs, tt.ortho_count, bda, len(bd), C.byref(out)))
        return RefTrain(out.value)


def _as_train(tt) -> RefTrain:
    return tt if isinstance(tt, RefTrain) else RefTrain.from_oracle(tt)


def _report(r: _Report) -> O.UpdateReport:
    n = r.n_ranks
    rep = O.UpdateReport(
        increment_index=int(r.increment_index),
        obs_in_batch=int(r.obs_in_batch),
        obs_used=int(r.obs_used),
        ranks_before=[int(r.ranks_before[i]) for i in range(n)],
        ranks_after=[int(r.ranks_after[i]) for i in range(n)],
        eps_target=float(r.eps_target),
        batch_rel_error_estimate=float(r.batch_rel_error_estimate),
        seconds=float(r.wall_seconds),
        tolerance_clamped=bool(r.tolerance_clamped),
    )
    rep.cpu_seconds = float(r.seconds)  # the reference's own std::clock figure
    return rep


def _call_update(fn, *args, keep_handle: bool):
    rep, out = _Report(), C.c_void_p()
    _check(fn(*args, C.byref(rep), C.byref(out)))
    t = RefTrain(out.value)
    return (t if keep_handle else t.to_oracle()), _report(rep)


# ---- the hot path ----------------------------------------------------------------

def tt_ice_bootstrap(y: np.ndarray, eps_des: float, keep_handle: bool = False):
    """tt_ice.cpp:143-165 (-> tt_svd.cpp:9-66)."""
    f = _flat(y)
    s, sp = _i64(y.shape)
    return _call_update(lib().tref_bootstrap, _dptr(f), sp, len(s), float(eps_des), keep_handle=keep_handle)


def tt_ice_update(tt, y: np.ndarray, eps_des: float, keep_handle: bool = False):
    """tt_ice.cpp:131-141."""
    t = _as_train(tt)
    f = _flat(y)
    s, sp = _i64(y.shape)
    return _call_update(lib().tref_ice_update, t.h, _dptr(f), sp, len(s), float(eps_des), keep_handle=keep_handle)


def tt_ice_update_with_tolerances(tt, y: np.ndarray, deltas: Sequence[float], keep_handle: bool = False):
    """tt_ice.cpp:60-129."""
    t = _as_train(tt)
    f = _flat(y)
    s, sp = _i64(y.shape)
    d = np.ascontiguousarray(np.asarray(deltas, dtype=np.float64))
    return _call_update(lib().tref_ice_update_with_tolerances, t.h, _dptr(f), sp, len(s), _dptr(d), len(d),
                        keep_handle=keep_handle)


def _heur(cfg: Optional[O.HeuristicConfig]) -> _Heur:
    cfg = cfg or O.HeuristicConfig()
    stat = 1 if str(getattr(cfg, "skip_statistic", "mean")).lower() in ("full", "full_batch", "kfullbatch", "1") else 0
    return _Heur(float(cfg.occupancy_threshold), int(bool(cfg.skip_enabled)), int(bool(cfg.subselect_enabled)), stat,
                 int(bool(cfg.use_approx_tolerance)))


def tt_ice_star_update(tt, y: np.ndarray, eps_des: float, cfg: Optional[O.HeuristicConfig] = None,
                       keep_handle: bool = False):
    """tt_ice_star.cpp:171-303."""
    t = _as_train(tt)
    f = _flat(y)
    s, sp = _i64(y.shape)
    h = _heur(cfg)
    return _call_update(lib().tref_star_update, t.h, _dptr(f), sp, len(s), float(eps_des), C.byref(h),
                        keep_handle=keep_handle)


def tt_svd(y: np.ndarray, eps_rel: float) -> O.TensorTrain:
    """tt_svd.cpp:9-66."""
    f = _flat(y)
    s, sp = _i64(y.shape)
    out = C.c_void_p()
    _check(lib().tref_tt_svd(_dptr(f), sp, len(s), float(eps_rel), C.byref(out)))
    return RefTrain(out.value).to_oracle()


# ---- helpers -----------------------------------------------------------------------

def svd_trunc(a: np.ndarray, delta: float) -> O.TruncatedSvd:
    """truncated_svd.cpp:29-94."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    m, l = a.shape
    k = min(m, l)
    u = np.zeros(max(m * k, 1))
    s = np.zeros(max(k, 1))
    vt = np.zeros(max(k * l, 1))
    rank = C.c_int64()
    tail = C.c_double()
    _check(lib().tref_svd_trunc(_dptr(a), m, l, float(delta), _dptr(u), _dptr(s), _dptr(vt), C.byref(rank),
                                C.byref(tail)))
    r = int(rank.value)
    return O.TruncatedSvd(u=np.reshape(u[: m * r], (m, r), order="F"), s=s[:r].copy(),
                          vt=np.reshape(vt[: r * l], (r, l), order="F"), rank=r, tail_norm=float(tail.value))


def append_directions(u_pad: np.ndarray, u_new: np.ndarray) -> np.ndarray:
    """update_common.hpp:19-36."""
    up = np.asfortranarray(u_pad, dtype=np.float64)
    un = np.asfortranarray(u_new, dtype=np.float64)
    a, r0 = up.shape
    r1 = un.shape[1]
    out = np.zeros(a * (r0 + r1))
    _check(lib().tref_append_directions(_dptr(up), a, r0, _dptr(un), r1, _dptr(out)))
    return np.reshape(out, (a, r0 + r1), order="F")


def compute_residual(u_pad: np.ndarray, y: np.ndarray) -> np.ndarray:
    """tt_ice.cpp:34-41."""
    u = np.asfortranarray(u_pad, dtype=np.float64)
    yy = np.asfortranarray(y, dtype=np.float64)
    out = np.zeros(yy.size)
    _check(lib().tref_compute_residual(_dptr(u), u.shape[0], u.shape[1], _dptr(yy), yy.shape[1], _dptr(out)))
    return np.reshape(out, yy.shape, order="F")


def pad_core(u_next: np.ndarray, r_left_old: int, added_rank: int) -> np.ndarray:
    """tt_ice.cpp:43-58."""
    u = np.asfortranarray(u_next, dtype=np.float64)
    rows, cols = u.shape
    n = rows // max(r_left_old, 1)
    out = np.zeros(max((r_left_old + max(added_rank, 0)) * n * cols, 1))
    _check(lib().tref_pad_core(_dptr(u), rows, cols, int(r_left_old), int(added_rank), _dptr(out)))
    return np.reshape(out[: (r_left_old + added_rank) * n * cols], ((r_left_old + added_rank) * n, cols), order="F")


def per_obs_errors(tt, y: np.ndarray) -> np.ndarray:
    """tt_ice_star.cpp:84-86 (-> per_obs_stats :22-42)."""
    t = _as_train(tt)
    f = _flat(y)
    s, sp = _i64(y.shape)
    out = np.zeros(int(y.shape[-1]))
    _check(lib().tref_per_obs_errors(t.h, _dptr(f), sp, len(s), _dptr(out)))
    return out


def relaxed_tolerance(y: np.ndarray, errs: Sequence[float], eps_des: float):
    """tt_ice_star.cpp:121-158 on the split subselect(errs, eps) makes; returns (eps_upd, clamped)."""
    f = _flat(y)
    s, sp = _i64(y.shape)
    e = np.ascontiguousarray(np.asarray(errs, dtype=np.float64))
    out = C.c_double()
    cl = C.c_int32()
    _check(lib().tref_relaxed_tolerance(_dptr(f), sp, len(s), _dptr(e), float(eps_des), C.byref(out), C.byref(cl)))
    return float(out.value), bool(cl.value)


def relaxed_tolerance_approx(n_batch: int, n_rejected: int, mean_rejected_error: float, eps_des: float) -> float:
    """tt_ice_star.cpp:160-169."""
    out = C.c_double()
    _check(lib().tref_relaxed_tolerance_approx(int(n_batch), int(n_rejected), float(mean_rejected_error),
                                               float(eps_des), C.byref(out)))
    return float(out.value)


def tt_project(tt, y: np.ndarray) -> np.ndarray:
    """tensor_train.cpp:195-226."""
    t = _as_train(tt)
    ot = t.to_oracle()
    f = _flat(y)
    s, sp = _i64(y.shape)
    rd = ot.cores[-1].r_left
    out = np.zeros(rd * int(y.shape[-1]))
    _check(lib().tref_tt_project(t.h, _dptr(f), sp, len(s), _dptr(out)))
    return np.reshape(out, (rd, int(y.shape[-1])), order="F")


def tt_reconstruct(tt, obs_begin: int = 0, obs_end: Optional[int] = None) -> np.ndarray:
    """tensor_train.cpp:182-193."""
    t = _as_train(tt)
    ot = t.to_oracle()
    if obs_end is None:
        obs_end = ot.obs_count()
    spatial = ot.spatial_shape()
    out = np.zeros(int(np.prod(spatial)) * max(obs_end - obs_begin, 0))
    _check(lib().tref_tt_reconstruct(t.h, int(obs_begin), int(obs_end), _dptr(out)))
    return np.reshape(out, tuple(spatial) + (obs_end - obs_begin,), order="F")


def rre(tt, x_ref: np.ndarray, obs_begin: int = 0, obs_end: Optional[int] = None) -> float:
    """metrics.cpp:31-35 (relative_error :13-27)."""
    t = _as_train(tt)
    if obs_end is None:
        obs_end = t.to_oracle().obs_count()
    f = _flat(x_ref)
    s, sp = _i64(x_ref.shape)
    out = C.c_double()
    _check(lib().tref_rre(t.h, _dptr(f), sp, len(s), int(obs_begin), int(obs_end), C.byref(out)))
    return float(out.value)


def tt_norm(tt) -> float:
    """tensor_train.cpp:382-390."""
    t = _as_train(tt)
    out = C.c_double()
    _check(lib().tref_tt_norm(t.h, C.byref(out)))
    return float(out.value)
