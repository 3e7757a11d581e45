"""Python host mirror of the reference's public ingest/update/reconstruct API.

Same names, argument meaning and error behaviour as /root/reference/proj:

==============================  =============================================
this module                     reference
==============================  =============================================
``tt_ice_bootstrap``            tt_ice.hpp:48-49  (tt_ice.cpp:143-165)
``tt_ice_update``               tt_ice.hpp:38-39  (tt_ice.cpp:131-141)
``tt_ice_update_with_tolerances`` tt_ice.hpp:43-45 (tt_ice.cpp:60-129)
``tt_ice_star_update``          tt_ice_star.hpp:57-59 (tt_ice_star.cpp:171-303)
``HeuristicConfig``             tt_ice_star.hpp:14-20
``per_obs_errors``              tt_ice_star.hpp:24
``tt_project``                  tensor_train.hpp:103
``tt_reconstruct``              tensor_train.hpp:96-98
``UpdateReport``                tt_ice.hpp:10-20
``TensorTrain``                 tensor_train.hpp:51-93 (device-resident)
==============================  =============================================

Every call goes through the C ABI of ``libttg.so`` (include/ttg.h); there is
no CPU path.  One deliberate difference: a device ``TensorTrain`` is updated
IN PLACE (the reference returns a new train sharing buffers), and the update
functions return that same object — earlier observations' coefficients are
never rewritten, so Theorem 3.3 holds bit-for-bit.

Increments ``y`` are either numpy arrays (host; copied H2D inside the call,
first-index-fastest as the reference's DenseTensor) or torch CUDA tensors
(device-resident).  A torch tensor must be float64 and either 1-D with an
explicit ``shape=`` or N-D laid out first-index-fastest (``y.permute(*reversed
dims)`` contiguous, e.g. ``torch.empty(shape[::-1]).permute(...)``).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import STATUS_TO_ERROR, Error

TTG_HOST, TTG_DEVICE = 0, 1


def _check(rc: int, ctx: Optional["Context"]) -> None:
    if rc == 0:
        return
    msg = ""
    if ctx is None or ctx._h:  # ctx None: context-free entry points keep a per-thread message
        raw = _lib.load().ttg_last_error(ctx._h if ctx is not None else None)
        msg = raw.decode() if raw else ""
    raise STATUS_TO_ERROR.get(rc, Error)(msg or f"ttg status {rc}")


class Context:
    """One context per stream and GPU (include/ttg.h ``ttg_ctx``)."""

    def __init__(self, device: int = 0, *, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        lib = _lib.load()
        h = ctypes.c_void_p()
        if world > 1 or nccl_id is not None:  # an explicit id at world 1: NCCL transport on one GPU
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("multi-GPU context needs the 128-byte NCCL unique id")
            rc = lib.ttg_ctx_create_dist(device, rank, world, nccl_id, ctypes.byref(h))
        else:
            rc = lib.ttg_ctx_create(device, ctypes.byref(h))
        self._h = None
        _check(rc, None)
        self._h = h
        self.device = device

    @classmethod
    def with_host_collectives(cls, device: int, rank: int, world: int, allreduce, allgather) -> "Context":
        """Multi-rank context over caller-supplied host collectives
        (include/ttg.h ttg_ctx_create_hostcoll): ``allreduce(a)`` sums the
        float64 array ``a`` in place over the ranks; ``allgather(b)`` returns
        the uint8 arrays ``b`` of all ranks concatenated in rank order."""
        lib = _lib.load()
        self = cls.__new__(cls)
        self._h = None
        self.device = device

        def ar(_user, buf, n):
            try:
                allreduce(np.ctypeslib.as_array(buf, shape=(int(n),)))
                return 0
            except Exception:  # surfaces as TTG_E_NCCL
                return 1

        def ag(_user, send, nbytes, recv):
            try:
                nb = int(nbytes)
                snd = np.ctypeslib.as_array(ctypes.cast(send, ctypes.POINTER(ctypes.c_uint8)), shape=(nb,)).copy()
                rcv = np.ctypeslib.as_array(ctypes.cast(recv, ctypes.POINTER(ctypes.c_uint8)), shape=(nb * world,))
                rcv[:] = np.asarray(allgather(snd), dtype=np.uint8).reshape(-1)
                return 0
            except Exception:
                return 1

        self._callbacks = (_lib.HOST_ALLREDUCE_FN(ar), _lib.HOST_ALLGATHER_FN(ag))  # kept alive with the context
        h = ctypes.c_void_p()
        rc = lib.ttg_ctx_create_hostcoll(device, rank, world, ctypes.cast(self._callbacks[0], ctypes.c_void_p),
                                         ctypes.cast(self._callbacks[1], ctypes.c_void_p), None, ctypes.byref(h))
        _check(rc, None)
        self._h = h
        return self

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_lib.load().ttg_nccl_unique_id(buf), None)
        return buf.raw

    @property
    def rank(self) -> int:
        return _lib.load().ttg_ctx_rank(self._h)

    @property
    def world(self) -> int:
        return _lib.load().ttg_ctx_world(self._h)

    @property
    def stream_ptr(self) -> int:
        return _lib.load().ttg_ctx_stream(self._h) or 0

    @property
    def launch_count(self) -> int:
        return int(_lib.load().ttg_ctx_launch_count(self._h))

    def set_profiling(self, on: bool) -> None:
        _check(_lib.load().ttg_ctx_set_profiling(self._h, int(bool(on))), self)

    def reset_stats(self) -> None:
        _lib.load().ttg_ctx_reset_stats(self._h)

    def kernel_stats(self) -> list:
        """[{name, launches, ms, bytes, flops}] accumulated since reset_stats()."""
        lib = _lib.load()
        n = lib.ttg_ctx_num_kernel_stats(self._h)
        if n < 0:
            _check(-n, self)
        out = []
        for i in range(n):
            name = ctypes.create_string_buffer(64)
            la, ms, by, fl = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            _check(lib.ttg_ctx_kernel_stat(self._h, i, name, 64, ctypes.byref(la), ctypes.byref(ms), ctypes.byref(by),
                                           ctypes.byref(fl)), self)
            out.append(dict(name=name.value.decode(), launches=la.value, ms=ms.value, bytes=by.value, flops=fl.value))
        return out

    def reserve(self, nbytes: int) -> None:
        """Pre-map workspace memory (include/ttg.h ttg_ctx_reserve)."""
        _check(_lib.load().ttg_ctx_reserve(self._h, int(nbytes)), self)

    def io_bytes(self):
        h, d = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.load().ttg_ctx_io_bytes(self._h, ctypes.byref(h), ctypes.byref(d)), self)
        return h.value, d.value

    def spec_stats(self):
        """(speculative sweeps, of which repeated synchronously) -- ttg_ctx_spec_stats."""
        s, r = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.load().ttg_ctx_spec_stats(self._h, ctypes.byref(s), ctypes.byref(r)), self)
        return s.value, r.value

    def prefetch(self, y: np.ndarray) -> None:
        """include/ttg.h ttg_prefetch: start the H2D copy of host increment ``y``
        (float64, first-index-fastest, ideally pinned) on the copy stream; the
        next update / projection given the same array consumes it, so the PCIe
        transfer of increment k+1 overlaps the update of increment k.  ``y``
        must not be modified until that call returns."""
        if not isinstance(y, np.ndarray) or y.dtype != np.float64:
            raise TypeError("prefetch takes a float64 numpy array")
        arr = np.asfortranarray(y)
        if arr is not y:
            raise ValueError("prefetch needs the first-index-fastest array the update will be given")
        self._prefetched = (getattr(self, "_prefetched", ()) + (arr,))[-2:]  # keep alive while in flight
        _check(_lib.load().ttg_prefetch(self._h, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), arr.size), self)

    def synchronize(self) -> None:
        _check(_lib.load().ttg_ctx_synchronize(self._h), self)

    def close(self) -> None:
        if self._h:
            _lib.load().ttg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT_CTX: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


@dataclass
class UpdateReport:
    """tt_ice.hpp:10-20; ``seconds`` is wall time from CUDA events."""

    increment_index: int = 0
    obs_in_batch: int = 0
    obs_used: int = 0
    ranks_before: List[int] = field(default_factory=list)
    ranks_after: List[int] = field(default_factory=list)
    eps_target: float = 0.0
    batch_rel_error_estimate: float = 0.0
    seconds: float = 0.0
    tolerance_clamped: bool = False
    guard_reorthogonalised: int = 0
    modes_updated: int = 0
    accurate_modes: int = 0
    raw_fallbacks: int = 0
    gram_only_unstable: int = 0

    @staticmethod
    def _from(r: _lib.Report) -> "UpdateReport":
        n = r.n_ranks
        return UpdateReport(
            increment_index=r.increment_index, obs_in_batch=r.obs_in_batch, obs_used=r.obs_used,
            ranks_before=[int(r.ranks_before[i]) for i in range(n)],
            ranks_after=[int(r.ranks_after[i]) for i in range(n)],
            eps_target=r.eps_target, batch_rel_error_estimate=r.batch_rel_error_estimate,
            seconds=r.seconds, tolerance_clamped=bool(r.tolerance_clamped),
            guard_reorthogonalised=r.guard_reorthogonalised, modes_updated=r.modes_updated,
            accurate_modes=r.accurate_modes, raw_fallbacks=r.raw_fallbacks, gram_only_unstable=r.gram_only_unstable)


@dataclass
class HeuristicConfig:
    """tt_ice_star.hpp:14-20 (``skip_statistic``: "mean" = kMean, "full" = kFullBatch)."""

    occupancy_threshold: float = 0.8
    skip_enabled: bool = True
    subselect_enabled: bool = True
    skip_statistic: str = "mean"
    use_approx_tolerance: bool = False

    def _to(self) -> _lib.Heuristics:
        if self.skip_statistic not in ("mean", "full"):
            raise ValueError("skip_statistic must be 'mean' or 'full'")
        return _lib.Heuristics(float(self.occupancy_threshold), int(bool(self.skip_enabled)),
                               int(bool(self.subselect_enabled)), 0 if self.skip_statistic == "mean" else 1,
                               int(bool(self.use_approx_tolerance)))


class DeviceIncrement:
    """A device-resident increment (first-index-fastest float64) owned by an
    IncrementStream; valid until the stream's next ``next()``."""

    def __init__(self, ptr: int, shape: Sequence[int], stream: "IncrementStream"):
        self.ptr = int(ptr)
        self.shape = tuple(int(s) for s in shape)
        self._stream = stream


class _Input:
    """Resolves y (numpy host array, torch CUDA tensor or DeviceIncrement) to (pointer, where, shape).
    A torch tensor is ordered before the context's (non-blocking) stream reads
    it: the context stream waits on torch's current stream (ttg_ctx_wait_stream,
    no host sync)."""

    def __init__(self, y, shape: Optional[Sequence[int]] = None, ctx: Optional["Context"] = None):
        self.keep = None
        if isinstance(y, np.ndarray):
            if y.dtype != np.float64:
                raise TypeError("increments are float64 (SPEC.md:88)")
            arr = np.asfortranarray(y)
            self.keep = arr
            self.shape = tuple(int(s) for s in (shape if shape is not None else arr.shape))
            if int(np.prod(self.shape)) != arr.size:
                raise ValueError("shape does not match the buffer")
            self.ptr = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            self.where = TTG_HOST
            return
        if isinstance(y, DeviceIncrement):  # an increment delivered by IncrementStream
            self.keep = y
            self.shape = tuple(y.shape) if shape is None else tuple(int(s) for s in shape)
            if int(np.prod(self.shape)) != int(np.prod(y.shape)):
                raise ValueError("shape does not match the buffer")
            self.ptr = ctypes.cast(ctypes.c_void_p(y.ptr), ctypes.POINTER(ctypes.c_double))
            self.where = TTG_DEVICE
            return
        # torch tensor (duck-typed so torch is not a hard dependency of the host mirror)
        if not hasattr(y, "data_ptr") or not getattr(y, "is_cuda", False):
            raise TypeError("y must be a numpy array or a CUDA torch tensor")
        import torch

        if y.dtype != torch.float64:
            raise TypeError("increments are float64 (SPEC.md:88)")
        if shape is not None:
            if not y.is_contiguous():
                raise ValueError("flat device buffer must be contiguous")
            self.shape = tuple(int(s) for s in shape)
            if int(np.prod(self.shape)) != y.numel():
                raise ValueError("shape does not match the buffer")
        else:
            if not y.permute(*reversed(range(y.dim()))).is_contiguous():
                raise ValueError("device tensor must be first-index-fastest (pass a flat tensor with shape=)")
            self.shape = tuple(int(s) for s in y.shape)
        self.keep = y
        self.ptr = ctypes.cast(ctypes.c_void_p(y.data_ptr()), ctypes.POINTER(ctypes.c_double))
        self.where = TTG_DEVICE
        if ctx is not None:
            _check(_lib.load().ttg_ctx_wait_stream(ctx._h, torch.cuda.current_stream(y.device).cuda_stream), ctx)

    def shape_arr(self):
        return (ctypes.c_int64 * len(self.shape))(*self.shape), len(self.shape)


class TensorTrain:
    """Device-resident accumulation (include/ttg.h ``ttg_tt``).

    Accessors mirror tensor_train.hpp:51-93; ``core(i)`` downloads a compact
    (r_left, n, r_right) copy (first-index-fastest) for inspection.
    """

    def __init__(self, handle: ctypes.c_void_p, ctx: Context):
        self._h = handle
        self.ctx = ctx

    # -- construction from host data (TensorTrain ctor, tensor_train.cpp:60-93)
    @staticmethod
    def upload(cores: Sequence[np.ndarray], ortho_count: int, batch_boundaries: Sequence[int] = (),
               ctx: Optional[Context] = None) -> "TensorTrain":
        ctx = ctx or default_context()
        n = len(cores)
        rl = (ctypes.c_int64 * n)(*[c.shape[0] for c in cores])
        nn = (ctypes.c_int64 * n)(*[c.shape[1] for c in cores])
        rr = (ctypes.c_int64 * n)(*[c.shape[2] for c in cores])
        keep = [np.asfortranarray(c, dtype=np.float64) for c in cores]
        ptrs = (ctypes.POINTER(ctypes.c_double) * n)(*[k.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for k in keep])
        nb = len(batch_boundaries)
        bnd = (ctypes.c_int64 * max(nb, 1))(*batch_boundaries) if nb else None
        h = ctypes.c_void_p()
        _check(_lib.load().ttg_tt_upload(ctx._h, n, rl, nn, rr, ptrs, int(ortho_count), bnd, nb, ctypes.byref(h)), ctx)
        return TensorTrain(h, ctx)

    def _shape(self):
        nc = _lib.load().ttg_tt_num_cores(self._h)
        ranks = (ctypes.c_int64 * (nc + 1))()
        modes = (ctypes.c_int64 * nc)()
        oc = ctypes.c_int64()
        nb = ctypes.c_int64()
        _check(_lib.load().ttg_tt_shape(self._h, ranks, modes, ctypes.byref(oc), ctypes.byref(nb)), self.ctx)
        return list(ranks), list(modes), oc.value, nb.value

    def num_cores(self) -> int:
        return _lib.load().ttg_tt_num_cores(self._h)

    def spatial_dims(self) -> int:
        return self.num_cores() - 1

    def ranks(self) -> List[int]:
        return self._shape()[0]

    def mode_sizes(self) -> List[int]:
        return self._shape()[1]

    def spatial_shape(self) -> List[int]:
        return self._shape()[1][:-1]

    @property
    def ortho_count(self) -> int:
        return self._shape()[2]

    def fully_orthonormal(self) -> bool:
        return self.ortho_count == self.num_cores() - 1

    def obs_count(self) -> int:
        return self._shape()[1][-1]

    def batch_boundaries(self) -> List[int]:
        nb = self._shape()[3]
        out = (ctypes.c_int64 * max(nb, 1))()
        _check(_lib.load().ttg_tt_bounds(self._h, out), self.ctx)
        return list(out)[:nb]

    def num_increments(self) -> int:
        return self._shape()[3]

    def increment_range(self, k: int):
        """tensor_train.cpp:117-123."""
        from .errors import IndexError_

        bb = self.batch_boundaries()
        if k < 0 or k >= len(bb):
            raise IndexError_("increment index out of range")
        return (0 if k == 0 else bb[k - 1]), bb[k]

    def measure_ortho_count(self, tol: float = 1e-10) -> int:
        """tensor_train.cpp:135-146, measured on the device."""
        out = ctypes.c_int64()
        _check(_lib.load().ttg_tt_measure_ortho_count(self.ctx._h, self._h, float(tol), ctypes.byref(out)), self.ctx)
        return int(out.value)

    def core(self, i: int) -> np.ndarray:
        ranks, modes, _, _ = self._shape()
        shape = (ranks[i], modes[i], ranks[i + 1])
        buf = np.empty(int(np.prod(shape)), dtype=np.float64)
        _check(_lib.load().ttg_tt_download_core(self.ctx._h, self._h, i,
                                                 buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), self.ctx)
        return np.reshape(buf, shape, order="F")

    def cores(self) -> List[np.ndarray]:
        return [self.core(i) for i in range(self.num_cores())]

    def param_count(self) -> int:
        r, m, _, _ = self._shape()
        return sum(r[i] * m[i] * r[i + 1] for i in range(len(m)))

    def close(self) -> None:
        if self._h:
            _lib.load().ttg_tt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tt_ice_bootstrap(y, eps_des: float, ctx: Optional[Context] = None, shape=None) -> Tuple[TensorTrain, UpdateReport]:
    """tt_ice.cpp:143-165: TT-SVD of the first increment (tt_svd.cpp:9-66), on device."""
    ctx = ctx or default_context()
    inp = _Input(y, shape, ctx)
    sh, nd = inp.shape_arr()
    h = ctypes.c_void_p()
    rep = _lib.Report()
    _check(_lib.load().ttg_bootstrap(ctx._h, inp.ptr, inp.where, sh, nd, float(eps_des), ctypes.byref(h),
                                     ctypes.byref(rep)), ctx)
    return TensorTrain(h, ctx), UpdateReport._from(rep)


def tt_ice_update(tt: TensorTrain, y, eps_des: float, shape=None) -> Tuple[TensorTrain, UpdateReport]:
    """tt_ice.cpp:131-141 (uniform delta = eps_des |y|_F / sqrt(d)); updates ``tt`` in place."""
    inp = _Input(y, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    rep = _lib.Report()
    _check(_lib.load().ttg_tt_ice_update(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd, float(eps_des),
                                         ctypes.byref(rep)), tt.ctx)
    return tt, UpdateReport._from(rep)


def tt_ice_update_with_tolerances(tt: TensorTrain, y, deltas: Sequence[float], shape=None):
    """tt_ice.cpp:60-129 (one absolute threshold per spatial mode)."""
    inp = _Input(y, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    rep = _lib.Report()
    dl = (ctypes.c_double * max(len(deltas), 1))(*[float(x) for x in deltas])
    _check(_lib.load().ttg_tt_ice_update_with_tolerances(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd, dl,
                                                         len(deltas), ctypes.byref(rep)), tt.ctx)
    return tt, UpdateReport._from(rep)


def tt_ice_star_update(tt: TensorTrain, y, eps_des: float, cfg: Optional[HeuristicConfig] = None, shape=None):
    """tt_ice_star.cpp:171-303 (Algorithm 2); updates ``tt`` in place."""
    cfg = cfg or HeuristicConfig()
    inp = _Input(y, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    rep = _lib.Report()
    h = cfg._to()
    _check(_lib.load().ttg_tt_ice_star_update(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd, float(eps_des),
                                              ctypes.byref(h), ctypes.byref(rep)), tt.ctx)
    return tt, UpdateReport._from(rep)


def per_obs_errors(tt: TensorTrain, y, shape=None) -> np.ndarray:
    """tt_ice_star.cpp:86-88."""
    inp = _Input(y, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    out = np.empty(inp.shape[-1], dtype=np.float64)
    _check(_lib.load().ttg_per_obs_errors(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd,
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), tt.ctx)
    return out


def tt_project(tt: TensorTrain, y, shape=None) -> np.ndarray:
    """tensor_train.cpp:195-226: r_d x n_obs latent coefficients."""
    inp = _Input(y, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    r_d = tt.ranks()[-2]
    out = np.empty((r_d, inp.shape[-1]), dtype=np.float64, order="F")
    _check(_lib.load().ttg_project(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd,
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), tt.ctx)
    return out


def tt_reconstruct(tt: TensorTrain, obs_begin: int = 0, obs_end: Optional[int] = None, out=None):
    """tensor_train.cpp:182-193.  ``out`` may be a torch CUDA float64 tensor (device result)."""
    if obs_end is None:
        obs_end = tt.obs_count()
    spatial = tt.spatial_shape()
    m = obs_end - obs_begin
    if out is None:
        host = np.empty(int(np.prod(spatial)) * max(m, 0), dtype=np.float64)
        _check(_lib.load().ttg_reconstruct(tt.ctx._h, tt._h, int(obs_begin), int(obs_end),
                                           host.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), TTG_HOST), tt.ctx)
        return np.reshape(host, tuple(spatial) + (m,), order="F")
    import torch

    lib = _lib.load()
    ts = torch.cuda.current_stream(out.device).cuda_stream
    ptr = ctypes.cast(ctypes.c_void_p(out.data_ptr()), ctypes.POINTER(ctypes.c_double))
    _check(lib.ttg_ctx_wait_stream(tt.ctx._h, ts), tt.ctx)  # torch's pending use of ``out`` first
    _check(lib.ttg_reconstruct(tt.ctx._h, tt._h, int(obs_begin), int(obs_end), ptr, TTG_DEVICE), tt.ctx)
    _check(lib.ttg_ctx_join_stream(tt.ctx._h, ts), tt.ctx)  # torch reads ``out`` after the write
    return out


def occupancy(core: np.ndarray) -> float:
    """tensor_train.cpp:377-380 on a (r_left, n, r_right) core."""
    return core.shape[2] / float(core.shape[0] * core.shape[1])


def relaxed_tolerance_approx(n_batch: int, n_rejected: int, mean_rejected_error: float, eps_des: float) -> float:
    """tt_ice_star.cpp:160-169 (Eq. 3.20); scalar host helper of the public API."""
    from .errors import ConfigError

    n_selected = n_batch - n_rejected
    if n_selected < 1:
        raise ConfigError("relaxed tolerance needs a nonempty selection")
    return (eps_des * n_batch - mean_rejected_error * n_rejected) / n_selected


def subselect(errs: Sequence[float], eps_des: float):
    """tt_ice_star.cpp:90-100: (selected, rejected) with the strict '>' test."""
    sel = [i for i, e in enumerate(errs) if e > eps_des]
    rej = [i for i, e in enumerate(errs) if not (e > eps_des)]
    return sel, rej


# ---------------------------------------------------------------------------
# metrics (metrics.hpp / metrics.cpp:7-68), computed on the device
# ---------------------------------------------------------------------------


def compression_ratio(tt: TensorTrain) -> float:
    """metrics.cpp:7-11."""
    out = ctypes.c_double()
    _check(_lib.load().ttg_compression_ratio(tt._h, ctypes.byref(out)), tt.ctx)
    return float(out.value)


def rre(tt: TensorTrain, x_ref, obs_begin: int = 0, obs_end: Optional[int] = None, *, shape=None,
        with_flag: bool = False):
    """metrics.cpp:34-42: ||x_ref - reconstruct(range)|| / ||x_ref|| (0 for a zero-norm reference;
    ``with_flag`` returns (value, zero_reference))."""
    if obs_end is None:
        obs_end = tt.obs_count()
    inp = _Input(x_ref, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    val, zr = ctypes.c_double(), ctypes.c_int()
    _check(_lib.load().ttg_rre(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd, int(obs_begin), int(obs_end),
                               ctypes.byref(val), ctypes.byref(zr)), tt.ctx)
    return (float(val.value), bool(zr.value)) if with_flag else float(val.value)


def rpe(tt: TensorTrain, unseen, *, shape=None, with_flag: bool = False):
    """metrics.cpp:44-47: relative error of tt_expand(tt_project(unseen))."""
    inp = _Input(unseen, shape, tt.ctx)
    sh, nd = inp.shape_arr()
    val, zr = ctypes.c_double(), ctypes.c_int()
    _check(_lib.load().ttg_rpe(tt.ctx._h, tt._h, inp.ptr, inp.where, sh, nd, ctypes.byref(val), ctypes.byref(zr)),
           tt.ctx)
    return (float(val.value), bool(zr.value)) if with_flag else float(val.value)


@dataclass
class IncrementErrors:
    """metrics.hpp:27-30."""

    per_increment: List[float]
    mean: float = 0.0


def mean_rre_per_increment(tt: TensorTrain, refs: Sequence) -> IncrementErrors:
    """metrics.cpp:49-66."""
    from .errors import DimensionError

    if len(refs) != tt.num_increments():
        raise DimensionError("need one reference per stored increment")
    per = []
    for k in range(tt.num_increments()):
        begin, end = tt.increment_range(k)
        ref_shape = refs[k].shape
        if ref_shape[-1] != end - begin:
            raise DimensionError("reference observation count does not match increment")
        per.append(rre(tt, refs[k], begin, end))
    return IncrementErrors(per, (sum(per) / len(per)) if per else 0.0)


# ---------------------------------------------------------------------------
# TTC1 checkpoint (serialization.hpp / serialization.cpp:68-152)
# ---------------------------------------------------------------------------


def serialize(tt: TensorTrain) -> bytes:
    """serialization.cpp:68-87 (strided D2H of the device train)."""
    lib = _lib.load()
    n = ctypes.c_int64()
    _check(lib.ttg_tt_serialize(tt.ctx._h, tt._h, None, 0, ctypes.byref(n)), tt.ctx)
    buf = (ctypes.c_uint8 * n.value)()
    _check(lib.ttg_tt_serialize(tt.ctx._h, tt._h, buf, n.value, ctypes.byref(n)), tt.ctx)
    return bytes(buf)


def deserialize(data: bytes, ctx: Optional[Context] = None) -> TensorTrain:
    """serialization.cpp:89-129; ortho_count re-measured on the device."""
    ctx = ctx or default_context()
    h = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * len(data)).from_buffer_copy(data) if data else None
    _check(_lib.load().ttg_tt_deserialize(ctx._h, buf, len(data), ctypes.byref(h)), ctx)
    return TensorTrain(h, ctx)


def save_ttc(tt: TensorTrain, path) -> None:
    """serialization.cpp:131-139."""
    _check(_lib.load().ttg_tt_save_ttc(tt.ctx._h, tt._h, str(path).encode()), tt.ctx)


def load_ttc(path, ctx: Optional[Context] = None) -> TensorTrain:
    """serialization.cpp:141-152."""
    ctx = ctx or default_context()
    h = ctypes.c_void_p()
    _check(_lib.load().ttg_tt_load_ttc(ctx._h, str(path).encode(), ctypes.byref(h)), ctx)
    return TensorTrain(h, ctx)


# ---------------------------------------------------------------------------
# TTB1 ingest (stream_io.hpp:57-65 / stream_io.cpp:123-204)
# ---------------------------------------------------------------------------


def write_batch(t: np.ndarray, path) -> None:
    """stream_io.cpp:123-137 (first-index-fastest payload)."""
    arr = np.asfortranarray(t, dtype=np.float64)
    sh = (ctypes.c_int64 * arr.ndim)(*arr.shape)
    _check(_lib.load().ttg_write_batch(str(path).encode(), sh, arr.ndim,
                                       arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), None)


def read_batch(path) -> np.ndarray:
    """stream_io.cpp:139-187."""
    lib = _lib.load()
    sh = (ctypes.c_int64 * 255)()
    nd, cnt = ctypes.c_int(), ctypes.c_int64()
    _check(lib.ttg_read_batch(str(path).encode(), sh, ctypes.byref(nd), None, 0, ctypes.byref(cnt)), None)
    out = np.empty(cnt.value, dtype=np.float64)
    _check(lib.ttg_read_batch(str(path).encode(), sh, ctypes.byref(nd),
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cnt.value, ctypes.byref(cnt)), None)
    return np.reshape(out, tuple(sh[:nd.value]), order="F")


def list_stream(directory) -> List[str]:
    """stream_io.cpp:189-204: the .ttb files of a directory in lexicographic filename order."""
    import os

    from .errors import FormatError

    d = str(directory)
    if not os.path.isdir(d):
        raise FormatError("stream path is not a directory: " + d)
    files = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".ttb") and os.path.isfile(os.path.join(d, f))]
    return sorted(files, key=os.path.basename)


class IncrementStream:
    """A .ttb directory streamed to the device: a host thread reads the next
    file into pinned memory and copies it H2D on a side stream while the
    caller updates on the current one (include/ttg.h ``ttg_stream_*``).
    Iterating yields DeviceIncrement objects accepted by every update call."""

    def __init__(self, directory, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self._h = ctypes.c_void_p()
        _check(_lib.load().ttg_stream_open(self.ctx._h, str(directory).encode(), ctypes.byref(self._h)), self.ctx)

    def __len__(self) -> int:
        return int(_lib.load().ttg_stream_count(self._h))

    def next(self) -> DeviceIncrement:
        p = ctypes.POINTER(ctypes.c_double)()
        sh = (ctypes.c_int64 * 255)()
        nd = ctypes.c_int()
        _check(_lib.load().ttg_stream_next(self._h, ctypes.byref(p), sh, ctypes.byref(nd)), self.ctx)
        return DeviceIncrement(ctypes.cast(p, ctypes.c_void_p).value, sh[:nd.value], self)

    def __iter__(self):
        for _ in range(len(self)):
            yield self.next()

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().ttg_stream_close(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
