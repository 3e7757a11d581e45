"""CPU oracle: a numpy restatement of the reference's TT-ICE / TT-ICE* hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker or the timed CPU baseline.  The product path
(``paper_2211_12487_b200``) never imports it and fails loudly when its CUDA
library is missing.

What it restates (reference = /root/reference/proj, C++20 + Eigen):

* ``svd_trunc``                 src/truncated_svd.cpp:29-94  (+ sign rule :16-25)
* ``append_directions``         src/update_common.hpp:19-36  (1e-10 Gram guard)
* ``compute_residual``          src/tt_ice.cpp:34-41
* ``pad_core``                  src/tt_ice.cpp:43-58
* ``tt_ice_update_with_tolerances`` src/tt_ice.cpp:60-129
* ``tt_ice_update``             src/tt_ice.cpp:131-141
* ``tt_ice_bootstrap``          src/tt_ice.cpp:143-165 -> ``tt_svd`` src/tt_svd.cpp:9-66
* ``per_obs_stats`` / ``mean_statistic`` / ``full_batch_statistic`` /
  ``project_through`` / ``subselect`` / ``gather_obs`` / ``relaxed_tolerance`` /
  ``relaxed_tolerance_approx`` / ``tt_ice_star_update``
                                src/tt_ice_star.cpp:22-303
* ``tt_project`` / ``tt_expand`` / ``tt_reconstruct`` / ``spatial_chain`` /
  ``occupancy`` / ``tt_norm`` / ``measure_ortho_count``
                                src/tensor_train.cpp:135-226, 377-390
* ``compression_ratio`` / ``rre`` / ``rpe`` / ``mean_rre_per_increment``
                                src/metrics.cpp:7-68
* ``serialize`` / ``deserialize`` (TTC1)  src/serialization.cpp:68-129
* ``write_batch`` / ``read_batch`` (TTB1) / ``list_stream``
                                src/stream_io.cpp:123-204

Parity status: PINNED to the reference itself.  The reference library's own
sources (/root/reference/proj/src/*.cpp) compile unchanged against the
Eigen-API shim in oracle/eigen_shim (oracle/Makefile -> oracle/_ref/
libttref.so, bound by oracle/ref_binding.py with this module's names);
tests/test_ref_pin.py runs the same seeded bytes through both on cfg0, reduced
cfg1/2/3, every TT-ICE* heuristic variant, the Appendix-B eps = 1e-8 cases, the
edge cases and the SPEC known-answer examples, at the north-star bar.  The
committed cfg0 golden fixtures are the reference's output.  The GPU parity
tests use the reference library as their checker when it is present and this
restatement otherwise.

Eigen -> LAPACK mapping: Eigen::BDCSVD -> numpy.linalg.svd (LAPACK dgesdd,
the same divide-and-conquer family); Eigen::HouseholderQR -> numpy.linalg.qr
(dgeqrf + dorgqr, same Householder sign convention beta = -sign(x0)*|x|).
Results agree with Eigen to rounding level, not bitwise.

Layout: every tensor is a numpy array in Fortran (first-index-fastest) order,
exactly the reference's linearisation (dense_tensor.hpp:18-22).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

# --------------------------------------------------------------------------
# errors (include/ttstream/errors.hpp:9-55)
# --------------------------------------------------------------------------


class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class NumericError(Error):
    pass


class StateError(Error):
    pass


class FormatError(Error):
    pass


class IndexError_(Error):
    pass


class ConfigError(Error):
    pass


class ResourceError(Error):
    pass


def _as_matrix(t: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """DenseTensor::as_matrix (dense_tensor.cpp:106-111): zero-copy F-order view."""
    if rows * cols != t.size:
        raise DimensionError("matrix view extents do not cover the buffer")
    return np.reshape(t, (rows, cols), order="F")


def frobenius_norm(t: np.ndarray) -> float:
    """DenseTensor::frobenius_norm (dense_tensor.cpp:113-115)."""
    return float(np.linalg.norm(np.ravel(t, order="K")))


# --------------------------------------------------------------------------
# TT container (tensor_train.hpp:12-93)
# --------------------------------------------------------------------------


@dataclass
class TTCore:
    """r_left x n x r_right core, first-index-fastest (tensor_train.cpp:12-58)."""

    data: np.ndarray  # shape (r_left, n, r_right), Fortran order

    @property
    def r_left(self) -> int:
        return self.data.shape[0]

    @property
    def n(self) -> int:
        return self.data.shape[1]

    @property
    def r_right(self) -> int:
        return self.data.shape[2]

    def left_unfolding(self) -> np.ndarray:
        return np.reshape(self.data, (self.r_left * self.n, self.r_right), order="F")

    def right_unfolding(self) -> np.ndarray:
        return np.reshape(self.data, (self.r_left, self.n * self.r_right), order="F")

    @staticmethod
    def from_left_unfolding(u: np.ndarray, r_left: int, n: int) -> "TTCore":
        """tensor_train.cpp:32-40 (copy + finiteness scan of the ctor :20-24)."""
        if u.shape[0] != r_left * n:
            raise DimensionError("left unfolding rows do not factor as r_left * n")
        if not np.all(np.isfinite(u)):
            raise NumericError("non-finite element rejected at core construction")
        return TTCore(np.asfortranarray(np.reshape(u, (r_left, n, u.shape[1]), order="F")).copy(order="F"))

    @staticmethod
    def from_right_unfolding(m: np.ndarray, n: int, r_right: int) -> "TTCore":
        """tensor_train.cpp:42-50."""
        if m.shape[1] != n * r_right:
            raise DimensionError("right unfolding columns do not factor as n * r_right")
        if not np.all(np.isfinite(m)):
            raise NumericError("non-finite element rejected at core construction")
        return TTCore(np.asfortranarray(np.reshape(m, (m.shape[0], n, r_right), order="F")).copy(order="F"))


@dataclass
class TensorTrain:
    """tensor_train.hpp:51-93; ctor validation tensor_train.cpp:60-93."""

    cores: List[TTCore]
    ortho_count: int
    batch_boundaries: List[int] = field(default_factory=list)

    def __post_init__(self):
        if not self.cores:
            raise DimensionError("a train needs at least one core")
        if self.cores[0].r_left != 1 or self.cores[-1].r_right != 1:
            raise DimensionError("boundary ranks must be 1")
        for i in range(len(self.cores) - 1):
            if self.cores[i].r_right != self.cores[i + 1].r_left:
                raise DimensionError(f"bond rank mismatch between cores {i} and {i + 1}")
        if self.ortho_count < 0 or self.ortho_count > len(self.cores) - 1:
            raise StateError("ortho_count outside [0, D-1]")
        if not self.batch_boundaries:
            self.batch_boundaries = [self.obs_count()]
        prev = 0
        for b in self.batch_boundaries:
            if b < prev:
                raise DimensionError("batch boundaries must be nondecreasing")
            prev = b
        if self.batch_boundaries[-1] != self.obs_count():
            raise DimensionError("batch boundaries must end at the observation count")

    def num_cores(self) -> int:
        return len(self.cores)

    def spatial_dims(self) -> int:
        return len(self.cores) - 1

    def core(self, i: int) -> TTCore:
        return self.cores[i]

    def ranks(self) -> List[int]:
        return [self.cores[0].r_left] + [c.r_right for c in self.cores]

    def mode_sizes(self) -> List[int]:
        return [c.n for c in self.cores]

    def spatial_shape(self) -> List[int]:
        return [c.n for c in self.cores[:-1]]

    def fully_orthonormal(self) -> bool:
        return self.ortho_count == self.num_cores() - 1

    def obs_count(self) -> int:
        return self.cores[-1].n

    def num_increments(self) -> int:
        return len(self.batch_boundaries)

    def increment_range(self, k: int) -> Tuple[int, int]:
        if k < 0 or k >= self.num_increments():
            raise IndexError_("increment index out of range")
        begin = 0 if k == 0 else self.batch_boundaries[k - 1]
        return begin, self.batch_boundaries[k]

    def param_count(self) -> int:
        return sum(c.data.size for c in self.cores)

    def measure_ortho_count(self, tol: float = 1e-10) -> int:
        """tensor_train.cpp:135-146."""
        count = 0
        for i in range(self.num_cores() - 1):
            u = self.cores[i].left_unfolding()
            dev = np.max(np.abs(u.T @ u - np.eye(u.shape[1])))
            if dev > tol:
                break
            count += 1
        return count


@dataclass
class UpdateReport:
    """tt_ice.hpp:10-20. ``seconds`` is wall time here (the reference uses std::clock)."""

    increment_index: int = 0
    obs_in_batch: int = 0
    obs_used: int = 0
    ranks_before: List[int] = field(default_factory=list)
    ranks_after: List[int] = field(default_factory=list)
    eps_target: float = 0.0
    batch_rel_error_estimate: float = 0.0
    seconds: float = 0.0
    tolerance_clamped: bool = False


# --------------------------------------------------------------------------
# truncated SVD (truncated_svd.cpp)
# --------------------------------------------------------------------------

K_TALL_ASPECT = 2.0  # truncated_svd.cpp:14


@dataclass
class TruncatedSvd:
    u: np.ndarray
    s: np.ndarray
    vt: np.ndarray
    rank: int = 0
    tail_norm: float = 0.0

    def scaled_vt(self) -> np.ndarray:
        return self.s[:, None] * self.vt


def normalize_column_signs(u: np.ndarray, vt: np.ndarray) -> None:
    """truncated_svd.cpp:16-25: largest-|.| entry (first max index) made positive."""
    for j in range(u.shape[1]):
        imax = int(np.argmax(np.abs(u[:, j])))  # argmax returns the first max, like Eigen
        if u[imax, j] < 0.0:
            u[:, j] = -u[:, j]
            vt[j, :] = -vt[j, :]


def _householder_q(a: np.ndarray) -> np.ndarray:
    """Thin Q of Householder QR (Eigen::HouseholderQR + householderQ() applied to I)."""
    q, _ = np.linalg.qr(a, mode="reduced")
    return q


def svd_trunc(a: np.ndarray, delta: float) -> TruncatedSvd:
    """truncated_svd.cpp:29-94."""
    a = np.asarray(a, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise NumericError("svd_trunc: non-finite input matrix")
    if delta < 0.0:
        raise NumericError("svd_trunc: negative truncation threshold")
    m, l = a.shape
    if m == 0 or l == 0:
        return TruncatedSvd(np.zeros((m, 0)), np.zeros(0), np.zeros((0, l)), 0, 0.0)
    tall = float(m) > K_TALL_ASPECT * float(l)  # :51
    if tall:
        q, r = np.linalg.qr(a, mode="reduced")  # :53-56
        reduced = np.triu(r)
    else:
        reduced = a
    try:
        uu, sigma, vt = np.linalg.svd(reduced, full_matrices=False)  # :61 BDCSVD thin
    except np.linalg.LinAlgError as e:  # :62-67
        raise NumericError(f"svd_trunc: backend failed on {m}x{l} matrix") from e
    k = sigma.size
    tail_sq = 0.0
    rank = k
    for j in range(k - 1, -1, -1):  # :74-81, '>' test keeps the smaller rank on ties
        nxt = tail_sq + sigma[j] * sigma[j]
        if math.sqrt(nxt) > delta:
            break
        tail_sq = nxt
        rank = j
    u = uu[:, :rank].copy()
    if tall:
        u = q @ u
    out_vt = vt[:rank, :].copy()
    normalize_column_signs(u, out_vt)  # :92
    return TruncatedSvd(u, sigma[:rank].copy(), out_vt, rank, math.sqrt(tail_sq))


# --------------------------------------------------------------------------
# TT-ICE building blocks (tt_ice.cpp, update_common.hpp)
# --------------------------------------------------------------------------

K_GRAM_GUARD = 1e-10  # update_common.hpp:17


def append_directions(u_pad: np.ndarray, u_new: np.ndarray) -> np.ndarray:
    """update_common.hpp:19-36."""
    if u_new.shape[1] == 0:
        return u_pad
    combined = np.concatenate([u_pad, u_new], axis=1)
    gram = combined.T @ combined
    dev = np.max(np.abs(gram - np.eye(gram.shape[0])))
    if dev > K_GRAM_GUARD:
        corrected = u_new - u_pad @ (u_pad.T @ u_new)
        combined[:, u_pad.shape[1]:] = _householder_q(corrected)
    return combined


def compute_residual(u_pad: np.ndarray, y: np.ndarray) -> np.ndarray:
    """tt_ice.cpp:34-41."""
    if u_pad.shape[1] == 0:
        return y
    if u_pad.shape[0] != y.shape[0]:
        raise DimensionError("residual operands have mismatched row counts")
    return y - u_pad @ (u_pad.T @ y)


def pad_core(u_next: np.ndarray, r_left_old: int, added_rank: int) -> np.ndarray:
    """tt_ice.cpp:43-58 (Eq. 3.4)."""
    if added_rank < 0:
        raise DimensionError("added rank must be nonnegative")
    if r_left_old < 1 or u_next.shape[0] % r_left_old != 0:
        raise DimensionError("unfolding rows do not factor as r_left * n")
    if added_rank == 0:
        return u_next
    n = u_next.shape[0] // r_left_old
    r_right = u_next.shape[1]
    r_new = r_left_old + added_rank
    as_rows = np.reshape(u_next, (r_left_old, n * r_right), order="F")
    grown = np.zeros((r_new, n * r_right))
    grown[:r_left_old, :] = as_rows
    return np.reshape(grown, (r_new * n, r_right), order="F")


def _check_update_preconditions(tt: TensorTrain, y: np.ndarray) -> None:
    """tt_ice.cpp:16-30."""
    if not tt.fully_orthonormal():
        raise StateError("incremental update requires a fully orthonormal train")
    d = tt.spatial_dims()
    if y.ndim != d + 1:
        raise DimensionError("increment must carry the spatial shape plus an observation mode")
    for i, n in enumerate(tt.spatial_shape()):
        if y.shape[i] != n:
            raise DimensionError("increment spatial shape does not match the train")


def _check_finite(y: np.ndarray) -> None:
    """DenseTensor ctor finiteness scan (dense_tensor.cpp:48-52)."""
    if not np.all(np.isfinite(y)):
        raise NumericError("non-finite element rejected at tensor construction")


def tt_ice_update_with_tolerances(tt: TensorTrain, y: np.ndarray, deltas: Sequence[float]):
    """tt_ice.cpp:60-129 (Algorithm 1)."""
    t0 = time.perf_counter()
    _check_finite(y)
    _check_update_preconditions(tt, y)
    d = tt.spatial_dims()
    if len(deltas) != d:
        raise DimensionError("need one SVD tolerance per spatial dimension")
    n_obs = y.shape[d]
    y_norm = frobenius_norm(y)

    report = UpdateReport(
        increment_index=tt.num_increments(), obs_in_batch=n_obs, obs_used=n_obs,
        ranks_before=tt.ranks(), eps_target=(deltas[0] if len(deltas) else 0.0))

    new_cores: List[TTCore] = []
    cur = _as_matrix(y, y.shape[0], y.size // y.shape[0])  # :82
    u_pad = tt.core(0).left_unfolding()
    r_left_new = 1
    discarded_sq = 0.0
    for i in range(d):  # :87-109
        r_old = u_pad.shape[1]
        u_new = u_pad
        resid = compute_residual(u_pad, cur)
        svd = svd_trunc(resid, deltas[i])
        discarded_sq += svd.tail_norm * svd.tail_norm
        if svd.rank > 0:
            u_new = append_directions(u_pad, svd.u)
        r_new = u_new.shape[1]
        new_cores.append(TTCore.from_left_unfolding(u_new, r_left_new, tt.core(i).n))
        proj = u_new.T @ cur  # :100
        if i + 1 < d:
            u_pad = pad_core(tt.core(i + 1).left_unfolding(), r_old, r_new - r_old)
            rows = r_new * tt.core(i + 1).n
            cur = np.reshape(proj, (rows, proj.size // rows), order="F")
        else:
            cur = proj
        r_left_new = r_new

    last = tt.core(d)  # :111-118
    n_old = last.n
    new_last = np.zeros((r_left_new, n_old + n_obs))
    new_last[:last.r_left, :n_old] = last.right_unfolding()
    new_last[:, n_old:] = cur
    new_cores.append(TTCore.from_right_unfolding(new_last, n_old + n_obs, 1))
    boundaries = list(tt.batch_boundaries) + [n_old + n_obs]
    updated = TensorTrain(new_cores, d, boundaries)
    report.ranks_after = updated.ranks()
    report.batch_rel_error_estimate = 0.0 if y_norm == 0.0 else math.sqrt(discarded_sq) / y_norm
    report.seconds = time.perf_counter() - t0
    return updated, report


def tt_ice_update(tt: TensorTrain, y: np.ndarray, eps_des: float):
    """tt_ice.cpp:131-141: uniform delta = eps_des*|y|_F/sqrt(d) (Cor. 3.2)."""
    if eps_des <= 0.0:
        raise NumericError("eps_des must be positive")
    d = tt.spatial_dims()
    eps = eps_des * frobenius_norm(y) / math.sqrt(float(d))
    return tt_ice_update_with_tolerances(tt, y, [eps] * d)


def tt_svd(y: np.ndarray, eps_rel: float) -> TensorTrain:
    """tt_svd.cpp:9-66."""
    if eps_rel < 0.0 or eps_rel > 1.0:
        raise NumericError("tt_svd tolerance must lie in [0, 1]")
    _check_finite(y)
    nd = y.ndim
    norm = frobenius_norm(y)
    if nd <= 1:
        n = 1 if nd == 0 else y.shape[0]
        svd = svd_trunc(_as_matrix(y, n, 1), eps_rel * norm)
        buf = np.zeros(n)
        if svd.rank == 1:
            buf = (svd.u @ svd.scaled_vt())[:, 0]
        return TensorTrain([TTCore(np.reshape(buf, (1, n, 1), order="F"))], 0)
    delta = eps_rel / math.sqrt(float(nd - 1)) * norm  # :30
    cores: List[TTCore] = []
    r_prev = 1
    carry = _as_matrix(y, y.shape[0], y.size // y.shape[0])
    for i in range(nd - 1):  # :37-60
        n_i = y.shape[i]
        svd = svd_trunc(carry, delta)
        if svd.rank == 0:  # :42-47 unit-column placeholder
            u = np.zeros((carry.shape[0], 1))
            u[0, 0] = 1.0
            nxt = np.zeros((1, carry.shape[1]))
        else:
            u = svd.u
            nxt = svd.scaled_vt()
        cores.append(TTCore.from_left_unfolding(u, r_prev, n_i))
        r_prev = u.shape[1]
        if i + 2 < nd:
            rows = r_prev * y.shape[i + 1]
            carry = np.reshape(nxt, (rows, nxt.size // rows), order="F")
        else:
            carry = nxt
    cores.append(TTCore.from_left_unfolding(np.reshape(carry, (carry.size, 1), order="F"),
                                            r_prev, y.shape[nd - 1]))
    return TensorTrain(cores, nd - 1)


def tt_norm(tt: TensorTrain) -> float:
    """tensor_train.cpp:382-390 (orthonormal branch; the sweep fallback is not on the path)."""
    if tt.fully_orthonormal():
        return float(np.linalg.norm(tt.cores[-1].data.ravel(order="F")))
    return float(np.linalg.norm(tt_reconstruct(tt).ravel(order="F")))


def tt_ice_bootstrap(y: np.ndarray, eps_des: float):
    """tt_ice.cpp:143-165."""
    t0 = time.perf_counter()
    tt = tt_svd(y, eps_des)
    report = UpdateReport(increment_index=0, obs_in_batch=y.shape[-1], obs_used=y.shape[-1])
    report.ranks_after = tt.ranks()
    report.ranks_before = [1] * len(report.ranks_after)
    y_norm = frobenius_norm(y)
    report.eps_target = (eps_des * y_norm / math.sqrt(float(y.ndim - 1))) if y.ndim > 1 else eps_des * y_norm
    kept = tt_norm(tt)
    lost_sq = max(y_norm * y_norm - kept * kept, 0.0)
    report.batch_rel_error_estimate = 0.0 if y_norm == 0.0 else math.sqrt(lost_sq) / y_norm
    report.seconds = time.perf_counter() - t0
    return tt, report


# --------------------------------------------------------------------------
# projection / expansion (tensor_train.cpp:152-226)
# --------------------------------------------------------------------------


def spatial_chain(tt: TensorTrain) -> np.ndarray:
    """tensor_train.cpp:152-166: the (n_1..n_d) x r_d basis matrix."""
    d = tt.spatial_dims()
    if d == 0:
        return np.eye(1)
    acc = tt.core(0).left_unfolding()
    rows = tt.core(0).n
    for i in range(1, d):
        c = tt.core(i)
        nxt = acc @ c.right_unfolding()
        rows *= c.n
        acc = np.reshape(nxt, (rows, c.r_right), order="F")
    return acc


def tt_expand(tt: TensorTrain, coeffs: np.ndarray) -> np.ndarray:
    """tensor_train.cpp:170-180."""
    d = tt.spatial_dims()
    r_d = 1 if d == 0 else tt.core(d - 1).r_right
    if coeffs.shape[0] != r_d:
        raise DimensionError("coefficient rows do not match the train's last bond rank")
    dense = spatial_chain(tt) @ coeffs
    return np.reshape(dense, tuple(tt.spatial_shape()) + (coeffs.shape[1],), order="F")


def tt_reconstruct(tt: TensorTrain, obs_begin: int = 0, obs_end: Optional[int] = None) -> np.ndarray:
    """tensor_train.cpp:182-193."""
    if obs_end is None:
        obs_end = tt.obs_count()
    if obs_begin < 0 or obs_end > tt.obs_count() or obs_begin > obs_end:
        raise IndexError_("observation range out of bounds")
    coeffs = tt.cores[-1].right_unfolding()
    return tt_expand(tt, coeffs[:, obs_begin:obs_end])


def tt_project(tt: TensorTrain, y: np.ndarray) -> np.ndarray:
    """tensor_train.cpp:195-226: r_d x n_obs latent coefficients."""
    if not tt.fully_orthonormal():
        raise StateError("projection requires a fully orthonormal train")
    d = tt.spatial_dims()
    if y.ndim != d + 1:
        raise DimensionError("data must carry the spatial shape plus an observation mode")
    for i, n in enumerate(tt.spatial_shape()):
        if y.shape[i] != n:
            raise DimensionError("data spatial shape does not match the train")
    n_obs = y.shape[d]
    cur = _as_matrix(y, y.shape[0], y.size // y.shape[0])
    for i in range(d):
        u = tt.core(i).left_unfolding()
        nxt = u.T @ cur
        if i + 1 < d:
            rows = tt.core(i).r_right * tt.core(i + 1).n
            cur = np.reshape(nxt, (rows, nxt.size // rows), order="F")
        else:
            cur = nxt
    if cur.shape[1] != n_obs:
        raise DimensionError("projection produced inconsistent observation count")
    return cur


def occupancy(core: TTCore) -> float:
    """tensor_train.cpp:377-380."""
    return core.r_right / float(core.r_left * core.n)


# --------------------------------------------------------------------------
# TT-ICE* (tt_ice_star.cpp)
# --------------------------------------------------------------------------


@dataclass
class HeuristicConfig:
    """tt_ice_star.hpp:14-20."""

    occupancy_threshold: float = 0.8
    skip_enabled: bool = True
    subselect_enabled: bool = True
    skip_statistic: str = "mean"  # "mean" (kMean) | "full" (kFullBatch)
    use_approx_tolerance: bool = False


@dataclass
class PerObsStats:
    errs: np.ndarray
    resid_norms: np.ndarray
    obs_norms: np.ndarray


def per_obs_stats(tt: TensorTrain, y: np.ndarray) -> PerObsStats:
    """tt_ice_star.cpp:22-42."""
    coeffs = tt_project(tt, y)
    approx = tt_expand(tt, coeffs)
    n_obs = coeffs.shape[1]
    n_spatial = y.size // n_obs
    ym = _as_matrix(y, n_spatial, n_obs)
    am = _as_matrix(approx, n_spatial, n_obs)
    rn = np.linalg.norm(ym - am, axis=0)
    on = np.linalg.norm(ym, axis=0)
    errs = np.where(on == 0.0, 0.0, rn / np.where(on == 0.0, 1.0, on))
    return PerObsStats(errs, rn, on)


def per_obs_errors(tt: TensorTrain, y: np.ndarray) -> np.ndarray:
    return per_obs_stats(tt, y).errs


def mean_statistic(s: PerObsStats) -> float:
    """tt_ice_star.cpp:46-56: mean over nonzero-norm observations."""
    total = 0.0
    count = 0
    for e, on in zip(s.errs, s.obs_norms):
        if on > 0.0:
            total += float(e)
            count += 1
    return 0.0 if count == 0 else total / count


def full_batch_statistic(s: PerObsStats) -> float:
    """tt_ice_star.cpp:58-65 (Eq. 3.21)."""
    num = float(np.sum(s.resid_norms ** 2))
    den = float(np.sum(s.obs_norms ** 2))
    return 0.0 if den == 0.0 else math.sqrt(num / den)


def project_through(u_list: Sequence[np.ndarray], mode_sizes: Sequence[int], y: np.ndarray) -> np.ndarray:
    """tt_ice_star.cpp:68-82."""
    d = len(u_list)
    cur = _as_matrix(y, y.shape[0], y.size // y.shape[0])
    for i in range(d):
        nxt = u_list[i].T @ cur
        if i + 1 < d:
            rows = nxt.shape[0] * mode_sizes[i + 1]
            cur = np.reshape(nxt, (rows, nxt.size // rows), order="F")
        else:
            cur = nxt
    return cur


@dataclass
class SubselectSplit:
    selected: List[int] = field(default_factory=list)
    rejected: List[int] = field(default_factory=list)


def subselect(errs: Sequence[float], eps_des: float) -> SubselectSplit:
    """tt_ice_star.cpp:90-100 (strict '>')."""
    split = SubselectSplit()
    for i, e in enumerate(errs):
        (split.selected if e > eps_des else split.rejected).append(i)
    return split


def gather_obs(y: np.ndarray, idx: Sequence[int]) -> np.ndarray:
    """tt_ice_star.cpp:102-119."""
    if len(idx) == 0:
        raise DimensionError("cannot gather an empty observation set")
    n_obs = y.shape[-1]
    for i in idx:
        if i < 0 or i >= n_obs:
            raise IndexError_("observation index out of range")
    return np.asfortranarray(y[..., list(idx)])


def relaxed_tolerance(y: np.ndarray, split: SubselectSplit, errs: Sequence[float], eps_des: float):
    """tt_ice_star.cpp:121-158 (Eq. 3.19). Returns (eps_upd, clamped)."""
    if not split.selected:
        raise ConfigError("relaxed tolerance needs a nonempty selection")
    if not split.rejected:
        return eps_des, False
    n_obs = y.shape[-1]
    ym = _as_matrix(y, y.size // n_obs, n_obs)
    rejected_resid_sq = 0.0
    for i in split.rejected:
        on = float(np.linalg.norm(ym[:, i]))
        rn = float(errs[i]) * on
        rejected_resid_sq += rn * rn
    selected_sq = 0.0
    for i in split.selected:
        selected_sq += float(np.dot(ym[:, i], ym[:, i]))
    if selected_sq == 0.0:
        raise NumericError("selected observations carry no energy")
    budget = eps_des * frobenius_norm(y)
    radicand = (budget * budget - rejected_resid_sq) / selected_sq
    clamped = False
    if radicand < 0.0:
        radicand = 0.0
        clamped = True
    return math.sqrt(radicand), clamped


def relaxed_tolerance_approx(n_batch: int, n_rejected: int, mean_rejected_error: float, eps_des: float) -> float:
    """tt_ice_star.cpp:160-169 (Eq. 3.20)."""
    n_selected = n_batch - n_rejected
    if n_selected < 1:
        raise ConfigError("relaxed tolerance needs a nonempty selection")
    return (eps_des * n_batch - mean_rejected_error * n_rejected) / n_selected


def tt_ice_star_update(tt: TensorTrain, y: np.ndarray, eps_des: float, cfg: Optional[HeuristicConfig] = None):
    """tt_ice_star.cpp:171-303 (Algorithm 2)."""
    cfg = cfg or HeuristicConfig()
    t0 = time.perf_counter()
    if eps_des <= 0.0:
        raise NumericError("eps_des must be positive")
    if cfg.occupancy_threshold <= 0.0 or cfg.occupancy_threshold > 1.0:
        raise ConfigError("occupancy threshold must lie in (0, 1]")
    _check_finite(y)
    d = tt.spatial_dims()
    n_obs = y.shape[y.ndim - 1]
    y_norm = frobenius_norm(y)
    report = UpdateReport(increment_index=tt.num_increments(), obs_in_batch=n_obs, ranks_before=tt.ranks())

    stats = per_obs_stats(tt, y)
    skip_stat = mean_statistic(stats) if cfg.skip_statistic == "mean" else full_batch_statistic(stats)

    new_u: List[np.ndarray] = []
    modes = tt.mode_sizes()
    cores_changed = False
    split = SubselectSplit()
    if cfg.skip_enabled and skip_stat <= eps_des:  # :201-203
        report.obs_used = 0
    else:
        if cfg.subselect_enabled:
            split = subselect(stats.errs, eps_des)
        else:
            split.selected = list(range(n_obs))
        report.obs_used = len(split.selected)

    if report.obs_used == 0:
        for i in range(d):
            new_u.append(tt.core(i).left_unfolding())
    else:
        eps_upd = eps_des
        if split.rejected:
            if cfg.use_approx_tolerance:
                mean_rej = sum(float(stats.errs[i]) for i in split.rejected) / len(split.rejected)
                eps_upd = relaxed_tolerance_approx(n_obs, len(split.rejected), mean_rej, eps_des)
            else:
                eps_upd, report.tolerance_clamped = relaxed_tolerance(y, split, stats.errs, eps_des)
        selected = gather_obs(y, split.selected)
        delta = eps_upd / math.sqrt(float(d)) * frobenius_norm(selected)  # :235-236
        report.eps_target = delta
        cur = _as_matrix(selected, selected.shape[0], selected.size // selected.shape[0])
        u_pad = tt.core(0).left_unfolding()
        for i in range(d):  # :242-265
            r_old = u_pad.shape[1]
            u_new = u_pad
            occ = u_pad.shape[1] / float(u_pad.shape[0])
            if occ < cfg.occupancy_threshold:
                resid = compute_residual(u_pad, cur)
                svd = svd_trunc(resid, delta)
                if svd.rank > 0:
                    u_new = append_directions(u_pad, svd.u)
                    cores_changed = True
            r_new = u_new.shape[1]
            new_u.append(u_new)
            if i + 1 < d:
                nxt = new_u[-1].T @ cur
                rows = r_new * tt.core(i + 1).n
                cur = np.reshape(nxt, (rows, nxt.size // rows), order="F")
                u_pad = pad_core(tt.core(i + 1).left_unfolding(), r_old, r_new - r_old)

    coeffs = project_through(new_u, modes, y)  # :270
    new_cores: List[TTCore] = []
    r_left = 1
    for i in range(d):
        if not cores_changed:
            new_cores.append(tt.core(i))
        else:
            new_cores.append(TTCore.from_left_unfolding(new_u[i], r_left, tt.core(i).n))
        r_left = new_cores[-1].r_right
    last = tt.core(d)
    n_old = last.n
    new_last = np.zeros((r_left, n_old + n_obs))
    new_last[:last.r_left, :n_old] = last.right_unfolding()
    new_last[:, n_old:] = coeffs
    new_cores.append(TTCore.from_right_unfolding(new_last, n_old + n_obs, 1))
    boundaries = list(tt.batch_boundaries) + [n_old + n_obs]
    updated = TensorTrain(new_cores, d, boundaries)
    report.ranks_after = updated.ranks()
    kept_sq = float(np.sum(coeffs * coeffs))
    lost_sq = max(y_norm * y_norm - kept_sq, 0.0)
    report.batch_rel_error_estimate = 0.0 if y_norm == 0.0 else math.sqrt(lost_sq) / y_norm
    report.seconds = time.perf_counter() - t0
    return updated, report


# --------------------------------------------------------------------------
# parity helpers (tests/helpers.hpp:107-124 pattern)
# --------------------------------------------------------------------------


def interface_projectors(tt: TensorTrain) -> List[np.ndarray]:
    """Phi_k (prod n_{<=k} x r_k) for k = 1..d: basis-invariant core-subspace comparison."""
    out = []
    acc = tt.core(0).left_unfolding()
    out.append(acc)
    rows = tt.core(0).n
    for i in range(1, tt.spatial_dims()):
        c = tt.core(i)
        nxt = acc @ c.right_unfolding()
        rows *= c.n
        acc = np.reshape(nxt, (rows, c.r_right), order="F")
        out.append(acc)
    return out


def rel_diff(a: np.ndarray, b: np.ndarray) -> float:
    """helpers.hpp:119-124."""
    den = float(np.linalg.norm(np.ravel(a)))
    num = float(np.linalg.norm(np.ravel(a) - np.ravel(b)))
    return float(np.linalg.norm(np.ravel(b))) if den == 0.0 else num / den


# --------------------------------------------------------------------------
# metrics (src/metrics.cpp:7-68)
# --------------------------------------------------------------------------


def compression_ratio(tt: TensorTrain) -> float:
    """metrics.cpp:7-11: elements of the represented tensor / stored parameters."""
    elements = 1.0
    for n in tt.mode_sizes():
        elements *= float(n)
    return elements / float(tt.param_count())


def _relative_error(ref: np.ndarray, approx: np.ndarray):
    """metrics.cpp:15-29; returns (error, zero_reference)."""
    if ref.shape != approx.shape:
        raise DimensionError("reference shape does not match reconstruction")
    ref_norm = float(np.linalg.norm(np.ravel(ref, order="F")))
    if ref_norm == 0.0:
        return 0.0, True
    return float(np.linalg.norm(np.ravel(ref, order="F") - np.ravel(approx, order="F"))) / ref_norm, False


def rre(tt: TensorTrain, x_ref: np.ndarray, obs_begin: int = 0, obs_end: Optional[int] = None):
    """metrics.cpp:34-42 -> (rre, zero_reference)."""
    if obs_end is None:
        obs_end = tt.obs_count()
    return _relative_error(x_ref, tt_reconstruct(tt, obs_begin, obs_end))


def rpe(tt: TensorTrain, unseen: np.ndarray):
    """metrics.cpp:44-47 -> (rpe, zero_reference)."""
    coeffs = tt_project(tt, unseen)
    return _relative_error(unseen, tt_expand(tt, coeffs))


def mean_rre_per_increment(tt: TensorTrain, refs: Sequence[np.ndarray]):
    """metrics.cpp:49-66 -> (per-increment list, mean)."""
    if len(refs) != tt.num_increments():
        raise DimensionError("need one reference per stored increment")
    per = []
    for k in range(tt.num_increments()):
        begin, end = tt.increment_range(k)
        if refs[k].shape[-1] != end - begin:
            raise DimensionError("reference observation count does not match increment")
        per.append(rre(tt, refs[k], begin, end)[0])
    return per, (sum(per) / len(per) if per else 0.0)


# --------------------------------------------------------------------------
# TTC1 train image (src/serialization.cpp:68-129): "TTC1", u8 core count,
# per core u64 r_left, n, r_right + little-endian f64 payload, u64 boundary
# count + u64 boundaries.
# --------------------------------------------------------------------------


def serialize(tt: TensorTrain) -> bytes:
    """serialization.cpp:68-87."""
    out = bytearray(b"TTC1")
    out.append(tt.num_cores() & 0xFF)
    for c in tt.cores:
        out += np.array([c.r_left, c.n, c.r_right], dtype="<u8").tobytes()
        out += np.ravel(c.data, order="F").astype("<f8").tobytes()
    out += np.array([len(tt.batch_boundaries)], dtype="<u8").tobytes()
    out += np.array(tt.batch_boundaries, dtype="<u8").tobytes()
    return bytes(out)


def deserialize(data: bytes) -> TensorTrain:
    """serialization.cpp:89-129 (same checks, same messages)."""
    pos = 0

    def need(n):
        if pos + n > len(data):
            raise FormatError("truncated train data")

    def u64():
        nonlocal pos
        need(8)
        v = int.from_bytes(data[pos:pos + 8], "little")
        pos += 8
        return v

    need(4)
    if data[:4] != b"TTC1":
        raise FormatError("bad magic: not a TTC1 train file")
    pos = 4
    need(1)
    nd = data[pos]
    pos += 1
    if nd < 1:
        raise FormatError("train file declares zero cores")
    cores = []
    prev = 1
    for _ in range(nd):
        rl, n, rr = u64(), u64(), u64()
        if rl < 1 or n < 1 or rr < 1:
            raise FormatError("core extents must be positive")
        if rl != prev:
            raise FormatError("bond ranks of adjacent cores disagree")
        if rl * n * rr > len(data) // 8 + 1:
            raise FormatError("truncated train data")
        cnt = rl * n * rr
        need(8 * cnt)
        vals = np.frombuffer(data, dtype="<f8", count=cnt, offset=pos).astype(np.float64)
        pos += 8 * cnt
        if not np.all(np.isfinite(vals)):
            raise NumericError("non-finite element rejected at core construction")
        cores.append(TTCore(np.asfortranarray(np.reshape(vals, (rl, n, rr), order="F"))))
        prev = rr
    if prev != 1:
        raise FormatError("last core must close the chain with rank 1")
    nb = u64()
    bounds = [u64() for _ in range(nb)]
    if pos != len(data):
        raise FormatError("trailing bytes after train data")
    try:
        probe = TensorTrain(cores, 0, list(bounds))
        return TensorTrain(cores, probe.measure_ortho_count(), list(bounds))
    except DimensionError as e:
        raise FormatError(str(e)) from None


# --------------------------------------------------------------------------
# TTB1 batch file (src/stream_io.cpp:123-204): "TTB1", u8 mode count,
# u64 extents, little-endian f64 payload (first-index-fastest).
# --------------------------------------------------------------------------


def write_batch(t: np.ndarray, path: str) -> None:
    """stream_io.cpp:123-137."""
    out = bytearray(b"TTB1")
    out.append(t.ndim & 0xFF)
    out += np.array(t.shape, dtype="<u8").tobytes()
    out += np.ravel(t, order="F").astype("<f8").tobytes()
    with open(path, "wb") as f:
        f.write(bytes(out))


def read_batch(path: str) -> np.ndarray:
    """stream_io.cpp:139-187."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 4 or data[:4] != b"TTB1":
        if len(data) < 4:
            raise FormatError("truncated batch file " + path)
        raise FormatError("bad magic: " + path + " is not a TTB1 batch")
    if len(data) < 5:
        raise FormatError("truncated batch file " + path)
    nd = data[4]
    if nd < 1:
        raise FormatError("batch file declares zero modes")
    pos = 5
    if len(data) < pos + 8 * nd:
        raise FormatError("truncated batch file " + path)
    shape = [int.from_bytes(data[pos + 8 * i:pos + 8 * i + 8], "little") for i in range(nd)]
    pos += 8 * nd
    count = int(np.prod(shape)) if shape else 0
    if len(data) - pos != count * 8:
        raise FormatError("payload length disagrees with declared shape in " + path)
    vals = np.frombuffer(data, dtype="<f8", count=count, offset=pos).astype(np.float64)
    if any(e < 1 for e in shape):
        raise DimensionError("tensor extent must be >= 1")
    if not np.all(np.isfinite(vals)):
        raise NumericError("non-finite element rejected at tensor construction")
    return np.asfortranarray(np.reshape(vals, shape, order="F"))


def list_stream(directory: str) -> List[str]:
    """stream_io.cpp:189-204: .ttb files in lexicographic filename order."""
    import os

    if not os.path.isdir(directory):
        raise FormatError("stream path is not a directory: " + directory)
    files = [os.path.join(directory, f) for f in os.listdir(directory)
             if f.endswith(".ttb") and os.path.isfile(os.path.join(directory, f))]
    return sorted(files, key=lambda p: os.path.basename(p))
