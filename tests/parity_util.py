"""Helpers comparing the CUDA path (through the C ABI) with the CPU oracle.

Tolerances (BASELINE.json north_star: "identical TT-ranks after every
increment, and core subspaces, reconstructions and per-increment relative
errors within 1e-10 relative (FP64)"):

* ranks                     : identical
* core subspaces            : |Phi_k - Phi_k^ref (Phi_k^ref^T Phi_k)|_F / sqrt(r_k) <= 1e-10 for every
                              interface matrix Phi_k (basis-invariant subspace distance)
* reconstructions           : |rec - rec_ref|_F / |rec_ref|_F <= 1e-10 per increment
* per-increment rel. errors : |err - err_ref| <= 1e-10 (absolute difference of two relative errors)
"""
from __future__ import annotations

import numpy as np

from oracle import ttstream_oracle as O

TOL = 1e-10


def to_oracle(tt) -> O.TensorTrain:
    cores = [O.TTCore(np.asfortranarray(c)) for c in tt.cores()]
    return O.TensorTrain(cores, tt.ortho_count, tt.batch_boundaries())


def subspace_distance(phi: np.ndarray, phi_ref: np.ndarray) -> float:
    if phi.shape != phi_ref.shape:
        return float("inf")
    r = phi.shape[1]
    resid = phi - phi_ref @ (phi_ref.T @ phi)
    return float(np.linalg.norm(resid)) / max(1.0, np.sqrt(r))


def compare_trains(tt_gpu, tt_ref: O.TensorTrain, tol: float = TOL, check_obs=True):
    """Returns a dict of diagnostics; raises AssertionError on parity failure."""
    g = to_oracle(tt_gpu) if not isinstance(tt_gpu, O.TensorTrain) else tt_gpu
    assert g.ranks() == tt_ref.ranks(), f"ranks differ: gpu {g.ranks()} ref {tt_ref.ranks()}"
    assert g.batch_boundaries == tt_ref.batch_boundaries, "batch boundaries differ"
    out = {"subspace": 0.0, "core_entry": 0.0}
    for pg, pr in zip(O.interface_projectors(g), O.interface_projectors(tt_ref)):
        dist = subspace_distance(pg, pr)
        out["subspace"] = max(out["subspace"], dist)
    for cg, cr in zip(g.cores[:-1], tt_ref.cores[:-1]):
        out["core_entry"] = max(out["core_entry"], float(np.max(np.abs(cg.data - cr.data))))
    assert out["subspace"] <= tol, f"core subspace distance {out['subspace']:.3e} > {tol}"
    return out


def compare_reconstructions(tt_gpu_host: O.TensorTrain, tt_ref: O.TensorTrain, ys, tol: float = TOL):
    """Per-increment reconstruction agreement and relative-error agreement."""
    worst_rec, worst_err = 0.0, 0.0
    for k, y in ys:
        b, e = tt_ref.increment_range(k)
        rr = O.tt_reconstruct(tt_ref, b, e)
        rg = O.tt_reconstruct(tt_gpu_host, b, e)
        den = float(np.linalg.norm(rr))
        d = float(np.linalg.norm(rg - rr)) / (den if den > 0 else 1.0)
        worst_rec = max(worst_rec, d)
        ny = float(np.linalg.norm(y))
        if ny > 0:
            eg = float(np.linalg.norm(y - rg)) / ny
            er = float(np.linalg.norm(y - rr)) / ny
            worst_err = max(worst_err, abs(eg - er))
    assert worst_rec <= tol, f"reconstruction rel diff {worst_rec:.3e} > {tol}"
    assert worst_err <= tol, f"per-increment relative error diff {worst_err:.3e} > {tol}"
    return worst_rec, worst_err


def compare_reports(rg, rr, tol: float = TOL, star: bool = False):
    assert list(rg.ranks_after) == list(rr.ranks_after), f"report ranks {rg.ranks_after} vs {rr.ranks_after}"
    assert rg.obs_in_batch == rr.obs_in_batch
    assert rg.obs_used == rr.obs_used, f"obs_used {rg.obs_used} vs {rr.obs_used}"
    assert abs(rg.batch_rel_error_estimate - rr.batch_rel_error_estimate) <= max(tol, 1e-8 * rr.batch_rel_error_estimate if star else tol), \
        f"estimate {rg.batch_rel_error_estimate!r} vs {rr.batch_rel_error_estimate!r}"
    if rr.eps_target != 0.0:
        assert abs(rg.eps_target - rr.eps_target) <= 1e-10 * abs(rr.eps_target), f"eps_target {rg.eps_target} vs {rr.eps_target}"
    else:
        assert rg.eps_target == 0.0
    assert bool(rg.tolerance_clamped) == bool(rr.tolerance_clamped)
