"""Helpers comparing the CUDA path (through the C ABI) with the CPU oracle.

Tolerances (BASELINE.json north_star: "identical TT-ranks after every
increment, and core subspaces, reconstructions and per-increment relative
errors within 1e-10 relative (FP64)"):

* ranks                     : identical
* core subspaces            : |Phi_k - Phi_k^ref (Phi_k^ref^T Phi_k)|_F / sqrt(r_k) <= 1e-10 for every
                              interface matrix Phi_k (basis-invariant subspace distance)
* reconstructions           : |rec - rec_ref|_F / |rec_ref|_F <= 1e-10 per increment
* per-increment rel. errors : |err - err_ref| <= 1e-10 (absolute difference of two relative errors)
* report error estimates    : 1e-10 absolute; Pythagoras-form estimates on their square at 1e-13
                              (see estimates_agree)
"""
from __future__ import annotations

import numpy as np

from oracle import ref_binding as R
from oracle import ttstream_oracle as O

TOL = 1e-10

# The checker of the GPU parity tests: the reference library itself
# (oracle/_ref/libttref.so, proj/src compiled unchanged against the Eigen-API
# shim) when it was built, else the numpy restatement, which
# tests/test_ref_pin.py pins to the reference case by case.
REF = R if R.available() else O
REF_NAME = "reference (oracle/_ref)" if REF is R else "numpy oracle"


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


# Pythagoras-form estimates (bootstrap tt_ice.cpp:159-162 and TT-ICE*
# tt_ice_star.cpp:297-300) are sqrt(max(1 - |c|^2/|y|^2, 0)): the SQUARE is
# computed to a few ulps absolute, the root of a near-zero difference is not
# (a noiseless stream gives 0 in one rounding and 3e-8 in another).  They are
# compared on the square at 1e-13 absolute, i.e. 5e-11 in the estimate at the
# 1e-3 errors of configs[3]; TT-ICE's sqrt(sum tail^2)/|y| (tt_ice.cpp:125-126)
# at 1e-10 absolute.
EST2_TOL = 1e-13


def estimates_agree(a: float, b: float, pythagoras: bool, tol: float = TOL) -> bool:
    if abs(a - b) <= tol:
        return True
    return pythagoras and abs(a * a - b * b) <= EST2_TOL


def compare_reports(rg, rr, tol: float = TOL, star: bool = False):
    assert list(rg.ranks_after) == list(rr.ranks_after), f"report ranks {rg.ranks_after} vs {rr.ranks_after}"
    assert rg.obs_in_batch == rr.obs_in_batch
    assert rg.obs_used == rr.obs_used, f"obs_used {rg.obs_used} vs {rr.obs_used}"
    assert estimates_agree(rg.batch_rel_error_estimate, rr.batch_rel_error_estimate,
                           pythagoras=star or rr.increment_index == 0, tol=tol), \
        f"estimate {rg.batch_rel_error_estimate!r} vs {rr.batch_rel_error_estimate!r}"
    if rr.eps_target != 0.0:
        assert abs(rg.eps_target - rr.eps_target) <= 1e-10 * abs(rr.eps_target), f"eps_target {rg.eps_target} vs {rr.eps_target}"
    else:
        assert rg.eps_target == 0.0
    assert bool(rg.tolerance_clamped) == bool(rr.tolerance_clamped)
