"""CPU: pin the numpy oracle to the reference itself.

oracle/_ref/libttref.so is the reference library's own sources
(/root/reference/proj/src/*.cpp) compiled unchanged against the Eigen-API
shim (oracle/eigen_shim, oracle/Makefile); oracle/ref_binding.py binds it
with the oracle's names.  Every case runs the same seeded bytes through both
and holds them to the north-star bar (ranks identical; subspaces,
reconstructions and per-increment errors within 1e-10), plus the SPEC
known-answer examples through the reference.

Skipped only when the library is absent (it needs /root/reference to build;
build() makes it in this container and it travels to the GPU box).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import ref_binding as R
from oracle import ttstream_oracle as O
from paper_2211_12487_b200.streams import Stream, tt_chain
from tests.parity_util import TOL, compare_reconstructions, compare_trains, estimates_agree

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref/libttref.so not built (needs /root/reference)")

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _reports_match(ro, rr, star):
    assert ro.ranks_after == rr.ranks_after, (ro.ranks_after, rr.ranks_after)
    assert ro.ranks_before == rr.ranks_before
    assert ro.obs_in_batch == rr.obs_in_batch and ro.obs_used == rr.obs_used, (ro.obs_used, rr.obs_used)
    assert ro.increment_index == rr.increment_index
    assert bool(ro.tolerance_clamped) == bool(rr.tolerance_clamped)
    if rr.eps_target == 0.0:
        assert ro.eps_target == 0.0
    else:
        assert abs(ro.eps_target - rr.eps_target) <= 1e-12 * abs(rr.eps_target)
    assert estimates_agree(ro.batch_rel_error_estimate, rr.batch_rel_error_estimate,
                           pythagoras=star or rr.increment_index == 0), \
        (ro.batch_rel_error_estimate, rr.batch_rel_error_estimate)


def _run_both(ys, eps, algo, cfg=None):
    to, ro = O.tt_ice_bootstrap(ys[0], eps)
    tr, rr = R.tt_ice_bootstrap(ys[0], eps)
    _reports_match(ro, rr, False)
    compare_trains(to, tr)
    h = R.RefTrain.from_oracle(tr)
    for y in ys[1:]:
        if algo == "ice":
            to, ro = O.tt_ice_update(to, y, eps)
            h, rr = R.tt_ice_update(h, y, eps, keep_handle=True)
        else:
            to, ro = O.tt_ice_star_update(to, y, eps, cfg)
            h, rr = R.tt_ice_star_update(h, y, eps, cfg, keep_handle=True)
        _reports_match(ro, rr, algo != "ice")
    tr = h.to_oracle()
    compare_trains(to, tr)
    compare_reconstructions(to, tr, list(enumerate(ys)))
    return to, tr


# ---- SPEC known-answer examples through the reference --------------------------

def test_kat_through_reference():
    with open(os.path.join(GOLD, "kat.json")) as f:
        k = json.load(f)
    for case in k["svd_trunc"]:
        s = R.svd_trunc(np.array(case["a"], dtype=np.float64), case["delta"])
        assert s.rank == case["rank"], case["spec"]
        assert abs(s.tail_norm - case["tail"]) <= 1e-15, case["spec"]
    for case in k["relaxed_tolerance_approx"]:
        args = (case["n_batch"], case["n_rejected"], case["mean_rejected_error"], case["eps"])
        assert abs(R.relaxed_tolerance_approx(*args) - case["value"]) <= 1e-15, case["spec"]


@pytest.mark.parametrize("seed", range(12))
def test_svd_trunc_matches_reference(seed):
    """truncated_svd.cpp:29-94 incl. the tall QR branch (:51-59) and the sign rule (:16-25)."""
    rng = np.random.default_rng(seed)
    m, l = (int(v) for v in rng.integers(1, 60, size=2))
    if seed % 3 == 0:
        m, l = max(m, 3 * l), l  # tall: rows > 2 cols
    a = rng.standard_normal((m, l)) * np.logspace(0, -5, l)[None, :]
    delta = float(rng.uniform(0, 0.5) * np.linalg.norm(a))
    so, sr = O.svd_trunc(a, delta), R.svd_trunc(a, delta)
    assert so.rank == sr.rank
    assert abs(so.tail_norm - sr.tail_norm) <= 1e-12 * max(1.0, np.linalg.norm(a))
    assert np.allclose(so.s, sr.s, rtol=1e-12, atol=1e-14 * np.linalg.norm(a))
    # sign rule fixes the columns: entrywise agreement away from degenerate sigma
    gaps = np.diff(sr.s) if sr.rank > 1 else np.array([-1.0])
    if sr.rank and np.all(np.abs(gaps) > 1e-6 * sr.s[0]):
        assert np.max(np.abs(so.u - sr.u)) <= 1e-9


def test_append_directions_guard_matches_reference():
    """update_common.hpp:19-36: both branches (guard quiet, guard fires -> Householder Q)."""
    rng = np.random.default_rng(3)
    q = np.linalg.qr(rng.standard_normal((30, 9)))[0]
    up, un = q[:, :6], q[:, 6:]
    assert np.max(np.abs(O.append_directions(up, un) - R.append_directions(up, un))) == 0.0
    un_bad = un + 1e-6 * rng.standard_normal(un.shape)
    a, b = O.append_directions(up, un_bad), R.append_directions(up, un_bad)
    assert np.max(np.abs(a - b)) <= 1e-13


def test_residual_and_pad_match_reference():
    rng = np.random.default_rng(4)
    u = np.linalg.qr(rng.standard_normal((12, 5)))[0]
    y = rng.standard_normal((12, 40))
    assert np.max(np.abs(O.compute_residual(u, y) - R.compute_residual(u, y))) <= 1e-14
    core = rng.standard_normal((3 * 4, 5))
    assert np.array_equal(O.pad_core(core, 3, 2), R.pad_core(core, 3, 2))


# ---- whole streams --------------------------------------------------------------

@pytest.mark.parametrize("algo,seed", [("ice", 0), ("star", 1)])
def test_cfg0_stream(algo, seed):
    """BASELINE configs[0]: 64 increments of 8^4, batch 1, eps 0.1."""
    s = Stream(0, seed=seed)
    _run_both([np.asfortranarray(s.increment(k)) for k in range(64)], s.eps, algo)


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_cfg1_video_reduced(algo):
    """configs[1] shape (14,15,16,10,3), batch 10, 6 increments."""
    s = Stream(1, seed=0, batch=10)
    _run_both([s.increment(k) for k in range(6)], s.eps, algo)


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_cfg2_simulation_reduced(algo):
    """configs[2] generator on a 16^3 x 3 grid, batch 8, 5 increments."""
    s = Stream(2, seed=0, batch=8, grid=16)
    _run_both([s.increment(k) for k in range(5)], s.eps, algo)


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_cfg3_reduced(algo):
    """configs[3] generator (drift + in-span increments) at 6^6, batch 24, 8 increments."""
    s = Stream(3, seed=0, modes=(6,) * 6, batch=24, true_rank=6)
    _run_both([s.increment(k) for k in range(8)], s.eps, algo)


@pytest.mark.parametrize("variant", [
    dict(skip_enabled=False),
    dict(subselect_enabled=False),
    dict(skip_statistic="full"),
    dict(use_approx_tolerance=True),
    dict(occupancy_threshold=0.3),
    dict(occupancy_threshold=1.0),
])
def test_star_heuristic_variants(variant):
    s = Stream(3, seed=3, modes=(4,) * 5, batch=12, true_rank=5)
    _run_both([s.increment(k) for k in range(7)], s.eps, "star", O.HeuristicConfig(**variant))


def _appendix_b(ranks, seed, n_inc=20, batch=10):
    rng = np.random.default_rng(seed)
    modes = (10, 15, 20)
    cores = [np.linalg.qr(rng.standard_normal((ranks[i] * n, ranks[i + 1])))[0] for i, n in enumerate(modes)]
    phi = tt_chain(cores)
    return [np.reshape(phi @ rng.standard_normal((ranks[-1], batch)), modes + (batch,), order="F")
            for _ in range(n_inc)]


@pytest.mark.parametrize("ranks", [[1, 2, 3, 5], [1, 4, 10, 30]])
@pytest.mark.parametrize("algo", ["ice", "star"])
def test_appendix_b_small_eps(ranks, algo):
    """PAPER Appendix B: noiseless 10x15x20
    streams at eps = 1e-8; the second case has a 200-row third unfolding."""
    ys = _appendix_b(ranks, 7, batch=12 if ranks[-1] > 5 else 10)
    to, tr = _run_both(ys, 1e-8, algo)
    assert tr.ranks() == ranks + [1]


def test_edge_cases_match_reference():
    """Zero increment, in-span increment, rank-0 placeholder (tt_svd.cpp:42-47)."""
    s = Stream(0, seed=5)
    y0 = s.increment(0, batch=4)
    z = np.zeros((8, 8, 8, 8, 3))
    to, _ = O.tt_ice_bootstrap(y0, 0.1)
    tr, _ = R.tt_ice_bootstrap(y0, 0.1)
    for fo, fr in ((O.tt_ice_update, R.tt_ice_update), (O.tt_ice_star_update, R.tt_ice_star_update)):
        a, ra = fo(to, z, 0.1)
        b, rb = fr(tr, z, 0.1)
        _reports_match(ra, rb, True)
        compare_trains(a, b)
    coeff = np.random.default_rng(0).standard_normal((to.ranks()[-2], 5))
    y = O.tt_expand(to, coeff)
    a, ra = O.tt_ice_update(to, y, 0.1)
    b, rb = R.tt_ice_update(tr, y, 0.1)
    _reports_match(ra, rb, False)
    assert rb.ranks_after[:-1] == rb.ranks_before[:-1]
    a, ra = O.tt_ice_bootstrap(y0, 1.0)
    b, rb = R.tt_ice_bootstrap(y0, 1.0)
    _reports_match(ra, rb, False)
    compare_trains(a, b)


def test_error_classes_match_reference():
    s = Stream(0, seed=12)
    y = s.increment(0, batch=2)
    tr, _ = R.tt_ice_bootstrap(y, 0.1)
    with pytest.raises(O.NumericError):
        R.tt_ice_update(tr, y, 0.0)
    with pytest.raises(O.DimensionError):
        R.tt_ice_update(tr, np.zeros((8, 8, 4, 8, 2)), 0.1)
    with pytest.raises(O.ConfigError):
        R.tt_ice_star_update(tr, y, 0.1, O.HeuristicConfig(occupancy_threshold=1.5))
    with pytest.raises(O.NumericError):
        R.tt_ice_bootstrap(y, 1.5)
    with pytest.raises(O.DimensionError):
        R.tt_ice_update_with_tolerances(tr, y, [0.1, 0.1])
    bad = O.TensorTrain(tr.cores, 0, tr.batch_boundaries)
    with pytest.raises(O.StateError):
        R.tt_ice_update(bad, y, 0.1)
    with pytest.raises(O.StateError):
        R.tt_project(bad, y)
    nan = y.copy()
    nan[0, 0, 0, 0, 0] = math.nan
    with pytest.raises(O.NumericError):
        R.tt_ice_update(tr, nan, 0.1)


def test_project_reconstruct_rre_match_reference():
    s = Stream(3, seed=8, modes=(4,) * 5, batch=9, true_rank=4)
    y0, y = s.increment(0), s.increment(3)
    tr, _ = R.tt_ice_bootstrap(y0, 0.05)
    co, cr = O.tt_project(tr, y), R.tt_project(tr, y)
    assert np.linalg.norm(co - cr) <= 1e-13 * np.linalg.norm(cr)
    assert np.max(np.abs(O.per_obs_errors(tr, y) - R.per_obs_errors(tr, y))) <= 1e-13
    rec_o, rec_r = O.tt_reconstruct(tr, 2, 7), R.tt_reconstruct(tr, 2, 7)
    assert np.linalg.norm(rec_o - rec_r) <= 1e-13 * np.linalg.norm(rec_r)
    assert abs(O.rre(tr, y0)[0] - R.rre(tr, y0)) <= 1e-13
