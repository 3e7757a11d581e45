"""GPU parity: the CUDA path (through the C ABI, libttg.so) against the CPU
oracle (oracle/ttstream_oracle.py) on identical seeded inputs.

Tolerances are stated in tests/parity_util.py (ranks identical; subspaces,
reconstructions, per-increment relative errors within 1e-10).
"""
import math

import numpy as np
import pytest

from oracle import ttstream_oracle as O
from paper_2211_12487_b200 import (ConfigError, DimensionError, HeuristicConfig, NumericError, StateError,
                                   TensorTrain, per_obs_errors, tt_ice_bootstrap, tt_ice_star_update,
                                   tt_ice_update, tt_ice_update_with_tolerances, tt_project, tt_reconstruct)
from paper_2211_12487_b200.streams import Stream
from tests.parity_util import (REF, TOL, compare_reconstructions, compare_reports, compare_trains, subspace_distance,
                               to_oracle)

pytestmark = pytest.mark.gpu


def run_stream(ctx, stream, n_inc, algo="ice", cfg=None, check_every=1, eps=None):
    eps = eps if eps is not None else stream.eps
    y0 = stream.increment(0)
    tg, rg = tt_ice_bootstrap(y0, eps, ctx=ctx)
    tr, rr = REF.tt_ice_bootstrap(y0, eps)
    compare_reports(rg, rr)
    compare_trains(tg, tr)
    ys = [(0, y0)]
    for k in range(1, n_inc):
        y = stream.increment(k)
        ys.append((k, y))
        if algo == "ice":
            tg, rg = tt_ice_update(tg, y, eps)
            tr, rr = REF.tt_ice_update(tr, y, eps)
        else:
            ocfg = O.HeuristicConfig(**vars(cfg)) if cfg else O.HeuristicConfig()
            tg, rg = tt_ice_star_update(tg, y, eps, cfg)
            tr, rr = REF.tt_ice_star_update(tr, y, eps, ocfg)
        compare_reports(rg, rr, star=(algo != "ice"), n_elems=y.size)
        if k % check_every == 0 or k == n_inc - 1:
            compare_trains(tg, tr)
    gh = to_oracle(tg)
    compare_reconstructions(gh, tr, ys)
    return tg, tr


def test_cfg0_stream_tt_ice(ctx):
    """BASELINE configs[0]: 64 increments of 8x8x8x8, batch 1, eps 0.1."""
    run_stream(ctx, Stream(0, seed=0), 64, "ice")


def test_cfg0_stream_tt_ice_star(ctx):
    run_stream(ctx, Stream(0, seed=1), 64, "star")


@pytest.mark.parametrize("seed", [0, 1])
def test_cfg3_small_ice_and_star(ctx, seed):
    """cfg3 generator (drift TT, skip path on odd increments) at 4^6, batch 24."""
    s = Stream(3, seed=seed, modes=(4,) * 6, batch=24, true_rank=6)
    run_stream(ctx, s, 10, "ice")
    run_stream(ctx, s, 10, "star")


def test_cfg3_shape_star_midsize(ctx):
    """cfg3 shape 8^7 at batch 4 (2.1M entries / observation), TT-ICE*."""
    s = Stream(3, seed=2, batch=4)
    run_stream(ctx, s, 5, "star")


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_cfg3_shape_batch16(ctx, algo):
    """cfg3 shape 8^7 at batch 16 (268 MB increments), 6 increments: two drift
    increments and two in-span (skip) increments after the bootstrap."""
    s = Stream(3, seed=4, batch=16)
    run_stream(ctx, s, 6, algo)


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_wide_unfoldings(ctx, algo):
    """Unfoldings with 128 < r*n <= 256 rows (tensor-map SYRK, 32-column
    projection tiles) and odd/even row counts: modes 16^3 x 6, batch 16."""
    s = Stream(3, seed=4, modes=(16, 16, 16, 6), batch=16, true_rank=11)
    run_stream(ctx, s, 6, algo)


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_ranks_17_to_20(ctx, algo):
    """Bond ranks 17..19 (projections with two MMA n-blocks + DFMA rows, r8 = 24
    paths): modes 6^5, batch 40, true rank 17."""
    s = Stream(3, seed=21, modes=(6,) * 5, batch=40, true_rank=17)
    run_stream(ctx, s, 6, algo)


@pytest.mark.parametrize("true_rank", [22, 27])
def test_high_ranks_multi_cta_gram(ctx, true_rank):
    """Bond ranks 22..29 at n = 8: mode-3 unfoldings a = 176..232 (k-split
    SYRK with 2 or 3 CTAs per tile set, then the k_syrk2 fallback above
    a = 224) and the 512-row statistics projection with r > 18 (NB = 3 plans,
    DFMA tails); modes 8^5, batch 24, TT-ICE*."""
    s = Stream(3, seed=31, modes=(8,) * 5, batch=24, true_rank=true_rank)
    run_stream(ctx, s, 5, "star")


def test_cfg1_video_small_batch(ctx):
    """BASELINE configs[1] shape (14,15,16,10,3) at batch 10, 6 increments."""
    s = Stream(1, seed=0, batch=10)
    run_stream(ctx, s, 6, "ice")


def test_cfg2_simulation_small_grid(ctx):
    """configs[2] generator on a 16^3 x 3 grid -> (4,4,4,4,4,4,3), batch 8."""
    s = Stream(2, seed=0, batch=8, grid=16)
    run_stream(ctx, s, 4, "ice")


@pytest.mark.parametrize("variant", [
    dict(skip_enabled=False),
    dict(subselect_enabled=False),
    dict(skip_statistic="full"),
    dict(use_approx_tolerance=True),
    dict(occupancy_threshold=0.3),
    dict(occupancy_threshold=1.0),
])
def test_tt_ice_star_heuristic_variants(ctx, variant):
    s = Stream(3, seed=3, modes=(4,) * 5, batch=12, true_rank=5)
    run_stream(ctx, s, 7, "star", cfg=HeuristicConfig(**variant))


def test_appendix_b_rank_recovery(ctx):
    """SPEC.md:681 / PAPER Appendix B: noiseless 10x15x20, ranks [1,2,3,5,1], eps 1e-8."""
    rng = np.random.default_rng(7)
    modes, ranks = (10, 15, 20), [1, 2, 3, 5]
    cores = []
    for i, n in enumerate(modes):
        q, _ = np.linalg.qr(rng.standard_normal((ranks[i] * n, ranks[i + 1])))
        cores.append(q)
    from paper_2211_12487_b200.streams import tt_chain
    phi = tt_chain(cores)
    eps = 1e-8
    ys = [np.reshape(phi @ rng.standard_normal((5, 10)), modes + (10,), order="F") for _ in range(50)]
    for algo in ("ice", "star"):
        tg, rg = tt_ice_bootstrap(ys[0], eps, ctx=ctx)
        tr, _ = REF.tt_ice_bootstrap(ys[0], eps)
        for k in range(1, 50):
            if algo == "ice":
                tg, rg = tt_ice_update(tg, ys[k], eps)
                tr, rr = REF.tt_ice_update(tr, ys[k], eps)
            else:
                tg, rg = tt_ice_star_update(tg, ys[k], eps)
                tr, rr = REF.tt_ice_star_update(tr, ys[k], eps)
            assert rg.ranks_after == rr.ranks_after
        assert tg.ranks() == [1, 2, 3, 5, 1]
        gh = to_oracle(tg)
        for k in range(50):
            b, e = gh.increment_range(k)
            rec = O.tt_reconstruct(gh, b, e)
            assert np.linalg.norm(rec - ys[k]) <= (eps + 1e-9) * np.linalg.norm(ys[k])


def test_in_span_increment_adds_no_directions(ctx):
    """increment drawn from the current span -> all r_R = 0."""
    s = Stream(0, seed=4)
    tg, _ = tt_ice_bootstrap(s.increment(0, batch=8), 0.1, ctx=ctx)
    th = to_oracle(tg)
    coeff = np.random.default_rng(0).standard_normal((th.ranks()[-2], 5))
    y = O.tt_expand(th, coeff)
    before = tg.ranks()
    tg, rep = tt_ice_update(tg, y, 0.1)
    assert tg.ranks()[:-1] == before[:-1]
    assert rep.modes_updated == 0
    c = tt_project(tg, y)
    assert np.allclose(c, coeff, atol=1e-12)


def test_zero_increment(ctx):
    s = Stream(0, seed=5)
    tg, _ = tt_ice_bootstrap(s.increment(0, batch=4), 0.1, ctx=ctx)
    tr, _ = REF.tt_ice_bootstrap(s.increment(0, batch=4), 0.1)
    z = np.zeros((8, 8, 8, 8, 3))
    tg, rg = tt_ice_update(tg, z, 0.1)
    tr, rr = REF.tt_ice_update(tr, z, 0.1)
    compare_reports(rg, rr)
    tg, rg = tt_ice_star_update(tg, z, 0.1)
    tr, rr = REF.tt_ice_star_update(tr, z, 0.1)
    compare_reports(rg, rr)
    assert rg.obs_used == 0


def test_bootstrap_rank_zero_placeholder(ctx):
    """tt_svd.cpp:42-47: eps >= 1 -> every mode rank 0 -> unit-column placeholder."""
    y = Stream(0, seed=6).increment(0, batch=3)
    tg, rg = tt_ice_bootstrap(y, 1.0, ctx=ctx)
    tr, rr = REF.tt_ice_bootstrap(y, 1.0)
    compare_reports(rg, rr)
    compare_trains(tg, tr)


def test_with_tolerances_and_project_reconstruct(ctx):
    s = Stream(3, seed=8, modes=(4,) * 5, batch=9, true_rank=4)
    y0 = s.increment(0)
    tg, _ = tt_ice_bootstrap(y0, 0.05, ctx=ctx)
    tr, _ = REF.tt_ice_bootstrap(y0, 0.05)
    y = s.increment(2)
    deltas = [0.3, 0.2, 0.1, 0.05, 0.01]
    tg, rg = tt_ice_update_with_tolerances(tg, y, deltas)
    tr, rr = REF.tt_ice_update_with_tolerances(tr, y, deltas)
    compare_reports(rg, rr)
    compare_trains(tg, tr)
    y2 = s.increment(3)
    cg = tt_project(tg, y2)
    cr = REF.tt_project(tr, y2)
    assert np.linalg.norm(cg - cr) <= TOL * np.linalg.norm(cr)
    eg = per_obs_errors(tg, y2)
    er = REF.per_obs_errors(tr, y2)
    assert np.max(np.abs(eg - er)) <= 1e-9
    rec = tt_reconstruct(tg, 3, 12)
    rec_r = O.tt_reconstruct(tr, 3, 12)
    assert np.linalg.norm(rec - rec_r) <= TOL * np.linalg.norm(rec_r)


def test_device_resident_input_matches_host(ctx):
    import torch

    s = Stream(3, seed=9, modes=(4,) * 5, batch=6, true_rank=4)
    y0, y1 = s.increment(0), s.increment(2)
    ta, _ = tt_ice_bootstrap(y0, 0.01, ctx=ctx)
    tb, _ = tt_ice_bootstrap(torch.from_numpy(np.ravel(y0, order="F")).cuda(), 0.01, ctx=ctx, shape=y0.shape)
    ta, ra = tt_ice_update(ta, y1, 0.01)
    tb, rb = tt_ice_update(tb, torch.from_numpy(np.ravel(y1, order="F")).cuda(), 0.01, shape=y1.shape)
    assert ra.ranks_after == rb.ranks_after
    for ca, cb in zip(ta.cores(), tb.cores()):
        assert np.array_equal(ca, cb)  # deterministic: same bytes


def test_determinism_bitwise(ctx):
    s = Stream(0, seed=10)
    outs = []
    for _ in range(2):
        tg, _ = tt_ice_bootstrap(s.increment(0, batch=2), 0.1, ctx=ctx)
        for k in range(1, 6):
            tg, _ = tt_ice_star_update(tg, s.increment(k, batch=2), 0.1)
        outs.append([c.copy() for c in tg.cores()])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def _run_spec_stream(ctx, speculate, monkeypatch):
    """cfg3-type stream at 4^6 under TT-ICE* (every even increment adds one direction per bond, the
    odd ones are skipped: the per-mode ranks of consecutive sweeps repeat, so the sweeps are
    speculative from the third on), then one TT-ICE update of an in-span increment (the guess
    "one direction per mode" is wrong: flagged, undone, repeated), then TT-ICE* again."""
    if speculate:
        monkeypatch.delenv("TTG_NO_SPEC", raising=False)
    else:
        monkeypatch.setenv("TTG_NO_SPEC", "1")
    s = Stream(3, seed=5, modes=(4,) * 6, batch=24, true_rank=6)
    tg, _ = tt_ice_bootstrap(s.increment(0), s.eps, ctx=ctx)
    reps = []
    for k in range(1, 14):
        upd = tt_ice_update if k == 11 else tt_ice_star_update
        tg, rep = upd(tg, s.increment(k), s.eps)
        reps.append((tuple(rep.ranks_after), rep.obs_used, rep.batch_rel_error_estimate, rep.modes_updated))
    return [c.copy() for c in tg.cores()], reps


def test_speculative_sweep_is_bitwise_the_synchronous_sweep(ctx, monkeypatch):
    """A sweep that sizes its launches from the previous update's ranks and
    verifies once (ttg.cu sweep(), ttg_ctx_spec_stats) must produce the same
    bytes as the sweep that reads every mode's rank on the host -- both when
    the guess holds and when it is rejected and the sweep repeated."""
    s0, r0 = ctx.spec_stats()
    cores_spec, reps_spec = _run_spec_stream(ctx, True, monkeypatch)
    s1, r1 = ctx.spec_stats()
    cores_sync, reps_sync = _run_spec_stream(ctx, False, monkeypatch)
    s2, r2 = ctx.spec_stats()
    assert s1 - s0 >= 2, "no sweep speculated"
    assert r1 - r0 >= 1, "no speculative sweep was rejected: the undo-and-repeat path is untested by this stream"
    assert r1 - r0 < s1 - s0, "every speculative sweep was rejected: the verified path is untested"
    assert (s2, r2) == (s1, r1), "TTG_NO_SPEC=1 still speculated"
    assert reps_spec == reps_sync
    for a, b in zip(cores_spec, cores_sync):
        assert a.shape == b.shape and np.array_equal(a, b)


def test_theorem_3_3_no_regression(ctx):
    """Earlier increments' reconstructions are unchanged (1e-12)."""
    s = Stream(3, seed=11, modes=(4,) * 5, batch=5, true_rank=4)
    tg, _ = tt_ice_bootstrap(s.increment(0), 0.01, ctx=ctx)
    prev = tt_reconstruct(tg)
    for k in range(1, 6):
        tg, _ = tt_ice_update(tg, s.increment(k), 0.01)
        now = tt_reconstruct(tg, 0, prev.shape[-1])
        assert np.linalg.norm(now - prev) <= 1e-12 * max(1.0, np.linalg.norm(prev))
        prev = tt_reconstruct(tg)


def test_errors_mirror_reference(ctx):
    s = Stream(0, seed=12)
    y = s.increment(0, batch=2)
    tg, _ = tt_ice_bootstrap(y, 0.1, ctx=ctx)
    with pytest.raises(NumericError):
        tt_ice_update(tg, y, 0.0)  # tt_ice.cpp:133-135
    with pytest.raises(DimensionError):
        tt_ice_update(tg, np.zeros((8, 8, 4, 8, 2)), 0.1)  # tt_ice.cpp:24-28
    bad = y.copy()
    bad[0, 0, 0, 0, 0] = np.nan
    with pytest.raises(NumericError):
        tt_ice_update(tg, bad, 0.1)
    with pytest.raises(ConfigError):
        tt_ice_star_update(tg, y, 0.1, HeuristicConfig(occupancy_threshold=1.5))
    with pytest.raises(NumericError):
        tt_ice_bootstrap(y, 1.5, ctx=ctx)  # tt_svd.cpp:10-12
    with pytest.raises(DimensionError):
        tt_ice_update_with_tolerances(tg, y, [0.1, 0.1])
    cores = [c for c in tg.cores()]
    nonortho = TensorTrain.upload(cores, 0, tg.batch_boundaries(), ctx=ctx)
    with pytest.raises(StateError):
        tt_ice_update(nonortho, y, 0.1)  # tt_ice.cpp:17-19
    with pytest.raises(StateError):
        tt_project(nonortho, y)


def test_upload_roundtrip_and_update(ctx):
    """A host train (oracle) uploaded through the ABI updates like the oracle."""
    s = Stream(0, seed=13)
    tr, _ = REF.tt_ice_bootstrap(s.increment(0, batch=3), 0.1)
    tg = TensorTrain.upload([c.data for c in tr.cores], tr.ortho_count, tr.batch_boundaries, ctx=ctx)
    for a, b in zip(tg.cores(), tr.cores):
        assert np.array_equal(a, b.data)
    y = s.increment(1, batch=3)
    tg, rg = tt_ice_star_update(tg, y, 0.1)
    tr, rr = REF.tt_ice_star_update(tr, y, 0.1)
    compare_reports(rg, rr, star=True)
    compare_trains(tg, tr)


@pytest.mark.parametrize("R", [24, 48, 64, 128])
def test_project_fixed_cores_high_rank(ctx, R):
    """tt_project through pre-built orthonormal cores with bond ranks up to 128
    (BASELINE configs[4] companion sweep shapes at batch 2): the r > 34 paths
    (k_project_ws with streamed W fragments, the DMMA GEMM, the fusion cost model)
    against the oracle, coefficients within 1e-10 relative."""
    modes, b = (8,) * 7, 2
    rng = np.random.default_rng(100 + R)
    r = [1]
    for i in range(1, len(modes) + 1):
        r.append(min(R, 8 ** i, 8 ** (len(modes) - i) * b))
    cores = []
    for i, n in enumerate(modes):
        q, _ = np.linalg.qr(rng.standard_normal((r[i] * n, r[i + 1])))
        cores.append(np.reshape(q, (r[i], n, r[i + 1]), order="F"))
    cores.append(np.reshape(rng.standard_normal((r[-1], 1)), (r[-1], 1, 1), order="F"))
    tg = TensorTrain.upload(cores, ortho_count=len(modes), batch_boundaries=[1], ctx=ctx)
    tr = O.TensorTrain([O.TTCore(np.asfortranarray(c)) for c in cores], len(modes), [1])
    y = np.asfortranarray(rng.standard_normal(modes + (b,)))
    cg = tt_project(tg, y)
    cr = REF.tt_project(tr, y)
    assert cg.shape == cr.shape
    assert np.linalg.norm(cg - cr) <= TOL * np.linalg.norm(cr)


@pytest.mark.parametrize("modes,ranks,b", [
    ((5, 3, 7, 2, 3), (3, 5, 4, 3, 2), 3),        # odd row counts (rows % 4 != 0), odd column counts
    ((6, 4, 3, 5, 2, 2, 3), (4, 6, 5, 7, 3, 2, 2), 5),  # six modes in the tail
    ((9, 8, 8, 8), (7, 19, 23, 11), 17),          # ranks 17-23 (r8 padding), 64-column blocks
    ((2, 2, 2), (2, 3, 1), 1),                    # tiny: the whole chain after the first mode
])
def test_project_chain_tail_shapes(ctx, modes, ranks, b, monkeypatch):
    """The last modes of tt_project in one launch (k_project_tail, tensor_train.cpp:195-226):
    shapes the m8n8k4 tiling has to pad or clamp, against the reference and against the
    per-mode kernels (TTG_NO_TAIL=1), coefficients within 1e-10 relative."""
    rng = np.random.default_rng(1000 + len(modes))
    r = [1] + list(ranks)
    cores = []
    for i, n in enumerate(modes):
        assert r[i] * n >= r[i + 1]
        q, _ = np.linalg.qr(rng.standard_normal((r[i] * n, r[i + 1])))
        cores.append(np.reshape(q, (r[i], n, r[i + 1]), order="F"))
    cores.append(np.reshape(rng.standard_normal((r[-1], 1)), (r[-1], 1, 1), order="F"))
    tg = TensorTrain.upload(cores, ortho_count=len(modes), batch_boundaries=[1], ctx=ctx)
    tr = O.TensorTrain([O.TTCore(np.asfortranarray(c)) for c in cores], len(modes), [1])
    y = np.asfortranarray(rng.standard_normal(tuple(modes) + (b,)))
    cr = REF.tt_project(tr, y)
    launches0 = ctx.launch_count
    cg = tt_project(tg, y)
    n_tail = ctx.launch_count - launches0
    monkeypatch.setenv("TTG_NO_TAIL", "1")
    launches0 = ctx.launch_count
    cm = tt_project(tg, y)
    n_modes = ctx.launch_count - launches0
    assert n_tail < n_modes, "k_project_tail did not take over the tail of this chain"
    assert cg.shape == cr.shape
    assert np.linalg.norm(cg - cr) <= TOL * np.linalg.norm(cr)
    assert np.linalg.norm(cg - cm) <= TOL * np.linalg.norm(cr)


def test_bootstrap_tall_unfolding_full_solver(ctx):
    """a = 2048 rows: the block-8 subspace vectors no longer fit shared memory
    (2 a 8 doubles > the opt-in limit), so the solver goes straight from the
    failed block-4 attempt to the full tridiagonal solver (configs[1] reaches
    a ~ 2000 at its bootstrap)."""
    rng = np.random.default_rng(7)
    u = np.linalg.qr(rng.standard_normal((2048, 40)))[0]
    v = rng.standard_normal((40, 300)) * np.logspace(0, -2, 40)[:, None]
    y = np.asfortranarray(u @ v + 1e-4 * rng.standard_normal((2048, 300)))
    tg, rg = tt_ice_bootstrap(y, 0.05, ctx=ctx)
    tr, rr = REF.tt_ice_bootstrap(y, 0.05)
    compare_reports(rg, rr)
    compare_trains(tg, tr)
    assert tg.ranks()[1] > 8


def test_update_large_append_guard_path(ctx):
    """a = 2048 rows, r_old ~ 150 kept directions + ~20 new ones: the appended
    block [U_pad U_R] has a r_new^2 >= 5e7, so its Gram guard runs through
    the DMMA GEMM + the grid deviation reduction (k_gram_dev) and the
    eigen-solve through the multi-CTA tridiagonalisation (k_sytrd_grid);
    TT-ICE against the reference."""
    rng = np.random.default_rng(11)
    basis = np.linalg.qr(rng.standard_normal((2048, 190)))[0]
    spec = np.logspace(0, -1.5, 190)[:, None]
    y0 = np.asfortranarray(basis[:, :150] @ (rng.standard_normal((150, 400)) * spec[:150]) +
                           1e-6 * rng.standard_normal((2048, 400)))
    y1 = np.asfortranarray(basis[:, 20:190] @ (rng.standard_normal((170, 300)) * spec[20:190]) +
                           1e-6 * rng.standard_normal((2048, 300)))
    tg, rg = tt_ice_bootstrap(y0, 1e-3, ctx=ctx)
    tr, rr = REF.tt_ice_bootstrap(y0, 1e-3)
    compare_reports(rg, rr)
    tg, rg = tt_ice_update(tg, y1, 1e-3)
    tr, rr = REF.tt_ice_update(tr, y1, 1e-3)
    compare_reports(rg, rr)
    compare_trains(tg, tr)
    r = tg.ranks()[1]
    assert 2048 * r * r >= 5e7, r


def test_prefetch_host_increments(ctx):
    """ttg_prefetch: host increments staged on the copy stream and consumed by
    the next update give bit-identical trains and reports to the plain host
    path (and a prefetch of a different array is ignored)."""
    st = Stream(3, seed=4, modes=(4,) * 5, batch=12)
    ys = [np.asfortranarray(st.increment(k)) for k in range(5)]
    ta, _ = tt_ice_bootstrap(ys[0], st.eps, ctx=ctx)
    tb, _ = tt_ice_bootstrap(ys[0], st.eps, ctx=ctx)
    other = np.asfortranarray(ys[1] + 1.0)
    for k in range(1, 5):
        ta, ra = tt_ice_star_update(ta, ys[k], st.eps)
        if k < 4:
            ctx.prefetch(ys[k + 1] if k % 2 else other)
        if k == 1:
            ctx.prefetch(ys[1])
        tb, rb = tt_ice_star_update(tb, ys[k], st.eps)
        assert ra.ranks_after == rb.ranks_after and ra.batch_rel_error_estimate == rb.batch_rel_error_estimate
    for ca, cb in zip(ta.cores(), tb.cores()):
        assert np.array_equal(ca, cb)


def test_prefetch_refilled_buffer_is_not_stale(ctx):
    """ttg_prefetch of a buffer that is never consumed, then refilled and
    prefetched again: the update must read the NEW contents (only the newest
    prefetch of a host pointer may be consumed)."""
    st = Stream(3, seed=6, modes=(4,) * 5, batch=8)
    y0, y1, y2 = (np.asfortranarray(st.increment(k)) for k in range(3))
    ta, _ = tt_ice_bootstrap(y0, st.eps, ctx=ctx)
    tb, _ = tt_ice_bootstrap(y0, st.eps, ctx=ctx)
    buf = np.asfortranarray(y1.copy())
    ctx.prefetch(buf)           # slot A <- y1 (never consumed)
    buf[...] = y2               # the caller refills the same host buffer
    ctx.prefetch(buf)           # slot B <- y2; slot A must be invalidated
    ta, ra = tt_ice_star_update(ta, buf, st.eps)
    tb, rb = tt_ice_star_update(tb, y2, st.eps)
    assert ra.ranks_after == rb.ranks_after
    for ca, cb in zip(ta.cores(), tb.cores()):
        assert np.array_equal(ca, cb)


def test_device_io_ordered_against_torch_stream(ctx):
    """Device increments produced by torch and device results consumed by torch
    without any host synchronisation (ttg_ctx_wait_stream / ttg_ctx_join_stream):
    a large torch kernel queue in front of the update and a torch read right
    after tt_reconstruct(out=...) see the same bytes as the host path."""
    import torch

    s = Stream(3, seed=13, modes=(6,) * 5, batch=24, true_rank=5)
    ys = [s.increment(k) for k in range(3)]
    th, _ = tt_ice_bootstrap(ys[0], s.eps, ctx=ctx)
    for y in ys[1:]:
        th, _ = tt_ice_update(th, y, s.eps)
    ref = tt_reconstruct(th, 0, th.obs_count())
    cores_h = th.cores()
    th.close()
    td = None
    for k, y in enumerate(ys):
        src = torch.from_numpy(np.ravel(y, order="F")).cuda()
        torch.cuda.synchronize()
        dev = torch.zeros_like(src)  # the increment's bytes are written only by the queued copy below
        big = torch.randn(1 << 26, device="cuda", dtype=torch.float64)  # keeps torch's stream busy
        for _ in range(4):
            big.mul_(1.0000001)
        dev.copy_(src)  # queued behind the big kernels: an update reading early sees zeros
        if k == 0:
            td, _ = tt_ice_bootstrap(dev, s.eps, ctx=ctx, shape=y.shape)
        else:
            td, _ = tt_ice_update(td, dev, s.eps, shape=y.shape)
        del big
    for a, b in zip(td.cores(), cores_h):
        assert np.array_equal(a, b)
    out = torch.full((ref.size,), float("nan"), device="cuda", dtype=torch.float64)
    tt_reconstruct(td, 0, td.obs_count(), out=out)
    got = out.mul(1.0).cpu().numpy()  # a torch kernel reads the result first
    assert np.array_equal(got, np.ravel(ref, order="F"))
    td.close()
