"""CPU: pin the oracle to the reference's SPEC known-answer examples and
property tests (the reference ships no golden vectors).

Each test cites the SPEC line it restates.
"""
import math

import numpy as np
import pytest

from oracle import ttstream_oracle as O
from paper_2211_12487_b200.streams import Stream, tt_chain


def _random_tt(rng, modes, ranks):
    cores = []
    for i, n in enumerate(modes):
        q, _ = np.linalg.qr(rng.standard_normal((ranks[i] * n, ranks[i + 1])))
        cores.append(q)
    return cores


def test_svd_trunc_diag_example():
    """diag(10,1,0.1), delta=0.5 -> rank 2, tail 0.1."""
    s = O.svd_trunc(np.diag([10.0, 1.0, 0.1]), 0.5)
    assert s.rank == 2
    assert abs(s.tail_norm - 0.1) < 1e-15


def test_svd_trunc_zero_matrix():
    """zero matrix, delta 0 -> rank 0."""
    s = O.svd_trunc(np.zeros((4, 5)), 0.0)
    assert s.rank == 0 and s.u.shape == (4, 0)


def test_svd_trunc_delta_zero_full_rank():
    """delta = 0 -> full numerical rank, reconstruction error <= 1e-10 |A|."""
    a = np.random.default_rng(0).standard_normal((7, 5))
    s = O.svd_trunc(a, 0.0)
    assert s.rank == 5
    assert np.linalg.norm(a - s.u @ np.diag(s.s) @ s.vt) <= 1e-10 * np.linalg.norm(a)


@pytest.mark.parametrize("seed", range(20))
def test_svd_trunc_eckart_young_and_minimality(seed):
    """|A - U S Vt| == tail within 1e-10; rank minimal; U orthonormal 1e-12."""
    rng = np.random.default_rng(seed)
    m, l = rng.integers(1, 40, size=2)
    a = rng.standard_normal((m, l)) * np.logspace(0, -6, l)[None, :]
    delta = rng.uniform(0, 1) * np.linalg.norm(a)
    s = O.svd_trunc(a, delta)
    err = np.linalg.norm(a - s.u @ np.diag(s.s) @ s.vt)
    assert abs(err - s.tail_norm) <= 1e-10 * max(1.0, np.linalg.norm(a))
    assert s.tail_norm <= delta + 1e-12
    if s.rank >= 1:
        assert math.sqrt(s.tail_norm ** 2 + s.s[-1] ** 2) > delta
    assert np.max(np.abs(s.u.T @ s.u - np.eye(s.rank))) <= 1e-12
    # sign rule: largest-|.| entry of each column positive (truncated_svd.cpp:16-25)
    for j in range(s.rank):
        assert s.u[np.argmax(np.abs(s.u[:, j])), j] > 0


def test_occupancy_examples():
    """SPEC.md:212-214."""
    assert O.occupancy(O.TTCore(np.zeros((1, 4, 2)))) == 0.5
    assert O.occupancy(O.TTCore(np.zeros((3, 5, 15)))) == 1.0


def test_subselect_example():
    """SPEC.md:395-397."""
    sp = O.subselect([0.2, 0.05], 0.1)
    assert sp.selected == [0] and sp.rejected == [1]
    assert O.subselect([0.1, 0.1], 0.1).selected == []  # strict '>'


def test_relaxed_tolerance_examples():
    """SPEC.md:404-406, 413-415."""
    assert O.relaxed_tolerance_approx(10, 5, 0.05, 0.1) == pytest.approx(0.15)
    assert O.relaxed_tolerance_approx(10, 0, 0.0, 0.1) == 0.1
    y = np.random.default_rng(0).standard_normal((3, 4, 5))
    eps, clamped = O.relaxed_tolerance(y, O.SubselectSplit([0, 1, 2, 3, 4], []), [0.5] * 5, 0.1)
    assert eps == 0.1 and not clamped
    # rejected perfectly represented: eps_upd = eps |y| / |D|
    split = O.SubselectSplit([0, 1], [2, 3, 4])
    eps, _ = O.relaxed_tolerance(y, split, [0.3, 0.3, 0.0, 0.0, 0.0], 0.1)
    d = y[..., [0, 1]]
    assert eps == pytest.approx(0.1 * np.linalg.norm(y) / np.linalg.norm(d), rel=1e-14)
    with pytest.raises(O.ConfigError):
        O.relaxed_tolerance(y, O.SubselectSplit([], [0]), [0.0] * 5, 0.1)


def test_pad_core_properties():
    """orthonormality kept; zero rows carry no content."""
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((3 * 4, 5)))
    p = O.pad_core(q, 3, 2)
    assert p.shape == (5 * 4, 5)
    assert np.max(np.abs(p.T @ p - np.eye(5))) <= 1e-12
    assert O.pad_core(q, 3, 0) is q


def test_compute_residual_properties():
    """SPEC.md:318-323."""
    rng = np.random.default_rng(2)
    u, _ = np.linalg.qr(rng.standard_normal((10, 3)))
    y = rng.standard_normal((10, 7))
    r = O.compute_residual(u, y)
    assert np.max(np.abs(u.T @ r)) <= 1e-12
    assert np.linalg.norm(O.compute_residual(u, u @ rng.standard_normal((3, 4)))) <= 1e-12 * 10
    assert O.compute_residual(np.zeros((10, 0)), y) is y


@pytest.mark.parametrize("seed", range(10))
def test_theorems_3_1_and_3_3(seed):
    """SPEC.md:344-347 (acceptance 1-2, reduced count): error <= eps + 1e-9 per
    increment; earlier reconstructions unchanged within 1e-12; orthonormal cores."""
    rng = np.random.default_rng(seed)
    modes = tuple(int(x) for x in rng.integers(2, 9, size=3))
    eps = [0.3, 0.1, 0.01][seed % 3]
    b = int(rng.integers(1, 6))
    ys = [rng.standard_normal(modes + (b,)) for _ in range(6)]
    tt, _ = O.tt_ice_bootstrap(ys[0], eps)
    for k in range(1, 6):
        prev = O.tt_reconstruct(tt)
        tt, rep = O.tt_ice_update(tt, ys[k], eps)
        now = O.tt_reconstruct(tt, 0, prev.shape[-1])
        assert np.linalg.norm(now - prev) <= 1e-12 * max(1.0, np.linalg.norm(prev))
        b0, e0 = tt.increment_range(k)
        rec = O.tt_reconstruct(tt, b0, e0)
        assert np.linalg.norm(ys[k] - rec) <= (eps + 1e-9) * np.linalg.norm(ys[k])
        assert tt.measure_ortho_count(1e-12) == tt.spatial_dims()


def test_in_span_increment_zero_new_directions():
    """SPEC.md:321."""
    rng = np.random.default_rng(3)
    y0 = rng.standard_normal((4, 5, 6, 3))
    tt, _ = O.tt_ice_bootstrap(y0, 0.1)
    y = O.tt_expand(tt, rng.standard_normal((tt.ranks()[-2], 4)))
    tt2, rep = O.tt_ice_update(tt, y, 0.1)
    assert tt2.ranks()[:-1] == tt.ranks()[:-1]


def test_appendix_b_rank_recovery_oracle():
    """noiseless 10x15x20, ranks [1,2,3,5,1], eps 1e-8."""
    rng = np.random.default_rng(5)
    cores = _random_tt(rng, (10, 15, 20), [1, 2, 3, 5])
    phi = tt_chain(cores)
    eps = 1e-8
    ys = [np.reshape(phi @ rng.standard_normal((5, 10)), (10, 15, 20, 10), order="F") for _ in range(50)]
    for upd in (O.tt_ice_update, O.tt_ice_star_update):
        tt, _ = O.tt_ice_bootstrap(ys[0], eps)
        for k in range(1, 50):
            tt, rep = upd(tt, ys[k], eps)
            b0, e0 = tt.increment_range(k)
            assert np.linalg.norm(ys[k] - O.tt_reconstruct(tt, b0, e0)) <= (eps + 1e-9) * np.linalg.norm(ys[k])
        assert tt.ranks() == [1, 2, 3, 5, 1]


def test_tt_ice_star_economy():
    """SPEC.md:682 (acceptance 4): in-span-heavy stream -> obs_used <= 0.5 x TT-ICE's."""
    s = Stream(3, seed=0, modes=(4,) * 5, batch=10, true_rank=4)
    ys = [s.increment(k) for k in range(10)]
    t1, _ = O.tt_ice_bootstrap(ys[0], s.eps)
    t2 = t1
    used1 = used2 = 0
    for y in ys[1:]:
        t1, r1 = O.tt_ice_update(t1, y, s.eps)
        t2, r2 = O.tt_ice_star_update(t2, y, s.eps)
        used1 += r1.obs_used
        used2 += r2.obs_used
    assert used2 <= 0.5 * used1


def test_per_obs_errors_pythagoras():
    """err^2 = 1 - |coeff|^2/|y|^2 within 1e-10."""
    rng = np.random.default_rng(6)
    tt, _ = O.tt_ice_bootstrap(rng.standard_normal((5, 6, 7, 4)), 0.3)
    y = rng.standard_normal((5, 6, 7, 3))
    e = O.per_obs_errors(tt, y)
    c = O.tt_project(tt, y)
    ym = np.reshape(y, (-1, 3), order="F")
    pyth = 1 - np.sum(c * c, axis=0) / np.sum(ym * ym, axis=0)
    assert np.max(np.abs(e * e - pyth)) <= 1e-10


def test_tt_svd_error_bound():
    """SPEC.md:687 acceptance 6: tt_svd relative error <= eps + 1e-9."""
    rng = np.random.default_rng(8)
    for eps in (0.1, 0.01, 0.3):
        y = rng.standard_normal((6, 5, 4, 3))
        tt = O.tt_svd(y, eps)
        assert np.linalg.norm(y - O.tt_reconstruct(tt)) <= (eps + 1e-9) * np.linalg.norm(y)
        assert tt.measure_ortho_count(1e-12) == 3


def test_append_directions_guard():
    """update_common.hpp:19-36: a non-orthogonal U_R triggers Householder re-orthogonalisation."""
    rng = np.random.default_rng(9)
    u, _ = np.linalg.qr(rng.standard_normal((12, 4)))
    v = rng.standard_normal((12, 2))
    v /= np.linalg.norm(v, axis=0)
    c = O.append_directions(u, v)
    assert np.max(np.abs(c.T @ c - np.eye(6))) <= 1e-12
    assert np.array_equal(c[:, :4], u)


def test_errors():
    y = np.ones((3, 4, 2))
    tt, _ = O.tt_ice_bootstrap(y, 0.1)
    with pytest.raises(O.NumericError):
        O.tt_ice_update(tt, y, 0.0)
    with pytest.raises(O.DimensionError):
        O.tt_ice_update(tt, np.ones((3, 5, 2)), 0.1)
    with pytest.raises(O.ConfigError):
        O.tt_ice_star_update(tt, y, 0.1, O.HeuristicConfig(occupancy_threshold=0.0))
    bad = O.TensorTrain(tt.cores, 0, tt.batch_boundaries)
    with pytest.raises(O.StateError):
        O.tt_ice_update(bad, y, 0.1)
