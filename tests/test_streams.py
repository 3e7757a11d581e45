"""CPU: seeded generators of the BASELINE configs (shapes, determinism,
noise levels, cfg3's in-span / new-direction alternation)."""
import numpy as np
import pytest

from oracle import ttstream_oracle as O
from paper_2211_12487_b200.streams import CONFIGS, Stream, capped_ranks, tt_chain


def test_config_shapes():
    assert CONFIGS[0].modes == (8, 8, 8, 8) and CONFIGS[0].batch == 1
    assert CONFIGS[1].modes == (14, 15, 16, 10, 3) and CONFIGS[1].batch == 100
    assert CONFIGS[2].modes == (8,) * 6 + (3,) and CONFIGS[2].batch == 32
    assert CONFIGS[3].modes == (8,) * 7 and CONFIGS[3].batch == 256
    assert CONFIGS[4].batch == 2048
    assert capped_ranks((8,) * 7, 12) == [1, 8, 12, 12, 12, 12, 12, 12]


@pytest.mark.parametrize("cfg,kw", [(0, {}), (1, dict(batch=3)), (2, dict(batch=2, grid=16)),
                                    (3, dict(modes=(4,) * 5, batch=5, true_rank=4))])
def test_deterministic_and_shaped(cfg, kw):
    a = Stream(cfg, seed=3, **kw).increment(2)
    b = Stream(cfg, seed=3, **kw).increment(2)
    assert np.array_equal(a, b)
    assert a.flags.f_contiguous or a.ndim == 1
    s = Stream(cfg, seed=3, **kw)
    assert a.shape == tuple(s.modes) + (s.batch,)
    assert not np.array_equal(a, Stream(cfg, seed=4, **kw).increment(2))


def test_cfg0_noise_level():
    s = Stream(0, seed=0)
    y = s.increment(5, batch=50)
    ym = np.reshape(y, (-1, 50), order="F")
    p = s.phi @ (s.phi.T @ ym)
    rel = np.linalg.norm(ym - p) / np.linalg.norm(p)
    assert 0.005 < rel < 0.02  # 1 % noise


def test_cfg3_in_span_and_new_directions():
    s = Stream(3, seed=1, modes=(4,) * 5, batch=8, true_rank=4)
    tt, _ = O.tt_ice_bootstrap(s.increment(0), s.eps)
    e_red = O.per_obs_errors(tt, s.increment(1))  # redundant: within noise
    assert np.mean(e_red) < s.eps
    e_new = O.per_obs_errors(tt, s.increment(2))  # new drift direction
    assert np.mean(e_new) > 10 * s.eps
    assert s.is_redundant(1) and not s.is_redundant(2)


def test_tt_chain_orthonormal():
    s = Stream(3, seed=2, modes=(3, 4, 5), batch=2, true_rank=4)
    phi = tt_chain(s.cores)
    assert np.allclose(phi.T @ phi, np.eye(phi.shape[1]), atol=1e-12)
