"""GPU parity at the BASELINE configs' FULL sizes against the reference
itself (fixtures written by tools/make_fullsize_fixtures.py with
oracle/_ref/libttref.so; format and tolerances in tests/fullsize_util.py).

* cfg3_full_{star,ice}: configs[3] at 8^7 x 256 (4.29 GB per increment) on
  bench.py's own stream (DeviceStream(seed=0)): bootstrap + 9 TT-ICE*
  increments (the benchmarked algorithm; update and skip steps) and
  bootstrap + 4 TT-ICE increments.
* cfg1_full_{ice,star}: configs[1], all 40 increments of 80.6 MB.
* cfg2_full_{ice,star}: configs[2], the first 8 increments of 201 MB.

Per increment: the input bytes' SHA-256 equals the fixture's (same stream);
ranks identical; obs_used, eps_target, clamp flag and the error estimate as
compare_reports; the increment's relative reconstruction error (device RRE
kernel) within 1e-10 of the reference's metrics.cpp RRE; every interface
subspace within 1e-10 (chained bases where they fit, fingerprints always);
the increment's reconstructions within 1e-10 (probe form).  At the end, when
the fixture holds the final train: coefficients of every observation agree
within 1e-10 inside the GPU subspace.
"""
import os

import numpy as np
import pytest

from oracle import ttstream_oracle as O
from paper_2211_12487_b200 import rre, tt_ice_bootstrap, tt_ice_star_update, tt_ice_update
from tests import fullsize_util as F
from tests.parity_util import TOL, compare_reports, subspace_distance

pytestmark = pytest.mark.gpu

NAMES = ["cfg3_full_star", "cfg3_full_ice", "cfg1_full_ice", "cfg1_full_star", "cfg2_full_ice", "cfg2_full_star"]
PHI_MAX = 60_000_000  # chain the interface bases explicitly while they stay this small (elements)


def _present(name):
    return os.path.exists(os.path.join(F.GOLD, name + ".npz"))


def _inputs(name, n):
    if name.startswith("cfg3"):
        import torch

        from paper_2211_12487_b200.streams import DeviceStream

        gen = DeviceStream(seed=0, modes=(8,) * 7)
        for k in range(n):
            y = gen.increment(k, 256)
            torch.cuda.synchronize()
            yield y, (8,) * 7 + (256,)
        return
    from paper_2211_12487_b200.streams import Stream

    s = Stream(1 if name.startswith("cfg1") else 2, seed=0)
    for k in range(n):
        y = np.asfortranarray(s.increment(k))
        yield y, y.shape


def _chained(cores, d):
    phis, acc = [], None
    for i in range(d):
        c = cores[i]
        if acc is None:
            acc = np.reshape(c, (c.shape[1], c.shape[2]), order="F")
        else:
            rows = acc.shape[0] * c.shape[1]
            if rows * c.shape[2] > PHI_MAX:
                break
            acc = np.reshape(acc @ np.reshape(c, (c.shape[0], -1), order="F"), (rows, c.shape[2]), order="F")
        phis.append(acc)
    return phis


def _report(fx, k, b):
    return O.UpdateReport(increment_index=k, obs_in_batch=b, obs_used=int(fx["obs_used"][k]),
                          ranks_after=[int(v) for v in fx["ranks_after"][k]], eps_target=float(fx["eps_target"][k]),
                          batch_rel_error_estimate=float(fx["estimate"][k]), tolerance_clamped=bool(fx["clamped"][k]))


@pytest.mark.parametrize("name", NAMES)
def test_fullsize_against_reference(ctx, name):
    if not _present(name):
        pytest.skip(f"fixture {name} not generated")
    fx = F.load(name)
    algo = str(fx["algo"])
    eps = float(fx["eps"])
    modes = tuple(int(v) for v in fx["modes"])
    d = len(modes)
    n = int(fx["n_inc"])
    tg = None
    worst = {"rre": 0.0, "fp": 0.0, "subspace": 0.0, "recp": 0.0}
    for k, (y, shape) in enumerate(_inputs(name, n)):
        if F.sha256_of(y) != bytes(fx["sha256"][k]):
            if not name.startswith("cfg3"):
                # configs[1]/[2] come from the numpy host generators, whose cos / FFT
                # kernels are CPU-dispatched: on another host CPU the bytes differ
                # (the fixtures were generated on the GPU pool's hosts)
                pytest.skip(f"{name}: host generator bytes differ on this CPU (increment {k})")
            raise AssertionError(f"{name}: increment {k} bytes differ from the fixture's")
        if k == 0:
            tg, rg = tt_ice_bootstrap(y, eps, ctx=ctx, shape=shape)
        elif algo == "ice":
            tg, rg = tt_ice_update(tg, y, eps, shape=shape)
        else:
            tg, rg = tt_ice_star_update(tg, y, eps, shape=shape)
        compare_reports(rg, _report(fx, k, shape[-1]), star=(algo != "ice"), n_elems=int(np.prod(shape)))
        b, e = tg.increment_range(k)
        err = rre(tg, y, b, e, shape=shape)
        worst["rre"] = max(worst["rre"], abs(err - float(fx["rre"][k])))
        assert abs(err - float(fx["rre"][k])) <= TOL, (k, err, float(fx["rre"][k]))
        cores = tg.cores()
        fr = F.fingerprints_agree(F.fingerprints(cores, modes), fx["fp"][k])
        worst["fp"] = max(worst["fp"], fr)
        assert fr <= 1.0, f"{name} k={k}: subspace fingerprint off by {fr:.2f} x its 1e-10 bound"
        if "recp" in fx:
            pr = F.recon_probes_agree(F.recon_probes(cores, modes, b, e)[0], fx["recp"][k], fx["recn"][k], fx["zn"])
            worst["recp"] = max(worst["recp"], pr)
            assert pr <= 1.0, f"{name} k={k}: reconstruction probe off by {pr:.2f} x its 1e-10 bound"
        if f"k{k}_core0" in fx:
            for pg, pr in zip(_chained(cores, d), _chained(F.step_cores(fx, k), d)):
                dist = subspace_distance(pg, pr)
                worst["subspace"] = max(worst["subspace"], dist)
                assert dist <= TOL, (k, dist)
        del y
    assert tg.batch_boundaries() == [int(v) for v in fx["batch_boundaries"]]
    assert "recp" in fx or "final_core0" in fx, "fixture carries no reconstruction check"
    coef = float("nan")
    if "final_core0" in fx:
        final_g = tg.cores()
        final_r = F.final_cores(fx)
        assert [c.shape for c in final_g] == [c.shape for c in final_r]
        coef = F.coefficient_agreement(final_g, final_r, d, 0, tg.obs_count())
        assert coef <= TOL, coef
    print(f"{name}: worst |rre - rre_ref| {worst['rre']:.2e}, fingerprint {worst['fp']:.3f} and reconstruction "
          f"probes {worst['recp']:.3f} of their 1e-10 bounds, subspace {worst['subspace']:.2e}, coefficients {coef:.2e}")
    tg.close()
