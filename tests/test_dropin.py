"""GPU: the C++ drop-in (include/ttstream/*.hpp over libttg.so) driven like a
reference caller (tests/cpp/test_dropin.cpp) agrees with the CPU oracle."""
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle import ttstream_oracle as O
from paper_2211_12487_b200.streams import Stream
from tests.parity_util import REF, estimates_agree

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRV = os.path.join(ROOT, "tests", "cpp", "test_dropin")

pytestmark = pytest.mark.gpu


def _run(tmp_path, ys, eps, algo):
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    shape = ys[0].shape
    with open(inp, "wb") as f:
        f.write(struct.pack("<q", len(shape)))
        f.write(struct.pack(f"<{len(shape)}q", *shape))
        f.write(struct.pack("<q", len(ys)))
        f.write(struct.pack("<d", eps))
        f.write(struct.pack("<q", algo))
        for y in ys:
            f.write(np.asfortranarray(y).tobytes(order="F"))
    res = subprocess.run([DRV, str(inp), str(out)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr
    buf = open(out, "rb").read()
    pos = 0

    def rd(fmt):
        nonlocal pos
        v = struct.unpack_from(fmt, buf, pos)
        pos += struct.calcsize(fmt)
        return v

    reps = []
    for _ in ys:
        (n,) = rd("<q")
        ranks = list(rd(f"<{n}q"))
        (used,) = rd("<q")
        est, tgt = rd("<dd")
        reps.append((ranks, used, est, tgt))
    (nc,) = rd("<q")
    cores = []
    for _ in range(nc):
        rl, n, rr = rd("<3q")
        data = np.array(rd(f"<{rl * n * rr}d"))
        cores.append(O.TTCore(np.reshape(data, (rl, n, rr), order="F")))
    (checks,) = rd("<q")
    return reps, cores, checks


@pytest.mark.parametrize("algo", [0, 1])
def test_dropin_cpp_api_matches_oracle(tmp_path, algo):
    if not os.path.exists(DRV):
        import __graft_entry__

        __graft_entry__.build()
    s = Stream(3, seed=21, modes=(4,) * 5, batch=6, true_rank=4)
    ys = [s.increment(k) for k in range(6)]
    reps, cores, checks = _run(tmp_path, ys, s.eps, algo)
    tr, rr = REF.tt_ice_bootstrap(ys[0], s.eps)
    assert reps[0][0] == rr.ranks_after
    for k in range(1, len(ys)):
        tr, rr = (REF.tt_ice_update if algo == 0 else REF.tt_ice_star_update)(tr, ys[k], s.eps)
        assert reps[k][0] == rr.ranks_after
        assert reps[k][1] == rr.obs_used
        assert estimates_agree(reps[k][2], rr.batch_rel_error_estimate, pythagoras=algo == 1)
    gh = O.TensorTrain(cores, len(cores) - 1, tr.batch_boundaries)
    rec_g, rec_r = O.tt_reconstruct(gh), O.tt_reconstruct(tr)
    assert np.linalg.norm(rec_g - rec_r) <= 1e-10 * np.linalg.norm(rec_r)
    assert checks == 6  # the error classes and the stale-generation re-upload
