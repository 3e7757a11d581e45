"""CPU: the §8(f) rows' oracle against the SPEC's known answers (metrics
SPEC.md:508-540, TTC1 SPEC.md:224-248, TTB1 stream_io.hpp:57-61) and the
context-free TTB1 entry points of libttg.so against the oracle's bytes."""
import os

import numpy as np
import pytest

from oracle import ttstream_oracle as O


def _random_tt(rng, modes, ranks, nobs, ortho=True):
    cores = []
    r = [1] + list(ranks)
    if ortho:  # an orthonormal left unfolding needs r_{i+1} <= r_i n_i
        for i, n in enumerate(modes):
            r[i + 1] = min(r[i + 1], r[i] * n)
    for i, n in enumerate(modes):
        a = rng.standard_normal((r[i] * n, r[i + 1]))
        if ortho:
            a = np.linalg.qr(a)[0]
        cores.append(O.TTCore.from_left_unfolding(a, r[i], n))
    cores.append(O.TTCore(np.asfortranarray(rng.standard_normal((r[-1], nobs, 1)))))
    return O.TensorTrain(cores, len(modes) if ortho else 0)


def test_compression_ratio_spec_example():
    """3 modes of extent 4, ranks [1,2,2,1] -> 64 / (8+16+8) = 2.0."""
    rng = np.random.default_rng(0)
    cores = [O.TTCore(np.asfortranarray(rng.standard_normal(s))) for s in [(1, 4, 2), (2, 4, 2), (2, 4, 1)]]
    assert O.compression_ratio(O.TensorTrain(cores, 0)) == 2.0


def test_compression_ratio_below_one_is_legal():
    rng = np.random.default_rng(1)
    tt = _random_tt(rng, (2, 2), (2, 4), 1, ortho=False)
    assert O.compression_ratio(tt) < 1.0


def test_rre_known_answers():
    rng = np.random.default_rng(2)
    tt = _random_tt(rng, (4, 5), (3, 2), 6)
    rec = O.tt_reconstruct(tt)
    assert O.rre(tt, rec)[0] == pytest.approx(0.0, abs=1e-15)
    # reference orthogonal to the reconstruction with equal norm -> sqrt(2)
    flat = np.ravel(rec, order="F")
    v = rng.standard_normal(flat.size)
    v -= flat * (flat @ v) / (flat @ flat)
    v *= np.linalg.norm(flat) / np.linalg.norm(v)
    e, zero = O.rre(tt, np.reshape(v, rec.shape, order="F"))
    assert e == pytest.approx(np.sqrt(2.0), rel=1e-12) and not zero
    e, zero = O.rre(tt, np.zeros_like(rec))
    assert e == 0.0 and zero
    with pytest.raises(O.DimensionError):
        O.rre(tt, rec[..., :3])


def test_rpe_properties():
    rng = np.random.default_rng(3)
    tt = _random_tt(rng, (4, 5, 3), (4, 6, 5), 4)
    in_span = O.tt_expand(tt, rng.standard_normal((5, 7)))
    assert O.rpe(tt, in_span)[0] <= 1e-12
    x = rng.standard_normal((4, 5, 3, 7))
    x /= np.linalg.norm(x)
    c = O.tt_project(tt, x)
    e = O.rpe(tt, x)[0]
    assert e <= 1.0 + 1e-12
    assert e * e + float(np.sum(c * c)) == pytest.approx(1.0, abs=1e-10)


def test_mean_rre_per_increment():
    rng = np.random.default_rng(4)
    tt = _random_tt(rng, (4, 5), (3, 2), 6)
    tt = O.TensorTrain(tt.cores, tt.ortho_count, [2, 6])
    refs = [O.tt_reconstruct(tt, 0, 2) + 0.01, O.tt_reconstruct(tt, 2, 6)]
    per, mean = O.mean_rre_per_increment(tt, refs)
    assert per[0] == pytest.approx(O.rre(tt, refs[0], 0, 2)[0]) and per[1] == pytest.approx(0.0, abs=1e-15)
    assert mean == pytest.approx(sum(per) / 2)
    with pytest.raises(O.DimensionError):
        O.mean_rre_per_increment(tt, refs[:1])


@pytest.mark.parametrize("seed", range(8))
def test_ttc1_round_trip_bit_exact(seed):
    """serialize / deserialize round trips are bit-exact."""
    rng = np.random.default_rng(100 + seed)
    d = int(rng.integers(1, 5))
    modes = tuple(int(x) for x in rng.integers(1, 6, d))
    ranks = tuple(int(x) for x in rng.integers(1, 4, d))
    tt = _random_tt(rng, modes, ranks, int(rng.integers(1, 9)), ortho=bool(seed % 2))
    b = O.serialize(tt)
    t2 = O.deserialize(b)
    assert O.serialize(t2) == b
    assert t2.ortho_count == tt.measure_ortho_count()


def test_ttc1_format_errors():
    rng = np.random.default_rng(5)
    b = O.serialize(_random_tt(rng, (3, 4), (2, 2), 3))
    cases = [(b"XXC1" + b[4:], "bad magic"), (b[:20], "truncated"), (b + b"\0", "trailing"),
             (b[:4] + b"\0" + b[5:], "zero cores")]
    for data, what in cases:
        with pytest.raises(O.FormatError):
            O.deserialize(data)
    # adjacent rank mismatch: bump core 1's r_left
    bad = bytearray(b)
    off = 5 + 24 + 8 * (1 * 3 * 2)
    bad[off:off + 8] = (3).to_bytes(8, "little")
    with pytest.raises(O.FormatError):
        O.deserialize(bytes(bad))


def test_ttb1_round_trip_and_errors(tmp_path):
    rng = np.random.default_rng(6)
    t = np.asfortranarray(rng.standard_normal((3, 4, 2)))
    p = tmp_path / "a.ttb"
    O.write_batch(t, str(p))
    assert np.array_equal(O.read_batch(str(p)), t)
    raw = p.read_bytes()
    (tmp_path / "bad.ttb").write_bytes(b"TTB2" + raw[4:])
    with pytest.raises(O.FormatError):
        O.read_batch(str(tmp_path / "bad.ttb"))
    (tmp_path / "short.ttb").write_bytes(raw[:-8])
    with pytest.raises(O.FormatError):
        O.read_batch(str(tmp_path / "short.ttb"))
    (tmp_path / "z.txt").write_bytes(raw)
    assert [os.path.basename(f) for f in O.list_stream(str(tmp_path))] == ["a.ttb", "bad.ttb", "short.ttb"]


def test_ttb1_through_the_c_abi(tmp_path):
    """The context-free TTB1 entry points of libttg.so (no GPU needed) write
    the oracle's bytes and read the oracle's files."""
    from paper_2211_12487_b200 import FormatError, read_batch, write_batch

    rng = np.random.default_rng(7)
    t = np.asfortranarray(rng.standard_normal((5, 2, 3, 4)))
    write_batch(t, tmp_path / "lib.ttb")
    O.write_batch(t, str(tmp_path / "ora.ttb"))
    assert (tmp_path / "lib.ttb").read_bytes() == (tmp_path / "ora.ttb").read_bytes()
    assert np.array_equal(read_batch(tmp_path / "ora.ttb"), t)
    (tmp_path / "bad.ttb").write_bytes(b"NOPE" + b"\0" * 20)
    with pytest.raises(FormatError, match="bad magic"):
        read_batch(tmp_path / "bad.ttb")
    raw = (tmp_path / "ora.ttb").read_bytes()
    (tmp_path / "short.ttb").write_bytes(raw[:-1])
    with pytest.raises(FormatError, match="payload length"):
        read_batch(tmp_path / "short.ttb")
