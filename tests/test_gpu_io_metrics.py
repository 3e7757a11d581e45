"""GPU: the SURVEY §8(f) rows through the C ABI against the oracle —
device RRE / RPE / mean RRE (metrics.cpp), device measure_ortho_count, the
TTC1 checkpoint (serialization.cpp; byte-identical images, resume parity) and
the prefetching TTB1 stream reader (stream_io.cpp) feeding the update."""
import numpy as np
import pytest

from oracle import ttstream_oracle as O
from paper_2211_12487_b200 import (FormatError, IncrementStream, NumericError, TensorTrain, compression_ratio,
                                   deserialize, load_ttc, mean_rre_per_increment, rpe, rre, save_ttc, serialize,
                                   tt_ice_bootstrap, tt_ice_star_update, tt_ice_update, write_batch)
from paper_2211_12487_b200.streams import Stream
from tests.parity_util import REF, TOL, compare_trains, to_oracle

pytestmark = pytest.mark.gpu


def _stream_train(ctx, stream, n_inc, star=False):
    ys = [stream.increment(k) for k in range(n_inc)]
    tg, _ = tt_ice_bootstrap(ys[0], stream.eps, ctx=ctx)
    for y in ys[1:]:
        tg, _ = (tt_ice_star_update if star else tt_ice_update)(tg, y, stream.eps)
    return tg, ys


def test_rre_rpe_cr_match_oracle(ctx):
    s = Stream(3, seed=11, modes=(4,) * 5, batch=12, true_rank=5)
    tg, ys = _stream_train(ctx, s, 6)
    th = to_oracle(tg)  # the same cores on the host
    assert compression_ratio(tg) == pytest.approx(O.compression_ratio(th), rel=1e-15)
    for k, y in enumerate(ys):
        b, e = tg.increment_range(k)
        got = rre(tg, y, b, e)
        ref = O.rre(th, y, b, e)[0]
        assert abs(got - ref) <= 1e-12 * max(1.0, ref), (k, got, ref)
    unseen = Stream(3, seed=12, modes=(4,) * 5, batch=7, true_rank=5).increment(3)
    assert abs(rpe(tg, unseen) - O.rpe(th, unseen)[0]) <= 1e-12
    per = mean_rre_per_increment(tg, ys)
    per_ref, mean_ref = O.mean_rre_per_increment(th, ys)
    assert np.allclose(per.per_increment, per_ref, rtol=1e-12, atol=1e-14)
    assert per.mean == pytest.approx(mean_ref, rel=1e-12)


def test_rre_known_answers_on_device(ctx):
    s = Stream(0, seed=3)
    tg, ys = _stream_train(ctx, s, 4)
    th = to_oracle(tg)
    rec = O.tt_reconstruct(th, 1, 3)
    assert rre(tg, rec, 1, 3) <= 1e-14
    val, zero = rre(tg, np.zeros_like(rec), 1, 3, with_flag=True)
    assert val == 0.0 and zero
    from paper_2211_12487_b200 import DimensionError, IndexError_

    with pytest.raises(DimensionError):
        rre(tg, rec, 0, 3)
    with pytest.raises(IndexError_):
        rre(tg, rec, 3, 99)


def test_device_measure_ortho_count(ctx):
    s = Stream(0, seed=4)
    tg, _ = _stream_train(ctx, s, 3)
    assert tg.measure_ortho_count() == to_oracle(tg).measure_ortho_count() == tg.ortho_count
    rng = np.random.default_rng(1)
    cores = [c.copy(order="F") for c in tg.cores()]
    cores[1] = cores[1] * 1.01  # break orthonormality of core 1 only
    bad = TensorTrain.upload(cores, 0, tg.batch_boundaries(), ctx=ctx)
    assert bad.measure_ortho_count() == 1
    del rng


def test_ttc1_image_byte_identical_and_resume(ctx, tmp_path):
    s = Stream(3, seed=13, modes=(4,) * 5, batch=12, true_rank=5)
    tg, ys = _stream_train(ctx, s, 4, star=True)
    img = serialize(tg)
    assert img == O.serialize(to_oracle(tg))  # same bytes as the reference layout of the same cores
    t2 = deserialize(img, ctx=ctx)
    assert serialize(t2) == img and t2.ortho_count == tg.ortho_count == O.deserialize(img).ortho_count
    save_ttc(tg, tmp_path / "ckpt.ttc")
    assert (tmp_path / "ckpt.ttc").read_bytes() == img
    t3 = load_ttc(tmp_path / "ckpt.ttc", ctx=ctx)
    # resume: the next update from the checkpoint equals the update from the live train
    y = s.increment(4)
    ta, ra = tt_ice_star_update(t3, y, s.eps)
    tr, rr = REF.tt_ice_star_update(O.deserialize(img), y, s.eps)
    assert list(ra.ranks_after) == list(rr.ranks_after)
    compare_trains(ta, tr)


def test_ttc1_errors(ctx):
    s = Stream(0, seed=5)
    tg, _ = _stream_train(ctx, s, 2)
    img = serialize(tg)
    with pytest.raises(FormatError, match="bad magic"):
        deserialize(b"TTX1" + img[4:], ctx=ctx)
    with pytest.raises(FormatError, match="truncated"):
        deserialize(img[:40], ctx=ctx)
    with pytest.raises(FormatError, match="trailing"):
        deserialize(img + b"\0", ctx=ctx)
    bad = bytearray(img)
    bad[5 + 24:5 + 32] = np.float64(np.nan).tobytes()  # first payload value of core 0
    with pytest.raises(NumericError):
        deserialize(bytes(bad), ctx=ctx)


def test_stream_reader_feeds_the_update(ctx, tmp_path):
    """A .ttb directory streamed through the pinned double-buffered reader gives
    the same train as passing the host arrays (same bytes, same kernels)."""
    s = Stream(3, seed=14, modes=(4,) * 5, batch=12, true_rank=5)
    ys = [s.increment(k) for k in range(6)]
    for k, y in enumerate(ys):
        write_batch(y, tmp_path / f"inc_{k:04d}.ttb")
    (tmp_path / "notes.txt").write_text("ignored")
    st = IncrementStream(tmp_path, ctx=ctx)
    assert len(st) == 6
    it = iter(st)
    first = next(it)
    assert first.shape == ys[0].shape
    tg, _ = tt_ice_bootstrap(first, s.eps, ctx=ctx)
    for y in it:
        tg, _ = tt_ice_star_update(tg, y, s.eps)
    st.close()
    th, _ = tt_ice_bootstrap(ys[0], s.eps, ctx=ctx)
    for y in ys[1:]:
        th, _ = tt_ice_star_update(th, y, s.eps)
    assert serialize(tg) == serialize(th)
    tr, _ = REF.tt_ice_bootstrap(ys[0], s.eps)
    for y in ys[1:]:
        tr, _ = REF.tt_ice_star_update(tr, y, s.eps)
    compare_trains(tg, tr)
    assert TOL > 0


def test_cpp_dropin_stream_checkpoint_metrics(tmp_path):
    """tests/cpp/test_io_dropin.cpp: a C++ caller of include/ttstream streams a
    .ttb directory through DeviceStreamReader + the device-pointer overloads,
    checkpoints (save_ttc / load_ttc) and reports RRE / CR; the checkpoint and
    the metrics agree with the oracle run on the same files."""
    import os
    import subprocess

    drv = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "cpp", "test_io_dropin")
    s = Stream(3, seed=15, modes=(4,) * 5, batch=12, true_rank=5)
    ys = [s.increment(k) for k in range(5)]
    d = tmp_path / "stream"
    d.mkdir()
    for k, y in enumerate(ys):
        O.write_batch(y, str(d / f"{k:03d}.ttb"))
    res = subprocess.run([drv, str(d), repr(s.eps), str(tmp_path / "out.ttc")], capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    lines = dict()
    for ln in res.stdout.splitlines():
        parts = ln.split()
        lines[(parts[0], parts[1] if len(parts) == 3 else "")] = float(parts[-1]) if parts[0] != "errors" else parts[1]
    tg = O.deserialize((tmp_path / "out.ttc").read_bytes())
    tr, _ = REF.tt_ice_bootstrap(ys[0], s.eps)
    for y in ys[1:]:
        tr, _ = REF.tt_ice_star_update(tr, y, s.eps)
    compare_trains(tg, tr)
    per_ref, _ = O.mean_rre_per_increment(tg, ys)
    for k, e in enumerate(per_ref):
        assert abs(lines[("rre", str(k))] - e) <= 1e-12 * max(1.0, e)
    assert lines[("cr", "")] == pytest.approx(O.compression_ratio(tg), rel=1e-15)
