"""Measurement of the SURVEY §8(f) rows on the GPU (companion to bench.py):

* device RRE of a cfg3 increment against its reference (metrics.cpp:34-42):
  GB/s of reference data and the HBM roofline of k_rre_partial (reads X and
  Phi once: 8 S (m + r) bytes per launch);
* TTC1 checkpoint save / load (serialization.cpp) of the cfg3 train;
* the prefetching TTB1 stream reader feeding TT-ICE* (stream_io.cpp): increments
  per second from files vs. the same updates on device-resident input;
* the oracle's RRE on a bounded sample as the CPU baseline.

usage: python tools/bench_io.py [--batch 64] [--steps 4] > profiles/r01_io_bench.json
"""
import argparse
import json
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_12487_b200 import (Context, IncrementStream, load_ttc, rre, save_ttc, tt_ice_bootstrap,  # noqa: E402
                                   tt_ice_star_update)
from paper_2211_12487_b200.streams import DeviceStream  # noqa: E402

MODES = (8,) * 7
EPS = 0.01


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    b = args.batch
    ctx = Context(0)
    gen = DeviceStream(seed=0, modes=MODES)
    shape = MODES + (b,)
    S = int(np.prod(MODES))
    ys = [gen.increment(k, b) for k in range(1 + args.steps)]
    tt, _ = tt_ice_bootstrap(ys[0], EPS, ctx=ctx, shape=shape)
    for y in ys[1:]:
        tt, _ = tt_ice_star_update(tt, y, EPS, shape=shape)
    torch.cuda.synchronize()
    out = {}

    # device RRE of the last increment against its reference
    k = len(ys) - 1
    b0, e0 = tt.increment_range(k)
    ref = ys[k]
    rre(tt, ref, b0, e0, shape=shape)  # warm
    ctx.reset_stats()
    ctx.set_profiling(True)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        val = rre(tt, ref, b0, e0, shape=shape)
    el = (time.perf_counter() - t0) / reps
    ks = {s["name"]: s for s in ctx.kernel_stats()}
    ctx.set_profiling(False)
    kp = ks.get("k_rre_partial")
    r = tt.ranks()[len(MODES)]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6550.0))
    ach = kp["bytes"] / (kp["ms"] * 1e-3) / 1e9 if kp else None
    out["rre"] = {"value": 8.0 * S * b / el / 1e9, "unit": "GB/s of reference data (whole call, incl. Phi chain)",
                  "rre": val, "rank": r, "obs": b,
                  "kernel": {"name": "k_rre_partial", "ms_per_launch": kp["ms"] / kp["launches"] if kp else None,
                             "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                                          "frac": (ach / hbm) if ach else None,
                                          "algorithmic_bytes_per_launch": kp["bytes"] / kp["launches"] if kp else None}}}

    # CPU baseline: oracle RRE on a bounded sample (8 observations)
    from oracle import ttstream_oracle as O

    from tests.parity_util import to_oracle

    th = to_oracle(tt)
    m = min(8, e0 - b0)
    refh = np.asfortranarray(ref[:, :m].cpu().numpy() if ref.dim() == 2 else
                             np.reshape(ref.cpu().numpy().ravel(order="C"), shape, order="F")[..., :m])
    t0 = time.perf_counter()
    cv = O.rre(th, refh, b0, b0 + m)[0]
    ct = time.perf_counter() - t0
    out["rre"]["cpu_baseline"] = {"value": 8.0 * S * m / ct / 1e9, "unit": "GB/s", "kind": "port", "cores": os.cpu_count(),
                                  "sample": f"oracle rre on {m} of {b} observations ({ct:.2f} s)", "rre_sample": cv}

    # TTC1 checkpoint
    tmp = tempfile.mkdtemp()
    try:
        p = os.path.join(tmp, "ckpt.ttc")
        t0 = time.perf_counter()
        save_ttc(tt, p)
        ts = time.perf_counter() - t0
        sz = os.path.getsize(p)
        t0 = time.perf_counter()
        t2 = load_ttc(p, ctx=ctx)
        tl = time.perf_counter() - t0
        out["ttc1"] = {"bytes": sz, "save_ms": ts * 1e3, "load_ms": tl * 1e3, "ortho_count": t2.ortho_count,
                       "ranks": tt.ranks()}
        t2.close()

        # stream reader: write the increments as .ttb, stream them into TT-ICE*
        from paper_2211_12487_b200 import write_batch

        sd = os.path.join(tmp, "stream")
        os.makedirs(sd)
        for i, y in enumerate(ys):
            write_batch(np.reshape(y.cpu().numpy().ravel(order="C"), shape, order="F"), os.path.join(sd, f"{i:04d}.ttb"))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = IncrementStream(sd, ctx=ctx)
        it = iter(st)
        ts_, _ = tt_ice_bootstrap(next(it), EPS, ctx=ctx)
        for y in it:
            ts_, _ = tt_ice_star_update(ts_, y, EPS)
        torch.cuda.synchronize()
        tstream = time.perf_counter() - t0
        st.close()
        t0 = time.perf_counter()
        td, _ = tt_ice_bootstrap(ys[0], EPS, ctx=ctx, shape=shape)
        for y in ys[1:]:
            td, _ = tt_ice_star_update(td, y, EPS, shape=shape)
        torch.cuda.synchronize()
        tdev = time.perf_counter() - t0
        nbytes = 8.0 * S * b * len(ys)
        out["stream"] = {"files": len(ys), "bytes_per_file": 8 * S * b,
                         "from_files_GBs": nbytes / tstream / 1e9, "device_resident_GBs": nbytes / tdev / 1e9,
                         "note": "files on the box's local disk (page cache warm after writing); the reader "
                                 "overlaps read + pinned H2D of increment k+1 with the update of k"}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    out["config"] = {"modes": list(MODES), "batch": b, "increments": len(ys), "eps": EPS,
                     "data": "synthetic cfg3 generator (DESIGN.md §6)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
