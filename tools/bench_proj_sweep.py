"""Companion projection-only sweep (BASELINE.json configs[4]):
tt_project (tensor_train.cpp:195-226) of one cfg3-shaped increment through
fixed, pre-built orthonormal cores with bond ranks R = 8 / 32 / 64 / 128
(capped by the unfolding sizes: r_i = min(R, 8^i, 8^(7-i) b)), spanning the
memory-bound to FP64-compute-bound crossover.

Per R: GB/s ingested (8 N bytes per call / device time of the call), the
SURVEY §8(d) projection roofline (F_proj = sum_i 2 r_i M_i flops, B_proj = 8 N
bytes, T_roof = max(B / BW, F / P)), and the launched kernels with their
CUDA-event times from a profiled replay.  Input is device-resident (a torch
CUDA tensor); the call returns the r_7 x b coefficients to the host.

usage: python tools/bench_proj_sweep.py [--batch 256] [--reps 5] > profiles/r01_proj_sweep.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_12487_b200 import Context, TensorTrain, tt_project  # noqa: E402
from paper_2211_12487_b200.streams import DeviceStream  # noqa: E402

MODES = (8,) * 7
P_FP64 = 37.0e12   # measured DMMA peak (profiles/r01_box_probe.log)
BW = 8.0e12        # north-star HBM figure (BASELINE.json)


def ranks_for(R, b):
    d = len(MODES)
    r = [1]
    for i in range(1, d + 1):
        left = int(np.prod(MODES[:i]))
        right = int(np.prod(MODES[i:])) * b
        r.append(min(R, left, right))
    return r


def build_train(R, b, ctx, rng):
    r = ranks_for(R, b)
    cores = []
    for i, n in enumerate(MODES):
        m = r[i] * n
        q, _ = np.linalg.qr(rng.standard_normal((m, r[i + 1])))
        cores.append(np.reshape(q, (r[i], n, r[i + 1]), order="F"))
    cores.append(np.reshape(rng.standard_normal((r[-1], 1)), (r[-1], 1, 1), order="F"))
    return TensorTrain.upload(cores, ortho_count=len(MODES), batch_boundaries=[1], ctx=ctx), r


def flops_bytes(r, b):
    N = int(np.prod(MODES)) * b
    F = 0.0
    L = N
    for i, n in enumerate(MODES):
        a = r[i] * n
        L = L // n
        F += 2.0 * r[i + 1] * a * L  # 2 r_i M_i, M_i = a_i L_i
    return F, 8.0 * N


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ranks", default="8,32,64,128")
    args = ap.parse_args()
    b = args.batch
    ctx = Context(0)
    y = DeviceStream(seed=0, modes=MODES).increment(1, b)
    shape = MODES + (b,)
    rng = np.random.default_rng(1234)
    rows = []
    for R in [int(x) for x in args.ranks.split(",")]:
        tt, r = build_train(R, b, ctx, rng)
        tt_project(tt, y, shape=shape)  # warm-up (workspaces, caches)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        for _ in range(args.reps):
            e0.record(torch.cuda.current_stream())
            c = tt_project(tt, y, shape=shape)  # synchronous: coefficients on the host on return
            e1.record(torch.cuda.current_stream())
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(times))
        ctx.reset_stats()
        ctx.set_profiling(True)
        tt_project(tt, y, shape=shape)
        ks = sorted(ctx.kernel_stats(), key=lambda s: -s["ms"])
        ctx.set_profiling(False)
        F, B = flops_bytes(r, b)
        t_roof = max(B / BW, F / P_FP64)
        top = ks[0] if ks else None
        kern = None
        if top:
            kt = top["ms"] * 1e-3 / top["launches"]
            fl = top["flops"] / top["launches"]
            by = top["bytes"] / top["launches"]
            bound = "tensor" if fl / max(by, 1.0) > P_FP64 / 6.54e12 else "hbm"
            ach = (fl / kt / 1e12) if bound == "tensor" else (by / kt / 1e9)
            peak = 37.0 if bound == "tensor" else 6540.0
            kern = {"name": top["name"], "ms_per_launch": kt * 1e3, "bound": bound, "achieved": ach, "peak": peak,
                    "unit": "TFLOP/s" if bound == "tensor" else "GB/s", "frac": ach / peak}
        rows.append({"R": R, "ranks": r, "coeff_shape": list(c.shape), "ms": t * 1e3,
                     "GBs_ingested": B / t / 1e9, "flops": F, "bytes": B, "flop_per_byte": F / B,
                     "tflops_achieved": F / t / 1e12, "t_roof_ms": t_roof * 1e3, "roofline_frac": t_roof / t,
                     "bound": "fp64" if F / P_FP64 > B / BW else "hbm", "dominant_kernel": kern,
                     "kernels": [{"name": s["name"], "launches": s["launches"], "ms": round(s["ms"], 4)}
                                 for s in ks[:8]]})
        tt.close()
    out = {"sweep": "projection-only (tt_project) at fixed pre-built cores (BASELINE configs[4] companion)",
           "config": {"modes": list(MODES), "batch": b, "increment_bytes": 8 * int(np.prod(MODES)) * b,
                      "data": "synthetic cfg3 generator increment, random orthonormal cores (seed 1234)",
                      "bw_gbs": BW / 1e9, "p_fp64_tflops": P_FP64 / 1e12,
                      "timing": f"median of {args.reps} synchronous calls, CUDA events; input device-resident"},
           "rows": rows}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
