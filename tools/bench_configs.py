"""Full-size throughput of the other BASELINE stream configs (companion to
bench.py, which measures configs[3]):

* configs[1] video-like, (14,15,16,10,3) x 100 frames, 40 increments, eps 0.1;
* configs[2] simulation-like, (8,8,8,8,8,8,3) x 32 snapshots, 50 increments, eps 0.05.

Each stream is generated on the host by the seeded generators
(paper_2211_12487_b200/streams.py), copied to HBM once (outside the timed
region), bootstrapped (tt_svd) and then updated increment by increment with
TT-ICE and, separately, TT-ICE* (default heuristics).  Reported: GB/s
ingested over the updates (device-resident input, CUDA events around the
whole update sequence), final ranks, and the top kernels of a profiled replay.

usage: python tools/bench_configs.py [--cfg 1,2] [--increments N] > profiles/r01_configs.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_star_update, tt_ice_update  # noqa: E402
from paper_2211_12487_b200.streams import CONFIGS, Stream  # noqa: E402


def run(ctx, ys, shape, eps, algo, profiled=False):
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    tt, _ = tt_ice_bootstrap(ys[0], eps, ctx=ctx, shape=shape)
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.set_profiling(profiled)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps = []
    for y in ys[1:]:
        if algo == "ice":
            tt, r = tt_ice_update(tt, y, eps, shape=shape)
        else:
            tt, r = tt_ice_star_update(tt, y, eps, shape=shape)
        reps.append(r)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    ks = sorted(ctx.kernel_stats(), key=lambda s: -s["ms"]) if profiled else []
    ctx.set_profiling(False)
    ranks = tt.ranks()
    tt.close()
    return ms, ranks, reps, ks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="1,2")
    ap.add_argument("--increments", type=int, default=0, help="0 = the config's own count")
    args = ap.parse_args()
    ctx = Context(0)
    out = {"rows": []}
    for cfg in [int(x) for x in args.cfg.split(",")]:
        sc = CONFIGS[cfg]
        n_inc = args.increments or sc.increments
        st = Stream(cfg, seed=0)
        t0 = time.perf_counter()
        hs = [st.increment(k) for k in range(n_inc)]
        tgen = time.perf_counter() - t0
        shape = sc.modes + (sc.batch,)
        ys = [torch.from_numpy(np.ravel(h, order="F")).cuda() for h in hs]
        del hs
        torch.cuda.synchronize()
        inc_bytes = 8 * int(np.prod(shape))
        for algo in ("ice", "star"):
            run(ctx, ys[:3], shape, sc.eps, algo)  # warm-up (workspaces, module loads)
            ms, ranks, reps, _ = run(ctx, ys, shape, sc.eps, algo)
            _, _, _, ks = run(ctx, ys, shape, sc.eps, algo, profiled=True)
            upd = n_inc - 1
            out["rows"].append({
                "cfg": cfg, "name": sc.name, "algo": "tt_ice" if algo == "ice" else "tt_ice_star",
                "shape": list(shape), "eps": sc.eps, "increments": n_inc, "increment_bytes": inc_bytes,
                "update_ms_total": ms, "ms_per_update": ms / upd, "GBs_ingested": inc_bytes * upd / (ms * 1e-3) / 1e9,
                "final_ranks": ranks, "obs_used": sum(r.obs_used for r in reps),
                "max_batch_rel_error_estimate": max(r.batch_rel_error_estimate for r in reps),
                "top_kernels": [{"name": s["name"], "launches": s["launches"], "ms": round(s["ms"], 3)} for s in ks[:6]],
                "host_generation_s": tgen})
            print(json.dumps(out["rows"][-1]), file=sys.stderr, flush=True)
        del ys
        torch.cuda.empty_cache()
    out["note"] = ("device-resident increments (host generation and H2D outside the timed region); "
                   "GB/s = increment bytes x updates / device time of the update sequence (CUDA events)")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
