"""Run the REFERENCE (oracle/_ref/libttref.so: proj/src compiled unchanged
against the Eigen-API shim) over BASELINE configs at their full sizes and
write the per-increment fixtures tests/test_gpu_fullsize_parity.py checks
the CUDA path against (format: tests/fullsize_util.py).

  cfg1   configs[1] video-like (14,15,16,10,3) x 100, all 40 increments,
         TT-ICE and TT-ICE* (host generator, runs anywhere)
  cfg2   configs[2] simulation-like (8,8,8,8,8,8,3) x 32, first 8 increments,
         TT-ICE and TT-ICE* (host generator)
  cfg3   configs[3] at full size, 8^7 x 256 = 4.29 GB per increment: the
         bench's own stream (DeviceStream(seed=0), generated on the GPU and
         copied to host), bootstrap + 9 TT-ICE* increments and bootstrap +
         4 TT-ICE increments.  Needs a CUDA device (run under gpurun).

usage: python tools/make_fullsize_fixtures.py cfg1|cfg2|cfg3 [--out DIR] [--threads N]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref_binding as R  # noqa: E402
from tests import fullsize_util as F  # noqa: E402

CORE_BUDGET = 1 << 20   # store per-increment spatial cores while they stay this small (bytes per increment)
FINAL_BUDGET = 4 << 20  # store the final train when it is this small (bytes)
STEP_CORES_FIRST = 10   # per-increment cores for the first increments and the last one


def run(name, ys, eps, algo, modes, out_dir, cfg_desc, n_inc):
    """ys: iterable of host arrays (first-index-fastest)."""
    d = len(modes)
    fx = {"eps": np.float64(eps), "algo": np.array(algo), "config": np.array(cfg_desc),
          "generator": np.array("reference proj/src via oracle/_ref/libttref.so")}
    sha, ranks, used, epst, est, clamped, rre, fps, secs, recp, recn = [], [], [], [], [], [], [], [], [], [], []
    zn = None
    h = None
    per_step_cores = True
    for k, y in enumerate(ys):
        t0 = time.time()
        sha.append(np.frombuffer(F.sha256_of(y), dtype=np.uint8))
        if k == 0:
            h, rep = R.tt_ice_bootstrap(y, eps, keep_handle=True)
        elif algo == "ice":
            h, rep = R.tt_ice_update(h, y, eps, keep_handle=True)
        else:
            h, rep = R.tt_ice_star_update(h, y, eps, keep_handle=True)
        t_upd = time.time() - t0
        tt = h.to_oracle()
        b, e = tt.increment_range(k)
        rre.append(R.rre(h, y, b, e))
        cores = [c.data for c in tt.cores]
        fps.append(F.fingerprints(cores, modes))
        p, nrm, zn = F.recon_probes(cores, modes, b, e)
        recp.append(p)
        recn.append(nrm)
        if not (k < STEP_CORES_FIRST or k == n_inc - 1):
            pass  # fingerprints and reconstruction probes still cover this increment
        elif per_step_cores and sum(c.nbytes for c in cores[:d]) <= CORE_BUDGET:
            for i in range(d):
                fx[f"k{k}_core{i}"] = np.asfortranarray(cores[i])
        else:
            per_step_cores = False
        ranks.append(rep.ranks_after)
        used.append(rep.obs_used)
        epst.append(rep.eps_target)
        est.append(rep.batch_rel_error_estimate)
        clamped.append(rep.tolerance_clamped)
        secs.append(t_upd)
        print(f"{name} k={k} ranks={rep.ranks_after} used={rep.obs_used} est={rep.batch_rel_error_estimate:.6e} "
              f"rre={rre[-1]:.6e} ref {t_upd:.1f}s total {time.time() - t0:.1f}s", flush=True)
    tt = h.to_oracle()
    fx.update({
        "n_inc": np.int64(len(sha)),
        "sha256": np.stack(sha),
        "ranks_after": np.array(ranks, dtype=np.int64),
        "obs_used": np.array(used, dtype=np.int64),
        "eps_target": np.array(epst),
        "estimate": np.array(est),
        "clamped": np.array(clamped, dtype=bool),
        "rre": np.array(rre),
        "fp": np.stack(fps),
        "recp": np.stack(recp),
        "recn": np.stack(recn),
        "zn": zn,
        "ref_seconds": np.array(secs),
        "per_step_cores": np.bool_(per_step_cores),
        "n_cores": np.int64(len(tt.cores)),
        "ortho_count": np.int64(tt.ortho_count),
        "batch_boundaries": np.array(tt.batch_boundaries, dtype=np.int64),
        "modes": np.array(modes, dtype=np.int64),
    })
    if sum(c.data.nbytes for c in tt.cores) <= FINAL_BUDGET:
        for i, c in enumerate(tt.cores):
            fx[f"final_core{i}"] = np.asfortranarray(c.data)
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, name + ".npz")
    np.savez_compressed(path, **fx)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.1f} MB)", flush=True)


def host_stream(cfg, n, **kw):
    from paper_2211_12487_b200.streams import Stream

    s = Stream(cfg, seed=0, **kw)
    return s, (np.asfortranarray(s.increment(k)) for k in range(n))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg1", "cfg2", "cfg3"])
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    R.set_threads(args.threads)
    if args.which in ("cfg1", "cfg2"):
        cfg, n = (1, 40) if args.which == "cfg1" else (2, 8)
        for algo in ("ice", "star"):
            s, ys = host_stream(cfg, n)
            run(f"{args.which}_full_{algo}", ys, s.eps, algo, s.modes, args.out,
                f"configs[{cfg}] full size, seed 0, {n} increments, Stream({cfg}, seed=0)", n)
        return
    import torch

    from paper_2211_12487_b200.streams import DeviceStream

    modes, b, eps = (8,) * 7, 256, 0.01
    gen = DeviceStream(seed=0, modes=modes)

    def dev_incs(n):
        for k in range(n):
            y = gen.increment(k, b)
            torch.cuda.synchronize()
            a = np.reshape(y.cpu().numpy(), modes + (b,), order="F")
            del y
            yield a

    for algo, n in (("star", 10), ("ice", 5)):
        run(f"cfg3_full_{algo}", dev_incs(n), eps, algo, modes, args.out,
            f"configs[3] full size 8^7 x 256, DeviceStream(seed=0) = bench.py's stream, {n} increments", n)


if __name__ == "__main__":
    main()
