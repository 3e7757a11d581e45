"""Generate the committed golden fixtures under tests/golden/.

The reference ships no golden vectors of its own (its test TUs are one-line
stubs), so the fixtures here are:

* kat.json   -- the SPEC known-answer examples for the path's helper
               operations, each with the SPEC.md line it restates (inputs and
               expected outputs written from the SPEC text, not computed);
* cfg0_ice.npz, cfg0_star.npz -- the REFERENCE ITSELF (oracle/_ref/libttref.so:
               /root/reference/proj/src compiled unchanged against the
               Eigen-API shim, see oracle/Makefile) run over BASELINE
               configs[0] (64 increments of 8x8x8x8, batch 1, eps 0.1; seeds 0
               and 1): per-increment reports and the final train, plus a
               SHA-256 of the generated input bytes so a change of the seeded
               generator is caught.  They pin the numpy oracle and the CUDA
               path to the reference's answer.

usage: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref_binding as R  # noqa: E402
from paper_2211_12487_b200.streams import Stream  # noqa: E402

N_INC = 64


def kat():
    return {
        "svd_trunc": [
            {"spec": "SPEC.md:121", "a": [[10, 0, 0], [0, 1, 0], [0, 0, 0.1]], "delta": 0.5, "rank": 2, "tail": 0.1},
            {"spec": "SPEC.md:123", "a": [[0, 0, 0, 0, 0]] * 4, "delta": 0.0, "rank": 0, "tail": 0.0},
        ],
        "occupancy": [
            {"spec": "SPEC.md:213", "shape": [1, 4, 2], "value": 0.5},
            {"spec": "SPEC.md:214", "shape": [3, 5, 15], "value": 1.0},
        ],
        "subselect": [
            {"spec": "SPEC.md:397", "errs": [0.2, 0.05], "eps": 0.1, "selected": [0], "rejected": [1]},
            {"spec": "SPEC.md:395", "errs": [0.01, 0.05, 0.1], "eps": 0.1, "selected": [], "rejected": [0, 1, 2]},
            {"spec": "SPEC.md:396", "errs": [0.5, 0.2], "eps": 0.1, "selected": [0, 1], "rejected": []},
        ],
        "relaxed_tolerance_approx": [
            {"spec": "SPEC.md:414", "n_batch": 10, "n_rejected": 5, "mean_rejected_error": 0.05, "eps": 0.1,
             "value": 0.15},
            {"spec": "SPEC.md:413", "n_batch": 10, "n_rejected": 0, "mean_rejected_error": 0.0, "eps": 0.1,
             "value": 0.1},
        ],
        "compression_ratio": [
            {"spec": "SPEC.md:514", "modes": [4, 4, 4], "ranks": [1, 2, 2, 1], "value": 2.0},
        ],
    }


def stream_fixture(algo, seed):
    s = Stream(0, seed=seed)
    h = hashlib.sha256()
    ys = []
    for k in range(N_INC):
        y = np.asfortranarray(s.increment(k))
        h.update(y.tobytes(order="F"))
        ys.append(y)
    tt, rep = R.tt_ice_bootstrap(ys[0], s.eps)
    reps = [rep]
    for k in range(1, N_INC):
        tt, rep = (R.tt_ice_update if algo == "ice" else R.tt_ice_star_update)(tt, ys[k], s.eps)
        reps.append(rep)
    out = {
        "input_sha256": np.frombuffer(h.digest(), dtype=np.uint8),
        "eps": np.float64(s.eps),
        "ranks_after": np.array([r.ranks_after for r in reps], dtype=np.int64),
        "obs_used": np.array([r.obs_used for r in reps], dtype=np.int64),
        "estimate": np.array([r.batch_rel_error_estimate for r in reps]),
        "eps_target": np.array([r.eps_target for r in reps]),
        "batch_boundaries": np.array(tt.batch_boundaries, dtype=np.int64),
        "ortho_count": np.int64(tt.ortho_count),
        "n_cores": np.int64(len(tt.cores)),
        "generator": np.array("reference proj/src via oracle/_ref/libttref.so"),
    }
    for i, c in enumerate(tt.cores):
        out[f"core{i}"] = np.asfortranarray(c.data)
    np.savez_compressed(os.path.join(HERE, f"cfg0_{algo}.npz"), **out)
    return out


def main():
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat(), f, indent=1)
    for algo, seed in (("ice", 0), ("star", 1)):
        o = stream_fixture(algo, seed)
        print(algo, "final ranks", list(o["ranks_after"][-1]), "sha", bytes(o["input_sha256"]).hex()[:16])


if __name__ == "__main__":
    main()
