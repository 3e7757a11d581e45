"""One cfg3 TT-ICE* update step (+ one skip step) at batch 256, for ncu captures.

usage: python tools/profile_step.py [--batch 256] [--steps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_star_update  # noqa: E402
from paper_2211_12487_b200.streams import DeviceStream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()
modes = (8,) * 7
shape = modes + (args.batch,)
gen = DeviceStream(seed=0, modes=modes)
ctx = Context(0)
y0 = gen.increment(0, args.batch)
tt, _ = tt_ice_bootstrap(y0, 0.01, ctx=ctx, shape=shape)
del y0
for k in range(1, 1 + args.steps):
    y = gen.increment(k + 1, args.batch)  # even first: update path, then skip
    tt, rep = tt_ice_star_update(tt, y, 0.01, shape=shape)
    print("step", k, "obs_used", rep.obs_used, "ranks", rep.ranks_after, "ms", round(rep.seconds * 1e3, 3), flush=True)
    del y
torch.cuda.synchronize()
