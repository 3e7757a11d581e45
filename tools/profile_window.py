"""Run the bench's cfg3 TT-ICE* stream (DeviceStream(seed=0), batch 256) to a
given increment, then K more steps inside an NVTX range "prof", for ncu
launch-list captures at the ranks the bench reaches:

  ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none \\
      --csv --log-file launches.csv python tools/profile_window.py --skip 18 --steps 2

Prints the per-step device time (CUDA events, outside ncu these are real).
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
ap.add_argument("--skip", type=int, default=18, help="increments updated before the profiled window")
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()
modes = (8,) * 7
shape = modes + (args.batch,)
gen = DeviceStream(seed=0, modes=modes)
ctx = Context(0)
y = gen.increment(0, args.batch)
tt, _ = tt_ice_bootstrap(y, 0.01, ctx=ctx, shape=shape)
for k in range(1, 1 + args.skip):
    y = gen.increment(k, args.batch)
    tt, rep = tt_ice_star_update(tt, y, 0.01, shape=shape)
ys = [gen.increment(k, args.batch) for k in range(1 + args.skip, 1 + args.skip + args.steps)]
torch.cuda.synchronize()
stream = torch.cuda.ExternalStream(ctx.stream_ptr)
torch.cuda.nvtx.range_push("prof")
for i, y in enumerate(ys):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tt, rep = tt_ice_star_update(tt, y, 0.01, shape=shape)
    e1.record(stream)
    e1.synchronize()
    print(f"step {1 + args.skip + i}: obs_used {rep.obs_used} ranks {rep.ranks_after} device {e0.elapsed_time(e1):.3f} ms "
          f"launches so far {ctx.launch_count}", flush=True)
torch.cuda.nvtx.range_pop()
ctx.close()
