import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_star_update, tt_ice_update
upd = tt_ice_update if os.environ.get('ALGO') == 'ice' else tt_ice_star_update
K0 = int(os.environ.get('K0', '12'))
from paper_2211_12487_b200.streams import Stream
s = Stream(1, seed=0)
ctx = Context(0)
ys = [torch.from_numpy(np.ravel(s.increment(k), order="F")).cuda() for k in range(0, K0 + 2)]
shape = tuple(s.increment(0).shape)
tt, _ = tt_ice_bootstrap(ys[0], s.eps, ctx=ctx, shape=shape)
for k in range(1, K0):
    tt, rep = upd(tt, ys[k], s.eps, shape=shape)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
for k in (K0, K0 + 1):
    tt, rep = upd(tt, ys[k], s.eps, shape=shape)
    print(k, rep.obs_used, rep.ranks_after, rep.seconds)
torch.cuda.nvtx.range_pop()
