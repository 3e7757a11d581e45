import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_update
from paper_2211_12487_b200.streams import CONFIGS, Stream
sc = CONFIGS[2]; st = Stream(2, seed=0)
hs = [st.increment(k) for k in range(3)]
shape = sc.modes + (sc.batch,)
ys = [torch.from_numpy(np.ravel(h, order="F")).cuda() for h in hs]
ctx = Context(0)
torch.cuda.synchronize(); t0 = time.perf_counter()
tt, r = tt_ice_bootstrap(ys[0], sc.eps, ctx=ctx, shape=shape)
torch.cuda.synchronize(); print("bootstrap", time.perf_counter() - t0, tt.ranks(), flush=True)
ctx.reset_stats(); ctx.set_profiling(True)
for y in ys[1:]:
    t0 = time.perf_counter()
    tt, r = tt_ice_update(tt, y, sc.eps, shape=shape)
    torch.cuda.synchronize(); print("update", time.perf_counter() - t0, tt.ranks(), flush=True)
for s in sorted(ctx.kernel_stats(), key=lambda s: -s["ms"])[:10]: print(s)
