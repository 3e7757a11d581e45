"""Debug: configs[2] TT-ICE* in lockstep with the reference; first divergence."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import ref_binding as R
from oracle import ttstream_oracle as O
from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_star_update, per_obs_errors, rre
from paper_2211_12487_b200.streams import Stream
from tests.parity_util import to_oracle

R.set_threads(os.cpu_count())
n = int(os.environ.get("N_INC", "5"))
s = Stream(2, seed=0)
ctx = Context(0)
ys = [np.asfortranarray(s.increment(k)) for k in range(n)]
tg, rg = tt_ice_bootstrap(ys[0], s.eps, ctx=ctx)
tr, rr = R.tt_ice_bootstrap(ys[0], s.eps)
print("k=0", rg.ranks_after, rr.ranks_after, flush=True)
for k in range(1, n):
    eg = per_obs_errors(tg, ys[k])
    er = O.per_obs_errors(tr, ys[k])
    print(f"k={k} per-obs err max diff {np.max(np.abs(eg-er)):.3e} (max err {er.max():.3e})", flush=True)
    tg, rg = tt_ice_star_update(tg, ys[k], s.eps)
    tr, rr = R.tt_ice_star_update(tr, ys[k], s.eps)
    go = to_oracle(tg)
    b, e = go.increment_range(k)
    print(f"k={k} gpu {rg.ranks_after} used {rg.obs_used} est {rg.batch_rel_error_estimate:.6e} rre {rre(tg, ys[k], b, e):.6e} "
          f"acc {rg.accurate_modes} unst {rg.gram_only_unstable} guard {rg.guard_reorthogonalised}", flush=True)
    print(f"     ref {rr.ranks_after} used {rr.obs_used} est {rr.batch_rel_error_estimate:.6e} rre {R.rre(tr, ys[k], b, e):.6e}", flush=True)
    orth = go.measure_ortho_count(1e-10)
    print(f"     gpu ortho_count measured {orth} of {go.spatial_dims()}", flush=True)
    if rg.ranks_after != rr.ranks_after:
        break
