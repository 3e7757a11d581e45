"""GPU, world_size 2 on ONE device: the library's own multi-rank host logic
(batch shards, all-reduced Grams / norms / TT-ICE* decision sums, all-gathered
coefficient columns, per-rank identical eigen-solves) run end to end.

Two processes share cuda:0, each with a context created by
ttg_ctx_create_hostcoll whose collectives are torch.distributed gloo calls on
host buffers (no NCCL: NCCL needs one GPU per rank).  The ranks' kernels never
wait on one another; only the host exchanges synchronise them.  The result
must equal the unsharded CPU oracle: ranks identical after every increment,
subspaces / reconstructions / error estimates within 1e-10 (the Gram summation
order differs from the unsharded run, so bitwise equality is not expected).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_INC = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _increment(s, k, algo):
    """Full (unsharded) increment k.  "star_skew": the first half of every
    update increment is re-sampled inside the current span (rejected by the
    subselection) and the second half carries the drift (selected), so with two
    ranks one shard contributes no selected observation at all and the other
    all of them (per-rank |D| = 0 / b/2)."""
    y = s.increment(k)
    if algo == "star_skew" and k >= 2 and k % 2 == 0:
        h = s.batch // 2
        y = np.concatenate([s.increment(k - 1)[..., :h], y[..., h:]], axis=-1)
    return np.asfortranarray(y)


def _n_inc(algo):
    return 1 if algo == "boot" else N_INC


def _worker(rank, world, port, algo, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_star_update, tt_ice_update
        from paper_2211_12487_b200.streams import Stream

        def allreduce(a):
            dist.all_reduce(torch.from_numpy(a))  # in place on the library's host buffer

        def allgather(b):
            t = torch.from_numpy(b)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return np.concatenate([p.numpy() for p in parts])

        ctx = Context.with_host_collectives(0, rank, world, allreduce, allgather)
        assert ctx.world == world and ctx.rank == rank
        s = Stream(3, seed=5, modes=(6,) * 4, batch=16, true_rank=5)
        bl = s.batch // world
        reps = []
        tt = None
        for k in range(_n_inc(algo)):
            y = np.asfortranarray(_increment(s, k, algo)[..., rank * bl:(rank + 1) * bl])
            if k == 0:
                tt, rep = tt_ice_bootstrap(y, s.eps, ctx=ctx)
            elif algo == "ice":
                tt, rep = tt_ice_update(tt, y, s.eps)
            else:
                tt, rep = tt_ice_star_update(tt, y, s.eps)
            reps.append((list(rep.ranks_after), rep.obs_used, rep.batch_rel_error_estimate))
        if rank == 0:
            q.put(("ok", reps, [np.array(c) for c in tt.cores()], tt.ortho_count, tt.batch_boundaries()))
        tt.close()
        ctx.close()
    except Exception as e:  # report instead of hanging the parent
        q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo,world", [("ice", 2), ("star", 2), ("star", 4), ("star_skew", 2), ("boot", 2),
                                        ("boot", 4)])
def test_ranks_on_one_gpu_match_unsharded_oracle(algo, world):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ttstream_oracle as O
    from paper_2211_12487_b200.streams import Stream
    from tests.parity_util import REF, TOL, compare_reconstructions, compare_trains, estimates_agree

    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, algo, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert res[0] == "ok", res
    _, reps, cores, ortho, bounds = res
    s = Stream(3, seed=5, modes=(6,) * 4, batch=16, true_rank=5)
    ys = [_increment(s, k, algo) for k in range(_n_inc(algo))]
    tr, rr = REF.tt_ice_bootstrap(ys[0], s.eps)
    ref = [rr]
    for y in ys[1:]:
        tr, rr = (REF.tt_ice_update if algo == "ice" else REF.tt_ice_star_update)(tr, y, s.eps)
        ref.append(rr)
    for (ranks, used, est), r in zip(reps, ref):
        assert ranks == list(r.ranks_after)
        assert used == r.obs_used
        assert estimates_agree(est, r.batch_rel_error_estimate, pythagoras=(algo != "ice" or r.increment_index == 0))
    if algo == "star_skew":  # the skew really happened: half the batch drove the update
        assert any(used == s.batch // 2 for _, used, _ in reps[1:])
    tg = O.TensorTrain([O.TTCore(np.asfortranarray(c)) for c in cores], ortho, bounds)
    compare_trains(tg, tr)
    compare_reconstructions(tg, tr, list(enumerate(ys)))
    for p in procs:
        assert p.exitcode == 0


def _mismatch_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2211_12487_b200 import Context, DimensionError, tt_ice_bootstrap
        from paper_2211_12487_b200.streams import Stream

        ctx = Context.with_host_collectives(0, rank, world, lambda a: dist.all_reduce(torch.from_numpy(a)),
                                            lambda b: b)
        y = np.asfortranarray(Stream(3, seed=5, modes=(6,) * 4, batch=8 + 2 * rank, true_rank=5).increment(0))
        try:
            tt_ice_bootstrap(y, 0.01, ctx=ctx)
            q.put((rank, "no error"))
        except DimensionError as e:
            q.put((rank, str(e)))
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_unequal_shard_sizes_rejected_on_every_rank():
    """Shard sizes ride on the |Y|^2 all-reduce (global_obs): unequal per-rank
    batches raise DimensionError on EVERY rank before anything is mutated (no
    rank continues into collectives the others skip)."""
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_mismatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    assert set(got) == {0, 1}
    for r in (0, 1):
        assert "same batch shard size" in got[r], got


@pytest.mark.parametrize("algo", ["ice", "star"])
def test_nccl_transport_single_rank_matches_oracle(algo):
    """The production NCCL transport (ttg_ctx_create_dist, ttg.cu allreduce_sum /
    allgather) on a one-rank communicator: every exchange step of the multi-GPU
    path runs through ncclAllReduce / ncclAllGather (an NCCL context always
    takes them, world 1 included) with PDL off as on N > 1 GPUs.  Ranks after
    every increment identical to the oracle, subspaces / reconstructions /
    estimates within 1e-10."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ttstream_oracle as O
    from paper_2211_12487_b200 import Context, tt_ice_bootstrap, tt_ice_star_update, tt_ice_update
    from paper_2211_12487_b200.streams import Stream
    from tests.parity_util import REF, TOL, compare_reconstructions, compare_trains, estimates_agree

    ctx = Context(0, rank=0, world=1, nccl_id=Context.nccl_unique_id())
    assert ctx.world == 1 and ctx.rank == 0
    s = Stream(3, seed=5, modes=(6,) * 4, batch=16, true_rank=5)
    ys = [s.increment(k) for k in range(N_INC)]
    tt, rep = tt_ice_bootstrap(ys[0], s.eps, ctx=ctx)
    tr, rr = REF.tt_ice_bootstrap(ys[0], s.eps)
    pairs = [(rep, rr)]
    for y in ys[1:]:
        tt, rep = (tt_ice_update if algo == "ice" else tt_ice_star_update)(tt, y, s.eps)
        tr, rr = (REF.tt_ice_update if algo == "ice" else REF.tt_ice_star_update)(tr, y, s.eps)
        pairs.append((rep, rr))
    for rg, r in pairs:
        assert list(rg.ranks_after) == list(r.ranks_after)
        assert rg.obs_used == r.obs_used
        assert estimates_agree(rg.batch_rel_error_estimate, r.batch_rel_error_estimate,
                               pythagoras=(algo != "ice" or r.increment_index == 0))
    tg = O.TensorTrain([O.TTCore(np.asfortranarray(c)) for c in tt.cores()], tt.ortho_count, tt.batch_boundaries())
    compare_trains(tg, tr)
    compare_reconstructions(tg, tr, list(enumerate(ys)))
    tt.close()
    ctx.close()
