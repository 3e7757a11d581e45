"""CPU, world_size 2 over gloo: the multi-GPU exchange plan of DESIGN.md §5
(batch-axis shards; all-reduce of |Y|^2, of each mode's residual Gram and of
the TT-ICE* decision sums; identical eigen-solve on every rank; all-gather of
the coefficient columns) reproduces the unsharded reference algorithm
(oracle) — ranks identical, subspaces / reconstructions within 1e-10.

The GPU path implements exactly these exchange points with NCCL (ttg.cu:
allreduce_sum / ncclAllGather); this test pins the decomposition itself on
CPU, where several ranks can run.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ttstream_oracle as O
from paper_2211_12487_b200.streams import Stream


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _gram_eig_rank(G, delta, kmax):
    lam, V = np.linalg.eigh(G)
    order = np.argsort(-lam, kind="stable")
    lam, V = lam[order], V[:, order]
    lam = np.maximum(lam, 0.0)
    tail, rank = 0.0, min(kmax, len(lam))
    for j in range(rank - 1, -1, -1):
        nxt = tail + lam[j]
        if math.sqrt(nxt) > delta:
            break
        tail, rank = nxt, j
    U = V[:, :rank].copy()
    for j in range(rank):  # sign rule (truncated_svd.cpp:16-25)
        i = int(np.argmax(np.abs(U[:, j])))
        if U[i, j] < 0:
            U[:, j] = -U[:, j]
    return U, rank, tail


def sharded_tt_ice_update(tt: O.TensorTrain, y_local: np.ndarray, eps: float, world: int):
    d = tt.spatial_dims()
    b_local = y_local.shape[-1]
    ysq = float(_allreduce(np.array([np.sum(y_local * y_local)]))[0])
    delta = eps * math.sqrt(ysq) / math.sqrt(d)
    cur = np.reshape(y_local, (y_local.shape[0], -1), order="F")
    u_pad = tt.core(0).left_unfolding()
    r_left = 1
    new_cores = []
    disc = 0.0
    for i in range(d):
        r_old = u_pad.shape[1]
        R = O.compute_residual(u_pad, cur)
        G = _allreduce(R @ R.T)  # <- the per-mode exchange
        U_R, r_R, tail = _gram_eig_rank(G, delta, kmax=cur.shape[1] * world)
        disc += tail
        u_new = O.append_directions(u_pad, U_R) if r_R > 0 else u_pad
        r_new = u_new.shape[1]
        new_cores.append(O.TTCore.from_left_unfolding(u_new, r_left, tt.core(i).n))
        proj = u_new.T @ cur
        if i + 1 < d:
            u_pad = O.pad_core(tt.core(i + 1).left_unfolding(), r_old, r_new - r_old)
            rows = r_new * tt.core(i + 1).n
            cur = np.reshape(proj, (rows, -1), order="F")
        else:
            cur = proj
        r_left = r_new
    gathered = [torch.zeros(cur.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(cur)))  # <- coefficient columns
    coeffs = np.concatenate([g.numpy() for g in gathered], axis=1)
    last = tt.core(d)
    new_last = np.zeros((r_left, last.n + coeffs.shape[1]))
    new_last[:last.r_left, :last.n] = last.right_unfolding()
    new_last[:, last.n:] = coeffs
    new_cores.append(O.TTCore.from_right_unfolding(new_last, last.n + coeffs.shape[1], 1))
    out = O.TensorTrain(new_cores, d, list(tt.batch_boundaries) + [last.n + coeffs.shape[1]])
    return out, math.sqrt(disc) / math.sqrt(ysq)


def sharded_star_sums(tt, y_local, eps):
    """The 9 TT-ICE* decision sums of k_star_local, all-reduced (ttg_misc.cuh)."""
    st = O.per_obs_stats(tt, y_local)
    s = np.zeros(9)
    for e, rn, on in zip(st.errs, st.resid_norms, st.obs_norms):
        if on > 0:
            s[0] += e
            s[1] += 1
        s[2] += rn * rn
        s[3] += on * on
        if e > eps:
            s[5] += on * on
            s[6] += 1
        else:
            s[4] += (e * on) ** 2
            s[7] += 1
            s[8] += e
    return _allreduce(s)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = Stream(3, seed=5, modes=(4,) * 5, batch=8, true_rank=4)
        ys = [s.increment(k) for k in range(5)]
        shard = lambda y: np.asfortranarray(y[..., rank * 4:(rank + 1) * 4])  # noqa: E731
        tt, _ = O.tt_ice_bootstrap(ys[0], s.eps)  # bootstrap replicated
        ref = tt
        out = []
        for k in range(1, 5):
            sums = sharded_star_sums(tt, shard(ys[k]), s.eps)
            st_full = O.per_obs_stats(ref, ys[k])
            tt, est = sharded_tt_ice_update(tt, shard(ys[k]), s.eps, world)
            ref, rr = O.tt_ice_update(ref, ys[k], s.eps)
            dsub = max(float(np.linalg.norm(pg - pr @ (pr.T @ pg)))
                       for pg, pr in zip(O.interface_projectors(tt), O.interface_projectors(ref)))
            rec = float(np.linalg.norm(O.tt_reconstruct(tt) - O.tt_reconstruct(ref)) /
                        np.linalg.norm(O.tt_reconstruct(ref)))
            mean_full = float(np.mean(st_full.errs))
            out.append((tt.ranks(), ref.ranks(), dsub, rec, abs(est - rr.batch_rel_error_estimate),
                        abs(sums[0] / sums[1] - mean_full), sums[6], int(np.sum(st_full.errs > s.eps))))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_update_matches_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        for ranks_g, ranks_r, dsub, rec, dest, dmean, nsel, nsel_ref in results[rank]:
            assert ranks_g == ranks_r
            assert dsub <= 1e-10
            assert rec <= 1e-10
            assert dest <= 1e-10
            assert dmean <= 1e-12
            assert int(nsel) == nsel_ref
    assert results[0] == results[1] or all(a[0] == b[0] for a, b in zip(results[0], results[1]))
