"""Expert parallelism host logic, world_size 2 on CPU (gloo):
ownership partition, sharded fetch logs, and the all-reduce combine being
bit-identical to the single-GPU combine."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import routing_ref, sim_ref
from paper_2509_07379_b200 import ep as EP


def test_ownership_partition():
    for world in (1, 2, 4, 8):
        shards = [EP.owned_experts(8, r, world) for r in range(world)]
        assert sorted(sum(shards, [])) == list(range(8))
        assert all(EP.owner_mask(8, r, world) == sum(1 << e for e in shards[r]) for r in range(world))


def test_sharded_logs_cover_single_gpu_log():
    rng = np.random.default_rng(0)
    L, M = 4, 8
    paths = [tuple(tuple(sorted(rng.choice(M, 2, replace=False).tolist())) for _ in range(L)) for _ in range(6)]
    preds = [[None] + [tuple(sorted(rng.choice(M, 2, replace=False).tolist())) for _ in range(L - 1)] for _ in paths]
    full, cnt = sim_ref.cache_log_decode(paths, preds, L)
    for world in (2, 4):
        per = [sim_ref.cache_log_decode(paths, preds, L, owned=EP.owned_experts(M, r, world)) for r in range(world)]
        for i, rec in enumerate(full):
            for key in ("fetch", "pred", "refetch"):
                if key in rec:
                    assert sorted(sum((p[0][i][key] for p in per), [])) == rec[key]
        assert sum(p[1]["prefetch_misses"] for p in per) == cnt["prefetch_misses"]
        assert EP.shard_log(full, 1, world)[1]["gate"] == full[1]["gate"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = EP.EPConfig.from_env()
    g = torch.Generator().manual_seed(0)
    T, k, M, d = 37, 2, 8, 64
    idx = torch.stack([torch.randperm(M, generator=g)[:k].sort().values for _ in range(T)]).to(torch.int32)
    w = torch.rand((T, k), generator=g)
    y = torch.randn((T * k, d), generator=g)             # expert outputs (any rank could compute any)
    _, pos, _ = routing_ref.permute(idx.numpy(), M)
    pos = torch.from_numpy(pos).long().view(T, k)
    part = torch.zeros((T, d))
    for j in range(k):
        own = torch.tensor([cfg.owns(int(e)) for e in idx[:, j]])
        part = part + torch.where(own[:, None], w[:, j:j + 1] * y[pos[:, j]], torch.zeros(()))
    part2 = part.clone()
    cfg.all_reduce_(part)
    cfg.all_to_all_combine_(part2)
    full = torch.zeros((T, d))
    for j in range(k):
        full = full + w[:, j:j + 1] * y[pos[:, j]]
    q.put((rank, bool(torch.equal(part, full)) and bool(torch.equal(part2, full))))
    dist.destroy_process_group()


def test_all_reduce_and_all_to_all_combine_bit_identical_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _dispatch_worker(rank, world, port, q):
    """Tokens partitioned over the ranks, experts sharded: dispatch rows to the
    owners over all_to_all, compute there, return and combine — equal to one
    process computing everything (integer-valued data, so f32 sums are exact
    and row-independent)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = EP.EPConfig.from_env()
    g = torch.Generator().manual_seed(0)
    B_tok, k, M, d = 29, 2, 8, 32
    a_all = torch.randint(-4, 5, (B_tok * world, d), generator=g).to(torch.bfloat16)
    idx_all = torch.stack([torch.randperm(M, generator=g)[:k].sort().values for _ in range(B_tok * world)])
    w_all = torch.randint(1, 4, (B_tok * world, k), generator=g).float() / 4
    h_all = torch.randint(-8, 9, (B_tok * world, d), generator=g).to(torch.bfloat16)
    W = torch.randint(-2, 3, (M, d, d), generator=g).float()

    def ffn(e, rows):
        return rows.float() @ W[e]

    mine = slice(rank * B_tok, (rank + 1) * B_tok)
    out, st = EP.dispatch_combine(a_all[mine], idx_all[mine].to(torch.int32), w_all[mine], h_all[mine], cfg, ffn, M)
    ref = torch.zeros((B_tok, d))
    for j in range(k):
        for t in range(B_tok):
            tt = rank * B_tok + t
            ref[t] += w_all[tt, j] * ffn(int(idx_all[tt, j]), a_all[tt:tt + 1])[0]
    ref = (h_all[mine].float() + ref).to(torch.bfloat16)
    ok = bool(torch.equal(out, ref)) and all(EP.owner(e, world) == rank for e in st["experts_run"])
    ok = ok and sum(st["sent_rows"]) == B_tok * k
    q.put((rank, ok, st["recv_rows"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_token_dispatch_all_to_all(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dispatch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def test_all_reduce_and_all_to_all_combine_bit_identical_world4():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
