"""Replica ranks on one node share ONE pinned copy of the expert store
(engine._shared_pinned: a memfd created by rank 0, mapped by every rank);
world_size 2 on CPU (gloo) — the pinning (cudaHostRegister) needs a GPU and is
skipped here."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_07379_b200.engine import _shared_pinned
    t, creator = _shared_pinned((3, 2, 1000), dist.group.WORLD)
    if creator:
        t.copy_(torch.arange(6000, dtype=torch.int64).remainder(251).to(torch.uint8).view(3, 2, 1000))
    dist.barrier()
    ok = bool(torch.equal(t.flatten().long(), torch.arange(6000).remainder(251)))
    q.put((rank, creator, ok, t.data_ptr() != 0))
    dist.barrier()
    dist.destroy_process_group()


def test_shared_store_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, False]
    assert all(r[2] for r in res), res
