"""NUMA placement helpers (paper_2509_07379_b200/numa.py) and the per-socket
replica store sharing, world_size 4 on CPU (gloo): ranks are grouped by
(host, PID namespace, NUMA node); each group shares one memfd store, a group
of one rank keeps a private store."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_07379_b200 import numa


def test_parse_cpulist():
    assert numa.parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert numa.parse_cpulist("") == []


def test_bind_without_gpu_is_a_noop_or_valid():
    info = numa.bind_to_gpu_node(0)
    assert info["gpu"] == 0 and isinstance(info["node"], int)
    assert os.sched_getaffinity(0)


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
    # pretend ranks 0,1 sit on node 0, rank 2 on node 1 and rank 3 on node 1 of another host
    keys = {0: ("h", "ns", 0), 1: ("h", "ns", 0), 2: ("h", "ns", 1), 3: ("h2", "ns", 1)}
    grp, members = numa.store_sharing_group(0, key=keys[rank])
    res = {"members": members}
    if len(members) > 1:
        t, creator = _shared_pinned((2, 3, 500), grp)
        if creator:
            t.copy_((torch.arange(3000) * (rank + 3)).remainder(251).to(torch.uint8).view(2, 3, 500))
        dist.barrier(group=grp)
        res["creator"] = creator
        res["ok"] = bool(torch.equal(t.flatten().long(), (torch.arange(3000) * (members[0] + 3)).remainder(251)))
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_store_sharing_groups_world4():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0]["members"] == [0, 1] and res[1]["members"] == [0, 1]
    assert res[2]["members"] == [2] and res[3]["members"] == [3]
    assert res[0]["creator"] and not res[1]["creator"]
    assert res[0]["ok"] and res[1]["ok"]
    assert "ok" not in res[2] and "ok" not in res[3]
