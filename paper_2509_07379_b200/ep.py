"""Expert parallelism: the M experts of every layer are
sharded over G ranks (rank r owns experts e with e % G == r); each rank holds
only its shard in pinned host memory, its own `slot_count` HBM cache and its
own copy stream / link, so the aggregate host-link bandwidth grows with G.

Attention, norms and the gate stay replicated (batch-1 serving: every rank
sees the same tokens, and the deterministic kernels give the same routing on
every rank).  Each rank computes the routing-weighted sum of ITS selected
experts into an f32 partial [T, d]; one collective (NCCL over NVLink on B200;
gloo in the CPU tests) combines them — `combine="allreduce"` (one all-reduce)
or `combine="alltoall"` (the north star's all-to-all exchange: each rank
receives every rank's share of one 1/G slice of the partial through
all_to_all_single, sums the G contributions in rank order and the slices are
all-gathered back, i.e. reduce-scatter + all-gather spelt with all-to-all).  With top-k = 2 at most two ranks hold a
non-zero term per element and adding exact zeros is exact, so the EP result is
bit-identical to the single-GPU result (tests/test_ep.py).

The reference is single-GPU by design; this is
the scaling extension named in BASELINE.json's north star.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


def owner(expert: int, world: int) -> int:
    return expert % world


def owned_experts(M: int, rank: int, world: int) -> list:
    return [e for e in range(M) if owner(e, world) == rank]


def owner_mask(M: int, rank: int, world: int) -> int:
    m = 0
    for e in owned_experts(M, rank, world):
        m |= 1 << e
    return m


def shard_fetch(fetch: list, rank: int, world: int) -> list:
    """The part of a (single-GPU) fetch list this rank performs."""
    return [e for e in fetch if owner(e, world) == rank]


def shard_log(log: list, rank: int, world: int) -> list:
    """Restrict a single-GPU cache log to the transfers owned by `rank`:
    prefill fetch lists, decode on-demand fetches, predictions and re-fetches
    are filtered by ownership; the gate sets stay whole (replicated routing)."""
    out = []
    for r in log:
        r = dict(r)
        for key in ("fetch", "pred", "refetch"):
            if key in r:
                r[key] = shard_fetch(r[key], rank, world)
        out.append(r)
    return out


@dataclass
class EPConfig:
    rank: int
    world: int
    group: object = None          # torch.distributed ProcessGroup (None = default group)
    combine: str = "allreduce"    # "allreduce" | "alltoall"

    @classmethod
    def from_env(cls, combine: str = "allreduce") -> "EPConfig | None":
        import torch.distributed as dist
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
            return None
        return cls(dist.get_rank(), dist.get_world_size(), None, combine)

    def combine_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum of the ranks' partials with the configured collective."""
        if self.combine == "alltoall":
            return self.all_to_all_combine_(t)
        if self.combine != "allreduce":
            raise ValueError(f"unknown EP combine {self.combine!r}")
        return self.all_reduce_(t)

    def all_to_all_combine_(self, t: torch.Tensor) -> torch.Tensor:
        """Sum of the ranks' partials via all-to-all: slice j of every rank's
        partial goes to rank j, which adds the G slices in rank order, then the
        summed slices are all-gathered.  Per element at most k ranks hold a
        non-zero term, so this equals the all-reduce bit for bit."""
        import torch.distributed as dist
        G = self.world
        flat = t.reshape(-1)
        n = flat.numel()
        c = (n + G - 1) // G
        dev = t.device
        stage = t.is_cuda and dist.get_backend(self.group) == "gloo"
        send = torch.zeros(G * c, dtype=t.dtype, device="cpu" if stage else dev)
        send[:n].copy_(flat)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        parts = recv.view(G, c)
        mine = parts[0].clone()
        for j in range(1, G):
            mine += parts[j]
        if dist.get_backend(self.group) == "gloo":
            chunks = [torch.empty_like(mine) for _ in range(G)]
            dist.all_gather(chunks, mine, group=self.group)
            out = torch.cat(chunks)
        else:
            out = torch.empty(G * c, dtype=t.dtype, device=mine.device)
            dist.all_gather_into_tensor(out, mine, group=self.group)
        flat.copy_(out[:n])
        return t

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place SUM all-reduce (NCCL over NVLink for CUDA tensors; a gloo
        group stages CUDA tensors through host memory)."""
        import torch.distributed as dist
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def owns(self, expert: int) -> bool:
        return owner(expert, self.world) == self.rank
