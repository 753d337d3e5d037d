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


# ---------------------------------------------------------------------------
# Token dispatch / combine over all-to-all ("NCCL all-to-all
# dispatch of permuted rows ... plus an all-to-all combine").  For batch > 1
# the tokens are partitioned over the ranks (each rank owns some sequences,
# their attention and KV cache) and the experts are sharded by `owner`:
#
#   1. every rank groups its (token, slot) rows by destination rank (the
#      owner of the selected expert), stable in (expert, token, slot) order;
#   2. all_to_all_single exchanges the row counts, then the bf16 rows and
#      their expert ids (variable splits);
#   3. each owner runs its experts on the received rows, grouped by expert
#      (`ffn(expert, rows) -> f32 outputs`, the caller's K3/K4 launch);
#   4. a second all_to_all_single returns the outputs in the received order;
#   5. the source combines out[t] = h[t] + sum_j w[t, j] * y[t, j] in slot
#      order j — the single-GPU combine, so the result is bit-identical to one
#      rank computing every expert (given an ffn whose rows are independent).

def _exchange(send: torch.Tensor, send_counts: list, group) -> tuple:
    """Variable-split all_to_all_single of the rows of `send` (grouped by
    destination); returns (received rows, receive counts)."""
    import torch.distributed as dist
    G = len(send_counts)
    dev = send.device
    cnt = torch.tensor(send_counts, dtype=torch.int64)
    rcnt = torch.empty(G, dtype=torch.int64)
    stage = dist.get_backend(group) == "gloo"
    if stage:
        dist.all_to_all_single(rcnt, cnt, group=group)
    else:
        c_d, r_d = cnt.to(dev), rcnt.to(dev)
        dist.all_to_all_single(r_d, c_d, group=group)
        rcnt = r_d.cpu()
    recv_counts = [int(c) for c in rcnt.tolist()]
    width = send.shape[1:]
    src = send.cpu() if (stage and send.is_cuda) else send
    recv = torch.empty((sum(recv_counts), *width), dtype=send.dtype, device=src.device)
    dist.all_to_all_single(recv, src.contiguous(), output_split_sizes=recv_counts, input_split_sizes=send_counts,
                           group=group)
    return (recv.to(dev) if recv.device != dev else recv), recv_counts


def dispatch_combine(a: torch.Tensor, idx: torch.Tensor, w: torch.Tensor, resid: torch.Tensor, cfg: "EPConfig",
                     ffn, M: int) -> tuple:
    """One MoE layer with token dispatch: a [T, d] (bf16) normed activations
    of THIS rank's tokens, idx / w [T, k] their routing, resid [T, d] the
    residual.  ffn(expert, rows [n, d] bf16) -> [n, d] f32 for an expert this
    rank owns.  Returns (out [T, d] bf16 = resid + sum_j w_j y_j, stats)."""
    G, rank = cfg.world, cfg.rank
    T, k = idx.shape
    d = a.shape[1]
    dev = a.device
    idx_l = idx.to(torch.int64).cpu()
    flat_e = idx_l.reshape(-1)                                   # row r = (token r // k, slot r % k)
    dest = flat_e % G
    # stable order: destination, then expert, then (token, slot)
    key = (dest * M + flat_e) * (T * k) + torch.arange(T * k)
    order = torch.argsort(key)
    send_counts = [int((dest == g).sum()) for g in range(G)]
    rows = a.reshape(T, 1, d).expand(T, k, d).reshape(T * k, d)[order.to(dev)]
    ids = flat_e[order].to(torch.int32).reshape(-1, 1)
    recv_rows, recv_counts = _exchange(rows, send_counts, cfg.group)
    recv_ids, _ = _exchange(ids.to(dev) if dev.type == "cuda" and not _gloo(cfg) else ids, send_counts, cfg.group)
    recv_ids = recv_ids.reshape(-1).cpu()
    y = torch.empty((recv_rows.shape[0], d), dtype=torch.float32, device=dev)
    experts = sorted(set(recv_ids.tolist()))
    for e in experts:
        if owner(e, G) != rank:
            raise RuntimeError(f"rank {rank} received rows for expert {e} it does not own")
        sel = torch.nonzero(recv_ids == e).reshape(-1).to(dev)
        y[sel] = ffn(e, recv_rows[sel])
    back, _ = _exchange(y, recv_counts, cfg.group)              # outputs return in the sent order
    y_rows = torch.empty((T * k, d), dtype=torch.float32, device=dev)
    y_rows[order.to(dev)] = back
    y_tk = y_rows.view(T, k, d)
    acc = torch.zeros((T, d), dtype=torch.float32, device=dev)
    wf = w.to(torch.float32)
    for j in range(k):
        acc = acc + wf[:, j:j + 1] * y_tk[:, j]
    out = (resid.float() + acc).to(torch.bfloat16)
    return out, {"sent_rows": send_counts, "recv_rows": recv_counts, "experts_run": experts}


def _gloo(cfg: "EPConfig") -> bool:
    import torch.distributed as dist
    return dist.get_backend(cfg.group) == "gloo"
