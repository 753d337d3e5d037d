"""DuoServe-MoE inference runtime on one B200: expert store, HBM expert
cache and the prefill / decode expert schedules (cache
semantics SPEC.md:340-438, restated in oracle/sim_ref.py).

  HostExpertStore   all L x M W4 experts in pinned host memory (the "CPU
                    expert cache"), kernel-ready bytes: one
                    contiguous blob per expert, one H2D copy per fetch.
  ExpertCache       slot_count(policy) fixed slots in HBM (config.py:101-114),
                    a dedicated copy stream, per-slot ready/free cudaEvents,
                    and the fetch log that must equal the oracle's.
  Engine            prefill(ids) / decode_step() — the reference-facing serving
                    API.  Compute stream: attention, K1 gate, K2 permute,
                    K3/K4 expert FFN, combine.  Copy stream: expert H2D.
                    Predict stream: K5 predictor for layer l+1.

Schedules (policy "duoserve"):
  prefill, per layer l  the copy stream speculatively fetches expert 0 of
      layer l while attention runs (the first transfer overlaps the non-MoE
      compute); after the gate + permute the activated set A_l
      is read back and the rest of A_l is fetched ascending, each expert once,
      into a ring of slots — the compute stream runs expert e_i's grouped FFN
      (K3) as soon as its copy event fires while e_{i+1} streams in.
  decode, per token     layer 0 fetches after the gate; for l >= 1 the
      prediction P_l made during layer l-1 was prefetched; sync point 1
      compares the gate set E_l with P_l and re-fetches only the wrong slots;
      the predictor for l+1 runs on its own stream as soon as E_l is in the
      device history buffer; sync point 2 issues the prefetch of P_{l+1} into
      the two slots released by layer l-1.
Policy "oracle" replays a recorded routing as the prediction (the SPEC's
DuoServeOracle); "ondemand" fetches after the gate (ACC baseline);
"prefetchall" (MoESys baseline) streams all M experts of
every layer visit into one of two banks of M slots, the next visit's bank
filling while the current one computes.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .config import ModelShape, SchedulerPolicy, model_config_for_shape, slot_count
from .model import (DenseWeights, KVCache, KVCacheBatch, attention_block, attention_block_batch,
                    attention_decode_static, attention_decode_static_batch, decode_front_fused, init_dense_weights,
                    logits_last,
                    rms_norm, rope_tables)
from .ep import EPConfig, owned_experts, owner_mask
from .predictor import ExpertMLP, StatsOnDevice, _mode_code
from .stats import OnlineRoutingStats


class HostExpertStore:
    """Pinned host memory holding every expert blob: [L, M, blob_bytes] u8."""

    def __init__(self, shape: ModelShape, seed: int, device, layers: int | None = None, experts=None,
                 shared_group=None):
        """experts: the expert ids this process stores (expert parallelism);
        default all M.  Non-owned experts are never allocated.

        shared_group: a torch.distributed group of ranks on this node serving
        replicas of the same model: they share ONE copy of the store (an
        anonymous memfd mapped by every rank and pinned with cudaHostRegister),
        so host memory holds the 23.4 GB (8x7B) once, not once per GPU."""
        self.shape = shape
        self.seed = seed
        L = layers if layers is not None else shape.num_layers
        self.offsets, self.blob_bytes = ops.expert_layout(shape.hidden, shape.ffn, shape.group_size)
        self.experts = list(range(shape.num_experts)) if experts is None else sorted(experts)
        self.local = {e: i for i, e in enumerate(self.experts)}
        t0 = time.time()
        shape3 = (L, len(self.experts), self.blob_bytes)
        fill = True
        self._registered = None
        self.data = None
        if shared_group is not None:
            self.data, fill = _shared_pinned(shape3, shared_group)
            if self.data is None:                     # ranks cannot share: private store each
                shared_group, fill = None, True
            else:
                self._registered = self.data
        if self.data is None:
            self.data = torch.empty(shape3, dtype=torch.uint8, pin_memory=True)
        self.shared = shared_group is not None
        self.alloc_s = time.time() - t0
        if not fill:                                  # another rank generates the bytes
            import torch.distributed as dist
            dist.barrier(group=shared_group)
            self.fill_s = 0.0
            return
        # generate on the device (counter-based, bit-identical to oracle/w4_ref.py) then D2H
        t0 = time.time()
        stage = [torch.empty(self.blob_bytes, dtype=torch.uint8, device=device) for _ in range(2)]
        s = torch.cuda.current_stream(device)
        for l in range(L):
            for i, e in enumerate(self.experts):
                buf = stage[(l * len(self.experts) + i) % 2]
                ops.w4_generate(seed, l, e, shape.hidden, shape.ffn, shape.group_size, buf)
                self.data[l, i].copy_(buf, non_blocking=True)
        s.synchronize()
        self.fill_s = time.time() - t0
        if shared_group is not None:
            import torch.distributed as dist
            dist.barrier(group=shared_group)             # the bytes are in place for every rank

    def blob(self, layer: int, expert: int) -> torch.Tensor:
        return self.data[layer, self.local[expert]]

    def close(self) -> None:
        """Unpin a shared (cudaHostRegister'd) mapping; private stores are
        cudaHostAlloc memory freed with the tensor."""
        if self._registered is not None:
            _unregister(self._registered)
            self._registered = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def nbytes(self) -> int:
        return self.data.numel()


def _shared_pinned(shape3: tuple, group) -> tuple:
    """(u8 host tensor of shape3 shared by all ranks of `group`, is_creator),
    or (None, False) on every rank when the ranks cannot share.

    `group` must hold ranks of one host and one PID namespace (see
    numa.store_sharing_group): rank 0 of the group creates an anonymous memfd,
    the others map it through /proc/<pid>/fd.  If any rank fails to open the
    path (another host or PID namespace) every rank falls back to a private
    store.  Every rank pins its mapping with cudaHostRegister (a registered
    mapping is DMA-able like cudaHostAlloc memory); release it with
    _unregister."""
    import os
    import torch.distributed as dist
    nbytes = 1
    for v in shape3:
        nbytes *= int(v)
    rank = dist.get_rank(group)
    fd = None
    path = [None]
    if rank == 0:
        fd = os.memfd_create("duoserve-expert-store", 0)
        os.ftruncate(fd, nbytes)
        path[0] = f"/proc/{os.getpid()}/fd/{fd}"
    dist.broadcast_object_list(path, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    flat, ok = None, 1
    try:
        flat = torch.from_file(path[0], shared=True, size=nbytes, dtype=torch.uint8)
    except (RuntimeError, OSError):
        ok = 0
    okt = torch.tensor([ok], dtype=torch.int64)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN, group=group)       # every rank holds a mapping?
    if fd is not None:
        os.close(fd)
    if int(okt) == 0:
        return None, False
    if torch.cuda.is_available():
        rc = torch.cuda.cudart().cudaHostRegister(flat.data_ptr(), nbytes, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister of the shared expert store failed ({rc})")
    return flat.view(shape3), rank == 0


def _unregister(t: torch.Tensor) -> None:
    if t is not None and torch.cuda.is_available():
        torch.cuda.cudart().cudaHostUnregister(t.data_ptr())


class ExpertCache:
    """Fixed-capacity HBM expert slots fed by a dedicated copy stream."""

    def __init__(self, store: HostExpertStore, n_slots: int, device):
        self.store = store
        self.n_slots = n_slots
        self.device = device
        self.slots = torch.empty((n_slots, store.blob_bytes), dtype=torch.uint8, device=device)
        self.copy_stream = torch.cuda.Stream(device)
        self.ready = [torch.cuda.Event() for _ in range(n_slots)]
        self.free = [torch.cuda.Event() for _ in range(n_slots)]
        self.used = [False] * n_slots
        self.content = [None] * n_slots          # (layer, expert) resident or in flight
        self.bytes_copied = 0
        self.n_copies = 0
        self.trace = None                        # list of (ev0, ev1) timing pairs when tracing
        sh = store.shape
        self._structs = [ops.expert_struct(self.slots[i].data_ptr(), sh.hidden, sh.ffn, sh.group_size)
                         for i in range(n_slots)]

    @property
    def nbytes(self) -> int:
        return self.slots.numel()

    def load(self, slot: int, layer: int, expert: int) -> None:
        """Queue the H2D copy of expert (layer, expert) into slot (after its last use)."""
        with torch.cuda.stream(self.copy_stream):
            if self.used[slot]:
                self.copy_stream.wait_event(self.free[slot])
            if self.trace is not None:
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(self.copy_stream)
            self.slots[slot].copy_(self.store.blob(layer, expert), non_blocking=True)
            if self.trace is not None:
                t1.record(self.copy_stream)
                self.trace.append((t0, t1))
            self.ready[slot].record(self.copy_stream)
        self.content[slot] = (layer, expert)
        self.bytes_copied += self.store.blob_bytes
        self.n_copies += 1

    def acquire(self, slot: int) -> "object":
        """Make the current (compute) stream wait until the slot's copy landed."""
        torch.cuda.current_stream(self.device).wait_event(self.ready[slot])
        return self._structs[slot]

    def struct(self, slot: int) -> "object":
        """The slot's expert struct without a stream wait (the caller passes
        ready[slot] to a graph launch that waits on the device)."""
        return self._structs[slot]

    def release(self, slot: int) -> None:
        self.free[slot].record(torch.cuda.current_stream(self.device))
        self.used[slot] = True


class Transfer:
    __slots__ = ("slot", "layer", "expert", "ticket", "cancelled")

    def __init__(self, slot, layer, expert, ticket):
        self.slot, self.layer, self.expert, self.ticket = slot, layer, expert, ticket
        self.cancelled = False


class LinkQueue:
    """Decode-side view of the native expert link (csrc/link.cu, K6).

    Expert transfers are split into chunks and issued just in time by a C++
    scheduler thread (at most `depth` chunks queued on the copy engine), so a
    prefetch the gate proves wrong (sync point 1) is cancelled after its
    in-flight chunks instead of holding the link for the whole expert, and
    the link keeps streaming while the Python thread launches attention.
    With cancel=False and one chunk per expert it is exactly the paper's
    schedule (whole-expert prefetch, then blocking re-fetch)."""

    def __init__(self, cache: "ExpertCache", chunk_bytes: int, depth: int, cancel: bool,
                 spec_chunk_bytes: int = 2 << 20):
        import ctypes as C
        from . import _lib
        self.C, self.lib = C, _lib
        self.cache = cache
        blob = cache.store.blob_bytes
        self.chunk = blob if chunk_bytes <= 0 else min(chunk_bytes, blob)
        self.depth = depth
        self.cancel_enabled = cancel
        self.spec_chunk = min(self.chunk, spec_chunk_bytes)
        h = C.c_void_p()
        _lib.call("ds_link_create", C.c_void_p(cache.copy_stream.cuda_stream), self.chunk, depth, C.byref(h))
        self.handle = h
        # materialise the slot events so their raw handles can cross the ABI
        s = torch.cuda.current_stream(cache.device)
        for ev in cache.ready + cache.free:
            ev.record(s)
        s.synchronize()
        # raw handles resolved once: submit/promote/cancel sit between the gate
        # result and the miss transfer (the decode reaction window), so they
        # avoid per-call tensor indexing and name lookups
        self._slot_ptr = [C.c_void_p(t.data_ptr()) for t in cache.slots]
        self._ready_ev = [C.c_void_p(e.cuda_event) for e in cache.ready]
        self._free_ev = [C.c_void_p(e.cuda_event) for e in cache.free]
        st = cache.store.data
        self._store_base, self._store_s0, self._store_s1 = st.data_ptr(), st.stride(0), st.stride(1)
        lib = _lib.load()
        self._f_submit, self._f_submit_chunked = lib.ds_link_submit, lib.ds_link_submit_chunked
        self._f_promote, self._f_cancel = lib.ds_link_promote, lib.ds_link_cancel

    def _check(self, rc: int, name: str) -> None:
        if rc != 0:
            raise self.lib.DeviceError(name, rc, self.lib.load().ds_last_error().decode(errors="replace"))

    def close(self) -> None:
        """Stop the native scheduler thread (idempotent)."""
        if self.handle is not None:
            self.cache.copy_stream.synchronize()
            self.lib.call("ds_link_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def submit(self, slot: int, layer: int, expert: int, speculative: bool = False) -> Transfer:
        """Queue expert (layer, expert) into slot.  Speculative (predicted)
        transfers use small chunks until promote(), so cancelling leaves at
        most `depth` small chunks in flight."""
        c = self.cache
        C = self.C
        t = C.c_uint64()
        wait = self._free_ev[slot] if c.used[slot] else None
        src = self._store_base + layer * self._store_s0 + c.store.local[expert] * self._store_s1
        args = (self.handle, self._slot_ptr[slot], C.c_void_p(src), c.store.blob_bytes)
        if speculative and self.cancel_enabled and self.spec_chunk < self.chunk:
            self._check(self._f_submit_chunked(*args, self.spec_chunk, wait, self._ready_ev[slot], C.byref(t)),
                        "ds_link_submit_chunked")
        else:
            self._check(self._f_submit(*args, wait, self._ready_ev[slot], C.byref(t)), "ds_link_submit")
        c.content[slot] = (layer, expert)
        c.n_copies += 1
        return Transfer(slot, layer, expert, t.value)

    def promote(self, tr: Transfer) -> None:
        if self.cancel_enabled:
            self._check(self._f_promote(self.handle, tr.ticket), "ds_link_promote")

    def cancel(self, tr: Transfer) -> None:
        if not self.cancel_enabled:
            return
        tr.cancelled = True
        self._check(self._f_cancel(self.handle, tr.ticket, None), "ds_link_cancel")

    def flush(self, tr: Transfer) -> None:
        """Block until every chunk of tr has been issued (its ready event recorded)."""
        self.lib.call("ds_link_wait_issued", self.handle, tr.ticket)

    def wait_event(self, ev) -> None:
        ev.synchronize()

    def stats(self) -> dict:
        C = self.C
        a, b, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.call("ds_link_stats", self.handle, C.byref(a), C.byref(b), C.byref(n))
        return {"bytes_issued": a.value, "wasted_prefetch_bytes": b.value, "chunks": n.value}

    def reset_stats(self) -> None:
        self.lib.call("ds_link_reset_stats", self.handle)

    def set_trace(self, on: bool) -> None:
        self.lib.call("ds_link_trace", self.handle, int(on))

    def trace_read(self, ref_event) -> list:
        """Copy-busy (start, end) ms of the chunks issued since the last read, relative to ref_event."""
        C = self.C
        cap = 1 << 20
        a, b, n = (C.c_float * cap)(), (C.c_float * cap)(), C.c_size_t()
        self.lib.call("ds_link_trace_read", self.handle, C.c_void_p(ref_event.cuda_event), a, b, cap, C.byref(n))
        return [(a[i], b[i]) for i in range(n.value)]

    def set_chunk(self, chunk_bytes: int) -> None:
        """Recreate the native link with a new chunk size (idle link only)."""
        C = self.C
        self.cache.copy_stream.synchronize()
        self.lib.call("ds_link_destroy", self.handle)
        self.chunk = min(chunk_bytes, self.cache.store.blob_bytes)
        h = C.c_void_p()
        self.lib.call("ds_link_create", C.c_void_p(self.cache.copy_stream.cuda_stream), self.chunk, self.depth,
                      C.byref(h))
        self.handle = h


class MLPDriver:
    """K5 on the predict stream: P_{l+1} from the device history buffer."""

    def __init__(self, net: ExpertMLP, pop, aff, L: int, M: int, k: int, device, batch: int = 1):
        self.dev = net.device(device)
        self.stats = StatsOnDevice(pop, aff, device)
        self.mode = _mode_code(net.meta.get("affinity_mode", "pool"))
        self.L, self.M, self.k, self.B = L, M, k, batch
        self.stream = torch.cuda.Stream(device)
        self.targets = [torch.full((batch,), l, dtype=torch.int32, device=device) for l in range(L)]
        self.out = torch.empty((batch, k), dtype=torch.int32, device=device)
        self.probs = torch.empty((batch, M), dtype=torch.float64, device=device)
        self.host_out = torch.empty((batch, k), dtype=torch.int32, pin_memory=True)
        self.host_probs = torch.empty((batch, M), dtype=torch.float64, pin_memory=True)
        self.sets = None                 # per-sequence predicted sets of the last result()
        self.done = torch.cuda.Event()
        self.nbytes = self.dev.nbytes + self.stats.pop.nbytes + self.stats.aff.nbytes
        self.prof = None                 # KernelProfiler (set by the engine when profiling)
        import os
        # opt-in: a persisting L2 window over the 23.9 MB of weights measured no
        # gain (K5 in the loop 43.7 vs 44.5 us: bound by its 7 dependent layers,
        # not by bytes; profiles/r2/README.md)
        self.l2_persist = os.environ.get("DS_K5_L2PERSIST", "0") == "1"
        if self.l2_persist:              # the weights stay in L2 between the per-layer calls
            from . import _lib
            import ctypes as C
            try:
                _lib.call("ds_l2_persist_window", C.c_void_p(self.stream.cuda_stream),
                          C.c_void_p(self.dev.packed.data_ptr()), self.dev.packed.numel() * 8, 1.0)
            except Exception:
                self.l2_persist = False

    def launch(self, hist: torch.Tensor, after: torch.cuda.Event, target_layer: int) -> None:
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(after)
            timed = self.prof is not None
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
            self.dev.predict_state(hist, self.targets[target_layer], self.stats.pop, self.stats.aff, self.L,
                                   self.M, self.k, self.mode, self.k, out=self.out, probs=self.probs,
                                   stream=self.stream)
            if timed:
                e1.record(self.stream)
                self.prof.add("K5 predictor (fused f64 MLP)", e0, e1, self.dev.nbytes)
            self.host_out.copy_(self.out, non_blocking=True)
            self.host_probs.copy_(self.probs, non_blocking=True)
            self.done.record(self.stream)

    def result(self, link=None) -> tuple:
        """(sorted predicted set, transfer order = descending probability).
        With B sequences: the union of their sets, ordered by descending
        probability summed over the batch (ties: lower index); for B = 1 that
        is the single sequence's order."""
        if link is not None:
            link.wait_event(self.done)
        self.done.synchronize()
        rows = self.host_out.tolist()
        self.sets = [tuple(sorted(int(e) for e in r)) for r in rows]
        if self.B == 1:
            P = [int(e) for e in rows[0]]
            pr = self.host_probs[0].tolist()
            return P, sorted(P, key=lambda e: (-pr[e], e))
        P = sorted({e for r in self.sets for e in r})
        score = self.host_probs.sum(dim=0).tolist()
        return P, sorted(P, key=lambda e: (-score[e], e))


class TraceDriver:
    """Perfect predictor for policy 'oracle': replays recorded decode routing."""

    def __init__(self, paths):
        self.paths = paths     # paths[t][l] -> tuple
        self.t = 0
        self._next = None

    def launch(self, hist, after, target_layer: int) -> None:
        self._next = list(self.paths[self.t][target_layer])

    def result(self, link=None) -> tuple:
        return sorted(self._next), list(self._next)


@dataclass
class StepTiming:
    ms: float
    bytes_h2d: int


class Engine:
    """Reference-facing serving API: load -> prefill(ids) -> decode_step()*."""

    def __init__(self, shape: ModelShape, policy="duoserve", seed: int = 0, device="cuda",
                 dense: DenseWeights | None = None, store: HostExpertStore | None = None,
                 predictor: ExpertMLP | None = None, pop=None, aff=None, oracle_paths=None,
                 max_seq: int = 2048, max_prefill: int = 2048, cancel_mispredicted: bool = True,
                 chunk_mb: float = 256.0, link_depth: int = 2, use_graphs: bool = True,
                 ep: EPConfig | None = None, collect_stats: bool = False, spec_chunk_mb: float = 0.5,
                 pin_budget_bytes: int = 0):
        self.shape = shape
        self.policy = SchedulerPolicy(policy)
        self.device = torch.device(device)
        sh = shape
        self.L, self.M, self.k, self.d, self.ff, self.G = (sh.num_layers, sh.num_experts, sh.top_k, sh.hidden,
                                                           sh.ffn, sh.group_size)
        self.W = dense if dense is not None else init_dense_weights(sh, seed, device=self.device)
        if self.W.embed.device != self.device:
            self.W = self.W.to(self.device)
        self.ep = ep
        self.owned = owned_experts(sh.num_experts, ep.rank, ep.world) if ep else list(range(sh.num_experts))
        self.owned_set = set(self.owned)
        self.store = store if store is not None else HostExpertStore(sh, seed, self.device, experts=self.owned)
        cfg = model_config_for_shape(sh)
        self.B = getattr(self, "B", 1)           # sequences served together (BatchEngine sets B first)
        self.n_slots = self._slot_count(cfg)
        self.cache = ExpertCache(self.store, self.n_slots, self.device)
        self.cancel_mispredicted = cancel_mispredicted
        self.link = LinkQueue(self.cache, int(chunk_mb * 2**20) if cancel_mispredicted else 0,
                              link_depth if cancel_mispredicted else 2, cancel_mispredicted,
                              spec_chunk_bytes=int(spec_chunk_mb * 2**20))
        self.max_seq, self.max_prefill = int(max_seq), int(max_prefill)
        # K4 as one device-resident graph launch per expert (A/B: DS_K4_GRAPH=0)
        self.k4_graphs = os.environ.get("DS_K4_GRAPH", "1") != "0"
        self.front_fused = os.environ.get("DS_FRONT_FUSED", "1") != "0"
        self.kv = self._make_kv(max_seq)
        self.cos, self.sin = rope_tables(sh, max_seq, self.device)
        self.driver = None
        if self.policy is SchedulerPolicy.DUOSERVE:
            if predictor is None or pop is None or aff is None:
                raise ValueError("policy 'duoserve' needs predictor, pop and aff")
            self.driver = MLPDriver(predictor, pop, aff, self.L, self.M, self.k, self.device, batch=self.B)
        elif self.policy is SchedulerPolicy.DUOSERVE_ORACLE:
            if oracle_paths is None:
                raise ValueError("policy 'oracle' needs the recorded decode routing (oracle_paths)")
            self.driver = TraceDriver(oracle_paths)
        dev = self.device
        # residency-budget policy: the most popular experts
        # live in HBM for the whole request within the spare residency budget
        self.pinned = {}             # (layer, expert) -> W4Expert of an HBM-resident expert
        self._pinned_buf = None
        if pin_budget_bytes > 0:
            self.pin_experts(pop, int(pin_budget_bytes))
        # decode buffers (one row per sequence)
        B = self.B
        self.hist = torch.zeros((B, self.L * self.k), dtype=torch.int32, device=dev)
        self.idx1 = torch.empty((B, self.k), dtype=torch.int32, device=dev)
        self.w1 = torch.empty((B, self.k), dtype=torch.float32, device=dev)
        self.idx_host = torch.empty((B, self.k), dtype=torch.int32, pin_memory=True)
        self._idx_np = self.idx_host.numpy()        # same memory: read at sync point 1 without torch indexing
        self.h_buf = torch.empty((1, self.ff), dtype=torch.bfloat16, device=dev)
        self.acc = torch.zeros((1, self.d), dtype=torch.float32, device=dev)
        self.ev_gate = torch.cuda.Event()
        # prefill buffers
        P = max_prefill
        self.p_idx = torch.empty((P, self.k), dtype=torch.int32, device=dev)
        self.p_w = torch.empty((P, self.k), dtype=torch.float32, device=dev)
        self.p_off = torch.empty(self.M + 1, dtype=torch.int32, device=dev)
        self.p_off_host = torch.empty(self.M + 1, dtype=torch.int32, pin_memory=True)
        self.p_pos = torch.empty(P * self.k, dtype=torch.int32, device=dev)
        self.p_src = torch.empty(P * self.k, dtype=torch.int32, device=dev)
        self.p_xperm = torch.empty((P * self.k, self.d), dtype=torch.bfloat16, device=dev)
        self.p_h = torch.empty((P * self.k, self.ff), dtype=torch.bfloat16, device=dev)
        self.p_y = torch.empty((P * self.k, self.d), dtype=torch.float32, device=dev)
        self.owner_bits = owner_mask(self.M, ep.rank, ep.world) if ep else (1 << self.M) - 1
        self.p_part = torch.zeros((P, self.d), dtype=torch.float32, device=dev) if ep else None
        ws = max(ops.grouped_ffn_workspace(r, self.d, self.ff) for r in (P * self.k // 4, P * self.k))
        self.p_ws = torch.empty(max(ws, 256), dtype=torch.uint8, device=dev)
        self.prefill_idx_host = None
        # online routing statistics: device counters fed by the gate
        self.route_stats = OnlineRoutingStats(self.L, self.M, self.k, dev) if collect_stats else None
        self.p_paths = torch.empty((P, self.L, self.k), dtype=torch.int32, device=dev) if collect_stats else None
        self.capture = None          # debug/parity: list of (phase, layer, gate input, idx)
        self.capture_moe = None      # parity: set of layers whose MoE block in/out is recorded
        self.moe_records = []        # dicts: phase, layer, token, h_in, a, out, idx, w (host copies)
        self.use_graphs = use_graphs
        self.g_graphs = None
        self.prof = None             # KernelProfiler when enabled (bench)
        self.d2h_bytes = 0
        self._link_peak = None
        self.last_logits = None
        self.reset()

    def pin_experts(self, pop, budget: int) -> int:
        """Residency-budget policy: pin the (layer, expert) pairs with the
        highest popularity pop[l, e] (ties: lower layer, then lower expert)
        that fit in `budget` bytes.  They are copied once here, never streamed,
        and take no cache slot.  Replaces any earlier pin set (between
        requests only); returns the number of pinned experts."""
        from .preprocess import rank_popular
        if self.policy is SchedulerPolicy.PREFETCH_ALL:
            raise ValueError("pinning is not defined for 'prefetchall' (every expert is streamed by design)")
        if pop is None:
            raise ValueError("pin_budget_bytes needs the popularity matrix (pop)")
        self.pinned = {}
        self._pinned_buf = None
        n = min(max(int(budget), 0) // self.store.blob_bytes, self.L * len(self.owned))
        if n <= 0:
            return 0
        chosen = sorted(rank_popular(pop, self.owned)[:n])
        self._pinned_buf = torch.empty((n, self.store.blob_bytes), dtype=torch.uint8, device=self.device)
        for i, (l, e) in enumerate(chosen):
            self._pinned_buf[i].copy_(self.store.blob(l, e))
            self.pinned[(l, e)] = ops.expert_struct(self._pinned_buf[i].data_ptr(), self.d, self.ff, self.G)
        torch.cuda.synchronize(self.device)
        return n

    def _split_pinned(self, l: int, experts) -> tuple:
        """(streamed, pinned) experts of layer l, order kept."""
        if not self.pinned:
            return list(experts), []
        return [e for e in experts if (l, e) not in self.pinned], [e for e in experts if (l, e) in self.pinned]

    def _slot_count(self, cfg) -> int:
        return slot_count(self.policy, cfg)

    def _make_kv(self, max_seq: int):
        return KVCache(self.shape, max_seq, self.device)

    # ------------------------------------------------------------------ API
    def reset(self) -> None:
        if hasattr(self, "link"):
            self.link.reset_stats()
        self.kv.len = 0
        self.log: list = []
        self.paths_decode: list = []          # recorded routing per decode token
        self.paths_prefill = None
        self.token = None
        self.t_decode = 0
        self.cache.used = [False] * self.n_slots
        self.cache.content = [None] * self.n_slots
        self._spec = None                     # (slot, layer, expert) speculative prefill fetch
        self._ring = 0
        self._pred_next = None
        self._pa_v = 0                        # prefetchall: layer visits computed so far
        self._pa_queued = 0                   # prefetchall: layer visits queued on the copy stream
        self.hist.zero_()
        self.d2h_bytes = 0
        # host seconds blocked at sync points 1 / 2 (decode), and spent deciding
        # after sync point 1 (gate result -> the layer's transfers submitted)
        self.host_wait = {"sync1": 0.0, "sync2": 0.0, "decide": 0.0}
        if hasattr(self, "link"):
            self.cache.copy_stream.synchronize()

    def close(self) -> None:
        """Release the native link thread and the engine's device buffers.  The
        host expert store and the dense weights may be shared with another
        engine and are left alone (HostExpertStore.close unpins a shared store)."""
        torch.cuda.synchronize(self.device)
        self.link.close()
        self.g_graphs = None
        ops.w4_graph_cache_clear()                      # K4 graphs capture this engine's buffers
        for name in ("p_xperm", "p_h", "p_y", "p_ws", "p_part", "p_paths", "_pinned_buf"):
            setattr(self, name, None)
        self.pinned = {}

    def enable_profile(self) -> "KernelProfiler":
        self.prof = KernelProfiler()
        if isinstance(self.driver, MLPDriver):
            self.driver.prof = self.prof
        return self.prof

    @torch.no_grad()
    def prefill(self, ids) -> int:
        """Prompt pass; returns the first generated token (greedy)."""
        ids = torch.as_tensor(ids, dtype=torch.long, device=self.device).reshape(-1)
        T = ids.numel()
        if T < 1:
            raise ValueError("prefill needs at least one prompt token")
        if T > self.max_prefill:
            raise ValueError(f"prompt of {T} tokens exceeds max_prefill={self.max_prefill}")
        if T > self.max_seq:
            raise ValueError(f"prompt of {T} tokens exceeds max_seq={self.max_seq}")
        h = self.W.embed[ids]
        idx_all = []
        if self.policy is SchedulerPolicy.PREFETCH_ALL:
            self._pa_fill(self._pa_v + 2)
        else:
            self._spec_fetch(0)
        for l in range(self.L):
            h = attention_block(self.shape, self.W.layers[l], h, self.kv, l, 0, self.cos, self.sin)
            h, idx_host = self._moe_prefill(l, h, T)
            idx_all.append(idx_host)
        self.kv.len = T
        self.paths_prefill = np.stack(idx_all, axis=1)     # [T, L, k]
        if self.route_stats is not None:
            self.route_stats.add(self.p_paths[:T])
        lg = logits_last(self.shape, self.W, h[-1:])[0]
        self.last_logits = lg
        tok = int(torch.argmax(lg).item())
        self.token = tok
        self.t_decode = 0
        return tok

    @torch.no_grad()
    def decode_step(self) -> int:
        """One greedy decode token (feeds back the previous output token)."""
        if self.token is None:
            raise ValueError("decode_step before prefill")
        pos = self.kv.len
        if pos + 1 > self.max_seq:
            raise ValueError(f"decode position {pos} would exceed max_seq={self.max_seq}")
        if self.use_graphs:
            self._ensure_decode_graphs()
            self.g_pos.fill_(pos)
            self.g_mask.copy_(torch.where(self.g_ar <= pos, 0.0, float("-inf")).view_as(self.g_mask))
            self.g_tok.fill_(self.token)
            self.g_h.copy_(self.W.embed.index_select(0, self.g_tok))
        else:
            h = self.W.embed[torch.tensor([self.token], device=self.device)]
        path = []
        if isinstance(self.driver, TraceDriver):
            self.driver.t = self.t_decode
        self._pred_next = None
        for l in range(self.L):
            if self.use_graphs:
                self.g_graphs[l].replay()                          # attention + norm + K1 gate
                ops._count("ds_gate_topk")
                h, E = self._moe_decode(l, self.g_h1, pre=self.g_a2, out=self.g_h)
            else:
                h = attention_block(self.shape, self.W.layers[l], h, self.kv, l, pos, self.cos, self.sin)
                h, E = self._moe_decode(l, h)
            path.append(tuple(E))
        self.kv.len = pos + 1
        self.paths_decode.append(tuple(path))
        if self.route_stats is not None:                   # hist holds idx + 1 of every layer
            self.route_stats.add((self.hist.view(1, self.L, self.k) - 1).to(torch.int32))
        lg = logits_last(self.shape, self.W, h)[0]
        self.last_logits = lg
        tok = int(torch.argmax(lg).item())
        self.token = tok
        self.t_decode += 1
        return tok

    def _attn_decode(self, l: int):
        return attention_decode_static(self.shape, self.W.layers[l], self.g_h, self.kv, l, self.g_pos, self.g_mask,
                                       self.cos, self.sin)

    def _decode_layer_front(self, l: int) -> None:
        """attention(l) + rms_norm + K1 gate on static buffers (captured per layer).
        Batch 1 with W4 attention: the fused front (csrc/front.cu, A/B:
        DS_FRONT_FUSED=0); otherwise the torch ops."""
        if self.front_fused and isinstance(self.kv, KVCache) and self.W.layers[l].get("wqkv") is not None:
            decode_front_fused(self.shape, self.W.layers[l], self.g_h, self.kv, l, self.g_pos, self.g_mask, self.cos,
                               self.sin, self.g_h1, self.g_a2)
        else:
            h1 = self._attn_decode(l)
            self.g_h1.copy_(h1)
            self.g_a2.copy_(rms_norm(h1, self.W.layers[l]["ln2"], self.shape.rms_eps))
        ops.gate_topk(self.g_a2, self.W.layers[l]["wg"], self.k, self.idx1, self.w1, hist=self.hist, layer=l)

    def _ensure_decode_graphs(self) -> None:
        if self.g_graphs is not None:
            return
        dev, d = self.device, self.d
        max_seq = self.kv.k.shape[-2]
        B = self.B
        self.g_pos = torch.zeros(1, dtype=torch.long, device=dev)
        self.g_tok = torch.zeros(B, dtype=torch.long, device=dev)
        self.g_ar = torch.arange(max_seq, device=dev)
        self.g_mask = torch.zeros((1, 1, 1, max_seq), dtype=torch.bfloat16, device=dev)
        self.g_h = torch.zeros((B, d), dtype=torch.bfloat16, device=dev)
        self.g_h1 = torch.zeros((B, d), dtype=torch.bfloat16, device=dev)
        self.g_a2 = torch.zeros((B, d), dtype=torch.bfloat16, device=dev)
        kv_k, kv_v = self.kv.k.clone(), self.kv.v.clone()
        hist = self.hist.clone()
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for l in range(self.L):                                 # warm-up outside capture
                self._decode_layer_front(l)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.g_graphs = []
        for l in range(self.L):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._decode_layer_front(l)
            self.g_graphs.append(g)
        torch.cuda.synchronize(dev)
        self.kv.k.copy_(kv_k)                                       # undo the warm-up writes
        self.kv.v.copy_(kv_v)
        self.hist.copy_(hist)
        del kv_k, kv_v

    def generate(self, ids, n_new: int) -> list:
        out = [self.prefill(ids)]
        for _ in range(n_new - 1):
            out.append(self.decode_step())
        return out

    # -------------------------------------------------------------- prefill
    def _next_ring_slot(self) -> int:
        s = self._ring
        self._ring = (self._ring + 1) % self.n_slots
        return s

    # ---------------------------------------------------------- prefetchall
    def _pa_slot(self, v: int, e: int) -> int:
        """Bank v % 2 of M slots, one per (owned) expert."""
        return (v % 2) * len(self.owned) + self.store.local[e]

    def _pa_fill(self, upto: int) -> None:
        """Queue every owned expert of the layer visits [queued, upto) (visit v
        is layer v % L: prefill layers then each decode token's layers)."""
        while self._pa_queued < upto:
            v = self._pa_queued
            for e in self.owned:
                self.cache.load(self._pa_slot(v, e), v % self.L, e)
            self._pa_queued += 1

    def _pa_done(self) -> None:
        """The current visit's compute is queued: free its bank and stream the visit after next into it."""
        v = self._pa_v
        for e in self.owned:
            self.cache.release(self._pa_slot(v, e))
        self._pa_v += 1
        self._pa_fill(self._pa_v + 2)

    def _spec_fetch(self, layer: int) -> None:
        """Speculative first transfer of layer `layer` (expert 0) to overlap attention."""
        if layer >= self.L or self.policy in (SchedulerPolicy.ON_DEMAND, SchedulerPolicy.PREFETCH_ALL):
            self._spec = None
            return
        cand = [e for e in self.owned if (layer, e) not in self.pinned]
        if not cand:                             # every expert of the layer is pinned in HBM
            self._spec = None
            return
        slot = self._next_ring_slot()
        first = cand[0]                          # lowest (owned, streamed) expert; 0 on a single GPU
        if self.link.cancel_enabled:
            # through the native link in small chunks: if the gate leaves `first`
            # out of A_l its remaining chunks are dropped (the log is unchanged)
            self.cache.content[slot] = (layer, first)
            self._spec = (slot, layer, first, self.link.submit(slot, layer, first, speculative=True))
        else:
            self.cache.load(slot, layer, first)
            self._spec = (slot, layer, first, None)

    def _moe_prefill(self, l: int, h: torch.Tensor, T: int):
        sh = self.shape
        a = rms_norm(h, self.W.layers[l]["ln2"], sh.rms_eps)
        idx, w = self.p_idx[:T], self.p_w[:T]
        ops.gate_topk(a, self.W.layers[l]["wg"], self.k, idx, w)
        if self.p_paths is not None:
            self.p_paths[:T, l].copy_(idx)
        if self.capture is not None:
            self.capture.append(("prefill", l, a.cpu(), idx.cpu()))
        ops.permute(idx, a, self.M, self.p_off, self.p_pos[:T * self.k], self.p_src[:T * self.k],
                    self.p_xperm[:T * self.k])
        self.p_off_host.copy_(self.p_off, non_blocking=True)
        idx_host = torch.empty((T, self.k), dtype=torch.int32, pin_memory=True)
        idx_host.copy_(idx, non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        done.synchronize()                                  # activated set -> host
        self.d2h_bytes += self.p_off_host.nbytes + idx_host.nbytes
        off = self.p_off_host.tolist()
        A_all = [e for e in range(self.M) if off[e + 1] > off[e]]
        A = [e for e in A_all if e in self.owned_set]       # this rank's share (all on one GPU)
        A, A_pin = self._split_pinned(l, A)                 # pinned experts are already in HBM
        plan = []                                           # (expert, slot, already_queued)
        if self.policy is SchedulerPolicy.PREFETCH_ALL:
            return self._moe_prefill_all(l, h, T, A, A_all, off, w, idx, idx_host)
        if self.policy is SchedulerPolicy.ON_DEMAND:
            plan = [(e, i % self.n_slots, False) for i, e in enumerate(A)]
        else:
            spec = self._spec if (self._spec is not None and self._spec[1] == l) else None
            if spec is not None:
                plan.append((spec[2], spec[0], True))
                tr = spec[3]
                if tr is not None:
                    if spec[2] in A:
                        self.link.promote(tr)          # confirmed: finish with large chunks
                        self.link.flush(tr)            # all chunks issued before later copies queue
                    else:
                        self.link.cancel(tr)           # wrong guess: drop its remaining chunks
            plan += [(e, self._next_ring_slot(), False) for e in A if not (spec and e == spec[2])]
        self.log.append({"phase": "prefill", "layer": l, "fetch": [e for e, _, _ in plan], "activated": A_all,
                         **({"pinned": A_pin} if self.pinned else {})})
        self._prefill_pinned(l, A_pin, off)
        # sliding window over the slot ring: the copy into a slot is queued only
        # after the compute that last used it has been queued (its free event)
        window = self.n_slots if self.policy is not SchedulerPolicy.ON_DEMAND else self.n_slots
        for i in range(min(window, len(plan))):
            e, slot, queued = plan[i]
            if not queued:
                self.cache.load(slot, l, e)
        for i, (e, slot, _) in enumerate(plan):
            if off[e + 1] > off[e]:
                self._prefill_ffn(e, slot, off)
            self.cache.release(slot)
            if i + window < len(plan):
                e2, slot2, queued2 = plan[i + window]
                if not queued2:
                    self.cache.load(slot2, l, e2)
        # next layer's first expert streams while this layer combines + next attention runs
        self._spec_fetch(l + 1)
        out = self._prefill_combine(h, T, w, idx)
        self._record_moe("prefill", l, h, a, out, idx_host, w)
        return out, idx_host.numpy()

    def _prefill_ffn(self, e: int, slot, off, st=None) -> None:
        lo, hi = off[e], off[e + 1]
        if st is None:
            st = self.cache.acquire(slot)
        evs = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if self.prof else (None, None)
        ops.grouped_ffn(self.p_xperm[lo:hi], [0, hi - lo], [st], self.d, self.ff, self.G,
                        self.p_h[lo:hi], self.p_y[lo:hi], self.p_ws, *evs)
        if self.prof:
            self.prof.add("K3 w4_grouped_ffn (tcgen05)", evs[0], evs[1], self.store.blob_bytes,
                          6.0 * (hi - lo) * self.d * self.ff)

    def _prefill_pinned(self, l: int, A_pin, off) -> None:
        """The layer's HBM-resident pinned experts in ONE grouped K3 launch
        (their rows are segments of the permuted buffer)."""
        self._prefill_group([e for e in A_pin if off[e + 1] > off[e]], off,
                            lambda e: self.pinned[(l, e)])

    def _prefill_group(self, es, off, struct_of) -> None:
        """Experts `es` (all resident) in one grouped K3 launch over their row
        segments; one launch per expert when the split-K workspace of the
        grouped call would not fit the preallocated one."""
        if not es:
            return
        segs = [(off[e], off[e + 1] - off[e]) for e in es]
        if len(es) == 1 or len(es) > 16 or \
                ops.grouped_ffn_segments_workspace(segs, self.d, self.ff, self.G) > self.p_ws.numel():
            for e in es:
                self._prefill_ffn(e, None, off, st=struct_of(e))
            return
        structs = [struct_of(e) for e in es]
        evs = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if self.prof else (None, None)
        ops.grouped_ffn_segments(self.p_xperm, segs, structs, self.d, self.ff, self.G, self.p_h, self.p_y, self.p_ws,
                                 *evs)
        if self.prof:
            self.prof.add("K3 w4_grouped_ffn (tcgen05)", evs[0], evs[1], len(es) * self.store.blob_bytes,
                          6.0 * sum(r for _, r in segs) * self.d * self.ff)

    def _prefill_combine(self, h, T, w, idx):
        out = torch.empty_like(h)
        if self.ep is None:
            ops.unpermute_combine(self.p_y[:T * self.k], self.p_pos[:T * self.k], w, h, out)
        else:
            part = self.p_part[:T]
            ops.unpermute_partial(self.p_y[:T * self.k], self.p_pos[:T * self.k], w, idx, self.owner_bits, part)
            self.ep.combine_(part)                          # sum of the ranks' expert terms
            ops.combine_finalize(part, h, out)
        return out

    def _moe_prefill_all(self, l, h, T, A, A_all, off, w, idx, idx_host):
        """prefetchall: the whole layer was queued two visits ago; compute the activated experts."""
        self.log.append({"phase": "prefill", "layer": l, "fetch": list(self.owned), "activated": A_all})
        # the whole bank is resident: the layer's activated experts in one grouped launch
        self._prefill_group([e for e in A if off[e + 1] > off[e]], off,
                            lambda e: self.cache.acquire(self._pa_slot(self._pa_v, e)))
        self._pa_done()
        out = self._prefill_combine(h, T, w, idx)
        self._record_moe("prefill", l, h, rms_norm(h, self.W.layers[l]["ln2"], self.shape.rms_eps), out, idx_host, w)
        return out, idx_host.numpy()

    def _record_moe(self, phase: str, l: int, h, a, out, idx_host, w) -> None:
        """Parity hook (tests / bench checker only): host copies of one MoE
        block's input h, its normed gate input a, its output and the routing."""
        if not self.capture_moe or l not in self.capture_moe:
            return
        self.moe_records.append({"phase": phase, "layer": l, "token": self.t_decode if phase == "decode" else None,
                                 "h_in": h.cpu(), "a": a.cpu(), "out": out.cpu(),
                                 "idx": torch.as_tensor(np.asarray(idx_host)).clone(), "w": w.cpu()})

    # --------------------------------------------------------------- decode
    def _moe_decode(self, l: int, h: torch.Tensor, pre: torch.Tensor | None = None, out: torch.Tensor | None = None):
        sh = self.shape
        link = self.link
        if pre is None:
            a = rms_norm(h, self.W.layers[l]["ln2"], sh.rms_eps)
            ops.gate_topk(a, self.W.layers[l]["wg"], self.k, self.idx1, self.w1, hist=self.hist, layer=l)
        else:
            a = pre                                                # gate already ran inside the layer graph
        self.ev_gate.record()
        self.idx_host.copy_(self.idx1, non_blocking=True)
        ev_idx = torch.cuda.Event()
        ev_idx.record()
        use_pred = self.driver is not None
        if use_pred and l + 1 < self.L:
            self.driver.launch(self.hist, self.ev_gate, l + 1)     # predict stream, overlapped
        t_w = time.perf_counter()
        link.wait_event(ev_idx)                                    # sync point 1: E_l on the host
        t_d = time.perf_counter()
        self.host_wait["sync1"] += t_d - t_w
        self.d2h_bytes += self.idx_host.nbytes + ((4 * self.k + 8 * self.M) if use_pred else 0)
        E = self._idx_np[0].tolist()
        if self.capture is not None:
            self.capture.append(("decode", l, a.cpu(), self.idx_host.clone()))
        slot_of, trs = {}, {}
        miss = []
        mine = [e for e in E if e in self.owned_set]
        mine, mine_pin = self._split_pinned(l, mine)           # pinned experts are already in HBM
        if self.policy is SchedulerPolicy.PREFETCH_ALL:
            self.log.append({"phase": "decode", "token": self.t_decode, "layer": l, "fetch": list(self.owned),
                             "kind": "prefetchall"})
            for e in mine:
                sl = self._pa_slot(self._pa_v, e)
                self._decode_ffn(a, self.cache.struct(sl), E.index(e), wait=self.cache.ready[sl])
            self._pa_done()
            out = self._decode_combine(h, out)
            self._record_moe("decode", l, h, a, out, self.idx_host, self.w1)
            return out, E
        if l == 0 or not use_pred:
            base = 0 if (l % 2 == 0 or self.n_slots < 2 * self.k) else self.k
            for j, e in enumerate(mine):
                slot = (base + j) % self.n_slots
                trs[e] = link.submit(slot, l, e)
                slot_of[e] = slot
            self.log.append({"phase": "decode", "token": self.t_decode, "layer": l, "fetch": mine,
                             "kind": "ondemand", **({"pinned": sorted(mine_pin)} if self.pinned else {})})
        else:
            P, order, pending = self._pred_next              # pending: this rank's predicted experts
            miss = sorted(set(mine) - set(P))
            spare = [pending[p][0] for p in order if p in pending and p not in E]
            confirmed = []
            for p in order:
                if p not in pending:
                    continue
                if p in E:
                    slot_of[p], trs[p] = pending[p]
                    confirmed.append(trs[p])
                else:
                    link.cancel(pending[p][1])                 # drop its not-yet-issued chunks
            used = set(slot_of.values())
            spare += [s_ for s_ in range(self.n_slots) if s_ not in used and s_ not in spare]
            for e, s_ in zip(miss, spare):
                trs[e] = link.submit(s_, l, e)                 # re-fetch into a wrong (or free) slot
                slot_of[e] = s_
            for tr in confirmed:                               # after the re-fetches: they wait on no promote
                link.promote(tr)                               # confirmed: finish with large chunks
            self.log.append({"phase": "decode", "token": self.t_decode, "layer": l,
                             "pred": sorted(p for p in P if p in self.owned_set),
                             "gate": sorted(E), "refetch": miss, **({"pinned": sorted(mine_pin)} if self.pinned else {})})
        # host time from the gate result to every transfer of this layer submitted
        self.host_wait["decide"] += time.perf_counter() - t_d
        # expert compute: pinned, then hits (already resident or in flight), then re-fetched ones
        for e in mine_pin:
            self._decode_ffn(a, self.pinned[(l, e)], E.index(e))
        for e in [x for x in mine if x not in miss] + miss:
            j = E.index(e)
            link.flush(trs[e])
            self._decode_ffn(a, self.cache.struct(slot_of[e]), j, wait=self.cache.ready[slot_of[e]])
            self.cache.release(slot_of[e])
        out = self._decode_combine(h, out)
        self._record_moe("decode", l, h, a, out, self.idx_host, self.w1)
        # sync point 2: prediction for l+1 ready -> prefetch into the slots layer l-1 used
        if use_pred and l + 1 < self.L:
            t_w = time.perf_counter()
            Pn, order = self.driver.result(link)
            self.host_wait["sync2"] += time.perf_counter() - t_w
            cur = set(slot_of.values())
            free = [s_ for s_ in range(self.n_slots) if s_ not in cur][: self.k]
            pending = {}
            for e, s_ in zip([e for e in order if e in self.owned_set and (l + 1, e) not in self.pinned], free):
                pending[e] = (s_, link.submit(s_, l + 1, e, speculative=True))
            self._pred_next = (Pn, order, pending)
        return out, E

    def _decode_ffn(self, a, st, j: int, wait=None) -> None:
        """K4: acc += w_j * W2 (silu(a W1) * (a W3)) for the expert in slot struct st,
        once `wait` (the slot's ready event; None for a pinned expert) fired.

        Default: one launch of a cached device-resident graph [wait -> span
        events -> K4] (ops.expert_gemv_graph): while the copy engine streams
        the next expert, host-submitted commands reach the GPU ~25-30 us late,
        graph-internal ones do not (profiles/r2/k4_ce_timeline.json)."""
        ev0 = ev1 = None
        timed = self.prof is not None
        if timed:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if self.k4_graphs:
            ops.expert_gemv_graph(a, st, self.d, self.ff, self.G, self.h_buf, self.w1[0, j:], 1, self.acc,
                                  wait, ev0, ev1)
        else:
            if wait is not None:
                torch.cuda.current_stream(self.device).wait_event(wait)
            ops.expert_gemv(a, st, self.d, self.ff, self.G, self.h_buf, self.w1[0, j:], 1, self.acc, ev0, ev1)
        if timed:
            self.prof.add("K4 w4_swiglu_gemv+down_gemv", ev0, ev1, self.store.blob_bytes)

    def _decode_combine(self, h, out):
        if out is None:
            out = torch.empty_like(h)
        if self.ep is not None:
            self.ep.combine_(self.acc)                         # sum of the ranks' expert terms
        ops.combine_finalize(self.acc, h, out)
        return out

    # -------------------------------------------------------------- metrics
    def link_peak_gbs(self) -> float:
        """Measured pinned H2D bandwidth (copy engine), 1 expert blob x 16."""
        if self._link_peak is None:
            src = self.store.data[0, 0]
            dst = self.cache.slots[0]
            s = self.cache.copy_stream
            with torch.cuda.stream(s):
                for _ in range(2):
                    dst.copy_(src, non_blocking=True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(16):
                    dst.copy_(src, non_blocking=True)
                e1.record(s)
            e1.synchronize()
            self._link_peak = 16 * src.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
            self.cache.used[0] = False
        return self._link_peak

    def enable_timeline(self) -> "Timeline":
        """Device timeline of copy-busy intervals and expert-FFN spans (needs enable_profile())."""
        if self.prof is None:
            self.enable_profile()
        return Timeline(self)

    def h2d_bytes(self) -> int:
        """Expert bytes moved host->device so far (prefill copies + decode link chunks)."""
        return self.cache.bytes_copied + self.link.stats()["bytes_issued"]

    def prefill_bytes_floor(self) -> int:
        """sum_l |A_l| * expert bytes of the last prefill."""
        n = sum(len(r["activated"]) for r in self.log if r["phase"] == "prefill")
        return n * self.store.blob_bytes

    def decode_bytes_floor(self) -> int:
        """L * k * expert bytes per token (perfect prediction)."""
        return self.L * self.k * self.store.blob_bytes

    def streamed_bytes_floor(self) -> dict:
        """Bytes any schedule must move over the link for the last request
        given the pinned experts (they never cross the link): prefill
        sum_l |A_l minus pinned|, decode per token sum_l |E_l minus pinned|,
        times the expert bytes (this rank's experts under EP)."""
        pre = dec = 0
        n_tok = 0
        for r in self.log:
            pins = set(r.get("pinned", []))
            if r["phase"] == "prefill":
                pre += len([e for e in r["activated"] if e in self.owned_set and e not in pins])
            elif "gate" in r:
                dec += len([e for e in r["gate"] if e in self.owned_set and e not in pins])
            elif r.get("kind") == "ondemand":
                dec += len(r["fetch"])
            if r["phase"] == "decode" and r["layer"] == 0:
                n_tok += 1
        b = self.store.blob_bytes
        return {"prefill_bytes": pre * b, "decode_bytes_per_token": dec * b / max(n_tok, 1)}

    def hit_summary(self) -> dict:
        """Prediction counters over the decode log, counted like
        oracle/sim_ref.cache_log_decode: prediction and gate sets restricted to
        this rank's streamed experts (owned, not pinned), so a pinned expert is
        never a prefetch hit and under EP a rank scores only its own experts."""
        dec = [r for r in self.log if r["phase"] == "decode" and "pred" in r]

        def streamed(r, key):
            pins = {e for (ll, e) in self.pinned if ll == r["layer"]}
            return {e for e in r[key] if e in self.owned_set and e not in pins}

        hits = sum(len(streamed(r, "pred") & streamed(r, "gate")) for r in dec)
        miss = sum(len(r["refetch"]) for r in dec)
        exact = sum(streamed(r, "pred") == streamed(r, "gate") for r in dec)
        n = len(dec)
        return {"policy": self.policy.value, "cancel_mispredicted": self.cancel_mispredicted,
                "chunk_bytes": self.link.chunk, "spec_chunk_bytes": self.link.spec_chunk, **self.link.stats(),
                "prefetch_hits": hits, "prefetch_misses": miss,
                "topk_hit_rate": round(exact / n, 4) if n else None,
                "at_least_one_rate": round(sum(bool(streamed(r, "pred") & streamed(r, "gate")) for r in dec) / n, 4)
                if n else None}

    def resident_bytes(self) -> dict:
        pred = self.driver.nbytes if isinstance(self.driver, MLPDriver) else 0
        out = {"non_moe": self.W.nbytes(), "expert_slots": self.cache.nbytes, "predictor": pred,
               "kv_cache": self.kv.nbytes, "model_total": self.shape.total_bytes}
        if self._pinned_buf is not None:
            out["pinned_experts"] = self._pinned_buf.numel()
        return out


class BatchEngine(Engine):
    """B sequences of equal prompt length served together (BASELINE config 4:
    batch 1-32 x prompt 128-2048, the dense-prefill vs sparse-decode
    crossover).  A build extension — the reference's simulator excludes
    batching; its cache semantics are extended to the batch's
    union of selections (oracle/sim_ref.cache_log_decode_batch):

      prefill   the B*P tokens are routed together: A_l = the union over the
                batch, fetched once per layer exactly as for one sequence;
      decode    per layer the activated set A_l = the union of the B gate
                selections; for l >= 1 the predicted set P_l = the union of
                the B predictions (K5 on B rows), prefetched during layer l-1
                in order of probability summed over the batch; sync point 1
                re-fetches A_l minus P_l; the expert rows are grouped by the
                permute kernel (K2) and each expert runs the K4 GEMV on its
                rows (<= 16) or the tcgen05 GEMM (K3) above that;
      capacity  2 * min(M, k*B) slots (duoserve/oracle: one bank for the
                layer's working set, one for the next layer's prefetch;
                ondemand: min(M, k*B)); B = 1 gives the SPEC's 2k / k.

    The API mirrors Engine: prefill(ids [B, P]) -> B first tokens,
    decode_step() -> B tokens; paths_decode[t][b] is sequence b's path."""

    GEMV_ROWS = 16          # K4 up to this many rows per expert, K3 (tcgen05) above

    def __init__(self, shape: ModelShape, policy="duoserve", batch: int = 1, max_prompt: int = 512,
                 max_seq: int = 2048, **kw):
        if batch < 1:
            raise ValueError("batch must be >= 1")
        if SchedulerPolicy(policy) in (SchedulerPolicy.DUOSERVE_ORACLE, SchedulerPolicy.PREFETCH_ALL):
            raise ValueError(f"BatchEngine serves 'duoserve' and 'ondemand' (got {policy!r})")
        if kw.get("ep") is not None and SchedulerPolicy(policy) is not SchedulerPolicy.ON_DEMAND:
            raise ValueError("BatchEngine with expert parallelism (token dispatch) serves policy 'ondemand'")
        self.B = int(batch)
        self.max_prompt = int(max_prompt)
        super().__init__(shape, policy, max_seq=max_seq, max_prefill=self.B * self.max_prompt, **kw)
        dev, B, k, d, ff = self.device, self.B, self.k, self.d, self.ff
        self.d_off = torch.empty(self.M + 1, dtype=torch.int32, device=dev)
        self.d_off_host = torch.empty(self.M + 1, dtype=torch.int32, pin_memory=True)
        self.d_pos = torch.empty(B * k, dtype=torch.int32, device=dev)
        self.d_src = torch.empty(B * k, dtype=torch.int32, device=dev)
        self.d_xperm = torch.empty((B * k, d), dtype=torch.bfloat16, device=dev)
        self.d_y = torch.zeros((B * k, d), dtype=torch.float32, device=dev)
        self.d_h = torch.empty((B * k, ff), dtype=torch.bfloat16, device=dev)
        self.ones = torch.ones(1, dtype=torch.float32, device=dev)
        self.d_ws = torch.empty(max(ops.grouped_ffn_workspace(B * k, d, ff), 256), dtype=torch.uint8, device=dev)
        self.tokens = None

    def _slot_count(self, cfg) -> int:
        cap = min(self.M, self.k * self.B)
        if self.policy is SchedulerPolicy.ON_DEMAND:
            return cap
        return 2 * cap

    def _make_kv(self, max_seq: int):
        return KVCacheBatch(self.shape, self.B, max_seq, self.device)

    def _attn_decode(self, l: int):
        return attention_decode_static_batch(self.shape, self.W.layers[l], self.g_h, self.kv, l, self.g_pos,
                                             self.g_mask, self.cos, self.sin)

    @torch.no_grad()
    def prefill(self, ids) -> list:
        """Prompt pass of the B sequences (ids [B, P]); returns their first tokens."""
        ids = torch.as_tensor(ids, dtype=torch.long, device=self.device)
        if ids.dim() != 2 or ids.shape[0] != self.B:
            raise ValueError(f"prefill needs ids of shape [{self.B}, P], got {tuple(ids.shape)}")
        P = ids.shape[1]
        T = self.B * P
        if P < 1:
            raise ValueError("prefill needs at least one prompt token")
        if P > self.max_prompt or P > self.max_seq:
            raise ValueError(f"prompt of {P} tokens exceeds max_prompt={self.max_prompt} / max_seq={self.max_seq}")
        h = self.W.embed[ids]                                     # [B, P, d]
        idx_all = []
        self._spec_fetch(0)
        for l in range(self.L):
            h = attention_block_batch(self.shape, self.W.layers[l], h, self.kv, l, 0, self.cos, self.sin)
            if self.ep is not None:
                hf, idx_host = self._moe_ep(l, "prefill", h.reshape(T, self.d), T)
            else:
                hf, idx_host = self._moe_prefill(l, h.reshape(T, self.d), T)
            h = hf.view(self.B, P, self.d)
            idx_all.append(idx_host)
        self.kv.len = P
        self.paths_prefill = np.stack(idx_all, axis=1)           # [B*P, L, k], sequence-major
        if self.route_stats is not None:
            self.route_stats.add(self.p_paths[:T])
        lg = logits_last(self.shape, self.W, h[:, -1])
        self.last_logits = lg
        toks = [int(t) for t in torch.argmax(lg, dim=-1).tolist()]
        self.tokens = toks
        self.token = toks[0]
        self.t_decode = 0
        return toks

    @torch.no_grad()
    def decode_step(self) -> list:
        """One greedy token for each of the B sequences."""
        if self.tokens is None:
            raise ValueError("decode_step before prefill")
        pos = self.kv.len
        if pos + 1 > self.max_seq:
            raise ValueError(f"decode position {pos} would exceed max_seq={self.max_seq}")
        self._ensure_decode_graphs()
        self.g_pos.fill_(pos)
        self.g_mask.copy_(torch.where(self.g_ar <= pos, 0.0, float("-inf")).view_as(self.g_mask))
        self.g_tok.copy_(torch.as_tensor(self.tokens, dtype=torch.long), non_blocking=True)
        self.g_h.copy_(self.W.embed.index_select(0, self.g_tok))
        paths = [[] for _ in range(self.B)]
        self._pred_next = None
        h = self.g_h
        for l in range(self.L):
            self.g_graphs[l].replay()                              # attention + norm + K1 gate (B rows)
            ops._count("ds_gate_topk")
            if self.ep is not None:
                out, idx_host = self._moe_ep(l, "decode", self.g_h1, self.B, a=self.g_a2)
                self.g_h.copy_(out)
                h = self.g_h
                rows = [tuple(int(e) for e in r) for r in idx_host.tolist()]
            else:
                h, rows = self._moe_decode_batch(l, self.g_h1, self.g_a2, self.g_h)
            for b in range(self.B):
                paths[b].append(rows[b])
        self.kv.len = pos + 1
        self.paths_decode.append(tuple(tuple(p) for p in paths))
        if self.route_stats is not None:
            self.route_stats.add((self.hist.view(self.B, self.L, self.k) - 1).to(torch.int32))
        lg = logits_last(self.shape, self.W, h)
        self.last_logits = lg
        toks = [int(t) for t in torch.argmax(lg, dim=-1).tolist()]
        self.tokens = toks
        self.t_decode += 1
        return toks

    def generate(self, ids, n_new: int) -> list:
        """[n_new][B] tokens."""
        out = [self.prefill(ids)]
        for _ in range(n_new - 1):
            out.append(self.decode_step())
        return out

    def _moe_ep(self, l: int, phase: str, h, T: int, a=None):
        """Expert parallelism with token dispatch (batch > 1):
        this rank's T rows are routed here, dispatched to the expert owners
        over all-to-all (ep.dispatch_combine), each owner fetches the experts
        it received rows for (on demand, ascending, through its own slot ring
        and copy stream) and runs them (K4 for <= 16 rows, K3 above), the
        outputs come back and are combined in slot order.  Log per layer:
        the owned experts fetched = (union of every rank's selections) ∩
        owned (oracle: sim_ref.cache_log_ep_dispatch)."""
        from .ep import dispatch_combine
        sh = self.shape
        if a is None:
            a = rms_norm(h, self.W.layers[l]["ln2"], sh.rms_eps)
            idx, w = self.p_idx[:T], self.p_w[:T]
            ops.gate_topk(a, self.W.layers[l]["wg"], self.k, idx, w)
            if self.p_paths is not None:
                self.p_paths[:T, l].copy_(idx)
        else:
            idx, w = self.idx1, self.w1
        idx_host = idx.cpu()
        if self.capture is not None:
            self.capture.append((phase, l, a.cpu(), idx_host.clone()))
        ran = []

        def ffn(e: int, rows: torch.Tensor) -> torch.Tensor:
            n = rows.shape[0]
            slot = self._next_ring_slot()
            self.cache.load(slot, l, e)
            st = self.cache.acquire(slot)
            y = torch.zeros((n, self.d), dtype=torch.float32, device=self.device)
            hb = torch.empty((n, self.ff), dtype=torch.bfloat16, device=self.device)
            if n <= self.GEMV_ROWS:
                ops.expert_gemv(rows.contiguous(), st, self.d, self.ff, self.G, hb, self.ones, 0, y)
            else:
                ws = torch.empty(max(ops.grouped_ffn_workspace(n, self.d, self.ff), 256), dtype=torch.uint8,
                                 device=self.device)
                ops.grouped_ffn(rows.contiguous(), [0, n], [st], self.d, self.ff, self.G, hb, y, ws)
            self.cache.release(slot)
            ran.append(e)
            return y

        out, _ = dispatch_combine(a, idx, w, h, self.ep, ffn, self.M)
        rec = {"phase": phase, "layer": l, "fetch": sorted(ran), "kind": "ep-dispatch"}
        if phase == "decode":
            rec = {"phase": phase, "token": self.t_decode, "layer": l, "fetch": sorted(ran), "kind": "ep-dispatch"}
        self.log.append(rec)
        return out, (idx_host.numpy() if phase == "prefill" else idx_host)

    def _batch_ffn(self, e: int, off, st) -> None:
        lo, hi = off[e], off[e + 1]
        R = hi - lo
        prof = self.prof
        evs = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if prof else (None, None)
        if R <= self.GEMV_ROWS:
            ops.expert_gemv(self.d_xperm[lo:hi], st, self.d, self.ff, self.G, self.d_h[:R], self.ones, 0,
                            self.d_y[lo:hi], *evs)
            if prof:
                prof.add("K4 w4_swiglu_gemv+down_gemv", evs[0], evs[1], self.store.blob_bytes)
        else:
            ops.grouped_ffn(self.d_xperm[lo:hi], [0, R], [st], self.d, self.ff, self.G, self.d_h[lo:hi],
                            self.d_y[lo:hi], self.d_ws, *evs)
            if prof:
                prof.add("K3 w4_grouped_ffn (tcgen05)", evs[0], evs[1], self.store.blob_bytes,
                         6.0 * R * self.d * self.ff)

    def _moe_decode_batch(self, l: int, h, a, out):
        link = self.link
        B, k, M = self.B, self.k, self.M
        ops.permute(self.idx1, a, M, self.d_off, self.d_pos, self.d_src, self.d_xperm)
        self.ev_gate.record()
        self.idx_host.copy_(self.idx1, non_blocking=True)
        self.d_off_host.copy_(self.d_off, non_blocking=True)
        ev_idx = torch.cuda.Event()
        ev_idx.record()
        use_pred = self.driver is not None
        if use_pred and l + 1 < self.L:
            self.driver.launch(self.hist, self.ev_gate, l + 1)    # predict stream, overlapped
        link.wait_event(ev_idx)                                    # sync point 1: the batch's selections on the host
        self.d2h_bytes += self.idx_host.nbytes + self.d_off_host.nbytes + \
            ((4 * k + 8 * M) * B if use_pred else 0)
        off = self.d_off_host.tolist()
        rows = [tuple(int(e) for e in r) for r in self.idx_host.tolist()]
        if self.capture is not None:
            self.capture.append(("decode", l, a.cpu(), self.idx_host.clone()))
        A = [e for e in range(M) if off[e + 1] > off[e]]
        mine, mine_pin = self._split_pinned(l, A)
        slot_of, trs, miss = {}, {}, []
        cap = min(M, k * B)
        if l == 0 or not use_pred:
            base = 0 if (l % 2 == 0 or self.n_slots < 2 * cap) else cap
            for j, e in enumerate(mine):
                slot = (base + j) % self.n_slots
                trs[e] = link.submit(slot, l, e)
                slot_of[e] = slot
            self.log.append({"phase": "decode", "token": self.t_decode, "layer": l, "fetch": mine,
                             "kind": "ondemand", **({"pinned": sorted(mine_pin)} if self.pinned else {})})
        else:
            P, order, pending = self._pred_next
            miss = sorted(set(mine) - set(P))
            spare = [pending[p][0] for p in order if p in pending and p not in A]
            for p in order:
                if p not in pending:
                    continue
                if p in A:
                    slot_of[p], trs[p] = pending[p]
                    link.promote(trs[p])
                else:
                    link.cancel(pending[p][1])
            used = set(slot_of.values())
            spare += [s_ for s_ in range(self.n_slots) if s_ not in used and s_ not in spare]
            for e, s_ in zip(miss, spare):
                trs[e] = link.submit(s_, l, e)
                slot_of[e] = s_
            self.log.append({"phase": "decode", "token": self.t_decode, "layer": l, "pred": sorted(P),
                             "gate": A, "refetch": miss, **({"pinned": sorted(mine_pin)} if self.pinned else {})})
            self._batch_sets.append((l, self._pred_sets, rows))
        self.d_y[:B * k].zero_()
        for e in mine_pin:
            self._batch_ffn(e, off, self.pinned[(l, e)])
        for e in [x for x in mine if x not in miss] + miss:
            link.flush(trs[e])
            self._batch_ffn(e, off, self.cache.acquire(slot_of[e]))
            self.cache.release(slot_of[e])
        ops.unpermute_combine(self.d_y[:B * k], self.d_pos[:B * k], self.w1, h, out)
        self._record_moe("decode", l, h, a, out, self.idx_host, self.w1)
        if use_pred and l + 1 < self.L:                            # sync point 2
            Pn, order = self.driver.result(link)
            self._pred_sets = list(self.driver.sets)
            cur = set(slot_of.values())
            free = [s_ for s_ in range(self.n_slots) if s_ not in cur]
            pending = {}
            for e, s_ in zip([e for e in order if (l + 1, e) not in self.pinned], free):
                pending[e] = (s_, link.submit(s_, l + 1, e, speculative=True))
            self._pred_next = (Pn, order, pending)
        return out, rows

    def reset(self) -> None:
        super().reset()
        self.tokens = None
        self._pred_sets = None
        self._batch_sets = []          # (layer, per-sequence predicted sets, per-sequence gate sets)

    def hit_summary(self) -> dict:
        """Per-sequence prediction counters (top-k exact / at least one) and
        the union-level prefetch hits / misses of the cache log."""
        dec = [r for r in self.log if r["phase"] == "decode" and "pred" in r]
        hits = sum(len(set(r["pred"]) & set(r["gate"])) for r in dec)
        miss = sum(len(r["refetch"]) for r in dec)
        n = exact = any_ = 0
        for _, preds, gates in self._batch_sets:
            for p, g in zip(preds, gates):
                n += 1
                exact += set(p) == set(g)
                any_ += bool(set(p) & set(g))
        return {"policy": self.policy.value, "batch": self.B, **self.link.stats(),
                "prefetch_hits": hits, "prefetch_misses": miss,
                "topk_hit_rate": round(exact / n, 4) if n else None,
                "at_least_one_rate": round(any_ / n, 4) if n else None}


def _union(iv: list) -> list:
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def _covered(a: float, b: float, union: list) -> float:
    return sum(max(0.0, min(b, y) - max(a, x)) for x, y in union)


class Timeline:
    """Per-step device timeline (CUDA timing events, common reference event):
    copy-busy intervals of every expert transfer (ExpertCache copies and the
    native link's chunks, csrc/link.cu trace mode) and the expert-FFN spans
    (K3/K4, from the KernelProfiler).  Reports the link busy fraction, the
    achieved GB/s while busy and the copy/compute overlap fraction =
    (expert compute time that runs while a transfer is in flight) / (total
    expert compute time) — SURVEY.md §8d."""

    def __init__(self, eng: "Engine"):
        self.eng = eng
        eng.cache.trace = []
        eng.link.set_trace(True)
        self.ref = None

    def begin(self) -> None:
        torch.cuda.synchronize(self.eng.device)
        self.ref = torch.cuda.Event(enable_timing=True)
        self.ref.record()
        self.eng.cache.trace.clear()
        self.eng.link.trace_read(self.ref)                # drop spans of earlier steps
        self.k0 = {n: len(v) for n, v in self.eng.prof.spans.items()}

    def end(self) -> dict:
        end = torch.cuda.Event(enable_timing=True)
        end.record()
        torch.cuda.synchronize(self.eng.device)
        ref = self.ref
        copies = [(ref.elapsed_time(a), ref.elapsed_time(b)) for a, b in self.eng.cache.trace]
        copies += self.eng.link.trace_read(ref)
        comp = []
        for n, v in self.eng.prof.spans.items():
            comp += [(ref.elapsed_time(a), ref.elapsed_time(b)) for a, b, _, _ in v[self.k0.get(n, 0):]]
        u = _union(copies)
        busy = sum(b - a for a, b in u)
        total = ref.elapsed_time(end)
        ct = sum(b - a for a, b in comp)
        hidden = sum(_covered(a, b, u) for a, b in comp)
        return {"step_ms": total, "copy_busy_ms": busy, "copy_busy_frac": busy / total if total else None,
                "expert_compute_ms": ct, "overlap_frac": hidden / ct if ct else None,
                "n_copy_spans": len(copies), "n_compute_spans": len(comp)}


class KernelProfiler:
    """CUDA-event spans around hot-path launches, on the launching stream.

    Used by bench.py for the live roofline: algorithmic bytes / FLOPs per
    launch divided by the event-measured duration."""

    def __init__(self):
        self.spans = {}          # name -> list of (ev0, ev1, bytes, flops)
        self.launch0 = ops.launch_total()

    def reset(self):
        self.spans = {}
        self.launch0 = ops.launch_total()

    def start(self):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def add(self, name: str, ev0, ev1, nbytes: float, flops: float = 0.0):
        """A span whose events were recorded elsewhere (natively, around the launches)."""
        self.spans.setdefault(name, []).append((ev0, ev1, nbytes, flops))

    def stop(self, name: str, ev0, nbytes: float, flops: float = 0.0):
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        self.spans.setdefault(name, []).append((ev0, ev1, nbytes, flops))

    def summary(self, peaks: dict) -> dict:
        torch.cuda.synchronize()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        # a K3 launch is timed inside a seconds-long serving step: its roofline
        # is the SUSTAINED bf16 figure when the driver measured one
        tf = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0)))
        tf_kind = "sustained" if "bf16_tflops_sustained" in peaks else "burst"
        out = []
        for name, sp in self.spans.items():
            t = sum(a.elapsed_time(b) for a, b, _, _ in sp) / 1e3
            nb = sum(x[2] for x in sp)
            fl = sum(x[3] for x in sp)
            if fl > 0:
                ach = fl / t / 1e12
                out.append({"kernel": name, "bound": "tensor", "achieved": round(ach, 1), "peak": tf,
                            "peak_kind": tf_kind, "unit": "TFLOP/s", "frac": round(ach / tf, 4), "traffic": None,
                            "launches": len(sp), "avg_us": round(1e6 * t / len(sp), 2),
                            "total_ms": round(1e3 * t, 2), "bytes_per_launch": nb / len(sp),
                            "flops_per_launch": fl / len(sp)})
            else:
                ach = nb / t / 1e9
                out.append({"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm,
                            "unit": "GB/s", "frac": round(ach / hbm, 4), "traffic": None,
                            "launches": len(sp), "avg_us": round(1e6 * t / len(sp), 2),
                            "total_ms": round(1e3 * t, 2), "bytes_per_launch": nb / len(sp)})
        out.sort(key=lambda r: -r["total_ms"])
        dom = dict(out[0]) if out else None
        return {"dominant": dom, "all": out, "launches": ops.launch_total() - self.launch0}
