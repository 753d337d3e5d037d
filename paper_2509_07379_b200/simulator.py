"""Deterministic discrete-event simulator of the DuoServe-MoE runtime — the
reference's specified-but-unshipped ``duoserve.simulator`` module
(``/root/reference/SPEC.md:340-438``).

It models what the B200 runtime (``engine.Engine``) executes, at the level of
the SPEC: three serial streams (``comm`` = the one host->device link,
``predict``, ``compute``), a fixed-capacity device expert cache of
``slot_count(policy)`` slots, the prefill two-stream pipeline and the decode
pipeline with its two synchronisation points and blocking re-fetch of
mispredicted experts, plus the OnDemand (ACC) and PrefetchAll (MoESys)
baselines.  Time is integer nanoseconds; ties are ordered by
(time, stream priority comm < predict < compute, sequence number)
(SPEC.md:433).

Decisions — which experts are fetched, hit, missed and re-fetched — are
emitted in the same cache-log format as ``Engine.log`` (and the test oracle
``oracle/sim_ref.py``), so one predictor run can be replayed here and on the
GPU and the logs compared record for record.  The time model is the
reference ``CostModel`` (config.py:62-85); ``presets/*-b200.json`` carry a
cost model calibrated from this repo's B200 measurements
(``scripts/calibrate_cost.py``), so simulated TTFT / decode latency can be
set against measured ones.

Public API:
  DeviceExpertCache, EventTimeline, RequestMetrics, SimReport,
  simulate_request, schedule_prefill_layer, schedule_decode_layer,
  compute_peak_memory, run_experiment, SimulationError.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import asdict, dataclass, field

import numpy as np

from .config import ConfigError, CostModel, ModelConfig, SchedulerPolicy, config_to_json, slot_count
from .trace import ActivationTrace, TraceDataset, TraceError

STREAMS = ("comm", "predict", "compute")   # tie-break priority
_PRIO = {s: i for i, s in enumerate(STREAMS)}


class SimulationError(RuntimeError):
    """A simulator invariant was violated (a bug surface)."""


def _ns(seconds: float) -> int:
    return int(round(seconds * 1e9))


# --------------------------------------------------------------- timeline
@dataclass(frozen=True)
class Event:
    start_ns: int
    end_ns: int
    stream: str
    kind: str            # transfer | refetch | op | gate | non_moe | predict
    seq: int
    layer: int = -1
    expert: int = -1
    token: int = -1      # decode token index; -1 for prefill
    phase: str = ""

    def to_dict(self) -> dict:
        return asdict(self)


class EventTimeline:
    """Ordered interval events per stream."""

    def __init__(self):
        self.events: list[Event] = []
        self.cache_log: list = []         # filled by simulate_request (B200 addition)

    def add(self, stream: str, kind: str, start: int, end: int, **payload) -> Event:
        if stream not in _PRIO:
            raise SimulationError(f"unknown stream {stream!r}")
        if end < start:
            raise SimulationError(f"{kind} ends before it starts ({start} > {end})")
        ev = Event(int(start), int(end), stream, kind, len(self.events), **payload)
        self.events.append(ev)
        return ev

    def ordered(self) -> list[Event]:
        return sorted(self.events, key=lambda e: (e.start_ns, _PRIO[e.stream], e.seq))

    def points(self) -> list[tuple]:
        """Flattened (time, stream, kind_start|kind_end, seq) in tie-break order."""
        pts = []
        for e in self.events:
            pts.append((e.start_ns, _PRIO[e.stream], e.seq, 0, e.stream, e.kind + "_start"))
            pts.append((e.end_ns, _PRIO[e.stream], e.seq, 1, e.stream, e.kind + "_end"))
        pts.sort(key=lambda p: (p[0], p[3], p[1], p[2]))
        return [(p[0], p[4], p[5], p[2]) for p in pts]

    def check(self, slots: int | None = None) -> None:
        """stream seriality, weight correctness, fetch-once."""
        by_stream: dict = {}
        for e in self.events:
            by_stream.setdefault(e.stream, []).append(e)
        for s, evs in by_stream.items():
            evs = sorted(evs, key=lambda e: (e.start_ns, e.seq))
            for a, b in zip(evs, evs[1:]):
                if b.start_ns < a.end_ns:
                    raise SimulationError(f"stream {s}: {a.kind}@{a.start_ns}-{a.end_ns} overlaps "
                                          f"{b.kind}@{b.start_ns}")
        arrived: dict = {}
        fetched_prefill: dict = {}
        for e in self.events:
            if e.kind in ("transfer", "refetch"):
                key = (e.phase, e.token, e.layer, e.expert)
                arrived[key] = min(arrived.get(key, e.end_ns), e.end_ns)
                if e.phase == "prefill":
                    k2 = (e.layer, e.expert)
                    fetched_prefill[k2] = fetched_prefill.get(k2, 0) + 1
                    if fetched_prefill[k2] > 1:
                        raise SimulationError(f"prefill layer {e.layer}: expert {e.expert} fetched twice")
        for e in self.events:
            if e.kind == "op":
                t = arrived.get((e.phase, e.token, e.layer, e.expert))
                if t is None or t > e.start_ns:
                    raise SimulationError(f"{e.phase} token {e.token} layer {e.layer}: expert {e.expert} "
                                          f"computes at {e.start_ns} before its weights arrived ({t})")

    def to_jsonl(self) -> str:
        return "".join(json.dumps(e.to_dict(), sort_keys=True, separators=(",", ":")) + "\n"
                       for e in self.ordered())


# ------------------------------------------------------------ expert cache
class DeviceExpertCache:
    """slot_count slots; each holds one (layer, expert) from the start of its
    transfer (loading) through ready and in_use until its last compute ends
    (SPEC.md:345-349).  A slot is handed to the next transfer only at or after
    its release time, so |resident| <= slot_count holds at every instant."""

    def __init__(self, slots: int):
        if slots < 1:
            raise SimulationError("the expert cache needs at least one slot")
        self.slot_count = slots
        self.free_at = [0] * slots                 # release time of each slot's current tenant
        self.tenant: list = [None] * slots
        self.history: list = []                    # (slot, key, t_load, t_ready, t_release)

    def acquire(self, bank: range | None = None) -> tuple[int, int]:
        """Earliest-released slot (lowest index on ties) -> (slot, release time)."""
        idx = range(self.slot_count) if bank is None else bank
        s = min(idx, key=lambda i: (self.free_at[i], i))
        return s, self.free_at[s]

    def load(self, slot: int, key: tuple, t_load: int, t_ready: int) -> None:
        if t_load < self.free_at[slot]:
            raise SimulationError(f"slot {slot} reused at {t_load} before its release {self.free_at[slot]}")
        self.tenant[slot] = key
        self.history.append([slot, key, t_load, t_ready, t_ready])
        self.free_at[slot] = t_ready

    def use(self, slot: int, t_end: int) -> None:
        """An op on the slot's expert ends at t_end (extends its residency)."""
        self.free_at[slot] = max(self.free_at[slot], t_end)
        self.history[self._last(slot)][4] = self.free_at[slot]

    def _last(self, slot: int) -> int:
        for i in range(len(self.history) - 1, -1, -1):
            if self.history[i][0] == slot:
                return i
        raise SimulationError(f"slot {slot} never loaded")

    def max_resident(self) -> int:
        pts = []
        for _, _, t0, _, t1 in self.history:
            pts.append((t0, 1))
            pts.append((t1, -1))
        pts.sort(key=lambda p: (p[0], p[1]))
        cur = best = 0
        for _, d in pts:
            cur += d
            best = max(best, cur)
        return best


# ----------------------------------------------------------------- metrics
@dataclass
class RequestMetrics:
    request_id: int
    ttft_s: float
    e2e_s: float
    decode_tokens: int
    throughput_tokens_per_s: float
    peak_mem_bytes: int
    prefetch_hits: int
    prefetch_misses: int
    refetch_count: int
    link_busy_s: float = 0.0
    link_bytes: int = 0

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass
class SimReport:
    policy: str
    seed: int
    config_digest: str
    requests: list = field(default_factory=list)

    def aggregates(self) -> dict:
        if not self.requests:
            return {}
        keys = ("ttft_s", "e2e_s", "throughput_tokens_per_s")
        return {f"mean_{k}": float(np.mean([getattr(r, k) for r in self.requests])) for k in keys}

    def throughput_cdf(self) -> list:
        v = np.array([r.throughput_tokens_per_s for r in self.requests], dtype=np.float64)
        return [float(x) for x in np.percentile(v, np.arange(101))] if v.size else []

    def to_dict(self) -> dict:
        return {"schema_version": 1, "policy": self.policy, "seed": self.seed,
                "config_digest": self.config_digest, "requests": [r.to_dict() for r in self.requests],
                "aggregates": self.aggregates(), "throughput_cdf": self.throughput_cdf()}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2) + "\n"


def compute_peak_memory(policy, cfg: ModelConfig) -> int:
    """non_moe + slot_count * expert_bytes + predictor (DuoServe) + kv reserve
    (SPEC.md:392-400).  Mixtral-8x7B preset, duoserve: 3.909 GB."""
    p = SchedulerPolicy(policy)
    pred = cfg.predictor_mem_bytes if p.needs_predictor else 0
    return cfg.non_moe_bytes + slot_count(p, cfg) * cfg.expert_bytes + pred + cfg.kv_reserve_bytes


def gpu_only_memory(cfg: ModelConfig) -> int:
    return cfg.total_param_bytes + cfg.kv_reserve_bytes


# ----------------------------------------------------------------- engine
class _State:
    """Mutable per-request simulation state: stream clocks, cache, log."""

    def __init__(self, policy: SchedulerPolicy, cfg: ModelConfig, cost: CostModel,
                 prefill_non_moe_s: float | None = None, cancel_chunk_bytes: int | None = None):
        self.policy, self.cfg, self.cost = policy, cfg, cost
        # B200 extension (engine.LinkQueue): a prefetch the gate proves wrong is
        # cancelled after its in-flight chunk instead of completing (SPEC.md:429
        # models no cancellation; None keeps the SPEC semantics)
        self.cancel_ns = None if cancel_chunk_bytes is None else _ns(
            cost.link_latency_s + min(cancel_chunk_bytes, cfg.expert_bytes) / cost.link_bandwidth_bytes_per_s)
        self.lazy: list = []           # cancel mode: (expert, earliest start) of the next layer's prefetch
        self.tl = EventTimeline()
        self.cache = DeviceExpertCache(slot_count(policy, cfg))
        self.t_compute = 0
        self.t_link = 0
        self.t_predict = 0
        self.T = _ns(cost.transfer_time_s(cfg.expert_bytes))
        self.nm = _ns(cost.non_moe_compute_per_layer_s)
        # B200 extension: the reference CostModel has one non-MoE time per layer;
        # a calibrated model may give the (T-token) prefill pass its own
        self.nm_prefill = self.nm if prefill_non_moe_s is None else _ns(prefill_non_moe_s)
        self.gate = _ns(cost.gate_compute_s)
        self.pred = _ns(cost.predictor_latency_s)
        self.log: list = []
        self.hits = self.misses = self.refetches = 0
        self.link_busy = 0
        self.link_bytes = 0
        self.visit = 0                 # PrefetchAll layer-visit counter (bank = visit % 2)
        self.pending: dict = {}        # decode prefetch of the next layer: expert -> (slot, ready)

    def C(self, n_tokens: int) -> int:
        return _ns(self.cost.expert_compute_base_s + n_tokens * self.cost.expert_compute_per_token_s)

    def transfer(self, key: tuple, earliest: int, kind: str, bank: range | None = None,
                 slot: int | None = None, **payload) -> tuple[int, int]:
        if slot is None:
            slot, free = self.cache.acquire(bank)
        else:
            free = self.cache.free_at[slot]
        start = max(self.t_link, earliest, free)
        end = start + self.T
        self.tl.add("comm", kind, start, end, expert=key[1], layer=key[0], **payload)
        self.cache.load(slot, key, start, end)
        self.t_link = end
        self.link_busy += self.T
        self.link_bytes += self.cfg.expert_bytes
        return slot, end

    def compute(self, slot: int, ready: int, earliest: int, dur: int, **payload) -> int:
        start = max(self.t_compute, ready, earliest)
        end = start + dur
        self.tl.add("compute", "op", start, end, **payload)
        self.cache.use(slot, end)
        self.t_compute = end
        return end

    def non_moe_and_gate(self, **payload) -> tuple[int, int]:
        t0 = self.t_compute
        nm = self.nm_prefill if payload.get("phase") == "prefill" else self.nm
        self.tl.add("compute", "non_moe", t0, t0 + nm, **payload)
        self.tl.add("compute", "gate", t0 + nm, t0 + nm + self.gate, **payload)
        self.t_compute = t0 + nm + self.gate
        return t0, self.t_compute


def schedule_prefill_layer(st: _State, l: int, activated: dict) -> dict:
    """One prefill MoE layer.  activated: expert -> number
    of routed (token, slot) rows.  Returns the layer's cache-log record."""
    pol = st.policy
    M = st.cfg.num_experts
    A = sorted(activated)
    t0, g = st.non_moe_and_gate(layer=l, phase="prefill")
    if pol in (SchedulerPolicy.DUOSERVE, SchedulerPolicy.DUOSERVE_ORACLE):
        # the first transfer (expert 0, speculative) overlaps the non-MoE compute;
        # the rest of A_l streams ascending, one fetch each (fetch-once)
        fetch = [0] + [e for e in A if e != 0]
        for i, e in enumerate(fetch):
            if i == 0 and e not in activated and st.cancel_ns is not None:
                # B200 extension: the speculative first transfer is dropped one
                # chunk after the gate proves it unneeded (log unchanged)
                slot, free = st.cache.acquire()
                start = max(st.t_link, t0, free)
                end = max(start, min(start + st.T, g + st.cancel_ns))
                st.tl.add("comm", "cancelled", start, end, expert=e, layer=l, phase="prefill")
                st.cache.load(slot, (l, e), start, end)
                st.t_link = end
                st.link_busy += end - start
                st.link_bytes += int(round(st.cfg.expert_bytes * (end - start) / st.T))
                continue
            slot, ready = st.transfer((l, e), t0 if i == 0 else g, "transfer", phase="prefill")
            if e in activated:
                st.compute(slot, ready, g, st.C(activated[e]), layer=l, expert=e, phase="prefill")
    elif pol is SchedulerPolicy.ON_DEMAND:
        fetch = A
        for e in A:   # serial fetch-then-compute after the gate
            slot, ready = st.transfer((l, e), max(g, st.t_compute), "transfer", phase="prefill")
            st.compute(slot, ready, g, st.C(activated[e]), layer=l, expert=e, phase="prefill")
    else:  # PREFETCH_ALL: all M experts of every layer visit, eagerly, into bank visit % 2
        fetch = list(range(M))
        _prefetchall_visit(st, l, activated, g, phase="prefill")
    return {"phase": "prefill", "layer": l, "fetch": fetch, "activated": A}


def _prefetchall_visit(st: _State, l: int, activated: dict, g: int, **payload) -> None:
    M = st.cfg.num_experts
    bank = range((st.visit % 2) * M, (st.visit % 2) * M + M)
    st.visit += 1
    slots = {}
    for e in range(M):
        slots[e] = st.transfer((l, e), 0, "transfer", bank=bank, **payload)
    for e in sorted(activated):
        slot, ready = slots[e]
        st.compute(slot, ready, g, st.C(activated[e]), layer=l, expert=e, **payload)
    for e in range(M):   # the whole bank stays resident until the visit's compute is done
        st.cache.use(slots[e][0], st.t_compute)


def schedule_decode_layer(st: _State, t: int, l: int, E: tuple, P_next: tuple | None,
                          pred_ready: int | None = None) -> dict:
    """One decode layer of token t.  E: the gate's true
    selection; the prediction for this layer (if any) was prefetched into
    st.pending during layer l-1.  P_next: the prediction for layer l+1 (None
    at the last layer / for non-predicting policies).  Returns the log record."""
    pol = st.policy
    k = len(E)
    E = tuple(sorted(E))
    t0, g = st.non_moe_and_gate(layer=l, token=t, phase="decode")
    kw = dict(token=t, phase="decode")
    if pol is SchedulerPolicy.PREFETCH_ALL:
        _prefetchall_visit(st, l, {e: 1 for e in E}, g, **kw)
        return {"phase": "decode", "token": t, "layer": l, "fetch": list(range(st.cfg.num_experts)),
                "kind": "prefetchall"}
    if pol is SchedulerPolicy.ON_DEMAND:
        for e in E:   # serial fetch-then-compute (ACC)
            slot, ready = st.transfer((l, e), max(g, st.t_compute), "transfer", **kw)
            st.compute(slot, ready, g, st.C(1), layer=l, expert=e, **kw)
        return {"phase": "decode", "token": t, "layer": l, "fetch": list(E), "kind": "ondemand"}

    # DuoServe / oracle
    if l == 0:
        # layer 0: fetched after the gate, not predicted
        ready = {e: st.transfer((l, e), g, "transfer", **kw) for e in E}
        rec = {"phase": "decode", "token": t, "layer": l, "fetch": list(E), "kind": "ondemand"}
    else:
        if st.cancel_ns is not None:
            _place_cancellable(st, l, E, g, kw)
        pf = st.pending
        P = tuple(sorted(pf))
        hit = [e for e in E if e in pf]
        miss = [e for e in E if e not in pf]
        wrong = [e for e in P if e not in E]
        st.hits += len(hit)
        st.misses += len(miss)
        st.refetches += len(miss)
        ready = {e: pf[e] for e in hit}
        # sync point 1: each wrong slot is re-fetched with the right expert (blocking)
        for e, w in zip(miss, wrong):
            ready[e] = st.transfer((l, e), g, "refetch", slot=pf[w][0], **kw)
        rec = {"phase": "decode", "token": t, "layer": l, "pred": list(P), "gate": list(E), "refetch": miss}
    # correct prefetched experts compute immediately; re-fetched ones when they land
    for e in sorted(E, key=lambda e: (ready[e][1], e)):
        slot, rdy = ready[e]
        st.compute(slot, rdy, g, st.C(1), layer=l, expert=e, **kw)
    st.pending = {}
    if P_next is not None:
        # prediction for l+1 on its own stream, from the gate of layer l;
        # sync point 2: its prefetch starts when the prediction is done, the
        # link is free and a slot has been released
        p0 = max(st.t_predict, g)
        p1 = p0 + (st.pred if pred_ready is None else pred_ready)
        st.tl.add("predict", "predict", p0, p1, layer=l + 1, **kw)
        st.t_predict = p1
        if st.cancel_ns is not None:
            st.lazy = [(e, p1) for e in sorted(P_next)]      # placed at the next gate
        else:
            for e in sorted(P_next):
                st.pending[e] = st.transfer((l + 1, e), p1, "transfer", **kw)
    return rec


def _place_cancellable(st: _State, l: int, E: tuple, g: int, kw: dict) -> None:
    """Place layer l's prefetches on the link knowing the gate time g: a
    correct one runs to completion; a wrong one stops one chunk after the gate
    (or never starts if the link reached it only after the gate)."""
    st.pending = {}
    taken: set = set()
    for e, earliest in st.lazy:
        c = st.cache
        slot = min((i for i in range(c.slot_count) if i not in taken), key=lambda i: (c.free_at[i], i))
        free = c.free_at[slot]
        taken.add(slot)
        start = max(st.t_link, earliest, free)
        if e in E:
            end = start + st.T
            kind = "transfer"
        elif start >= g:
            st.pending[e] = (slot, start)          # never issued: its slot takes the re-fetch
            continue
        else:
            end = min(start + st.T, g + st.cancel_ns)
            kind = "cancelled"
        st.tl.add("comm", kind, start, end, expert=e, layer=l, **kw)
        st.cache.load(slot, (l, e), start, end)
        st.t_link = end
        st.link_busy += end - start
        st.link_bytes += int(round(st.cfg.expert_bytes * (end - start) / st.T))
        st.pending[e] = (slot, end)
    st.lazy = []


def _requests(traces) -> list:
    by: dict = {}
    for tr in traces:
        by.setdefault(tr.request_id, []).append(tr)
    out = []
    for rid in sorted(by):
        trs = by[rid]
        pre = sorted([x for x in trs if x.phase == "prefill"], key=lambda x: x.token_index)
        dec = sorted([x for x in trs if x.phase == "decode"], key=lambda x: x.token_index)
        out.append((rid, pre, dec))
    return out


def simulate_request(policy, traces, cfg: ModelConfig, cost: CostModel, net=None, pop=None, aff=None,
                     seed: int = 0, check: bool = True, prefill_non_moe_s: float | None = None,
                     cancel_chunk_bytes: int | None = None, return_log: bool = False):
    """Simulate one request (its prefill + decode traces) under a policy.

    net: a predictor object with ``predict(trace, l) -> tuple`` (the
    reference protocol, predictor.py:424-510); required by ``duoserve``;
    ``oracle`` predicts the true selection with zero prediction latency.
    prefill_non_moe_s: optional non-MoE time of a prefill layer (B200
    calibration; default: cost.non_moe_compute_per_layer_s as in the SPEC).
    cancel_chunk_bytes: model the B200 runtime's cancellable chunked prefetch
    (a wrong prefetch stops one chunk after the gate); None = SPEC semantics.
    Returns (RequestMetrics, EventTimeline) as SPEC.md:365 specifies; with
    return_log=True also the cache log (a third element), which the timeline
    carries as ``EventTimeline.cache_log`` in either case."""
    pol = SchedulerPolicy(policy)
    traces = list(traces)
    reqs = _requests(traces)
    if len(reqs) != 1:
        raise TraceError(f"simulate_request needs exactly one request, got {len(reqs)}")
    rid, pre, dec = reqs[0]
    if not dec:
        raise TraceError(f"request {rid}: at least one decode token is required")
    if not pre:
        raise TraceError(f"request {rid}: no prefill tokens")
    L, M, k = cfg.num_layers, cfg.num_experts, cfg.top_k
    for tr in traces:
        tr.validate(L, M, k)
    if pol is SchedulerPolicy.DUOSERVE:
        if net is None:
            raise ConfigError("policy duoserve needs a predictor")
        if hasattr(net, "input_dim") and not hasattr(net, "predict"):
            raise ConfigError("pass a predictor object (MLPPredictor / PrecomputedPredictor), not a raw network")
    st = _State(pol, cfg, cost, prefill_non_moe_s, cancel_chunk_bytes)
    for l in range(L):
        act: dict = {}
        for tr in pre:
            for e in tr.path[l]:
                act[e] = act.get(e, 0) + 1
        st.log.append(schedule_prefill_layer(st, l, act))
    ttft = st.t_compute
    for tr in dec:
        for l in range(L):
            P_next = None
            if pol in (SchedulerPolicy.DUOSERVE, SchedulerPolicy.DUOSERVE_ORACLE) and l + 1 < L:
                if pol is SchedulerPolicy.DUOSERVE:
                    P_next = tuple(int(e) for e in net.predict(tr, l + 1))
                else:
                    P_next = tuple(tr.path[l + 1])
            st.log.append(schedule_decode_layer(st, tr.token_index, l, tr.path[l], P_next,
                                                pred_ready=0 if pol is SchedulerPolicy.DUOSERVE_ORACLE
                                                else None))
    e2e = st.t_compute
    if check:
        st.tl.check()
        if st.cache.max_resident() > st.cache.slot_count:
            raise SimulationError("resident set exceeded the slot count")
    n_dec = len(dec)
    m = RequestMetrics(request_id=rid, ttft_s=ttft / 1e9, e2e_s=e2e / 1e9, decode_tokens=n_dec,
                       throughput_tokens_per_s=n_dec / ((e2e - ttft) / 1e9),
                       peak_mem_bytes=compute_peak_memory(pol, cfg), prefetch_hits=st.hits,
                       prefetch_misses=st.misses, refetch_count=st.refetches, link_busy_s=st.link_busy / 1e9,
                       link_bytes=st.link_bytes)
    st.tl.cache_log = st.log
    if return_log:
        return m, st.tl, st.log
    return m, st.tl


def config_digest(cfg: ModelConfig, cost: CostModel) -> str:
    return hashlib.sha256(config_to_json(cfg, cost).encode()).hexdigest()[:16]


def run_experiment(policies, dataset: TraceDataset, cfg: ModelConfig, cost: CostModel, net=None,
                   seed: int = 0) -> dict:
    """SimReport per policy over the same requests."""
    if not dataset.traces:
        raise TraceError("empty dataset")
    reports = {}
    for p in policies:
        pol = SchedulerPolicy(p)
        rep = SimReport(policy=pol.value, seed=seed, config_digest=config_digest(cfg, cost))
        for rid, pre, dec in _requests(dataset.traces):
            m, _ = simulate_request(pol, pre + dec, cfg, cost, net=net, seed=seed)
            rep.requests.append(m)
        reports[pol.value] = rep
    return reports
