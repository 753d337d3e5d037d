"""Expert-cache simulator semantics (oracle) — CPU restatement of the
reference's SPEC-only simulator module (
the module itself is not shipped).

Two parts:
 1. cache_log_*: the hit / miss / refetch decisions, a pure function of the
    routing (gate selections E), the predictions P and the policy — this is
    what the B200 runtime's log must equal bit for bit:
      * capacity = slot_count(policy) (config.py:101-114)
      * prefill: per layer the activated
        set A_l = union_t E_{t,l}; every activated expert is fetched exactly
        once ("fetch-once").  The runtime overlaps the first transfer with
        the preceding non-MoE compute by speculatively fetching
        the lowest-index expert (0) before the gate is known, then the rest of
        A_l ascending — restated here as fetch = [0] + sorted(A_l - {0}).
      * decode: layer 0 is fetched after
        the gate, not predicted; for l >= 1 hits = P & E, misses = E - P and
        each miss is re-fetched (blocking); prefetch_hits + prefetch_misses
        = k*(L-1) per token.
      * ondemand: fetch E after the gate every layer (prefill: A_l).
      * prefetchall (MoESys baseline): every layer visit
        transfers all M experts (ascending) into one of two banks of M slots
        (2M = slot_count), eagerly and in visit order, whatever the gate says.
 2. timeline_*: integer-nanosecond event model used to pin the SPEC's
    hand-traced fixtures (32/48/40 ms prefill, 20/30/25 ms
    decode).  Interpretation of sync point 2 with 2k slots: the next layer's
    prefetch starts once the prediction is done, the link is free and its
    slots are released (with the paper's k-slot cache the slot condition is
    "after the first expert's compute").
"""

from __future__ import annotations


def _sorted(x):
    return [int(e) for e in sorted(x)]


def cache_log_prefill(E_by_token, L: int, policy: str = "duoserve", owned=None, M: int = 8, pinned=None):
    """E_by_token: list over prefill tokens of L-tuples of selections.
    owned: expert ids of this rank under expert parallelism (None = all);
    the speculative first transfer is then the rank's lowest owned expert.
    M: experts per layer (used by prefetchall only).
    pinned: (layer, expert) pairs resident in HBM for the whole request
    (residency-budget extension): never fetched, no
    speculative transfer, listed under "pinned" when activated."""
    log = []
    for l in range(L):
        A = set()
        for path in E_by_token:
            A.update(path[l])
        mine = A if owned is None else A & set(owned)
        pins = {e for (ll, e) in (pinned or ()) if ll == l}
        cand = [e for e in (range(M) if owned is None else sorted(owned)) if e not in pins]
        first = cand[0] if cand else None
        if policy in ("duoserve", "oracle"):
            fetch = ([first] if first is not None else []) + _sorted(mine - pins - {first})
        elif policy == "ondemand":
            fetch = _sorted(mine - pins)
        elif policy == "prefetchall":
            fetch = list(range(M)) if owned is None else _sorted(owned)
        else:
            raise ValueError(policy)
        log.append({"phase": "prefill", "layer": l, "fetch": fetch, "activated": _sorted(A)})
        if pinned:
            log[-1]["pinned"] = _sorted(mine & pins)
    return log


def cache_log_decode(paths, preds, L: int, policy: str = "duoserve", owned=None, M: int = 8, pinned=None):
    """paths[t][l] = gate selection of decode token t at layer l;
    preds[t][l] = predicted set for l >= 1 (ignored for ondemand/prefetchall).
    owned: expert ids of this rank under expert parallelism (None = all).
    M: experts per layer (used by prefetchall only).
    pinned: (layer, expert) pairs resident in HBM (see cache_log_prefill): never
    fetched or re-fetched, not counted as prefetch hits / misses."""
    own = None if owned is None else set(owned)
    keep = (lambda xs: _sorted(xs)) if own is None else (lambda xs: _sorted(set(xs) & own))
    log = []
    hits = misses = refetches = 0
    for t, path in enumerate(paths):
        for l in range(L):
            E = _sorted(path[l])
            pins = {e for (ll, e) in (pinned or ()) if ll == l}
            extra = {"pinned": _sorted(set(keep(E)) & pins)} if pinned else {}
            if policy == "prefetchall":
                log.append({"phase": "decode", "token": t, "layer": l,
                            "fetch": list(range(M)) if own is None else _sorted(own), "kind": "prefetchall"})
                continue
            if l == 0 or policy == "ondemand":
                log.append({"phase": "decode", "token": t, "layer": l,
                            "fetch": [e for e in keep(E) if e not in pins], "kind": "ondemand", **extra})
                continue
            P = keep(preds[t][l])
            Ed = set(keep(E)) - pins
            miss = _sorted(Ed - set(P))
            hits += len(Ed & set(P))
            misses += len(miss)
            refetches += len(miss)
            log.append({"phase": "decode", "token": t, "layer": l, "pred": P, "gate": E, "refetch": miss, **extra})
    return log, {"prefetch_hits": hits, "prefetch_misses": misses, "refetch_count": refetches}


def cache_log_decode_batch(paths_b, preds_b, L: int, policy: str = "duoserve", pinned=None):
    """Batch extension of cache_log_decode (a build extension: the SPEC's
    simulator excludes batching).  paths_b[t][b][l] = gate
    selection of sequence b at decode step t, layer l; preds_b[t][b][l] =
    its predicted set (l >= 1).  Per (t, l) the activated set is the union of
    the B selections and the predicted set the union of the B predictions;
    the record is then formed exactly as for one sequence:
      l = 0 (or ondemand): fetch the union (minus pinned experts);
      l >= 1: pred = union of predictions, gate = union of selections,
              refetch = gate minus pinned minus pred."""
    log = []
    hits = misses = 0
    for t, step in enumerate(paths_b):
        for l in range(L):
            A = _sorted({e for path in step for e in path[l]})
            pins = {e for (ll, e) in (pinned or ()) if ll == l}
            extra = {"pinned": _sorted(set(A) & pins)} if pinned else {}
            if l == 0 or policy == "ondemand":
                log.append({"phase": "decode", "token": t, "layer": l, "fetch": [e for e in A if e not in pins],
                            "kind": "ondemand", **extra})
                continue
            P = _sorted({e for pr in preds_b[t] for e in pr[l]})
            Ed = set(A) - pins
            miss = _sorted(Ed - set(P))
            hits += len(Ed & set(P))
            misses += len(miss)
            log.append({"phase": "decode", "token": t, "layer": l, "pred": P, "gate": A, "refetch": miss, **extra})
    return log, {"prefetch_hits": hits, "prefetch_misses": misses}


def cache_log_ep_dispatch(prefill_paths_by_rank, decode_paths_by_rank, L: int, owned):
    """Expert parallelism with token dispatch (engine.BatchEngine(ep=...),
    ondemand): per layer visit the owner fetches the experts it owns that ANY
    rank's tokens selected, ascending.  prefill_paths_by_rank[r] = that rank's
    prefill token paths; decode_paths_by_rank[r][t][b] = its sequence b's path
    at decode step t."""
    own = set(owned)
    log = []
    for l in range(L):
        sel = {e for paths in prefill_paths_by_rank for p in paths for e in p[l]}
        log.append({"phase": "prefill", "layer": l, "fetch": _sorted(sel & own), "kind": "ep-dispatch"})
    steps = len(decode_paths_by_rank[0])
    for t in range(steps):
        for l in range(L):
            sel = {e for rk in decode_paths_by_rank for p in rk[t] for e in p[l]}
            log.append({"phase": "decode", "token": t, "layer": l, "fetch": _sorted(sel & own), "kind": "ep-dispatch"})
    return log


# --------------------------------------------------------------------------
# integer-ns timelines for the SPEC fixtures

def timeline_prefill_layer(policy: str, n_act: int, T: int, C: int, non_moe: int, slots: int) -> int:
    """MoE-block time (end of last expert compute - end of non-MoE), ns."""
    t_moe = non_moe                       # non-MoE (and gate) runs [0, non_moe)
    link = 0
    comp = t_moe
    if policy == "ondemand":
        for _ in range(n_act):
            ready = comp + T              # fetch after the gate / previous compute, serial
            comp = ready + C
        return comp - t_moe
    ends = []
    for i in range(n_act):
        slot_free = ends[i - slots] if i >= slots else 0
        start = max(link, slot_free)      # first transfer overlaps non-MoE compute
        ready = start + T
        link = ready
        c0 = max(comp, ready, t_moe)
        comp = c0 + C
        ends.append(comp)
    return comp - t_moe


def timeline_decode(policy: str, n_layers: int, k: int, T: int, C: int, non_moe_gate: int,
                    miss_per_layer, pred_latency: int = 0):
    """Per-layer completion times of a decode token (ns); returns the list of
    layer durations.  Layer 0 fetches after the gate; layers >= 1 use the
    prefetch issued during the previous layer."""
    link = 0
    t = 0
    durations = []
    pf_ready = None        # time the prefetched experts of the next layer are resident
    for l in range(n_layers):
        start = t
        g = t + non_moe_gate
        if policy == "ondemand" or l == 0:
            comp = g
            if policy == "ondemand":
                for _ in range(k):
                    rdy = max(link, comp) + T
                    link = rdy
                    comp = rdy + C
                t = comp
                durations.append(t - start)
                continue
            link = max(link, g) + k * T
            ready = link
        else:
            ready = pf_ready
            m = miss_per_layer[l] if l < len(miss_per_layer) else 0
            if m:
                link = max(link, g) + m * T   # blocking re-fetch of the wrong slots
                ready = max(ready, link)
        # prediction for l+1 issued at g; prefetch starts when predicted, link free
        pred_done = g + pred_latency
        comp = max(g, ready)
        for _ in range(k):
            comp += C
        if l + 1 < n_layers and policy != "ondemand":
            link = max(link, pred_done) + k * T
            pf_ready = link
        t = comp
        durations.append(t - start)
    return durations
