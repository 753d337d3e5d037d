"""The paper's preprocess loop, run on the serving device (PAPER.md:106-148,
277: "data collection and inference serving ... simultaneously"; the
predictor "executable on the same device").

    collect_routing   serve prompts through an Engine with on-demand (ACC-like)
                      scheduling — the paper's collection schedule, PAPER.md:277 —
                      recording every token's routing path as ActivationTraces
                      (trace.py:30-126 wire format) while the gate's device
                      counters (OnlineRoutingStats, stats.py:52-71) accumulate
                      popularity / affinity;
    preprocess        collect -> pop/aff from the device counters -> split by
                      request -> train the ExpertMLP on the GPU (training.py,
                      predictor.py:339-370) -> held-out hit rates in the
                      paper's Table 3 format -> the
                      (net, pop, aff) triple the DuoServe engine serves with.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .predictor import ExpertMLP, HitRateReport, evaluate
from .stats import AffinityMatrix, PopularityMatrix
from .trace import DECODE, PREFILL, ActivationTrace, TraceDataset, split_dataset
from .training import TrainReport, train


def engine_traces(eng, request_id: int) -> list:
    """The last request served by `eng` as ActivationTraces: prefill tokens at
    positions 0..T-1, decode tokens after them (the gate emits sorted k-tuples)."""
    out = []
    pre = eng.paths_prefill
    if pre is None:
        raise ValueError("engine_traces: the engine has not served a prefill")
    T = pre.shape[0]
    for t in range(T):
        out.append(ActivationTrace(request_id, PREFILL, t, tuple(tuple(int(e) for e in pre[t, l])
                                                                  for l in range(pre.shape[1]))))
    for i, path in enumerate(eng.paths_decode):
        out.append(ActivationTrace(request_id, DECODE, T + i, tuple(tuple(int(e) for e in s) for s in path)))
    return out


def collect_routing(eng, prompts, decode_len: int, first_request_id: int = 0) -> TraceDataset:
    """Serve every prompt (prefill + decode_len tokens) and return the routing
    of all their tokens; the engine's online counters (if enabled) see the
    same selections."""
    traces = []
    for i, ids in enumerate(prompts):
        eng.reset()
        eng.generate(ids, decode_len + 1)
        traces += engine_traces(eng, first_request_id + i)
    return TraceDataset(eng.shape.name, eng.L, eng.M, eng.k, traces,
                        provenance={"kind": "served", "policy": eng.policy.value, "requests": len(prompts),
                                    "decode_len": decode_len})


@dataclass
class PreprocessResult:
    net: ExpertMLP
    pop: PopularityMatrix
    aff: AffinityMatrix
    train_report: TrainReport
    held_out: HitRateReport | None
    held_out_decode: HitRateReport | None
    timings_s: dict = field(default_factory=dict)
    n_traces: int = 0

    def table(self, model: str, dataset: str = "synthetic prompts") -> dict:
        """One row of the paper's predictor hit-rate table."""
        row = {"model": model, "dataset": dataset}
        for name, rep in (("all_tokens", self.held_out), ("decode_tokens", self.held_out_decode)):
            if rep is not None:
                row[name] = {"top2": round(rep.topk_hit_rate, 4), "at_least_one": round(rep.at_least_one_rate, 4),
                             "n": rep.n_evaluated}
        return row


def preprocess(eng, prompts, decode_len: int, epochs: int = 20, train_fraction: float = 0.75, seed: int = 0,
               batch_size: int = 256, learning_rate: float = 1e-3, hidden=None) -> PreprocessResult:
    """Collect on `eng` (built with collect_stats=True; any policy), derive
    pop/aff from its device counters, train on the requests of the training
    split and evaluate on the held-out requests."""
    if eng.route_stats is None:
        raise ValueError("preprocess needs an Engine built with collect_stats=True")
    t0 = time.time()
    eng.route_stats.reset()
    ds = collect_routing(eng, prompts, decode_len)
    t1 = time.time()
    pop, aff = eng.route_stats.matrices()                     # int64 device counts -> stats.py normalisation
    tr, te = split_dataset(ds, train_fraction, seed) if len(prompts) > 1 else (ds, None)
    net, rep = train(tr, pop, aff, epochs=epochs, batch_size=batch_size, learning_rate=learning_rate, seed=seed,
                     hidden=hidden, device=eng.device)
    t2 = time.time()
    held = held_dec = None
    if te is not None and te.traces:
        held = evaluate(net, te, pop, aff)
        dec = te.filter_phase(DECODE) if hasattr(te, "filter_phase") else None
        if dec is not None and dec.traces:
            held_dec = evaluate(net, dec, pop, aff)
    # the batched evaluation sized the cached device net's workspace for
    # thousands of rows; drop it so the serving engine starts from a fresh one
    net.invalidate_device()
    t3 = time.time()
    return PreprocessResult(net=net, pop=pop, aff=aff, train_report=rep, held_out=held, held_out_decode=held_dec,
                            timings_s={"collect": round(t1 - t0, 2), "train": round(t2 - t1, 2),
                                       "evaluate": round(t3 - t2, 2)},
                            n_traces=len(ds.traces))


def rank_popular(pop: PopularityMatrix, experts=None) -> list:
    """(layer, expert) pairs by descending popularity (ties: lower layer, then
    lower expert) — the residency-budget policy's pin order."""
    vals = np.asarray(pop.values, dtype=np.float64)
    L, M = vals.shape
    experts = range(M) if experts is None else experts
    return sorted(((l, e) for l in range(L) for e in experts), key=lambda le: (-vals[le[0], le[1]], le))
