"""Request-level parity checker (TEST INFRASTRUCTURE — called only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline/checker leg, never by the
product path).

Given what the B200 engine recorded while serving one request, recompute the
decisions on the CPU and compare them bit for bit:

  routing   teacher forced: the GPU's gate input a (bf16) of every routed layer
            through oracle/routing_ref (HF MixtralTopKRouter semantics, fixed
            f64 order) -> indices must be equal; the top-k logit margin of any
            mismatch is reported
  sets      every decode prediction P_{t,l} (l >= 1) from the reference's
            predictor restated in oracle/predictor_ref (predictor.py:53-232,
            419-421, PrecomputedPredictor.from_net :480-510) on the engine's
            recorded paths
  log       the whole cache log from oracle/sim_ref (SPEC.md:374-391,
            411-428) driven by the recorded routing and those predictions

The contract is the north star's: routing indices, predicted expert sets and
cache hit/miss sequences bit-exact.
"""

from __future__ import annotations

import numpy as np

from . import predictor_ref, routing_ref, sim_ref


def _bits(t) -> np.ndarray:
    import torch
    return t.to(torch.bfloat16).contiguous().view(torch.int16).numpy().view(np.uint16)


def check_routing(capture, gate_weights, k: int) -> dict:
    """capture: engine.capture entries (phase, layer, a [T, d] bf16 host, idx [T, k]);
    gate_weights[l]: the layer's router weight [M, d] (bf16, any device)."""
    n_tok = n_bad = 0
    worst = None
    wg_bits = {}
    for phase, l, a, idx in capture:
        if l not in wg_bits:
            wg_bits[l] = _bits(gate_weights[l].cpu())
        lg = routing_ref.gate_logits(_bits(a), wg_bits[l])
        ref, _ = routing_ref.topk_route(lg, k)
        got = np.asarray(idx, dtype=np.int32).reshape(ref.shape)
        bad = np.nonzero((got != ref).any(axis=1))[0]
        n_tok += ref.shape[0]
        n_bad += bad.size
        for t in bad:
            s = np.sort(lg[t])[::-1]
            m = float(s[k - 1] - s[k])
            if worst is None or m > worst["margin"]:
                worst = {"phase": phase, "layer": int(l), "row": int(t), "margin": m}
    return {"routed_tokens": n_tok, "mismatches": n_bad, "worst_mismatch": worst}


def predictions(net: predictor_ref.RefNet, paths_decode, L: int, pop_values, aff_values, k: int,
                mode: str = "pool") -> list:
    """preds[t][l] (None at l = 0) for the recorded decode paths, batched."""
    if not paths_decode:
        return []
    rows = [(t, l) for t in range(len(paths_decode)) for l in range(1, L)]
    sets, _ = predictor_ref.predict_sets(net, [paths_decode[t] for t, _ in rows], [l for _, l in rows],
                                         pop_values, aff_values, k, mode)
    out = [[None] * L for _ in paths_decode]
    for (t, l), s in zip(rows, sets):
        out[t][l] = tuple(int(e) for e in s)
    return out


def expected_log(paths_prefill, paths_decode, L: int, preds, policy: str = "duoserve", pinned=None,
                 owned=None, M: int = 8) -> list:
    """sim_ref cache log for one served request (paths_prefill [T, L, k])."""
    pre = [tuple(tuple(int(e) for e in paths_prefill[t, l]) for l in range(L)) for t in range(paths_prefill.shape[0])]
    pins = set(pinned) if pinned else None
    return (sim_ref.cache_log_prefill(pre, L, policy, owned=owned, M=M, pinned=pins)
            + sim_ref.cache_log_decode(paths_decode, preds, L, policy, owned=owned, M=M, pinned=pins)[0])


def check_request(eng_log, paths_prefill, paths_decode, L: int, k: int, net=None, pop_values=None,
                  aff_values=None, policy: str = "duoserve", pinned=None, mode: str = "pool") -> dict:
    """Predicted sets and the cache log of one request vs the oracle."""
    preds = None
    n_pred = bad_pred = 0
    if policy == "duoserve":
        preds = predictions(net, paths_decode, L, pop_values, aff_values, k, mode)
        got = [r for r in eng_log if r["phase"] == "decode" and "pred" in r]
        want = [(t, l) for t in range(len(paths_decode)) for l in range(1, L)]
        n_pred = len(want)
        for r, (t, l) in zip(got, want):
            if (r["token"], r["layer"]) != (t, l) or r["pred"] != sorted(preds[t][l]):
                bad_pred += 1
        bad_pred += abs(len(got) - n_pred)
    exp = expected_log(paths_prefill, paths_decode, L, preds, policy, pinned=pinned)
    n_rec = max(len(exp), len(eng_log))
    bad_log = sum(1 for a, b in zip(eng_log, exp) if a != b) + abs(len(exp) - len(eng_log))
    return {"predicted_sets": n_pred, "set_mismatches": bad_pred, "log_records": n_rec, "log_mismatches": bad_log,
            "log_equal": bad_log == 0}


def check_request_batch(eng_log, paths_prefill, paths_decode_b, batch_sets, L: int, k: int, net=None,
                        pop_values=None, aff_values=None, policy: str = "duoserve", pinned=None,
                        mode: str = "pool") -> dict:
    """Batched serving (engine.BatchEngine): every sequence's prediction at
    every decode step and layer >= 1 vs the reference predictor on that
    sequence's recorded path, and the whole cache log vs sim_ref's batch
    extension (prefill: the union over all B*P tokens, exactly the
    single-sequence rule; decode: unions over the batch).
    paths_decode_b[t][b] = sequence b's path at step t; batch_sets = the
    engine's (layer, per-sequence predicted sets, per-sequence gate sets)."""
    T = len(paths_decode_b)
    B = len(paths_decode_b[0]) if T else 0
    preds_b = [[None] * B for _ in range(T)]
    n_pred = bad_pred = 0
    if policy == "duoserve" and T:
        for b in range(B):
            pb = predictions(net, [paths_decode_b[t][b] for t in range(T)], L, pop_values, aff_values, k, mode)
            for t in range(T):
                preds_b[t][b] = pb[t]
        want = [(t, l) for t in range(T) for l in range(1, L)]
        n_pred = len(want) * B
        for (layer, sets, _), (t, l) in zip(batch_sets, want):
            for b in range(B):
                if layer != l or tuple(sets[b]) != tuple(sorted(preds_b[t][b][l])):
                    bad_pred += 1
        bad_pred += abs(len(batch_sets) - len(want)) * B
    pre = [tuple(tuple(int(e) for e in paths_prefill[t, l]) for l in range(L)) for t in range(paths_prefill.shape[0])]
    pins = set(pinned) if pinned else None
    exp = (sim_ref.cache_log_prefill(pre, L, policy, pinned=pins)
           + sim_ref.cache_log_decode_batch(paths_decode_b, preds_b, L, policy, pinned=pins)[0])
    n_rec = max(len(exp), len(eng_log))
    bad_log = sum(1 for a, b in zip(eng_log, exp) if a != b) + abs(len(exp) - len(eng_log))
    return {"predicted_sets": n_pred, "set_mismatches": bad_pred, "log_records": n_rec, "log_mismatches": bad_log,
            "log_equal": bad_log == 0}
