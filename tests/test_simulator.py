"""The product simulator (paper_2509_07379_b200/simulator.py) — the reference's
SPEC-only ``duoserve.simulator`` — against the SPEC's
hand-traced fixtures, its memory example,
its invariants and properties, and the test oracle's cache
log (oracle/sim_ref.py, which Engine.log equals on the GPU)."""

import json

import numpy as np
import pytest

from oracle import sim_ref
from paper_2509_07379_b200 import config as C, simulator as S, trace as T
from paper_2509_07379_b200.predictor import OraclePredictor, PopularityPredictor, PrecomputedPredictor
from paper_2509_07379_b200 import stats as ST

MS = 1_000_000


def _cfg(L, expert_bytes=9_999_000, M=8, k=2):
    non_moe = 1000
    return C.ModelConfig(name="fixture", num_layers=L, num_experts=M, top_k=k,
                         total_param_bytes=non_moe + L * M * expert_bytes, non_moe_bytes=non_moe,
                         predictor_mem_bytes=10, kv_reserve_bytes=10)


def _cost(T_ms, C_ms, nm_ms, gate_ms=0.0001, pred_ms=0.0001, eb=9_999_000):
    # transfer = 1 us + eb / bw = T_ms exactly; op = base + 1 token * 1 ns
    bw = eb / (T_ms * 1e-3 - 1e-6)
    return C.CostModel(link_bandwidth_bytes_per_s=bw, link_latency_s=1e-6,
                       expert_compute_base_s=C_ms * 1e-3 - 1e-9, expert_compute_per_token_s=1e-9,
                       non_moe_compute_per_layer_s=nm_ms * 1e-3 - gate_ms * 1e-3, gate_compute_s=gate_ms * 1e-3,
                       predictor_latency_s=pred_ms * 1e-3)


def _req(prefill_paths, decode_paths, rid=0):
    return ([T.ActivationTrace(rid, "prefill", i, p) for i, p in enumerate(prefill_paths)] +
            [T.ActivationTrace(rid, "decode", len(prefill_paths) + i, p) for i, p in enumerate(decode_paths)])


def _moe_block(tl, layer, phase="prefill"):
    g = max(e.end_ns for e in tl.events if e.kind == "gate" and e.layer == layer and e.phase == phase)
    end = max(e.end_ns for e in tl.events if e.kind == "op" and e.layer == layer and e.phase == phase)
    return end - g


@pytest.mark.parametrize("policy,Tm,Cm,expect", [("duoserve", 10, 2, 32), ("oracle", 10, 2, 32),
                                                 ("ondemand", 10, 2, 48), ("duoserve", 2, 10, 40)])
def test_prefill_fixtures(policy, Tm, Cm, expect):
    """E_act = 4 (experts 0..3, one row each), non-MoE >= T."""
    cfg = _cfg(1)
    cost = _cost(Tm, Cm, nm_ms=10)
    reqs = _req([((0, 1),), ((2, 3),)], [((0, 1),)])
    net = OraclePredictor()
    _, tl, log = S.simulate_request(policy, reqs, cfg, cost, net=net, return_log=True)
    assert _moe_block(tl, 0) == expect * MS
    assert log[0]["fetch"] == [0, 1, 2, 3]


def _decode_layer_durations(tl, token):
    ends = []
    for l in range(max(e.layer for e in tl.events) + 1):
        ends.append(max(e.end_ns for e in tl.events
                        if e.kind == "op" and e.layer == l and e.phase == "decode" and e.token == token))
    return [b - a for a, b in zip(ends, ends[1:])]


class _OneMissAt:
    """Predicts the true set except at one layer, where one expert is wrong."""
    name = "one-miss"

    def __init__(self, layer, M=8):
        self.layer, self.M = layer, M

    def predict(self, trace, l):
        E = tuple(trace.path[l])
        if l != self.layer:
            return E
        wrong = next(e for e in range(self.M) if e not in E)
        return tuple(sorted((E[0], wrong)))


def test_decode_fixtures():
    """k=2, T=10 ms, C=2 ms, non-MoE+gate = 1 ms: full hit
    20 ms/layer (link-bound); one wrong expert +T = 30 ms; OnDemand 25 ms."""
    L = 8
    cfg = _cfg(L)
    cost = _cost(10, 2, nm_ms=1)
    path = tuple((2 * (l % 4), 2 * (l % 4) + 1) for l in range(L))
    reqs = _req([path], [path])
    m, tl, log = S.simulate_request("duoserve", reqs, cfg, cost, net=OraclePredictor(), return_log=True)
    d = _decode_layer_durations(tl, 1)
    assert d[2:] == [20 * MS] * (L - 3)
    assert m.prefetch_hits == 2 * (L - 1) and m.prefetch_misses == 0
    m, tl, log = S.simulate_request("duoserve", reqs, cfg, cost, net=_OneMissAt(4), return_log=True)
    d = _decode_layer_durations(tl, 1)
    assert d[3] == 30 * MS and d[4] == 20 * MS and d[5] == 20 * MS   # layers 3->4 carries the re-fetch
    assert m.refetch_count == 1 and m.prefetch_misses == 1 and m.prefetch_hits == 2 * (L - 1) - 1
    m, tl, log = S.simulate_request("ondemand", reqs, cfg, cost, return_log=True)
    assert _decode_layer_durations(tl, 1) == [25 * MS] * (L - 1)


def _dataset(L=6, M=8, n=4, seed=3, alpha=0.8):
    cfg = _cfg(L, M=M)
    return T.generate_traces(T.default_generator_params(L, M, alpha, seed), cfg, n, 6, 5), cfg


def test_cache_log_equals_oracle():
    """Decisions (fetch / hit / miss / re-fetch) equal oracle/sim_ref for every policy."""
    ds, cfg = _dataset()
    cost = _cost(10, 2, nm_ms=1)
    pop = ST.build_popularity(ds)
    pp = PopularityPredictor(pop, cfg.top_k)
    L = cfg.num_layers
    for rid, trs in ds.by_request().items():
        pre = [t for t in trs if t.phase == "prefill"]
        dec = sorted([t for t in trs if t.phase == "decode"], key=lambda t: t.token_index)
        for pol in ("duoserve", "oracle", "ondemand", "prefetchall"):
            _, _, log = S.simulate_request(pol, trs, cfg, cost, net=pp, return_log=True)
            exp = sim_ref.cache_log_prefill([t.path for t in pre], L, pol)
            preds = [[None] + [pp.predict(t, l) if pol == "duoserve" else t.path[l] for l in range(1, L)]
                     for t in dec]
            dl, _ = sim_ref.cache_log_decode([t.path for t in dec], preds, L, pol)
            for r in dl:
                if "token" in r:
                    r["token"] = dec[r["token"]].token_index
            assert log == exp + dl, pol


def test_invariants_and_metrics():
    ds, cfg = _dataset(n=3)
    cost = _cost(10, 2, nm_ms=1)
    pp = PopularityPredictor(ST.build_popularity(ds), cfg.top_k)
    for rid, trs in ds.by_request().items():
        for pol in ("duoserve", "oracle", "ondemand", "prefetchall"):
            m, tl = S.simulate_request(pol, trs, cfg, cost, net=pp)
            tl.check()                                   # seriality, weight-correctness, fetch-once
            assert m.ttft_s <= m.e2e_s and m.throughput_tokens_per_s > 0
            n_dec = sum(t.phase == "decode" for t in trs)
            if pol in ("duoserve", "oracle"):
                assert m.prefetch_hits + m.prefetch_misses == cfg.top_k * (cfg.num_layers - 1) * n_dec
            # e2e = TTFT + sum of decode-step durations (contiguous compute stream)
            ends = sorted({max(e.end_ns for e in tl.events
                               if e.stream == "compute" and e.phase == "decode" and e.token == t.token_index)
                           for t in trs if t.phase == "decode"})
            ttft = round(m.ttft_s * 1e9)
            steps = np.diff([ttft] + ends)
            assert (steps > 0).all() and ttft + int(steps.sum()) == round(m.e2e_s * 1e9)


def test_zero_decode_rejected():
    cfg = _cfg(2)
    with pytest.raises(T.TraceError):
        S.simulate_request("ondemand", _req([((0, 1), (2, 3))], []), cfg, _cost(10, 2, 1))
    with pytest.raises(C.ConfigError):
        S.simulate_request("duoserve", _req([((0, 1), (2, 3))], [((0, 1), (2, 3))]), cfg, _cost(10, 2, 1))


def test_oracle_dominance_and_monotonicity():
    """DuoServeOracle e2e <= OnDemand e2e on every request; a faster link never
    increases e2e."""
    ds, cfg = _dataset(n=20, seed=11)
    pp = PopularityPredictor(ST.build_popularity(ds), cfg.top_k)
    for Tm, Cm in [(10, 2), (2, 10), (5, 5)]:
        cost = _cost(Tm, Cm, nm_ms=1)
        fast = _cost(Tm / 2, Cm, nm_ms=1)
        for rid, trs in ds.by_request().items():
            o = S.simulate_request("oracle", trs, cfg, cost)[0]
            od = S.simulate_request("ondemand", trs, cfg, cost)[0]
            assert o.e2e_s <= od.e2e_s
            for pol in ("duoserve", "oracle", "ondemand", "prefetchall"):
                assert S.simulate_request(pol, trs, cfg, fast, net=pp)[0].e2e_s <= \
                    S.simulate_request(pol, trs, cfg, cost, net=pp)[0].e2e_s


def test_capacity_never_exceeded():
    """|resident| <= slot_count at every event time (simulate_request checks it
    and raises SimulationError); here also re-derived from the cache history."""
    ds, cfg = _dataset(n=2)
    pp = PopularityPredictor(ST.build_popularity(ds), cfg.top_k)
    for pol in ("duoserve", "ondemand", "prefetchall"):
        for rid, trs in ds.by_request().items():
            st = S._State(C.SchedulerPolicy(pol), cfg, _cost(3, 7, 1))
            S.schedule_prefill_layer(st, 0, {0: 3, 5: 1, 6: 2})
            assert st.cache.max_resident() <= st.cache.slot_count == C.slot_count(pol, cfg)
            S.simulate_request(pol, trs, cfg, _cost(3, 7, 1), net=pp)


def test_peak_memory_and_ordering():
    cfg, _ = C.load_preset("mixtral-8x7b")
    assert abs(S.compute_peak_memory("duoserve", cfg) / 1e9 - 3.909) < 1e-3
    assert S.compute_peak_memory("ondemand", cfg) < S.compute_peak_memory("duoserve", cfg) < \
        S.compute_peak_memory("prefetchall", cfg)
    assert S.gpu_only_memory(cfg) > S.compute_peak_memory("prefetchall", cfg)


def test_run_experiment_deterministic_and_ordered():
    ds, cfg = _dataset(n=8, seed=5)
    cost = _cost(10, 2, nm_ms=1)
    pp = PrecomputedPredictor({(t.request_id, t.token_index, l): tuple(t.path[l])
                               for t in ds.traces for l in range(1, cfg.num_layers)})
    a = S.run_experiment(["duoserve", "ondemand", "prefetchall"], ds, cfg, cost, net=pp, seed=1)
    b = S.run_experiment(["duoserve", "ondemand", "prefetchall"], ds, cfg, cost, net=pp, seed=1)
    assert all(a[p].to_json() == b[p].to_json() for p in a)
    doc = json.loads(a["duoserve"].to_json())
    assert len(doc["throughput_cdf"]) == 101 and len(doc["requests"]) == 8
    # perfect predictions, link-bound: DuoServe beats both baselines on every request
    for rd, ro, rp in zip(a["duoserve"].requests, a["ondemand"].requests, a["prefetchall"].requests):
        assert rd.e2e_s < ro.e2e_s and rd.e2e_s < rp.e2e_s
    with pytest.raises(T.TraceError):
        S.run_experiment(["ondemand"], T.TraceDataset("fixture", 6, 8, 2, []), cfg, cost)


def test_cancellable_prefetch_extension():
    """B200 extension: with chunked cancellation a wrong prefetch (and an
    unneeded speculative prefill transfer) stops one chunk after the gate, so
    the request is never slower than the SPEC schedule, the decisions (cache
    log) are unchanged, and with perfect predictions the decode schedules
    coincide."""
    ds, cfg = _dataset(n=6, seed=4)
    cost = _cost(10, 2, nm_ms=1)
    pp = PopularityPredictor(ST.build_popularity(ds), cfg.top_k)
    chunk = cfg.expert_bytes // 8
    for rid, trs in ds.by_request().items():
        ms, tls, ls = S.simulate_request("duoserve", trs, cfg, cost, net=pp, return_log=True)
        mc, tlc, lc = S.simulate_request("duoserve", trs, cfg, cost, net=pp, cancel_chunk_bytes=chunk, return_log=True)
        assert lc == ls
        assert mc.e2e_s <= ms.e2e_s and mc.ttft_s <= ms.ttft_s
        assert mc.link_bytes <= ms.link_bytes
        tlc.check()
        mo, _ = S.simulate_request("oracle", trs, cfg, cost)
        mo2, _ = S.simulate_request("oracle", trs, cfg, cost, cancel_chunk_bytes=chunk)
        assert mo2.e2e_s <= mo.e2e_s
        # with perfect predictions only the speculative prefill transfer differs
        assert abs((mo2.e2e_s - mo2.ttft_s) - (mo.e2e_s - mo.ttft_s)) < 1e-6


def test_b200_calibrated_preset():
    """presets/mixtral-8x7b-b200.json: the reference schema with the W4 model's
    byte budget (uniform expert bytes = the 91,521,024-byte W4 blob) and a cost
    model measured on the B200 (scripts/calibrate_cost.py); the simulator runs
    on it and the link dominates (decode is link-bound on a PCIe host link)."""
    cfg, cost = C.load_preset("mixtral-8x7b-b200")
    assert cfg.expert_bytes == 91_521_024
    assert 40e9 < cost.link_bandwidth_bytes_per_s < 70e9
    L = cfg.num_layers
    ds = T.generate_traces(T.default_generator_params(L, 8, 0.8, 3), cfg, 1, 4, 16)
    trs = ds.traces
    m, tl = S.simulate_request("oracle", trs, cfg, cost)
    per_tok = (m.e2e_s - m.ttft_s) / m.decode_tokens
    floor = L * cfg.top_k * cost.transfer_time_s(cfg.expert_bytes)
    assert floor <= per_tok < 1.2 * floor


def test_oracle_pinned_extension_properties():
    """sim_ref's residency-budget extension: an empty pin
    set changes nothing; pinned experts never appear in a fetch / refetch
    list and are reported under "pinned" when the gate or prefill uses them;
    the speculative prefill transfer skips a pinned expert 0."""
    rng = np.random.default_rng(3)
    L, M, k = 4, 8, 2
    pre = [tuple(tuple(int(e) for e in rng.choice(M, k, replace=False)) for _ in range(L)) for _ in range(16)]
    paths = [tuple(tuple(int(e) for e in rng.choice(M, k, replace=False)) for _ in range(L)) for _ in range(6)]
    preds = [[None] + [tuple(int(e) for e in rng.choice(M, k, replace=False)) for _ in range(1, L)] for _ in paths]
    for pol in ("duoserve", "ondemand"):
        assert sim_ref.cache_log_prefill(pre, L, pol, pinned=set()) == sim_ref.cache_log_prefill(pre, L, pol)
        assert sim_ref.cache_log_decode(paths, preds, L, pol, pinned=set()) == \
            sim_ref.cache_log_decode(paths, preds, L, pol)
    pins = {(0, 0), (1, 3), (2, 5), (3, 1)}
    lp = sim_ref.cache_log_prefill(pre, L, "duoserve", pinned=pins)
    for r in lp:
        pl = {e for (ll, e) in pins if ll == r["layer"]}
        assert not pl & set(r["fetch"])
        assert set(r["pinned"]) == set(r["activated"]) & pl
    assert lp[0]["fetch"][0] == 1                         # expert 0 pinned at layer 0: speculate on 1
    ld, cnt = sim_ref.cache_log_decode(paths, preds, L, "duoserve", pinned=pins)
    _, cnt0 = sim_ref.cache_log_decode(paths, preds, L, "duoserve")
    n_pin = 0
    for r in ld:
        pl = {e for (ll, e) in pins if ll == r["layer"]}
        assert not pl & set(r.get("refetch", r.get("fetch", [])))
        n_pin += len(r["pinned"]) if r["layer"] > 0 else 0
    assert cnt["prefetch_hits"] + cnt["prefetch_misses"] + n_pin == cnt0["prefetch_hits"] + cnt0["prefetch_misses"]


def test_simulate_request_returns_spec_pair():
    """simulate_request -> (RequestMetrics, EventTimeline); the
    cache log is opt-in (return_log=True) and rides on the timeline."""
    cfg = _cfg(2)
    reqs = _req([((0, 1), (2, 3))], [((0, 1), (2, 3))])
    out = S.simulate_request("ondemand", reqs, cfg, _cost(10, 2, 1))
    assert len(out) == 2
    m, tl = out
    _, _, log = S.simulate_request("ondemand", reqs, cfg, _cost(10, 2, 1), return_log=True)
    assert tl.cache_log == log and log
