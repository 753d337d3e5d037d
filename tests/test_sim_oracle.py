"""The SPEC simulator restatement (oracle/sim_ref.py) against the SPEC's
hand-traced fixtures and memory example."""

import pytest

from oracle import sim_ref
from paper_2509_07379_b200 import config as C

MS = 1_000_000  # integer nanoseconds


def test_prefill_fixtures():
    # E_act=4, T=10 ms, C=2 ms, non-MoE >= T: DuoServe 32 ms, OnDemand 48 ms; C>T: 40 ms
    assert sim_ref.timeline_prefill_layer("duoserve", 4, 10 * MS, 2 * MS, 10 * MS, 4) == 32 * MS
    assert sim_ref.timeline_prefill_layer("duoserve", 4, 10 * MS, 2 * MS, 10 * MS, 2) == 32 * MS
    assert sim_ref.timeline_prefill_layer("ondemand", 4, 10 * MS, 2 * MS, 10 * MS, 2) == 48 * MS
    assert sim_ref.timeline_prefill_layer("duoserve", 4, 2 * MS, 10 * MS, 10 * MS, 4) == 40 * MS


def test_decode_fixtures():
    # k=2, T=10, C=2, non-MoE+gate=1: full hit 20 ms/layer; one miss 30; OnDemand 25
    d = sim_ref.timeline_decode("duoserve", 6, 2, 10 * MS, 2 * MS, 1 * MS, [0] * 6)
    assert d[2:] == [20 * MS] * 4
    d = sim_ref.timeline_decode("duoserve", 6, 2, 10 * MS, 2 * MS, 1 * MS, [0, 0, 0, 1, 0, 0])
    assert d[3] == 30 * MS and d[4] == 20 * MS
    d = sim_ref.timeline_decode("ondemand", 4, 2, 10 * MS, 2 * MS, 1 * MS, [0] * 4)
    assert d == [25 * MS] * 4


def test_cache_log_semantics():
    paths = [((0, 1), (2, 3), (4, 5)), ((1, 2), (3, 4), (5, 6))]
    preds = [[None, (2, 3), (4, 6)], [None, (0, 1), (5, 6)]]
    log, cnt = sim_ref.cache_log_decode(paths, preds, 3)
    assert log[0] == {"phase": "decode", "token": 0, "layer": 0, "fetch": [0, 1], "kind": "ondemand"}
    assert log[1]["refetch"] == [] and log[2]["refetch"] == [5]
    assert log[4]["refetch"] == [3, 4]
    assert cnt["prefetch_hits"] + cnt["prefetch_misses"] == 2 * 2 * 2
    pa, cnt = sim_ref.cache_log_decode(paths, None, 3, "prefetchall", M=8)
    assert all(r["fetch"] == list(range(8)) and r["kind"] == "prefetchall" for r in pa) and len(pa) == 6
    assert cnt["prefetch_hits"] == cnt["prefetch_misses"] == 0
    pa = sim_ref.cache_log_prefill([((0, 1), (2, 3))], 2, "prefetchall", owned=[1, 3, 5, 7])
    assert pa[1]["fetch"] == [1, 3, 5, 7] and pa[1]["activated"] == [2, 3]
    pre = sim_ref.cache_log_prefill([((0, 1), (2, 3)), ((1, 2), (3, 5))], 2)
    assert pre[0]["fetch"] == [0, 1, 2] and pre[1]["fetch"] == [0, 2, 3, 5] and pre[1]["activated"] == [2, 3, 5]


@pytest.mark.parametrize("preset", ["mixtral-8x7b", "mixtral-8x22b"])
def test_peak_memory_accounting(preset):
    """non_moe + slots*expert_bytes + (predictor if duoserve) + kv."""
    cfg, _ = C.load_preset(preset)
    peak = {p: cfg.non_moe_bytes + C.slot_count(p, cfg) * cfg.expert_bytes
            + (cfg.predictor_mem_bytes if p.needs_predictor else 0) + cfg.kv_reserve_bytes
            for p in C.SchedulerPolicy}
    P = C.SchedulerPolicy
    assert peak[P.ON_DEMAND] < peak[P.DUOSERVE] < peak[P.PREFETCH_ALL]
    if preset == "mixtral-8x7b":
        assert abs(peak[P.DUOSERVE] - 3.91e9) / 3.91e9 < 0.05
        assert peak[P.DUOSERVE] / cfg.total_param_bytes <= 0.16


def test_batch_extension_reduces_to_single_sequence_and_unions():
    """cache_log_decode_batch: B = 1 is exactly cache_log_decode; with B > 1
    the gate set is the union of the sequences' selections, the prediction
    the union of their predictions, refetch = gate - pred (hand-traced)."""
    import numpy as np
    from oracle import sim_ref
    rng = np.random.default_rng(3)
    L, M = 4, 8
    paths = [tuple(tuple(sorted(rng.choice(M, 2, replace=False).tolist())) for _ in range(L)) for _ in range(5)]
    preds = [[None] + [tuple(sorted(rng.choice(M, 2, replace=False).tolist())) for _ in range(L - 1)] for _ in paths]
    one, c1 = sim_ref.cache_log_decode(paths, preds, L)
    bat, cb = sim_ref.cache_log_decode_batch([[p] for p in paths], [[q] for q in preds], L)
    assert bat == one and cb["prefetch_misses"] == c1["prefetch_misses"]
    step = [((0, 1), (2, 5)), ((1, 3), (5, 6))]
    pr = [[None, (2, 4)], [None, (6, 7)]]
    log, cnt = sim_ref.cache_log_decode_batch([step], [pr], 2)
    assert log[0] == {"phase": "decode", "token": 0, "layer": 0, "fetch": [0, 1, 3], "kind": "ondemand"}
    assert log[1] == {"phase": "decode", "token": 0, "layer": 1, "pred": [2, 4, 6, 7], "gate": [2, 5, 6],
                      "refetch": [5]}
    assert cnt == {"prefetch_hits": 2, "prefetch_misses": 1}


def test_ep_dispatch_rule_is_owned_part_of_the_union():
    from oracle import sim_ref
    pre = [[((0, 1), (2, 3))], [((4, 5), (3, 6))]]          # rank 0 / rank 1 prefill tokens
    dec = [[[((1, 7), (0, 2))]], [[((2, 7), (5, 6))]]]        # one decode step, one sequence per rank
    log0 = sim_ref.cache_log_ep_dispatch(pre, dec, 2, owned=[0, 2, 4, 6])
    log1 = sim_ref.cache_log_ep_dispatch(pre, dec, 2, owned=[1, 3, 5, 7])
    assert [r["fetch"] for r in log0] == [[0, 4], [2, 6], [2], [0, 2, 6]]
    assert [r["fetch"] for r in log1] == [[1, 5], [3], [1, 7], [5]]
