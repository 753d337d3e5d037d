"""Host API mirror vs the reference's own outputs (golden files made by
oracle/gen_golden.py from /root/reference).  CPU only."""

import hashlib
import json

import numpy as np
import pytest

from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200 import predictor as P
from paper_2509_07379_b200 import stats as S
from paper_2509_07379_b200 import trace as T


def _cfg(name, L, M=8, k=2):
    return C.ModelConfig(name=name, num_layers=L, num_experts=M, top_k=k, total_param_bytes=10**9,
                         non_moe_bytes=10**8, predictor_mem_bytes=0, kv_reserve_bytes=0)


SHAPES = {"tiny": (4, 3, 16, 64), "mixtral-8x7b": (32, 1, 8, 8), "mixtral-8x22b": (56, 1, 4, 4)}


@pytest.mark.parametrize("name", list(SHAPES))
def test_generate_traces_byte_identical(name, golden, tmp_path):
    L, nreq, dec, pre = SHAPES[name]
    ds = T.generate_traces(T.default_generator_params(L, 8, 0.8, seed=7), _cfg(name, L), nreq, dec, pre)
    T.save_traces(ds, tmp_path / "t.jsonl")
    assert (tmp_path / "t.jsonl").read_bytes() == (golden / f"traces_{name}.jsonl").read_bytes()
    back = T.load_traces(tmp_path / "t.jsonl", _cfg(name, L))
    assert back == ds


def test_chain_and_toy_traces(golden, tmp_path):
    ds = T.generate_traces(T.chain_generator_params(4, 8, seed=3), _cfg("chain", 4), 2, 8, 8)
    T.save_traces(ds, tmp_path / "c.jsonl")
    assert (tmp_path / "c.jsonl").read_bytes() == (golden / "traces_chain.jsonl").read_bytes()
    toy, _ = C.load_preset("toy-4x2")
    ds = T.generate_traces(T.default_generator_params(4, 4, 0.5, seed=1), toy, 2, 4, 4)
    T.save_traces(ds, tmp_path / "t.jsonl")
    assert (tmp_path / "t.jsonl").read_bytes() == (golden / "traces_toy-4x2.jsonl").read_bytes()


@pytest.mark.parametrize("name", list(SHAPES))
def test_stats_match_reference(name, golden, tmp_path):
    L = SHAPES[name][0]
    ds = T.load_traces(golden / f"traces_{name}.jsonl", _cfg(name, L))
    pop, aff = S.build_popularity(ds), S.build_affinity(ds)
    S.save_matrices(pop, aff, tmp_path / "m.json")
    assert (tmp_path / "m.json").read_text() == (golden / f"matrices_{name}.json").read_text()


def test_known_answers(golden):
    known = json.loads((golden / "known_answers.json").read_text())
    A = T.ActivationTrace(0, "decode", 0, ((0, 1), (2, 3), (0, 2), (1, 3)))
    B = T.ActivationTrace(1, "decode", 0, ((0, 2), (2, 3), (0, 1), (1, 3)))
    ds = T.TraceDataset("toy-4x2", 4, 4, 2, [A, B])
    pop, aff = S.build_popularity(ds), S.build_affinity(ds)
    assert pop.values[0].tolist() == known["pop_layer0"] == [0.5, 0.25, 0.25, 0.0]
    assert aff.values[0][0].tolist() == known["aff_l0_row0"] == [0.0, 0.0, 0.5, 0.5]
    sv = P.construct_input(A, 1, pop, aff)
    assert sv.history.tolist() == known["construct_A_l1_history"] == [1, 2, 0, 0, 0, 0, 0, 0]
    assert sv.layer_pos == known["construct_A_l1_layer_pos"]
    assert list(P.topk_indices(np.array([.9, .1, .8, .2]), 2)) == known["topk_ex1"] == [0, 2]
    assert list(P.topk_indices(np.array([.5, .5, .5, .5]), 2)) == known["topk_equal"] == [0, 1]
    cfg8, _ = C.load_preset("mixtral-8x7b")
    assert {p.value: C.slot_count(p, cfg8) for p in C.SchedulerPolicy} == known["slot_counts_8x7b"]
    for n, b in known["expert_bytes"].items():
        assert C.load_preset(n)[0].expert_bytes == b


def test_config_validation_and_roundtrip(tmp_path):
    cfg, cost = C.load_preset("mixtral-8x7b")
    C.save_config(cfg, cost, tmp_path / "c.json")
    assert C.load_config(tmp_path / "c.json") == (cfg, cost)
    with pytest.raises(C.ConfigError):
        C.ModelConfig("x", 4, 8, 8, 100, 10, 0, 0)
    with pytest.raises(C.ConfigError):
        C.load_preset("nope")
    doc = json.loads((tmp_path / "c.json").read_text())
    doc["model"]["extra"] = 1
    (tmp_path / "bad.json").write_text(json.dumps(doc))
    with pytest.raises(C.ConfigError, match="unknown model fields"):
        C.load_config(tmp_path / "bad.json")


def test_trace_validation_errors(tmp_path):
    cfg = _cfg("x", 4)
    with pytest.raises(T.TraceError):
        T.TraceDataset("x", 4, 8, 2, [T.ActivationTrace(0, "decode", 0, ((0, 0), (1, 2), (1, 2), (1, 2)))])
    (tmp_path / "b.jsonl").write_text('{"model":"x","L":4,"M":8,"k":2}\n{"req":0}\n')
    with pytest.raises(T.TraceError, match=":2:"):
        T.load_traces(tmp_path / "b.jsonl", cfg)


@pytest.mark.parametrize("tag", ["tiny_full_s0", "mixtral-8x7b_full_s1", "mixtral-8x22b_full_s0"])
def test_expertmlp_init_and_features_match_reference(tag, golden):
    man = json.loads((golden / "MANIFEST.json").read_text())["fixtures"][f"pred_{tag}.npz"]
    net = P.ExpertMLP(man["net"]["input_dim"], 8, hidden=man["net"]["hidden"], seed=man["net"]["seed"],
                      meta=man["net"]["meta"])
    digest = hashlib.sha256(b"".join(np.ascontiguousarray(a, dtype="<f8").tobytes()
                                     for _, a in P._array_specs(net))).hexdigest()
    assert digest == man["weights_sha256"]
    name = tag.split("_full")[0]
    L = {"tiny": 4, "mixtral-8x7b": 32, "mixtral-8x22b": 56}[name]
    ds = T.load_traces(golden / f"traces_{name}.jsonl", _cfg(name, L))
    pop, aff = S.load_matrices(golden / f"matrices_{name}.json")
    g = np.load(golden / f"pred_{tag}.npz")
    by = {(t.request_id, t.token_index): t for t in ds.traces}
    for i, (rid, pos, l) in enumerate(g["keys"][:200]):
        x = P.construct_input(by[(rid, pos)], int(l), pop, aff).as_features(8)
        assert np.array_equal(x, g["features"][i])


def test_model_container_roundtrip(golden, tmp_path):
    net = P.load_model(golden / "model_trained_alpha08.bin")
    P.save_model(net, tmp_path / "m.bin")
    assert (tmp_path / "m.bin").read_bytes() == (golden / "model_trained_alpha08.bin").read_bytes()
    (tmp_path / "bad.bin").write_bytes(b'{"format":"other","version":1}\n')
    with pytest.raises(P.PredictorError):
        P.load_model(tmp_path / "bad.bin")


def test_stub_predictors():
    t = T.ActivationTrace(0, "decode", 0, ((0, 1), (2, 3), (4, 5)))
    assert P.OraclePredictor().predict(t, 1) == (2, 3)
    assert P.ComplementPredictor(8).predict(t, 1) == (0, 1)
    assert P.ComplementPredictor(8).predict(t, 2) == (0, 1)


def test_bench_arms_share_the_workload_config():
    """bench.py: the reference arm's `config` is the same dict as ours (the
    driver compares the two lines' configs)."""
    import argparse
    import bench
    from paper_2509_07379_b200.config import load_shape
    a = argparse.Namespace(prefill=512, decode=128)
    c = bench.workload_config(load_shape("mixtral-8x7b"), a)
    assert c == bench.workload_config(load_shape("mixtral-8x7b"), a, 1)
    assert c["seq_len"] == 640 and c["model"] == "mixtral-8x7b" and "l2" in c
