"""K5 on the B200 vs the reference's own predictions (golden, made by the
reference) — predicted SETS bit-exact; probabilities within 1e-12 (only the
dot-product summation order differs from BLAS)."""

import json

import numpy as np
import pytest

from oracle import predictor_ref as PR
from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200 import predictor as P
from paper_2509_07379_b200 import stats as S
from paper_2509_07379_b200 import trace as T

pytestmark = pytest.mark.gpu

TAGS = ["tiny_full_s0", "tiny_full_s1", "mixtral-8x7b_full_s0", "mixtral-8x7b_full_s1",
        "mixtral-8x22b_full_s0", "mixtral-8x22b_full_s1", "tiny_concat_s2"]
L_OF = {"tiny": 4, "mixtral-8x7b": 32, "mixtral-8x22b": 56}
PROB_TOL = 1e-12


def _cfg(name, L):
    return C.ModelConfig(name=name, num_layers=L, num_experts=8, top_k=2, total_param_bytes=10**9,
                         non_moe_bytes=10**8, predictor_mem_bytes=0, kv_reserve_bytes=0)


def _load(tag, golden):
    man = json.loads((golden / "MANIFEST.json").read_text())["fixtures"][f"pred_{tag}.npz"]
    name = tag.split("_full")[0].split("_concat")[0]
    L = L_OF[name]
    net = P.ExpertMLP(man["net"]["input_dim"], 8, hidden=man["net"]["hidden"], seed=man["net"]["seed"],
                      meta=man["net"]["meta"])
    ds = T.load_traces(golden / f"traces_{name}.jsonl", _cfg(name, L))
    pop, aff = S.load_matrices(golden / f"matrices_{name}.json")
    return net, ds, pop, aff, np.load(golden / f"pred_{tag}.npz")


def _check(sets, probs, g):
    ref_sets = [tuple(s) for s in g["sets"].tolist()]
    got = [tuple(int(e) for e in s) for s in sets]
    mism = [i for i, (a, b) in enumerate(zip(got, ref_sets)) if a != b]
    margins = [PR.topk_margin(g["probs"][i], 2) for i in mism]
    assert not mism or max(margins) < 1e-12, (mism[:5], margins[:5])
    assert not mism, f"{len(mism)} set mismatches with margins {margins[:5]}"
    if probs is not None:
        assert np.abs(probs - g["probs"]).max() <= PROB_TOL


@pytest.mark.parametrize("tag", TAGS)
def test_batched_sets_bit_exact(tag, golden, cuda):
    net, ds, pop, aff, g = _load(tag, golden)
    pred = P.MLPPredictor(net, pop, aff)
    by = {(t.request_id, t.token_index): t for t in ds.traces}
    traces = [by[(int(r), int(p))] for r, p, _ in g["keys"]]
    layers = [int(l) for _, _, l in g["keys"]]
    sets, probs = pred.predict_batch(traces, layers, with_probs=True)    # B > 8: tiled path
    _check(sets, probs, g)


@pytest.mark.parametrize("tag", ["tiny_full_s0", "mixtral-8x7b_full_s0", "mixtral-8x22b_full_s1",
                                 "tiny_concat_s2"])
@pytest.mark.parametrize("B", [1, 3, 8])
def test_fused_small_batch_sets(tag, B, golden, cuda):
    net, ds, pop, aff, g = _load(tag, golden)
    pred = P.MLPPredictor(net, pop, aff)
    by = {(t.request_id, t.token_index): t for t in ds.traces}
    n = min(len(g["keys"]), 48)
    sets, probs = [], []
    for s in range(0, n, B):
        keys = g["keys"][s:s + B]
        a, p = pred.predict_batch([by[(int(r), int(q))] for r, q, _ in keys], [int(l) for *_, l in keys],
                                  with_probs=True)
        sets += list(a)
        probs.append(p)
    sub = {k: g[k][:n] for k in ("sets", "probs")}
    _check(sets, np.concatenate(probs), sub)


def test_single_call_protocol(golden, cuda):
    net, ds, pop, aff, g = _load("mixtral-8x7b_full_s0", golden)
    pred = P.MLPPredictor(net, pop, aff)
    by = {(t.request_id, t.token_index): t for t in ds.traces}
    for i in range(len(g["single_sets"])):
        r, p, l = g["keys"][i]
        assert pred.predict(by[(int(r), int(p))], int(l)) == tuple(g["single_sets"][i])


@pytest.mark.parametrize("tag", ["trained_alpha08", "trained_chain"])
def test_trained_nets_and_evaluate(tag, golden, cuda):
    net = P.load_model(golden / f"model_{tag}.bin")
    pop, aff = S.load_matrices(golden / f"matrices_{tag}.json")
    g = np.load(golden / f"pred_{tag}.npz")
    probs = net.forward(g["features"])                      # ExpertMLP.forward on device
    assert np.abs(probs - g["probs"]).max() <= PROB_TOL
    src = "traces_tiny.jsonl" if tag == "trained_alpha08" else "traces_chain.jsonl"
    ds = T.load_traces(golden / src, _cfg("x", 4))
    rep = P.evaluate(net, ds, pop, aff).to_dict()
    ref = json.loads((golden / f"eval_{tag}.json").read_text())
    assert rep == ref


def test_zero_net_is_half(golden, cuda):
    net = P.load_model(golden / "model_zero.bin")
    out = net.forward(np.random.default_rng(0).random((5, net.input_dim)))
    assert np.all(out == 0.5)


def test_features_kernel_matches_reference_features(golden, cuda):
    """The fused State Constructor: probabilities from hist-path == from features-path."""
    net, ds, pop, aff, g = _load("mixtral-8x22b_full_s0", golden)
    p_feat = net.forward(g["features"])
    pred = P.MLPPredictor(net, pop, aff)
    by = {(t.request_id, t.token_index): t for t in ds.traces}
    _, p_state = pred.predict_batch([by[(int(r), int(p))] for r, p, _ in g["keys"]],
                                    [int(l) for *_, l in g["keys"]], with_probs=True)
    assert np.array_equal(p_feat, p_state)
