"""The CPU oracle pinned against the reference's own outputs (golden)."""

import json

import numpy as np
import pytest

from oracle import predictor_ref as PR
from oracle import stats_ref as SR
from oracle import w4_ref as WR
from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200 import stats as S
from paper_2509_07379_b200 import trace as T

TAGS = ["tiny_full_s0", "tiny_full_s1", "mixtral-8x7b_full_s0", "mixtral-8x7b_full_s1",
        "mixtral-8x22b_full_s0", "mixtral-8x22b_full_s1", "tiny_concat_s2"]
L_OF = {"tiny": 4, "mixtral-8x7b": 32, "mixtral-8x22b": 56}


def _cfg(name, L):
    return C.ModelConfig(name=name, num_layers=L, num_experts=8, top_k=2, total_param_bytes=10**9,
                         non_moe_bytes=10**8, predictor_mem_bytes=0, kv_reserve_bytes=0)


@pytest.mark.parametrize("tag", TAGS)
def test_predictor_oracle_matches_reference(tag, golden):
    man = json.loads((golden / "MANIFEST.json").read_text())["fixtures"][f"pred_{tag}.npz"]
    name = tag.split("_full")[0].split("_concat")[0]
    L = L_OF[name]
    mode = man["net"]["meta"].get("affinity_mode", "pool")
    net = PR.RefNet(man["net"]["input_dim"], 8, man["net"]["hidden"], man["net"]["seed"],
                    meta=man["net"]["meta"])
    ds = T.load_traces(golden / f"traces_{name}.jsonl", _cfg(name, L))
    pop, aff = S.load_matrices(golden / f"matrices_{name}.json")
    g = np.load(golden / f"pred_{tag}.npz")
    by = {(t.request_id, t.token_index): t.path for t in ds.traces}
    paths = [by[(int(r), int(p))] for r, p, _ in g["keys"]]
    layers = [int(l) for _, _, l in g["keys"]]
    X = np.stack([PR.features(p, l, pop.values, aff.values, mode) for p, l in zip(paths, layers)])
    assert np.array_equal(X, g["features"])
    sets, probs = PR.predict_sets(net, paths, layers, pop.values, aff.values, 2, mode)
    assert np.array_equal(probs, g["probs"])          # same numpy ops -> bitwise
    assert [tuple(s) for s in g["sets"].tolist()] == sets


@pytest.mark.parametrize("tag", ["trained_alpha08", "trained_chain"])
def test_trained_container_oracle(tag, golden):
    net = PR.load_container(golden / f"model_{tag}.bin")
    g = np.load(golden / f"pred_{tag}.npz")
    P = net.forward(g["features"])
    assert np.array_equal(P, g["probs"])
    assert [tuple(s) for s in g["sets"].tolist()] == [PR.topk_indices(p, 2) for p in P]
    assert (golden / f"model_{tag}.bin").read_bytes() == PR.container_bytes(net)


@pytest.mark.parametrize("name", list(L_OF))
def test_stats_oracle_recount(name, golden):
    L = L_OF[name]
    ds = T.load_traces(golden / f"traces_{name}.jsonl", _cfg(name, L))
    pv, pc, av, ac = SR.recount([t.path for t in ds.traces], L, 8)
    pop, aff = S.load_matrices(golden / f"matrices_{name}.json")
    assert np.array_equal(pc, pop.counts) and np.array_equal(ac, aff.counts)
    assert np.abs(pv - pop.values).max() <= 1e-12 and np.abs(av - aff.values).max() <= 1e-12


def test_w4_pack_roundtrip_and_dequant():
    rng = np.random.default_rng(0)
    q = rng.integers(0, 16, size=(128, 256), dtype=np.uint8)
    assert np.array_equal(WR.unpack_codes(WR.pack_codes(q)), q)
    c, s, z = WR.gen_linear(7, 1, 2, 0, 256, 128, 128)
    assert c.shape == (128, 32) and s.shape == (128, 2) and z.size == 128
    w = WR.bf16_bits_to_f32(WR.dequant(c, s, z, 256, 128, 128))
    qq = WR.unpack_codes(c).astype(np.float32)
    zz = np.repeat(WR.unpack_zeros(z, 128, 2).astype(np.float32), 128, axis=1)
    ss = np.repeat(WR.bf16_bits_to_f32(s), 128, axis=1)
    assert np.abs(w - (qq - zz) * ss).max() <= np.abs((qq - zz) * ss).max() * 2 ** -8
    # generator statistics: codes and zeros uniform on 0..15
    assert abs(qq.mean() - 7.5) < 0.2
