"""Third-party pins of the oracles the reference cannot pin:
fixtures produced by the installed transformers 5.5.0 / vLLM 0.22.0 code
(oracle/gen_thirdparty_golden.py; THIRDPARTY_MANIFEST.json) vs

  * oracle/routing_ref (gate): indices equal to HF MixtralTopKRouter's wherever
    the top-k logit margin exceeds ROUTER_MARGIN (HF takes top-k of float32
    softmax probabilities, which can only reorder logits closer than that;
    exact ties break to the lower index here, arbitrarily in torch.topk);
    renormalised weights within 1e-6 relative;
  * oracle/model_ref.moe_block (expert FFN + combine): equal to HF
    MixtralSparseMoeBlock to 1e-12 in float64 without the kernels' bf16
    rounding of h, within MOE_BF16_TOL with it;
  * oracle/w4_ref (W4 dequant): the codes, zeros and (q - z) s weights vLLM's
    AWQ loader reads from this build's blob converted to the AWQ checkpoint
    layout (oracle/awq_convert) are bit-identical to w4_ref's.
"""

import hashlib
import json

import numpy as np
import pytest
import torch

from oracle import model_ref, routing_ref, w4_ref

ROUTER_MARGIN = 1e-6
MOE_BF16_TOL = 4e-3      # measured 1.6e-3 (tiny)


def _load(golden, name):
    p = golden / name
    if not p.exists():
        pytest.skip(f"{name} not generated (oracle/gen_thirdparty_golden.py)")
    return np.load(p)


@pytest.mark.parametrize("name", ["tiny", "8x7b"])
def test_routing_ref_matches_hf_router(golden, name):
    f = _load(golden, f"hf_router_{name}.npz")
    lg = routing_ref.gate_logits(f["x_bits"], f["wg_bits"])
    idx, w = routing_ref.topk_route(lg, 2)
    s = np.sort(lg, axis=1)[:, ::-1]
    ok = (s[:, 1] - s[:, 2]) > ROUTER_MARGIN
    assert ok.mean() > 0.99
    assert np.array_equal(idx[ok], f["hf_idx"][ok])
    assert np.allclose(w[ok], f["hf_w"][ok], rtol=1e-6, atol=0)


def _experts(meta):
    d, ff, M, k, G, wseed = (int(v) for v in meta)
    out = []
    for e in range(M):
        W = []
        for m, (K, N) in enumerate([(d, ff), (d, ff), (ff, d)]):
            c, s, z = w4_ref.gen_linear(wseed, 0, e, m, K, N, G)
            W.append(torch.from_numpy(w4_ref.bf16_bits_to_f32(w4_ref.dequant(c, s, z, K, N, G))))
        out.append(W)
    return out


@pytest.mark.parametrize("name", ["tiny", "8x7b"])
def test_model_ref_moe_matches_hf_block(golden, name):
    f = _load(golden, f"hf_moe_{name}.npz")
    a = torch.from_numpy(w4_ref.bf16_bits_to_f32(f["a_bits"]))
    idx, w = routing_ref.topk_route(routing_ref.gate_logits(f["a_bits"], f["wg_bits"]), 2)
    ex = _experts(f["meta"])
    hf = torch.from_numpy(f["out"])
    exact = model_ref.moe_block(a, idx, w.astype(np.float64), ex, round_h=False, dtype=torch.float64)
    # HF renormalises the f32 softmax; routing_ref's f32 weights differ by ~1 ulp
    assert ((exact - hf).norm() / hf.norm()).item() < 1e-6
    kern = model_ref.moe_block(a, idx, w, ex, round_h=True, dtype=torch.float32).double()
    rel = ((kern - hf).norm() / hf.norm()).item()
    print(name, "bf16-h f32 moe_block vs HF rel-L2", rel)
    assert rel < MOE_BF16_TOL


def test_w4_ref_matches_vllm_awq_reading(golden):
    p = golden / "awq_vllm.json"
    if not p.exists():
        pytest.skip("awq_vllm.json not generated")
    for c in json.loads(p.read_text())["cases"]:
        seed, layer, expert, m, K, N, G = (c[x] for x in ("seed", "layer", "expert", "matrix", "K", "N", "G"))
        codes, sc, z = w4_ref.gen_linear(seed, layer, expert, m, K, N, G)
        q = w4_ref.unpack_codes(codes).T
        zz = w4_ref.unpack_zeros(z, N, K // G).T
        w = w4_ref.dequant_exact(codes, sc, z, K, N, G).T.astype(np.float32)
        assert hashlib.sha256(np.ascontiguousarray(q).tobytes()).hexdigest() == c["sha256_q"]
        assert hashlib.sha256(np.ascontiguousarray(zz).tobytes()).hexdigest() == c["sha256_z"]
        assert hashlib.sha256(np.ascontiguousarray(w).tobytes()).hexdigest() == c["sha256_w_f32"]
