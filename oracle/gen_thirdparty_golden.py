"""Pin the oracles the reference cannot pin (gate, W4 FFN,
model forward) against the THIRD-PARTY code whose semantics they restate, run
here in the build container where that code is installed:

  * transformers 5.5.0  models/mixtral/modeling_mixtral.py
      MixtralTopKRouter (:104-118)  -> tests/golden/hf_router_{tiny,8x7b}.npz
      MixtralSparseMoeBlock / MixtralExperts (:62-100, :121-137)
                                    -> tests/golden/hf_moe_{tiny,8x7b}.npz
  * vLLM 0.22.0  model_executor/layers/quantization/awq_marlin.py:74-156
      (_convert_awq_to_standard_format: AWQ nibble order + repack, pure torch)
                                    -> tests/golden/awq_vllm.json

    python oracle/gen_thirdparty_golden.py [--skip-8x7b]

Inputs are this build's own synthetic data: W4 experts from oracle/w4_ref.py
(the generator the GPU reproduces byte for byte), bf16 activations and router
weights from numpy seeds.  The third-party modules run in float64 on the
exact bf16/W4 values, so their outputs are the semantic reference the
oracle restatements (routing_ref, model_ref, w4_ref) and the GPU kernels are
checked against in tests/test_thirdparty_pins.py and
tests/test_gpu_thirdparty_pins.py.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tests" / "golden"

from oracle import awq_convert, w4_ref  # noqa: E402


def _bf16(rng, shape, std):
    return w4_ref.bf16_round_bits((rng.standard_normal(shape) * std).astype(np.float32))


def _hf_config(d, ff, M, k):
    from transformers import MixtralConfig
    return MixtralConfig(hidden_size=d, intermediate_size=ff, num_local_experts=M, num_experts_per_tok=k,
                         num_hidden_layers=1, num_attention_heads=4, num_key_value_heads=2,
                         router_jitter_noise=0.0)


def router_fixture(name, d, M, k, T, seed):
    from transformers.models.mixtral.modeling_mixtral import MixtralTopKRouter
    rng = np.random.default_rng(seed)
    x = _bf16(rng, (T, d), 1.0)
    wg = _bf16(rng, (M, d), 0.02)
    r = MixtralTopKRouter(_hf_config(d, 4 * d, M, k)).double()
    with torch.no_grad():
        r.weight.copy_(torch.from_numpy(w4_ref.bf16_bits_to_f32(wg).astype(np.float64)))
        probs, scores, idx = r(torch.from_numpy(w4_ref.bf16_bits_to_f32(x).astype(np.float64)))
    order = torch.argsort(idx, dim=-1)
    np.savez_compressed(OUT / f"hf_router_{name}.npz", x_bits=x, wg_bits=wg,
                        hf_idx=torch.gather(idx, -1, order).numpy().astype(np.int32),
                        hf_w=torch.gather(scores, -1, order).numpy().astype(np.float32),
                        hf_probs=probs.numpy())
    return f"MixtralTopKRouter (float64 module; softmax in float32 as shipped) on T={T}, d={d}, M={M}, k={k}"


def moe_fixture(name, d, ff, M, k, G, T, seed, wseed):
    from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock
    rng = np.random.default_rng(seed)
    a = _bf16(rng, (T, d), 1.0)
    wg = _bf16(rng, (M, d), 0.02)
    blk = MixtralSparseMoeBlock(_hf_config(d, ff, M, k)).double()
    with torch.no_grad():
        blk.gate.weight.copy_(torch.from_numpy(w4_ref.bf16_bits_to_f32(wg).astype(np.float64)))
        for e in range(M):
            W = []
            for m, (K, N) in enumerate([(d, ff), (d, ff), (ff, d)]):
                c, s, z = w4_ref.gen_linear(wseed, 0, e, m, K, N, G)
                W.append(torch.from_numpy(w4_ref.bf16_bits_to_f32(w4_ref.dequant(c, s, z, K, N, G)).astype(np.float64)))
            blk.experts.gate_up_proj[e].copy_(torch.cat([W[0], W[1]], dim=0))     # [2ff, d]: gate (W1) then up (W3)
            blk.experts.down_proj[e].copy_(W[2])                                  # [d, ff]
            del W
        out = blk(torch.from_numpy(w4_ref.bf16_bits_to_f32(a).astype(np.float64))[None])[0]
    np.savez_compressed(OUT / f"hf_moe_{name}.npz", a_bits=a, wg_bits=wg, out=out.numpy(),
                        meta=np.array([d, ff, M, k, G, wseed]))
    return (f"MixtralSparseMoeBlock (float64) with layer-0 W4 experts of w4_ref.gen_linear(seed={wseed}) "
            f"dequantised bf16_rn((q-z)s), T={T}, d={d}, ff={ff}")


def awq_fixture(cases):
    import vllm.model_executor.parameter as VP
    VP.get_tensor_model_parallel_rank = lambda: 0          # no TP group outside a vLLM engine
    VP.get_tensor_model_parallel_world_size = lambda: 1
    from vllm.model_executor.layers.quantization.awq_marlin import _convert_awq_to_standard_format
    out = []
    for (seed, layer, expert, m, K, N, G) in cases:
        c, s, z = w4_ref.gen_linear(seed, layer, expert, m, K, N, G)
        qw, qz, sc = awq_convert.to_awq(c, s, z, K, N, G)

        class Layer(torch.nn.Module):
            pass
        lay = Layer()
        lay.qweight = torch.nn.Parameter(torch.from_numpy(qw), requires_grad=False)
        lay.qzeros = torch.nn.Parameter(torch.from_numpy(qz), requires_grad=False)
        _convert_awq_to_standard_format(lay, "qweight", "qzeros", 4)
        # standard (GPTQ-like) layout: qweight [K/8, N], nibble j of row r = k 8r + j;
        # qzeros [N/8, K/G], nibble j of row r = column 8r + j
        sq = lay.qweight.data.numpy().view(np.uint32)
        q = np.stack([(sq >> np.uint32(4 * j)) & np.uint32(15) for j in range(8)], axis=1).reshape(K, N)
        szz = lay.qzeros.data.numpy().view(np.uint32)
        zz = np.stack([(szz >> np.uint32(4 * j)) & np.uint32(15) for j in range(8)], axis=1).reshape(N, K // G).T
        w = (q.astype(np.float32) - np.repeat(zz, G, axis=0).astype(np.float32)) * \
            np.repeat(sc.astype(np.float32), G, axis=0)                            # [K, N], exact products
        rec = {"seed": seed, "layer": layer, "expert": expert, "matrix": m, "K": K, "N": N, "G": G,
               "sha256_q": hashlib.sha256(q.astype(np.uint8).tobytes()).hexdigest(),
               "sha256_z": hashlib.sha256(np.ascontiguousarray(zz).astype(np.uint8).tobytes()).hexdigest(),
               "sha256_w_f32": hashlib.sha256(np.ascontiguousarray(w).tobytes()).hexdigest(),
               "w_f32_head": w[:2, :8].tolist()}
        out.append(rec)
    (OUT / "awq_vllm.json").write_text(json.dumps({
        "generator": "oracle/gen_thirdparty_golden.py",
        "source": "vLLM 0.22.0 awq_marlin._convert_awq_to_standard_format on oracle/awq_convert.to_awq(w4_ref blob); "
                  "w = (q - z) * s, [K, N]", "cases": out}, indent=1) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-8x7b", action="store_true")
    a = ap.parse_args()
    import transformers
    import vllm
    man = {"generator": "oracle/gen_thirdparty_golden.py", "transformers": transformers.__version__,
           "vllm": vllm.__version__, "fixtures": {}}
    man["fixtures"]["hf_router_tiny.npz"] = router_fixture("tiny", 256, 8, 2, 512, 11)
    man["fixtures"]["hf_moe_tiny.npz"] = moe_fixture("tiny", 256, 896, 8, 2, 128, 64, 12, 3)
    if not a.skip_8x7b:
        man["fixtures"]["hf_router_8x7b.npz"] = router_fixture("8x7b", 4096, 8, 2, 256, 13)
        man["fixtures"]["hf_moe_8x7b.npz"] = moe_fixture("8x7b", 4096, 14336, 8, 2, 128, 6, 14, 0)
    awq_fixture([(3, 0, 1, 0, 256, 896, 128), (3, 0, 1, 2, 896, 256, 128), (0, 3, 5, 0, 4096, 14336, 128),
                 (0, 7, 2, 2, 14336, 4096, 128)])
    man["fixtures"]["awq_vllm.json"] = "vLLM AWQ standard-format conversion of w4_ref linears (digests)"
    (OUT / "THIRDPARTY_MANIFEST.json").write_text(json.dumps(man, indent=1) + "\n")
    print(json.dumps(man, indent=1))


if __name__ == "__main__":
    main()
