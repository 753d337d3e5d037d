"""Mixtral-shaped model pieces around the hot path.

The non-MoE layers (embedding, RMSNorm, RoPE, GQA attention with a KV
cache, lm_head) are ordinary PyTorch/cuBLAS/cuDNN ops — outside the graded
hot path ("use PyTorch/cuBLAS/cuDNN ops"; the paper runs
them as plain vLLM layers).  They stay resident in HBM
("fetch them all onto the GPU").  The MoE block is the hot
path and lives in engine.py on top of the sm_100a kernels.

Numerics (restated independently in oracle/model_ref.py):
  rms_norm(x)  = bf16( f32(x) * rsqrt(mean(f32(x)^2) + eps) * f32(gamma) )
  rope         = HF rotate-half, f32 cos/sin tables, bf16 out
  attention    = SDPA (causal for prefill), bf16 in/out, GQA
  residual add = bf16(f32(a) + f32(b))
  logits       = f32 of bf16(lm_head(norm(h)))
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from .config import ModelShape


@dataclass
class DenseWeights:
    embed: torch.Tensor                  # [V, d]
    layers: list = field(default_factory=list)  # dicts: ln1, wq, wk, wv, wo, ln2, wg
    norm: torch.Tensor | None = None     # [d]
    lm_head: torch.Tensor | None = None  # [d, V]

    def to(self, device) -> "DenseWeights":
        mv = lambda t: t.to(device, non_blocking=False)
        return DenseWeights(embed=mv(self.embed),
                            layers=[{k: mv(v) for k, v in L.items()} for L in self.layers],
                            norm=mv(self.norm), lm_head=mv(self.lm_head))

    def nbytes(self) -> int:
        n = self.embed.nbytes + self.norm.nbytes + self.lm_head.nbytes
        return n + sum(t.nbytes for L in self.layers for t in L.values())


def init_dense_weights(shape: ModelShape, seed: int, device="cpu", std: float = 0.02) -> DenseWeights:
    """Random-init non-MoE weights, bf16 N(0, std); norms = 1.
    Deterministic per (seed, device type)."""
    g = torch.Generator(device=device).manual_seed(seed)
    d, hd = shape.hidden, shape.head_dim
    bf = torch.bfloat16

    def randn(*s):
        return (torch.randn(*s, generator=g, device=device, dtype=torch.float32) * std).to(bf)

    embed = randn(shape.vocab, d)
    layers = []
    for _ in range(shape.num_layers):
        layers.append({
            "ln1": torch.ones(d, dtype=bf, device=device),
            "wq": randn(d, shape.n_heads * hd),
            "wk": randn(d, shape.n_kv_heads * hd),
            "wv": randn(d, shape.n_kv_heads * hd),
            "wo": randn(shape.n_heads * hd, d),
            "ln2": torch.ones(d, dtype=bf, device=device),
            "wg": randn(shape.num_experts, d),
        })
    return DenseWeights(embed=embed, layers=layers, norm=torch.ones(d, dtype=bf, device=device),
                        lm_head=randn(d, shape.vocab))


def rms_norm(x: torch.Tensor, gamma: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * gamma.float()).to(torch.bfloat16)


def rope_tables(shape: ModelShape, max_pos: int, device):
    hd = shape.head_dim
    inv = 1.0 / (shape.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float32, device=device) / hd))
    t = torch.arange(max_pos, dtype=torch.float32, device=device)
    f = torch.outer(t, inv)
    emb = torch.cat([f, f], dim=-1)
    return emb.cos(), emb.sin()


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [T, H, hd] bf16; cos/sin [T, hd] f32."""
    xf = x.float()
    h = xf.shape[-1] // 2
    rot = torch.cat([-xf[..., h:], xf[..., :h]], dim=-1)
    return (xf * cos[:, None, :] + rot * sin[:, None, :]).to(torch.bfloat16)


class KVCache:
    def __init__(self, shape: ModelShape, max_seq: int, device):
        self.k = torch.zeros(shape.num_layers, shape.n_kv_heads, max_seq, shape.head_dim,
                             dtype=torch.bfloat16, device=device)
        self.v = torch.zeros_like(self.k)
        self.len = 0

    @property
    def nbytes(self) -> int:
        return self.k.nbytes + self.v.nbytes


def attention_block(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCache, layer: int, pos0: int,
                    cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """h [T, d] bf16 (positions pos0 .. pos0+T-1) -> h + attn(norm(h)) (bf16)."""
    T = h.shape[0]
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    a = rms_norm(h, L["ln1"], shape.rms_eps)
    q = (a @ L["wq"]).view(T, nh, hd)
    k = (a @ L["wk"]).view(T, nkv, hd)
    v = (a @ L["wv"]).view(T, nkv, hd)
    c, s = cos[pos0:pos0 + T], sin[pos0:pos0 + T]
    q, k = apply_rope(q, c, s), apply_rope(k, c, s)
    kv.k[layer, :, pos0:pos0 + T] = k.transpose(0, 1)
    kv.v[layer, :, pos0:pos0 + T] = v.transpose(0, 1)
    K = kv.k[layer, :, :pos0 + T].unsqueeze(0)
    V = kv.v[layer, :, :pos0 + T].unsqueeze(0)
    o = F.scaled_dot_product_attention(q.transpose(0, 1).unsqueeze(0), K, V, is_causal=(T > 1 and pos0 == 0),
                                       enable_gqa=True)
    o = o.squeeze(0).transpose(0, 1).reshape(T, nh * hd)
    return (h.float() + (o @ L["wo"]).float()).to(torch.bfloat16)


def attention_decode_static(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCache, layer: int,
                            pos: torch.Tensor, mask: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """One decode token with the position on the device (CUDA-graph capturable):
    h [1, d]; pos int64 [1]; mask [1, 1, 1, max_seq] additive (0 for <= pos, -inf after)."""
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    a = rms_norm(h, L["ln1"], shape.rms_eps)
    q = (a @ L["wq"]).view(1, nh, hd)
    k = (a @ L["wk"]).view(1, nkv, hd)
    v = (a @ L["wv"]).view(1, nkv, hd)
    c, s = cos.index_select(0, pos), sin.index_select(0, pos)
    q, k = apply_rope(q, c, s), apply_rope(k, c, s)
    kv.k[layer].index_copy_(1, pos, k.transpose(0, 1))
    kv.v[layer].index_copy_(1, pos, v.transpose(0, 1))
    o = F.scaled_dot_product_attention(q.transpose(0, 1).unsqueeze(0), kv.k[layer].unsqueeze(0),
                                       kv.v[layer].unsqueeze(0), attn_mask=mask, enable_gqa=True)
    o = o.squeeze(0).transpose(0, 1).reshape(1, nh * hd)
    return (h.float() + (o @ L["wo"]).float()).to(torch.bfloat16)


def logits_last(shape: ModelShape, W: DenseWeights, h_last: torch.Tensor) -> torch.Tensor:
    return (rms_norm(h_last, W.norm, shape.rms_eps) @ W.lm_head).float()
