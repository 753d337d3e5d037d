"""Mixtral-shaped model pieces around the hot path.

The non-MoE layers (embedding, RMSNorm, RoPE, GQA attention with a KV
cache, lm_head) stay resident in HBM ("fetch them all onto the GPU",
PAPER.md:163).  The attention projections are W4 like the experts (the
paper's W4 model: 2.15 GB of non-MoE weights; SURVEY.md §2.3
"W4 attention projections (may reuse K3/K4)"): q|k|v fused into one W4
linear and o, run by the repo's own kernels — the K4 decode GEMV for a few
rows, the tcgen05 GEMM (K3's down-projection kernel) for a prompt.  Norms,
RoPE, SDPA, the embedding and lm_head (bf16) are PyTorch ops.  The MoE block
is the hot path and lives in engine.py.

Numerics (restated independently in oracle/model_ref.py):
  rms_norm(x)  = bf16( f32(x) * rsqrt(mean(f32(x)^2) + eps) * f32(gamma) )
  q, k, v      = bf16( x Wqkv^T ) with f32 accumulation; W = bf16_rn((q-z)s)
                 for a prompt (GEMM), the exact (q-z)s for decode (GEMV)
  rope         = HF rotate-half, f32 cos/sin tables, bf16 out
  attention    = SDPA (causal for prefill), bf16 in/out, GQA
  o-proj + residual = bf16( f32(h) + o Wo^T ) (one rounding)
  logits       = f32 of bf16(lm_head(norm(h)))
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from . import ops
from .config import ModelShape

# generator identity of the W4 attention projections: tag 63 of the
# (seed, layer, tag, matrix, kind) key space (experts use tags 0..M-1)
ATTN_TAG, QKV_MATRIX, O_MATRIX = 63, 0, 1


def attn_linear_shapes(shape: ModelShape) -> dict:
    """{name: (matrix id, K, N)} of the W4 attention projections."""
    hd = shape.head_dim
    return {"wqkv": (QKV_MATRIX, shape.hidden, (shape.n_heads + 2 * shape.n_kv_heads) * hd),
            "wo": (O_MATRIX, shape.n_heads * hd, shape.hidden)}


@dataclass
class DenseWeights:
    embed: torch.Tensor                  # [V, d]
    layers: list = field(default_factory=list)  # dicts: ln1, wqkv, wo (ops.W4Lin | None on CPU), ln2, wg
    norm: torch.Tensor | None = None     # [d]
    lm_head: torch.Tensor | None = None  # [d, V]
    shape: ModelShape | None = None
    attn_seed: int = 0                   # generator seed of the W4 attention projections

    def to(self, device) -> "DenseWeights":
        """Move to `device`; the W4 attention linears are (re)generated there
        by the counter-based generator (identical bytes on any device;
        oracle/w4_ref.gen_linear regenerates them on the CPU)."""
        device = torch.device(device)
        mv = lambda t: t.to(device, non_blocking=False)
        layers = []
        for l, L in enumerate(self.layers):
            out = {}
            for k, v in L.items():
                if isinstance(v, torch.Tensor):
                    out[k] = mv(v)
                elif device.type == "cuda":
                    out[k] = v if (v is not None and v.blob.device == device) else \
                        _gen_attn(self.shape, self.attn_seed, l, k, device)
                else:
                    out[k] = None
            layers.append(out)
        return DenseWeights(embed=mv(self.embed), layers=layers, norm=mv(self.norm), lm_head=mv(self.lm_head),
                            shape=self.shape, attn_seed=self.attn_seed)

    def nbytes(self) -> int:
        n = self.embed.nbytes + self.norm.nbytes + self.lm_head.nbytes
        return n + sum(t.nbytes for L in self.layers for t in L.values() if t is not None)


def _gen_attn(shape: ModelShape, seed: int, layer: int, name: str, device) -> "ops.W4Lin":
    m, K, N = attn_linear_shapes(shape)[name]
    return ops.W4Lin.generate(seed, layer, ATTN_TAG, m, K, N, shape.group_size, device)


def init_dense_weights(shape: ModelShape, seed: int, device="cpu", std: float = 0.02) -> DenseWeights:
    """Random-init non-MoE weights: embedding, lm_head and router bf16
    N(0, std) (deterministic per (seed, device type)); norms = 1; attention
    projections W4 from the counter-based generator keyed by (seed, layer,
    ATTN_TAG, matrix) — device-independent bytes, generated on the GPU (None
    in a CPU copy)."""
    device = torch.device(device)
    g = torch.Generator(device=device).manual_seed(seed)
    d = shape.hidden
    bf = torch.bfloat16

    def randn(*s):
        return (torch.randn(*s, generator=g, device=device, dtype=torch.float32) * std).to(bf)

    embed = randn(shape.vocab, d)
    layers = []
    for l in range(shape.num_layers):
        layers.append({
            "ln1": torch.ones(d, dtype=bf, device=device),
            "wqkv": _gen_attn(shape, seed, l, "wqkv", device) if device.type == "cuda" else None,
            "wo": _gen_attn(shape, seed, l, "wo", device) if device.type == "cuda" else None,
            "ln2": torch.ones(d, dtype=bf, device=device),
            "wg": randn(shape.num_experts, d),
        })
    return DenseWeights(embed=embed, layers=layers, norm=torch.ones(d, dtype=bf, device=device),
                        lm_head=randn(d, shape.vocab), shape=shape, attn_seed=seed)


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


def _qkv(shape: ModelShape, L: dict, a: torch.Tensor):
    """a [T, d] bf16 -> q [T, nh, hd], k, v [T, nkv, hd] (bf16) through the W4 q|k|v linear."""
    T = a.shape[0]
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    lin = L["wqkv"]
    y = torch.empty((T, lin.N), dtype=torch.float32, device=a.device)
    ws = None
    if T > ops.GEMV_MAX_ROWS:
        nb = ops.linear_workspace(T, lin.K, lin.N)
        ws = torch.empty(nb, dtype=torch.uint8, device=a.device) if nb else None
    ops.w4_linear(a, lin, y, ws)
    y = y.to(torch.bfloat16)
    q = y[:, : nh * hd].view(T, nh, hd)
    k = y[:, nh * hd:(nh + nkv) * hd].view(T, nkv, hd)
    v = y[:, (nh + nkv) * hd:].view(T, nkv, hd)
    return q, k, v


def _o_proj_residual(L: dict, o: torch.Tensor, h: torch.Tensor) -> torch.Tensor:
    """bf16( f32(h) + o Wo^T ) with the W4 o linear (f32 accumulation, one rounding)."""
    T = o.shape[0]
    lin = L["wo"]
    y = torch.empty((T, lin.N), dtype=torch.float32, device=o.device)
    ws = None
    if T > ops.GEMV_MAX_ROWS:
        nb = ops.linear_workspace(T, lin.K, lin.N)
        ws = torch.empty(nb, dtype=torch.uint8, device=o.device) if nb else None
    ops.w4_linear(o.contiguous(), lin, y, ws)
    return (h.float() + y).to(torch.bfloat16)


def attention_block(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCache, layer: int, pos0: int,
                    cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """h [T, d] bf16 (positions pos0 .. pos0+T-1) -> h + attn(norm(h)) (bf16)."""
    T = h.shape[0]
    nh, hd = shape.n_heads, shape.head_dim
    a = rms_norm(h, L["ln1"], shape.rms_eps)
    q, k, v = _qkv(shape, L, a)
    c, s = cos[pos0:pos0 + T], sin[pos0:pos0 + T]
    q, k = apply_rope(q, c, s), apply_rope(k, c, s)
    kv.k[layer, :, pos0:pos0 + T] = k.transpose(0, 1)
    kv.v[layer, :, pos0:pos0 + T] = v.transpose(0, 1)
    K = kv.k[layer, :, :pos0 + T].unsqueeze(0)
    V = kv.v[layer, :, :pos0 + T].unsqueeze(0)
    o = F.scaled_dot_product_attention(q.transpose(0, 1).unsqueeze(0), K, V, is_causal=(T > 1 and pos0 == 0),
                                       enable_gqa=True)
    o = o.squeeze(0).transpose(0, 1).reshape(T, nh * hd)
    return _o_proj_residual(L, o, h)


def attention_decode_static(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCache, layer: int,
                            pos: torch.Tensor, mask: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """One decode token with the position on the device (CUDA-graph capturable):
    h [1, d]; pos int64 [1]; mask [1, 1, 1, max_seq] additive (0 for <= pos, -inf after)."""
    nh, hd = shape.n_heads, shape.head_dim
    a = rms_norm(h, L["ln1"], shape.rms_eps)
    q, k, v = _qkv(shape, L, a)
    c, s = cos.index_select(0, pos), sin.index_select(0, pos)
    q, k = apply_rope(q, c, s), apply_rope(k, c, s)
    kv.k[layer].index_copy_(1, pos, k.transpose(0, 1))
    kv.v[layer].index_copy_(1, pos, v.transpose(0, 1))
    o = F.scaled_dot_product_attention(q.transpose(0, 1).unsqueeze(0), kv.k[layer].unsqueeze(0),
                                       kv.v[layer].unsqueeze(0), attn_mask=mask, enable_gqa=True)
    o = o.squeeze(0).transpose(0, 1).reshape(1, nh * hd)
    return _o_proj_residual(L, o, h)


def decode_front_fused(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCache, layer: int, pos: torch.Tensor,
                       mask: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, h1: torch.Tensor,
                       a2: torch.Tensor) -> None:
    """attention_decode_static + the post-attention RMSNorm for one token, with
    the elementwise steps in csrc/front.cu: rmsnorm -> W4 q|k|v GEMV -> RoPE +
    KV write -> SDPA -> W4 o GEMV -> residual + rmsnorm.  Writes h1 (the
    residual stream after attention) and a2 (the MoE block input)."""
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    dev = h.device
    a = ops.rmsnorm(h, L["ln1"], shape.rms_eps, torch.empty_like(h))
    lin = L["wqkv"]
    y = torch.empty((1, lin.N), dtype=torch.float32, device=dev)
    ops.w4_linear(a, lin, y)
    q = torch.empty((nh, hd), dtype=torch.bfloat16, device=dev)
    ops.rope_kv_decode(y, nh, nkv, hd, cos, sin, pos, q, kv.k[layer], kv.v[layer])
    o = F.scaled_dot_product_attention(q.view(1, nh, 1, hd), kv.k[layer].unsqueeze(0), kv.v[layer].unsqueeze(0),
                                       attn_mask=mask, enable_gqa=True)
    o = o.reshape(1, nh * hd)
    lo = L["wo"]
    yo = torch.empty((1, lo.N), dtype=torch.float32, device=dev)
    ops.w4_linear(o, lo, yo)
    ops.residual_rmsnorm(h, yo, L["ln2"], shape.rms_eps, h1, a2)


def logits_last(shape: ModelShape, W: DenseWeights, h_last: torch.Tensor) -> torch.Tensor:
    return (rms_norm(h_last, W.norm, shape.rms_eps) @ W.lm_head).float()


# ------------------------------------------------------------- batched serving
# B sequences of equal prompt length served together (BASELINE config 4:
# batch 1-32 x prompt 128-2048).  Same numerics as the single-sequence path:
# the projections take the B*T rows at once (GEMV for <= GEMV_MAX_ROWS rows,
# else the tcgen05 GEMM), attention runs per sequence inside one SDPA call.

class KVCacheBatch:
    """[L, B, kv_heads, max_seq, head_dim] bf16 keys / values; every sequence
    of the batch sits at the same position (equal prompt lengths)."""

    def __init__(self, shape: ModelShape, batch: int, max_seq: int, device):
        self.k = torch.zeros(shape.num_layers, batch, shape.n_kv_heads, max_seq, shape.head_dim,
                             dtype=torch.bfloat16, device=device)
        self.v = torch.zeros_like(self.k)
        self.len = 0

    @property
    def nbytes(self) -> int:
        return self.k.nbytes + self.v.nbytes


def attention_block_batch(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCacheBatch, layer: int, pos0: int,
                          cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """h [B, T, d] bf16 (positions pos0 .. pos0+T-1 of every sequence) -> h + attn(norm(h))."""
    B, T, d = h.shape
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    hf = h.reshape(B * T, d)
    a = rms_norm(hf, L["ln1"], shape.rms_eps)
    q, k, v = _qkv(shape, L, a)                                  # [B*T, heads, hd]
    c, s = cos[pos0:pos0 + T].repeat(B, 1), sin[pos0:pos0 + T].repeat(B, 1)
    q, k = apply_rope(q, c, s), apply_rope(k, c, s)
    kv.k[layer, :, :, pos0:pos0 + T] = k.view(B, T, nkv, hd).transpose(1, 2)
    kv.v[layer, :, :, pos0:pos0 + T] = v.view(B, T, nkv, hd).transpose(1, 2)
    K = kv.k[layer, :, :, :pos0 + T]
    V = kv.v[layer, :, :, :pos0 + T]
    o = F.scaled_dot_product_attention(q.view(B, T, nh, hd).transpose(1, 2), K, V,
                                       is_causal=(T > 1 and pos0 == 0), enable_gqa=True)
    o = o.transpose(1, 2).reshape(B * T, nh * hd)
    return _o_proj_residual(L, o, hf).view(B, T, d)


def attention_decode_static_batch(shape: ModelShape, L: dict, h: torch.Tensor, kv: KVCacheBatch, layer: int,
                                  pos: torch.Tensor, mask: torch.Tensor, cos: torch.Tensor,
                                  sin: torch.Tensor) -> torch.Tensor:
    """One decode token per sequence with the position on the device (CUDA-graph
    capturable): h [B, d]; pos int64 [1]; mask [1, 1, 1, max_seq] additive."""
    B = h.shape[0]
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    a = rms_norm(h, L["ln1"], shape.rms_eps)
    q, k, v = _qkv(shape, L, a)                                  # [B, heads, hd]
    c, s = cos.index_select(0, pos).expand(B, -1), sin.index_select(0, pos).expand(B, -1)
    q, k = apply_rope(q, c, s), apply_rope(k, c, s)
    kv.k[layer].index_copy_(2, pos, k.unsqueeze(2))             # [B, nkv, 1, hd] at position pos
    kv.v[layer].index_copy_(2, pos, v.unsqueeze(2))
    o = F.scaled_dot_product_attention(q.unsqueeze(2), kv.k[layer], kv.v[layer], attn_mask=mask, enable_gqa=True)
    o = o.squeeze(2).reshape(B, nh * hd)
    return _o_proj_residual(L, o, h)
