"""Tiny Mixtral-style W4 model forward on the CPU (oracle, torch fp32).

PARITY UNPINNED BY THE REFERENCE: the reference computes no model forward
(PAPER.md:188-192 used third-party vLLM/AWQ, unpinned).
This restates the build's documented numerics from
their third-party sources so the B200 engine can be checked:
  * Mixtral decoder block: HF transformers 5.5.0 modeling_mixtral.py
    (RMSNorm, rotate-half RoPE, GQA attention, MixtralSparseMoeBlock
    :74-98 per-expert SiLU(gate)*up -> down, routing-weighted sum);
  * router: routing_ref (modeling_mixtral.py:109-116 semantics, fixed f64
    order, reference tie rule);
  * W4 dequant: w4_ref (vLLM awq_triton.py:54-101 rule).
Prefill experts use bf16-rounded dequantised weights (what the tcgen05 GEMM
consumes); decode experts use the exact (q - z) * s products (what the
factorised GEMV computes) — see oracle/w4_ref.py.  The W4 attention
projections (q|k|v fused, o; generator key (attn_seed, layer, ATTN_TAG,
matrix)) follow the same rule by row count: <= GEMV_MAX_ROWS rows take the
GEMV (exact products), more rows the GEMM (bf16-rounded weights); the o
projection adds to the residual in f32 with one bf16 rounding.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import routing_ref, w4_ref

BF = torch.bfloat16
ATTN_TAG, QKV_MATRIX, O_MATRIX = 63, 0, 1     # restated from paper_2509_07379_b200/model.py
GEMV_MAX_ROWS = 16                            # rows at or below which the product uses the GEMV


def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(BF).float()


def _bits(x: torch.Tensor) -> np.ndarray:
    return x.to(BF).contiguous().view(torch.int16).numpy().view(np.uint16)


class TinyMixtralRef:
    def __init__(self, shape, dense, seed: int, flash_p: bool = True):
        """shape: ModelShape-like (attributes), dense: DenseWeights on CPU (bf16).
        flash_p: emulate the fused attention kernels' bf16 probabilities."""
        self.s = shape
        self.flash_p = flash_p
        self.W = dense
        self.seed = seed
        d, ff, G = shape.hidden, shape.ffn, shape.group_size
        self.rounded, self.exact = {}, {}
        for l in range(shape.num_layers):
            for e in range(shape.num_experts):
                r, x = [], []
                for m, (K, N) in enumerate([(d, ff), (d, ff), (ff, d)]):
                    c, sc, z = w4_ref.gen_linear(seed, l, e, m, K, N, G)
                    r.append(torch.from_numpy(w4_ref.bf16_bits_to_f32(w4_ref.dequant(c, sc, z, K, N, G))))
                    x.append(torch.from_numpy(w4_ref.dequant_exact(c, sc, z, K, N, G)).float())
                self.rounded[(l, e)] = r          # [N, K] each
                self.exact[(l, e)] = x
        hd = shape.head_dim
        self.attn_w = {}                          # (layer, name) -> (rounded [N, K], exact [N, K])
        aseed = getattr(dense, "attn_seed", 0)
        for l in range(shape.num_layers):
            for name, m, K, N in (("wqkv", QKV_MATRIX, d, (shape.n_heads + 2 * shape.n_kv_heads) * hd),
                                  ("wo", O_MATRIX, shape.n_heads * hd, d)):
                c, sc, z = w4_ref.gen_linear(aseed, l, ATTN_TAG, m, K, N, G)
                self.attn_w[(l, name)] = (torch.from_numpy(w4_ref.bf16_bits_to_f32(w4_ref.dequant(c, sc, z, K, N, G))),
                                        torch.from_numpy(w4_ref.dequant_exact(c, sc, z, K, N, G)).float())
        hd = shape.head_dim
        inv = 1.0 / (shape.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
        f = torch.outer(torch.arange(4096, dtype=torch.float32), inv)
        emb = torch.cat([f, f], -1)
        self.cos, self.sin = emb.cos(), emb.sin()
        self.reset()

    def reset(self):
        L = self.s.num_layers
        self.K = [None] * L
        self.V = [None] * L
        self.pos = 0

    def norm(self, x, g):
        return _bf(x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.s.rms_eps) * g.float())

    def rope(self, x, p0):
        T = x.shape[0]
        c, s = self.cos[p0:p0 + T][:, None, :], self.sin[p0:p0 + T][:, None, :]
        h = x.shape[-1] // 2
        rot = torch.cat([-x[..., h:], x[..., :h]], -1)
        return _bf(x * c + rot * s)

    def _w(self, l, name, rows):
        r, x = self.attn_w[(l, name)]
        return x if rows <= GEMV_MAX_ROWS else r

    def attn(self, l, h):
        s = self.s
        Lw = self.W.layers[l]
        T = h.shape[0]
        a = self.norm(h, Lw["ln1"])
        nh, nkv, hd = s.n_heads, s.n_kv_heads, s.head_dim
        y = _bf(a @ self._w(l, "wqkv", T).T)
        q = y[:, : nh * hd].reshape(T, nh, hd)
        k = y[:, nh * hd:(nh + nkv) * hd].reshape(T, nkv, hd)
        v = y[:, (nh + nkv) * hd:].reshape(T, nkv, hd)
        q, k = self.rope(q, self.pos), self.rope(k, self.pos)
        self.K[l] = k if self.K[l] is None else torch.cat([self.K[l], k])
        self.V[l] = v if self.V[l] is None else torch.cat([self.V[l], v])
        Kx = self.K[l].repeat_interleave(s.n_heads // s.n_kv_heads, dim=1)
        Vx = self.V[l].repeat_interleave(s.n_heads // s.n_kv_heads, dim=1)
        S = torch.einsum("thd,shd->hts", q, Kx) / math.sqrt(s.head_dim)
        n = Kx.shape[0]
        causal = torch.arange(n)[None, :] <= (torch.arange(T)[:, None] + self.pos)
        S = S.masked_fill(~causal[None], float("-inf"))
        if self.flash_p:
            # the fused attention kernels' numerics: unnormalised probabilities
            # exp(S - rowmax) rounded to bf16 for the P V product (f32
            # accumulation), normalised by the f32 row sum afterwards
            m = S.amax(-1, keepdim=True)
            Pu = torch.exp(S - m)
            o = torch.einsum("hts,shd->thd", _bf(Pu), Vx) / Pu.sum(-1).transpose(0, 1)[..., None]
            o = _bf(o).reshape(T, -1)
        else:
            o = _bf(torch.einsum("hts,shd->thd", torch.softmax(S, -1), Vx)).reshape(T, -1)
        return _bf(h + o @ self._w(l, "wo", T).T)

    def gate(self, l, a):
        lg = routing_ref.gate_logits(_bits(a), _bits(self.W.layers[l]["wg"]))
        return routing_ref.topk_route(lg, self.s.top_k)

    def moe(self, l, h, decode: bool, idx_override=None):
        s = self.s
        a = self.norm(h, self.W.layers[l]["ln2"])
        idx, w = self.gate(l, a)
        if idx_override is not None:
            idx = idx_override
        experts = [(self.exact if decode else self.rounded)[(l, e)] for e in range(s.num_experts)]
        acc = moe_block(a, idx, w, experts)
        return _bf(h + acc), idx, a

    def forward(self, ids, decode: bool, idx_override=None):
        """ids: 1-D token ids at positions self.pos...; returns (logits of last, per-layer idx)."""
        h = _bf(self.W.embed[torch.as_tensor(ids)].float())
        idxs = []
        for l in range(self.s.num_layers):
            h = self.attn(l, h)
            h, idx, _ = self.moe(l, h, decode, None if idx_override is None else idx_override[l])
            idxs.append(idx)
        self.pos += len(ids)
        logits = _bf(self.norm(h[-1:], self.W.norm) @ self.W.lm_head.float())[0]
        return logits, idxs


def moe_block(a: torch.Tensor, idx: np.ndarray, w: np.ndarray, experts, round_h: bool = True,
              dtype=torch.float32) -> torch.Tensor:
    """Routing-weighted SwiGLU expert sum of HF MixtralSparseMoeBlock
    (modeling_mixtral.py:62-100: per selected expert SiLU(x W1^T) * (x W3^T),
    then W2, times the routing weight, summed over the k slots in j order).
    experts[e] = (W1 [ff, d], W3 [ff, d], W2 [d, ff]); round_h rounds the
    SwiGLU intermediate to bf16 as the kernels do (K3/K4 write bf16 h)."""
    T = a.shape[0]
    d = experts[0][2].shape[0]
    acc = torch.zeros((T, d), dtype=dtype)
    ws = torch.from_numpy(np.asarray(w)).to(dtype)
    x_all = a.to(dtype)
    for j in range(idx.shape[1]):
        for e in range(len(experts)):
            rows = np.nonzero(idx[:, j] == e)[0]
            if rows.size == 0:
                continue
            W1, W3, W2 = (m.to(dtype) for m in experts[e])
            x = x_all[rows]
            hh = torch.nn.functional.silu(x @ W1.T) * (x @ W3.T)
            if round_h:
                hh = _bf(hh).to(dtype)
            acc[rows] = acc[rows] + ws[rows, j:j + 1] * (hh @ W2.T)
    return acc
