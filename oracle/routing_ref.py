"""Gate top-k, permute and combine (oracle).

No reference code (routing is only sampled in the reference,
trace.py:178-242).  Semantics: HF MixtralTopKRouter (third-party
transformers 5.5.0, models/mixtral/modeling_mixtral.py:109-116: logits =
x W_g^T, softmax, top-k, renormalise) with the reference's tie rule
(predictor.py:419-421, lower index wins) and sorted k-tuples (trace.py:39-58).
The float64 accumulation order is the build's contract,
restated here so the indices are bit-exact:
  thread q in [0,256) sums 8-element vectors v = q, q+256, ... sequentially
  (bf16 x bf16 products are exact in f64); then P[q] += P[q+off] for
  off = 128, 64, ..., 1.
"""

from __future__ import annotations

import numpy as np

from .w4_ref import bf16_bits_to_f32


def gate_logits(x_bits: np.ndarray, wg_bits: np.ndarray) -> np.ndarray:
    """x_bits [T, d] uint16 (bf16), wg_bits [M, d] -> f64 logits [T, M]."""
    x = bf16_bits_to_f32(x_bits).astype(np.float64)
    w = bf16_bits_to_f32(wg_bits).astype(np.float64)
    T, d = x.shape
    M = w.shape[0]
    nvec = d // 8
    out = np.empty((T, M))
    for e in range(M):
        prod = x * w[e][None, :]                       # exact
        P = np.zeros((T, 256))
        for base in range(0, nvec, 256):
            vs = np.arange(base, min(base + 256, nvec))
            q = vs - base
            for j in range(8):
                P[:, q] = P[:, q] + prod[:, vs * 8 + j]
        off = 128
        while off:
            P[:, :off] = P[:, :off] + P[:, off:2 * off]
            off >>= 1
        out[:, e] = P[:, 0]
    return out


def topk_route(logits: np.ndarray, k: int):
    """(idx [T,k] ascending, w [T,k] f32) — lower index wins ties."""
    T, M = logits.shape
    idx = np.empty((T, k), dtype=np.int32)
    w = np.empty((T, k), dtype=np.float32)
    for t in range(T):
        order = np.argsort(-logits[t], kind="stable")[:k]
        top = logits[t][order[0]]
        sel = np.sort(order)
        ex = np.exp(logits[t][sel] - top)
        den = 0.0
        for v in ex:
            den = den + v
        idx[t] = sel
        w[t] = (ex / den).astype(np.float32)
    return idx, w


def permute(idx: np.ndarray, M: int):
    """Stable grouping by expert: (offsets [M+1], pos [T*k], src_token [T*k])."""
    flat = idx.reshape(-1)
    k = idx.shape[1]
    order = np.argsort(flat, kind="stable")
    pos = np.empty_like(order)
    pos[order] = np.arange(flat.size)
    offsets = np.zeros(M + 1, dtype=np.int32)
    offsets[1:] = np.cumsum(np.bincount(flat, minlength=M))
    return offsets, pos.astype(np.int32), (order // k).astype(np.int32)


def combine(y: np.ndarray, pos: np.ndarray, w: np.ndarray, resid_f32: np.ndarray) -> np.ndarray:
    """out = bf16(resid + sum_j w_j * y[pos_j]) with f32 mul/add in j order; returns f32 values."""
    from .w4_ref import bf16_round_bits
    T, k = w.shape
    acc = np.zeros_like(resid_f32, dtype=np.float32)
    for j in range(k):
        acc = (acc + (w[:, j:j + 1].astype(np.float32) * y[pos.reshape(T, k)[:, j]].astype(np.float32))).astype(np.float32)
    return bf16_bits_to_f32(bf16_round_bits((resid_f32.astype(np.float32) + acc).astype(np.float32)))
