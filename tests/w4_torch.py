"""Test helper: unpack a W4 expert blob into dense weights with torch (on the
blob's device), for the floating-point FFN parity checks at full shapes.

A restatement of oracle/w4_ref.unpack_codes / unpack_zeros / dequant /
dequant_exact on tensors, so 8x7B / 8x22B experts (58.7M / 100.7M weights per
matrix) unpack on the GPU in milliseconds.  It is pinned to w4_ref on the CPU
(tests/test_w4_torch.py, tiny shapes) and, at full size, to the C-ABI dequant
kernel which is pinned bit-exact to w4_ref (tests/test_gpu_parity_full.py).
"""

from __future__ import annotations

import torch

PERM = (0, 2, 4, 6, 1, 3, 5, 7)


def _sections(blob: torch.Tensor, d: int, ff: int, G: int):
    from oracle import w4_ref
    offs, total = w4_ref.expert_layout(d, ff, G)
    assert blob.numel() >= total
    KN = [(d, ff), (d, ff), (ff, d)]
    out = []
    for m, (K, N) in enumerate(KN):
        c = blob[offs[m]:offs[m] + N * K // 2].view(torch.int32).view(N, K // 8)
        s = blob[offs[3 + m]:offs[3 + m] + N * (K // G) * 2].view(torch.bfloat16).view(N, K // G)
        nz = (N * (K // G) + 1) // 2
        z = blob[offs[6 + m]:offs[6 + m] + nz]
        out.append((K, N, c, s, z))
    return out


def unpack_q(codes: torch.Tensor) -> torch.Tensor:
    """int32 [N, K/8] -> int32 [N, K] codes in logical k order."""
    N, W = codes.shape
    nib = torch.stack([(codes >> (4 * j)) & 15 for j in range(8)], dim=-1)
    q = torch.empty_like(nib)
    q[:, :, list(PERM)] = nib
    return q.reshape(N, W * 8)


def unpack_z(zeros: torch.Tensor, N: int, gpr: int) -> torch.Tensor:
    z = zeros.to(torch.int32)
    zz = torch.stack([z & 15, z >> 4], dim=-1).reshape(-1)
    return zz[: N * gpr].reshape(N, gpr)


def linear_weights(K: int, N: int, codes, scales, zeros, G: int, exact: bool, dtype=torch.float64) -> torch.Tensor:
    """[N, K] weights: exact (q - z) * s, or bf16_rn((q - z) * s) (as f32 product, one rounding)."""
    q = unpack_q(codes)
    z = unpack_z(zeros, N, K // G).repeat_interleave(G, dim=1)
    s = scales.float().repeat_interleave(G, dim=1)
    if exact:
        return (q - z).to(dtype) * s.to(dtype)
    return ((q - z).float() * s).to(torch.bfloat16).to(dtype)


def expert_weights(blob: torch.Tensor, d: int, ff: int, G: int, exact: bool, dtype=torch.float64):
    """(W1 [ff, d], W3 [ff, d], W2 [d, ff]) in y = x W^T form."""
    return [linear_weights(K, N, c, s, z, G, exact, dtype) for K, N, c, s, z in _sections(blob, d, ff, G)]


def expert_ffn(x: torch.Tensor, W, round_h: bool = True) -> torch.Tensor:
    """y = W2 (bf16(silu(x W1^T) * (x W3^T))) in W's dtype (x bf16 or float)."""
    xd = x.to(W[0].dtype)
    g = xd @ W[0].T
    u = xd @ W[1].T
    h = torch.nn.functional.silu(g) * u
    if round_h:
        h = h.to(torch.bfloat16).to(W[0].dtype)
    return h @ W[2].T
