"""This build's W4 blob linear <-> the AWQ checkpoint layout (oracle / test
infrastructure).

AWQ as read by the installed third-party vLLM 0.22.0
(vllm/model_executor/layers/quantization/awq.py:213-251, awq_triton.py:54-101,
awq_marlin.py:74-156):
    qweight int32 [K, N/8]   8 output columns per word; column 8c + i sits in
                             nibble j with AWQ_PACK[j] = i, i.e. vLLM unpacks
                             nibble j and reorders with [0, 4, 1, 5, 2, 6, 3, 7]
    qzeros  int32 [K/G, N/8] same packing
    scales  fp16  [K/G, N]
    w[k, n] = (q[k, n] - z[k/G, n]) * s[k/G, n]
This build stores the transpose (output-major, oracle/w4_ref.py): codes u32
[N, K/8], bf16 scales [N, K/G], u4 zeros [N*K/G].  The bf16 scales convert to
fp16 exactly (8 significant bits, exponents of the generator's range,
0.5/(8 sqrt(K)) .. 1.5/(8 sqrt(K)), are fp16 normals), so the conversion is
lossless and the vLLM-side dequantisation must give the same weights.
"""

from __future__ import annotations

import numpy as np

from . import w4_ref

AWQ_PACK = np.array([0, 2, 4, 6, 1, 3, 5, 7])      # nibble j holds column 8c + AWQ_PACK[j]


def _pack_awq(vals: np.ndarray) -> np.ndarray:
    """uint8 [R, N] (values < 16) -> int32 [R, N/8] in AWQ nibble order."""
    R, N = vals.shape
    v = vals.reshape(R, N // 8, 8).astype(np.uint32)
    out = np.zeros((R, N // 8), dtype=np.uint32)
    for j in range(8):
        out |= v[:, :, AWQ_PACK[j]] << np.uint32(4 * j)
    return out.view(np.int32)


def to_awq(codes: np.ndarray, scales_bits: np.ndarray, zeros: np.ndarray, K: int, N: int, G: int):
    """(qweight int32 [K, N/8], qzeros int32 [K/G, N/8], scales fp16 [K/G, N])."""
    q = w4_ref.unpack_codes(codes)                              # [N, K] logical order
    z = w4_ref.unpack_zeros(zeros, N, K // G)                   # [N, K/G]
    s = w4_ref.bf16_bits_to_f32(scales_bits)                    # [N, K/G] f32 (exact bf16 values)
    s16 = s.astype(np.float16)
    if not np.array_equal(s16.astype(np.float32), s):
        raise ValueError("scales not exactly representable in fp16")
    return _pack_awq(np.ascontiguousarray(q.T)), _pack_awq(np.ascontiguousarray(z.T)), np.ascontiguousarray(s16.T)
