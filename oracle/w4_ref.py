"""W4 expert format: counter-based generator + dequantisation (oracle).

No reference code exists for the expert FFN (PAPER.md:188,192 use vLLM's AWQ
operators, unpinned).  The dequant rule follows AWQ as shipped in the
installed third-party vLLM 0.22.0 (vllm/model_executor/layers/quantization/
awq_triton.py:54-101: w = (q - z) * s), with one rounding to bf16:
    w = bf16_rn(f32(q - z) * f32(s)).
Storage (include/duoserve_b200.h):
    codes u32 [N, K/8], nibble j of word w holds q[n, 8w + PERM[j]]
    scales bf16 [N, K/G];  zeros u4 [N*K/G], low nibble first.
The generator restates paper_2509_07379_b200/csrc/ds_common.cuh (mix64 /
stream_key / draw) and csrc/w4.cu (gen_*_kernel) bit-for-bit.
"""

from __future__ import annotations

import numpy as np

PERM = np.array([0, 2, 4, 6, 1, 3, 5, 7])
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _u64(x):
    return np.uint64(x & 0xFFFFFFFFFFFFFFFF)


def mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, layer: int, expert: int, matrix: int, kind: int) -> np.uint64:
    tag = np.array([(((layer * 64 + expert) * 4 + matrix) * 4 + kind)], dtype=np.uint64)
    s = np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return mix64(s ^ mix64(tag))[0]


def draw(key: np.uint64, counters: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return mix64((np.uint64(key) + counters.astype(np.uint64) * np.uint64(0xD1B54A32D192ED03)).astype(np.uint64))


def bf16_round_bits(f32: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern, round-to-nearest-even (finite inputs)."""
    u = np.asarray(f32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << np.uint32(16)).view(np.float32)


def gen_linear(seed, layer, expert, matrix, K, N, G):
    """(codes u32 [N, K/8], scales bf16-bits u16 [N, K/G], zeros u8 [ceil(N*K/G/2)])."""
    words = N * K // 8
    r = draw(stream_key(seed, layer, expert, matrix, 0), np.arange((words + 1) // 2, dtype=np.uint64))
    codes = np.empty(2 * r.size, dtype=np.uint32)
    codes[0::2] = (r & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    codes[1::2] = (r >> np.uint64(32)).astype(np.uint32)
    codes = codes[:words].reshape(N, K // 8)
    groups = N * (K // G)
    inv = np.float32(1.0) / (np.float32(8.0) * np.sqrt(np.float32(K)))
    u = (draw(stream_key(seed, layer, expert, matrix, 2), np.arange(groups, dtype=np.uint64))
         >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    scales = bf16_round_bits((np.float32(0.5) + u) * inv).reshape(N, K // G)
    nz = (groups + 1) // 2
    rz = draw(stream_key(seed, layer, expert, matrix, 1), np.arange((nz + 7) // 8, dtype=np.uint64))
    zb = np.stack([(rz >> np.uint64(8 * i)) & np.uint64(0xFF) for i in range(8)], axis=1).reshape(-1)
    zeros = zb[:nz].astype(np.uint8)
    return codes, scales, zeros


def unpack_codes(codes: np.ndarray) -> np.ndarray:
    """u32 [N, K/8] -> q uint8 [N, K] in logical k order."""
    N, W = codes.shape
    nib = np.stack([(codes >> np.uint32(4 * j)) & np.uint32(15) for j in range(8)], axis=-1)
    q = np.empty((N, W, 8), dtype=np.uint8)
    q[:, :, PERM] = nib
    return q.reshape(N, W * 8)


def pack_codes(q: np.ndarray) -> np.ndarray:
    """inverse of unpack_codes."""
    N, K = q.shape
    q = q.reshape(N, K // 8, 8).astype(np.uint32)
    out = np.zeros((N, K // 8), dtype=np.uint32)
    for j in range(8):
        out |= q[:, :, PERM[j]] << np.uint32(4 * j)
    return out


def unpack_zeros(zeros: np.ndarray, N: int, groups_per_row: int) -> np.ndarray:
    z = np.empty(zeros.size * 2, dtype=np.uint8)
    z[0::2] = zeros & 15
    z[1::2] = zeros >> 4
    return z[: N * groups_per_row].reshape(N, groups_per_row)


def dequant(codes, scales, zeros, K, N, G) -> np.ndarray:
    """bf16 bit patterns [N, K] of w = bf16_rn((q - z) * s)."""
    q = unpack_codes(codes).astype(np.int32)
    z = np.repeat(unpack_zeros(zeros, N, K // G).astype(np.int32), G, axis=1)
    s = np.repeat(bf16_bits_to_f32(scales), G, axis=1)
    return bf16_round_bits((q - z).astype(np.float32) * s)


def expert_layout(d: int, ff: int, G: int):
    """Section offsets {c1,c3,c2,s1,s3,s2,z1,z3,z2} + total (256-B aligned),
    restating ds_w4_expert_layout (csrc/w4.cu)."""
    al = lambda v: (v + 255) // 256 * 256
    sizes = [ff * d // 2, ff * d // 2, d * ff // 2, ff * (d // G) * 2, ff * (d // G) * 2,
             d * (ff // G) * 2, (ff * (d // G) + 1) // 2, (ff * (d // G) + 1) // 2,
             (d * (ff // G) + 1) // 2]
    offs, off = [], 0
    for s in sizes:
        offs.append(off)
        off = al(off + s)
    return offs, off


def gen_expert_blob(seed, layer, expert, d, ff, G) -> np.ndarray:
    offs, total = expert_layout(d, ff, G)
    blob = np.zeros(total, dtype=np.uint8)
    KN = [(d, ff), (d, ff), (ff, d)]
    for m, (K, N) in enumerate(KN):
        c, s, z = gen_linear(seed, layer, expert, m, K, N, G)
        for sec, arr in ((m, c), (3 + m, s), (6 + m, z)):
            b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
            blob[offs[sec]:offs[sec] + b.size] = b
    return blob


def expert_dense(seed, layer, expert, d, ff, G):
    """float32 dense weights (W1 [d, ff], W3 [d, ff], W2 [ff, d]) in x@W form."""
    out = []
    for m, (K, N) in enumerate([(d, ff), (d, ff), (ff, d)]):
        c, s, z = gen_linear(seed, layer, expert, m, K, N, G)
        out.append(bf16_bits_to_f32(dequant(c, s, z, K, N, G)).T.copy())
    return out


def dequant_exact(codes, scales, zeros, K, N, G) -> np.ndarray:
    """float64 [N, K] of (q - z) * s WITHOUT the bf16 rounding: the decode
    GEMV (K4) factorises the group scale out of the dot product,
        sum_k x_k (q_k - z) s = s * (sum_k x_k (128+q_k) - (128+z) sum_k x_k),
    so its reference weights are the exact products."""
    q = unpack_codes(codes).astype(np.float64)
    z = np.repeat(unpack_zeros(zeros, N, K // G).astype(np.float64), G, axis=1)
    s = np.repeat(bf16_bits_to_f32(scales).astype(np.float64), G, axis=1)
    return (q - z) * s
