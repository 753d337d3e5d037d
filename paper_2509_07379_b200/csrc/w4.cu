// W4 expert format, counter-based random init, dequantisation and the decode
// GEMV path (K4).
//
// The reference has no FFN (vLLM AWQ operators).  Format
// (DESIGN.md §W4): per linear y = x W with input K, output N, group G:
//   codes  u32 [N, K/8]  nibble j of word w holds q[n, 8w + kPerm[j]],
//                        kPerm = {0,2,4,6,1,3,5,7}, so (word >> 4i) & 0xF000F
//                        is the consecutive pair (q[2i], q[2i+1]);
//   scales bf16 [N, K/G]
//   zeros  u4  [N*K/G]   (nibble index n*K/G + g, low nibble first)
//   w[k, n] = bf16_rn( (q - z) * s )          (AWQ: awq_triton.py:54-101)
// N-major rows keep one output's K codes contiguous: 16-byte vector loads
// for the GEMV and 2-D TMA tiles for the tcgen05 grouped GEMM (w4_gemm.cu).
//
// Decode GEMV (K4): one warp per output row (x both W1 and W3 for SwiGLU),
// 128-bit streaming loads of codes, dequant in registers with the bf16
// exponent trick (0x4300 | q == 128 + q), mixed-precision FHFMA.BF16
// (f32 += bf16*bf16, no conversion instructions) and the group correction
//     sum_k x_k (q_k - z) s = s * ( sum_k x_k (128+q_k) - (128+z) sum_k x_k ),
// warp-shuffle reduction, SwiGLU / routing-weight epilogue fused.
#include "ds_common.cuh"
#include "sm100.cuh"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cstring>
#include <vector>

namespace ds {
namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

// ------------------------------------------------------------ generator
// kinds: 0 codes, 1 zeros, 2 scales.  matrix: 0 W1, 1 W3, 2 W2.
__global__ void gen_codes_kernel(uint64_t key, size_t n_words, uint32_t* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_words / 2;
         i += (size_t)gridDim.x * blockDim.x) {
        uint64_t r = draw(key, i);
        reinterpret_cast<uint2*>(out)[i] = make_uint2((uint32_t)r, (uint32_t)(r >> 32));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n_words & 1))
        out[n_words - 1] = (uint32_t)draw(key, n_words / 2);
}

__global__ void gen_zeros_kernel(uint64_t key, size_t n_bytes, uint8_t* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_bytes;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = (uint8_t)(draw(key, i >> 3) >> (8 * (i & 7)));
}

__global__ void gen_scales_kernel(uint64_t key, size_t n, int K, uint16_t* __restrict__ out) {
    const float inv = __fdiv_rn(1.0f, __fmul_rn(8.0f, __fsqrt_rn((float)K)));
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        float u = (float)(uint32_t)(draw(key, i) >> 40) * (1.0f / 16777216.0f);
        out[i] = f32_to_bf16_bits(__fmul_rn(__fadd_rn(0.5f, u), inv));
    }
}

// --------------------------------------------------------------- dequant
__global__ void dequant_kernel(const uint32_t* __restrict__ codes, const uint16_t* __restrict__ scales,
                               const uint8_t* __restrict__ zeros, int K, int N, int G,
                               __nv_bfloat16* __restrict__ out) {
    const size_t total = (size_t)N * K / 8;
    const int gpr = K / G;
    for (size_t wi = blockIdx.x * (size_t)blockDim.x + threadIdx.x; wi < total;
         wi += (size_t)gridDim.x * blockDim.x) {
        const int n = (int)(wi / (K / 8));
        const int k0 = (int)(wi % (K / 8)) * 8;
        const int g = k0 / G;
        const size_t zi = (size_t)n * gpr + g;
        const int z = (zeros[zi >> 1] >> ((zi & 1) * 4)) & 15;
        const float s = __uint_as_float((uint32_t)scales[zi] << 16);
        const uint32_t v = codes[wi];
        const int perm[8] = {0, 2, 4, 6, 1, 3, 5, 7};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int q = (v >> (4 * j)) & 15;
            out[(size_t)n * K + k0 + perm[j]] = __float2bfloat16_rn((float)(q - z) * s);
        }
    }
}

// -------------------------------------------------------------- GEMV (K4)
constexpr int kGemvThreads = 512;
constexpr int kRMax = 4;  // activation rows per pass (decode batch chunk)

struct W4Ptr {
    const uint32_t* codes;
    const uint16_t* scales;
    const uint8_t* zeros;
};

// Stage x [R, K] (bf16) in smem and the per-32 sums sum_k x_k (f32).
// 16-byte unit u of a row is stored at u ^ ((u >> 3) & 3): lane l reads the
// 4 units of its 32-k chunk c = 32*it + l, so without the swizzle 8 lanes of
// a quarter-warp phase would hit only 2 of the 8 16-byte bank groups.
__device__ __forceinline__ int swz_unit(int u) { return u ^ ((u >> 3) & 3); }

template <bool COHERENT = false>
__device__ __forceinline__ void stage_x(const __nv_bfloat16* __restrict__ x, int R, int K,
                                        uint32_t* xs, float* xsum) {
    const int words = K / 2;
    const int units = words / 4;                        // 16-byte units per row
    const uint4* xu = reinterpret_cast<const uint4*>(x);
    for (int i = threadIdx.x; i < R * units; i += blockDim.x) {
        const int r = i / units, u = i - r * units;
        // COHERENT: x was written earlier in the same kernel by other CTAs (L2 path, not .nc)
        *reinterpret_cast<uint4*>(xs + r * words + swz_unit(u) * 4) = COHERENT ? __ldcg(xu + i) : __ldg(xu + i);
    }
    __syncthreads();
    const int chunks = K / 32;
    for (int i = threadIdx.x; i < R * chunks; i += blockDim.x) {
        const uint32_t* p = xs + (size_t)i * 16;  // a chunk's 4 units stay inside the chunk
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) s += bf16_lo(p[j]) + bf16_hi(p[j]);
        xsum[i] = s;
    }
    __syncthreads();
}

// One warp per output row n (NMAT = 2: rows n of W1 and W3 for SwiGLU;
// NMAT = 1: row n of W2).  Lane l owns the 32-code chunks c = l + 32 i; the
// loads for U chunks x NMAT matrices (codes, scale, zero) are issued back to
// back before any math so each warp keeps U*NMAT*16 B per lane in flight.
// GUARD=false requires (K/32) % (32*U) == 0 (every lane owns exactly
// nchunks/32 chunks, batches of U) so the batch loop carries no predicates.
template <int R, int NMAT, int U, int G, bool GUARD>
__device__ __forceinline__ void gemv_row(const W4Ptr (&W)[NMAT], int n, int K,
                                         const uint32_t* __restrict__ xs, const float* __restrict__ xsum,
                                         float (&acc)[NMAT][R]) {
    constexpr int CPG_SHIFT = (G == 128) ? 2 : (G == 64 ? 1 : 0);   // log2(chunks per group)
    const int lane = threadIdx.x & 31;
    const int nchunks = K >> 5;
    const int gpr = K / G;
    const int zbase = n * gpr;                  // nibble index of group 0 of this row
    const uint4* crow[NMAT];
    const uint16_t* srow[NMAT];
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
        crow[m] = reinterpret_cast<const uint4*>(W[m].codes + (size_t)n * (K >> 3)) + lane;
        srow[m] = W[m].scales + zbase;
    }
#pragma unroll
    for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[m][r] = 0.f;
    for (int c0 = lane; c0 < nchunks; c0 += 32 * U) {
        uint4 cv[U][NMAT];
        uint16_t sv[U][NMAT];
        uint8_t zv[U][NMAT];
        const int cb = c0 - lane;               // batch base chunk (warp-uniform)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = c0 + 32 * u;
            if (!GUARD || c < nchunks) {
                const int g = c >> CPG_SHIFT;
#pragma unroll
                for (int m = 0; m < NMAT; ++m) {
                    cv[u][m] = ldg_nc_v4(crow[m] + cb + 32 * u);
                    sv[u][m] = __ldg(srow[m] + g);
                    zv[u][m] = __ldg(W[m].zeros + ((zbase + g) >> 1));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = c0 + 32 * u;
            if (!GUARD || c < nchunks) {
                const int zsh = ((zbase + (c >> CPG_SHIFT)) & 1) << 2;
                const int sw = (c >> 1) & 3;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t* xc = xs + r * (K >> 1) + (c << 4);
                    const float xsm = xsum[r * nchunks + c];
                    uint4 xv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const uint4*>(xc + 4 * (i ^ sw));
#pragma unroll
                    for (int m = 0; m < NMAT; ++m) {
                        const uint32_t cw[4] = {cv[u][m].x, cv[u][m].y, cv[u][m].z, cv[u][m].w};
                        float p[4] = {0.f, 0.f, 0.f, 0.f};   // 4 independent FHFMA chains
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint32_t xx[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint32_t pr = nib_pair_magic(cw[i] >> (4 * q));
                                fma_bf16_lo(p[(q & 1) * 2], pr, xx[q]);
                                fma_bf16_hi(p[(q & 1) * 2 + 1], pr, xx[q]);
                            }
                        }
                        // 128 + z as an f32 built from bits (no I2F on the XU pipe)
                        const float z128 = __uint_as_float(0x43000000u | ((((uint32_t)zv[u][m] >> zsh) & 15u) << 16));
                        const float sc = __uint_as_float((uint32_t)sv[u][m] << 16);
                        acc[m][r] = fmaf(sc, ((p[0] + p[1]) + (p[2] + p[3])) - z128 * xsm, acc[m][r]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[m][r] = warp_sum(acc[m][r]);
}

// h[r, n] = bf16( silu(x_r . W1[:, n]) * (x_r . W3[:, n]) )
template <int R, int G, int U, bool GUARD>
__global__ void __launch_bounds__(kGemvThreads, 2) swiglu_gemv_kernel(
    const __nv_bfloat16* __restrict__ x, W4Ptr w1, W4Ptr w3, int K, int N,
    __nv_bfloat16* __restrict__ h) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* xs = sm;
    float* xsum = reinterpret_cast<float*>(sm + R * K / 2);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the down GEMV may launch early
    stage_x(x, R, K, xs, xsum);
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const W4Ptr W[2] = {w1, w3};
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += warps) {
        float acc[2][R];
        gemv_row<R, 2, U, G, GUARD>(W, n, K, xs, xsum, acc);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (lane == r) {
                const float av = acc[0][r], bv = acc[1][r];
                h[(size_t)r * N + n] = __float2bfloat16_rn(av / (1.0f + expf(-av)) * bv);
            }
        }
    }
}

// acc[r, n] += route_w[r] * (h_r . W2[:, n])
template <int R, int G, int U, bool GUARD>
__global__ void __launch_bounds__(kGemvThreads, 2) down_gemv_kernel(
    const __nv_bfloat16* __restrict__ hin, W4Ptr w2, int K, int N, const float* __restrict__ route_w,
    int route_stride, float* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* xs = sm;
    float* xsum = reinterpret_cast<float*>(sm + R * K / 2);
    asm volatile("griddepcontrol.wait;" ::: "memory");   // h comes from the SwiGLU GEMV (PDL launch)
    stage_x(hin, R, K, xs, xsum);
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const W4Ptr W[1] = {w2};
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += warps) {
        float acc[1][R];
        gemv_row<R, 1, U, G, GUARD>(W, n, K, xs, xsum, acc);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (lane == r) {
                float* o = out + (size_t)r * N + n;
                *o = __fadd_rn(*o, __fmul_rn(route_w[(size_t)r * route_stride], acc[0][r]));
            }
        }
    }
}

// ------------------------------------------ GEMV v5 (K4, bulk-staged, R = 1)
// The v2 GEMV keeps its weight stream in registers: each warp issues one
// batch of 16-byte loads per row and then computes, so the bytes in flight
// per SM are bounded by the warps that are not computing (DRAM 34 % busy
// under ncu).  Here one producer thread per CTA streams blocks of RB rows
// (codes, scales, zero nibbles: all three are row-major, so a row block is
// three contiguous 1-D bulk copies per matrix) into an S-deep shared-memory
// ring with cp.async.bulk + mbarrier transaction counts, and 16 consumer
// warps run the same per-row FHFMA dot product as v2 from shared memory
// (same chunk order and operations: bit-identical results).  One CTA per SM,
// ~180 KB of weights in flight per SM independent of compute.
//
// Row blocks are handed out by a ticket counter (one atomicAdd per block,
// prefetched one block ahead by the producer), not by a static split: a CTA
// that becomes resident late — measured on B200: with one 213 KB CTA per SM
// the 148th CTA of a grid of 148 started 15 us after the others — or shares
// its SM with the predictor K5 on another stream takes fewer blocks instead
// of stretching the kernel.  The producer ends each consumer group's stream
// with a sentinel block; counters live in a ring of kTicketSlots (one slot
// per launch, round-robin on the host), reset by the last producer to finish.
namespace k4s {
constexpr int kConsumers = 16;
constexpr int kThreads = 32 * (kConsumers + 1);
constexpr int kSmemBudget = 220 * 1024;
constexpr int kTicketSlots = 64;

template <int NMAT, int CPL, int G, int RB>
struct Geo {
    static constexpr int K = CPL * 1024;                  // 32 lanes x CPL chunks x 32 codes
    static constexpr int GPR = K / G;                     // groups per row
    static constexpr int CODE_B = K / 2;
    static constexpr int SC_B = GPR * 2;
    static constexpr int Z_B = (RB * GPR / 2 + 32 + 15) & ~15;   // 16-aligned superset of the rows' nibbles
    static constexpr int MAT_B = RB * CODE_B + RB * SC_B + Z_B;
    static constexpr int STAGE_B = NMAT * MAT_B;
    static constexpr int X_B = (K * 2 + (K / 32) * 4 + 127) & ~127;
};
}  // namespace k4s

__device__ unsigned g_k4s_ticket[k4s::kTicketSlots];

__device__ unsigned g_k4s_done[k4s::kTicketSlots];

// stage_x for the consumer warps only (named barrier 1): all loads of a
// thread are issued before its shared-memory stores
template <int K>
__device__ __forceinline__ void stage_x_consumers(const __nv_bfloat16* __restrict__ x, uint32_t* xs, float* xsum) {
    constexpr int NT = 32 * k4s::kConsumers;
    constexpr int UNITS = K / 8;                           // 16-byte units
    constexpr int PER = (UNITS + NT - 1) / NT;
    const uint4* xu = reinterpret_cast<const uint4*>(x);
    uint4 v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int i = threadIdx.x + j * NT;
        if (i < UNITS) v[j] = __ldg(xu + i);
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int i = threadIdx.x + j * NT;
        if (i < UNITS) *reinterpret_cast<uint4*>(xs + swz_unit(i) * 4) = v[j];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    for (int i = threadIdx.x; i < K / 32; i += NT) {
        const uint32_t* p = xs + (size_t)i * 16;
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) s += bf16_lo(p[j]) + bf16_hi(p[j]);
        xsum[i] = s;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// The producer thread of a bulk-staged GEMV CTA: takes row blocks from the
// ticket counter, streams each into the next ring slot, and ends every
// consumer group's stream with a sentinel block (hdr = -1).
template <int NMAT, int CPL, int G, int RB>
__device__ __forceinline__ void k4s_produce(const W4Ptr (&W)[2], int N, int S, int NG, uint8_t* stages, uint64_t* full,
                                            uint64_t* empty, int* hdr, unsigned slot_id, unsigned long long* dbg) {
    using namespace ds::sm100;
    using Gm = k4s::Geo<NMAT, CPL, G, RB>;
    constexpr int GPR = Gm::GPR;
    const int T = (N + RB - 1) / RB;
    unsigned* tk = g_k4s_ticket + slot_id;
    const uint64_t pol = l2_evict_first_policy();
    const int first = (int)atomicAdd(tk, (unsigned)S);   // the first S blocks in one grab
    int pending = -1;
    int sentinels = 0;
    for (int s = 0; sentinels < NG; ++s) {
        const int slot = s % S;
        if (s >= S) mbar_wait(&empty[slot], ((s / S) - 1) & 1);
        int t = s < S ? first + s : pending;
        if (s >= S - 1 && t < T) pending = (int)atomicAdd(tk, 1u);   // next block, latency hidden
        if (t >= T || t < 0) t = -1;
        hdr[slot] = t;
        if (t < 0) {
            mbar_arrive(&full[slot]);
            ++sentinels;
            continue;
        }
        const int r0 = t * RB, rows = min(RB, N - r0);
        uint8_t* dst = stages + (size_t)slot * Gm::STAGE_B;
        const uint32_t zb0 = ((uint32_t)(r0 * GPR) >> 1) & ~15u;
        const uint32_t zb1 = (((uint32_t)((r0 + rows) * GPR) >> 1) + 15u) & ~15u;
        const uint32_t cb = rows * Gm::CODE_B, sb = rows * Gm::SC_B, zb = zb1 - zb0;
        mbar_expect_tx(&full[slot], NMAT * (cb + sb + zb));
#pragma unroll
        for (int m = 0; m < NMAT; ++m) {
            uint8_t* md = dst + m * Gm::MAT_B;
            bulk_load(md, reinterpret_cast<const uint8_t*>(W[m].codes) + (size_t)r0 * Gm::CODE_B, cb, &full[slot], pol);
            bulk_load(md + RB * Gm::CODE_B, reinterpret_cast<const uint8_t*>(W[m].scales) + (size_t)r0 * Gm::SC_B, sb,
                      &full[slot], pol);
            bulk_load(md + RB * (Gm::CODE_B + Gm::SC_B), W[m].zeros + zb0, zb, &full[slot], pol);
        }
        if (s == 0 && dbg) {
            unsigned long long ts;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
            atomicMax(dbg + blockIdx.x * 8 + 1, ts);
        }
    }
    if (dbg) {
        unsigned long long ts;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
        atomicMax(dbg + blockIdx.x * 8 + 3, ts);
    }
    __threadfence();                                       // every ticket of this CTA is taken
    if (atomicAdd(g_k4s_done + slot_id, 1u) == gridDim.x - 1) {
        atomicExch(tk, 0u);
        atomicExch(g_k4s_done + slot_id, 0u);
    }
}

template <int NMAT, int CPL, int G, int RB, bool SWIGLU>
__global__ void __launch_bounds__(k4s::kThreads, 1) staged_gemv_kernel(
    const __nv_bfloat16* __restrict__ x, W4Ptr wa, W4Ptr wb, int N, int S, __nv_bfloat16* __restrict__ hout,
    const float* __restrict__ route_w, float* __restrict__ out, unsigned slot_id, unsigned long long* dbg) {
    using namespace ds::sm100;
    using Gm = k4s::Geo<NMAT, CPL, G, RB>;
    constexpr int K = Gm::K, GPR = Gm::GPR;
    constexpr int CPG_SHIFT = G == 128 ? 2 : 1;
    constexpr int NG = k4s::kConsumers / RB;              // consumer groups (one stage each)
    auto stamp = [&](int i) {          // DS_K4_TIMELINE: per-CTA globaltimer stamps (diagnostics only)
        if (dbg) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(dbg + blockIdx.x * 8 + i, t);
        }
    };
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* xs = reinterpret_cast<uint32_t*>(smem);
    float* xsum = reinterpret_cast<float*>(smem + K * 2);
    uint8_t* stages = smem + Gm::X_B;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)S * Gm::STAGE_B);
    uint64_t* empty = full + S;
    int* hdr = reinterpret_cast<int*>(empty + S);         // row block of each ring slot (-1: end of stream)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const W4Ptr W[2] = {wa, wb};
    if (threadIdx.x == 0) {
        stamp(0);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], RB);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if constexpr (SWIGLU)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the down GEMV may launch early

    if (warp == k4s::kConsumers) {                        // producer
        if (lane == 0)
            k4s_produce<NMAT, CPL, G, RB>(W, N, S, NG, stages, full, empty, hdr, slot_id, dbg);
        return;
    }

    if constexpr (!SWIGLU)
        asm volatile("griddepcontrol.wait;" ::: "memory");   // h comes from the SwiGLU GEMV (PDL launch)
    stage_x_consumers<K>(x, xs, xsum);
    if (threadIdx.x == 0) stamp(2);
    const int grp = warp / RB, r = warp % RB;
    bool first_stage = true;
    for (int s = grp;; s += NG) {
        const int slot = s % S;
        mbar_wait(&full[slot], (s / S) & 1);
        const int t = hdr[slot];
        if (t < 0) break;                                  // end of this group's stream
        if (first_stage && lane == 0) stamp(4);
        first_stage = false;
        const int r0 = t * RB;
        const int n = r0 + r;
        if (n < N) {
            const uint8_t* base = stages + (size_t)slot * Gm::STAGE_B;
            const uint32_t zb0 = ((uint32_t)(r0 * GPR) >> 1) & ~15u;
            float acc[NMAT];
#pragma unroll
            for (int m = 0; m < NMAT; ++m) acc[m] = 0.f;
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int c = lane + 32 * i;
                const int g = c >> CPG_SHIFT;
                const int sw = (c >> 1) & 3;
                const uint32_t* xc = xs + (c << 4);
                const float xsm = xsum[c];
                uint4 xv[4];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) xv[ii] = *reinterpret_cast<const uint4*>(xc + 4 * (ii ^ sw));
                const uint32_t zn = (uint32_t)(n * GPR + g);          // global nibble index of the zero
#pragma unroll
                for (int m = 0; m < NMAT; ++m) {
                    const uint8_t* mb = base + m * Gm::MAT_B;
                    const uint4 c4 = *reinterpret_cast<const uint4*>(mb + r * Gm::CODE_B + c * 16);
                    const uint16_t sv = reinterpret_cast<const uint16_t*>(mb + RB * Gm::CODE_B + r * Gm::SC_B)[g];
                    const uint8_t zv = mb[RB * (Gm::CODE_B + Gm::SC_B) + (zn >> 1) - zb0];
                    const uint32_t cw[4] = {c4.x, c4.y, c4.z, c4.w};
                    float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        const uint32_t xx[4] = {xv[ii].x, xv[ii].y, xv[ii].z, xv[ii].w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t pr = nib_pair_magic(cw[ii] >> (4 * q));
                            fma_bf16_lo(p[(q & 1) * 2], pr, xx[q]);
                            fma_bf16_hi(p[(q & 1) * 2 + 1], pr, xx[q]);
                        }
                    }
                    const float z128 = __uint_as_float(0x43000000u | ((((uint32_t)zv >> ((zn & 1) << 2)) & 15u) << 16));
                    const float sc = __uint_as_float((uint32_t)sv << 16);
                    acc[m] = fmaf(sc, ((p[0] + p[1]) + (p[2] + p[3])) - z128 * xsm, acc[m]);
                }
            }
#pragma unroll
            for (int m = 0; m < NMAT; ++m) acc[m] = warp_sum(acc[m]);
            if (lane == 0) {
                if constexpr (SWIGLU) {
                    const float av = acc[0], bv = acc[NMAT - 1];
                    hout[n] = __float2bfloat16_rn(av / (1.0f + expf(-av)) * bv);
                } else {
                    out[n] = __fadd_rn(out[n], __fmul_rn(route_w[0], acc[0]));
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (lane == 0) stamp(5);
}

// ------------------------------------------------- GEMV v3 (K4, mma.sync)
// G = 128.  The int4 -> bf16 dequant stays on the CUDA cores (7 ALU ops per
// 8 codes: the (128 + q) exponent trick) but the multiply-accumulate moves to
// the tensor cores: one mma.m16n8k16 consumes 16 weight rows x 16 k with the
// activation rows (<= 8 tokens) on the N side.  A CTA owns one 16-row block
// of the output; its S warps split K into runs of whole groups, so every
// warp-step is exactly one quantisation group (4 lanes x 32 codes per row):
//   lane (g, t) = (lane / 4, lane % 4) loads the 16-byte code chunk t of
//   rows g and g + 8 of the group; its 32 codes are the A fragments of 8 mmas
//   and the same k positions of x (64 contiguous bytes) its B fragments:
//   mma j = (word w, half s): a = {P_g[w][2s], P_g+8[w][2s], P_g[w][2s+1],
//   P_g+8[w][2s+1]} with P_r[w][i] = (128 + q) pair i of word w of row r,
//   b = x[c0 + 32t + 8w + 4s .. +4).  The k permutation inside an mma is the
//   same for A and B, so the dot product is unchanged.
// A ninth fragment set with A = 1.0 gives sum_k x per token and group, so
//   sum_k x (q - z) s = s * ( D - (128 + z) * sum_k x )
// (the same factorisation as v2, exact products (q - z) s).  Loads run P
// groups ahead in a register ring; the S per-warp partials are reduced in
// shared memory in a fixed order (deterministic).
constexpr int kTok = 8;  // activation rows per pass (mma N)

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Per-lane stream pointers, positioned at the warp's first group.
template <int NMAT>
struct GroupPtrs {
    const uint4* c[NMAT][2];
    const uint4* x;
};

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// codes of group j -> this lane's ring slot (lane-private: no warp sync needed)
template <int NMAT>
__device__ __forceinline__ void issue_codes(uint32_t slot, const GroupPtrs<NMAT>& q, int j) {
#pragma unroll
    for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) cp_async16(slot + (uint32_t)(m * 2 + h) * 512u, q.c[m][h] + 4 * j);
}

// x[tok][c0 + 32 t .. + 32) of group j: re-read by every row block, so it
// comes from L1 / L2; loaded one group ahead of its use
__device__ __forceinline__ void load_x(uint4 (&xv)[4], const uint4* __restrict__ x, int j) {
#pragma unroll
    for (int w = 0; w < 4; ++w) xv[w] = __ldg(x + 16 * j + w);
}

template <int NMAT>
__device__ __forceinline__ void mma_group(const uint4 (&c)[NMAT][2], const uint4 (&xv)[4],
                                          const uint16_t* __restrict__ sm_s, const uint8_t* __restrict__ sm_z,
                                          int ngw, int g, int j, float (&acc)[NMAT][4]) {
    // CH independent accumulator chains per matrix (and for sum x) cut the
    // dependent-HMMA latency per group; with NMAT = 2 the W1 / W3 chains
    // already interleave
    constexpr int CH = NMAT == 1 ? 2 : 1;
    float dx[CH][4] = {};
    float d[NMAT][CH][4] = {};
    constexpr uint32_t kOne = 0x3F803F80u;  // bf16 {1.0, 1.0}
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t xw[4] = {xv[w].x, xv[w].y, xv[w].z, xv[w].w};
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            mma16816(dx[s % CH], kOne, kOne, kOne, kOne, xw[2 * s], xw[2 * s + 1]);
#pragma unroll
            for (int m = 0; m < NMAT; ++m) {
                const uint32_t* cg = reinterpret_cast<const uint32_t*>(&c[m][0]);
                const uint32_t* cg8 = reinterpret_cast<const uint32_t*>(&c[m][1]);
                mma16816(d[m][s % CH], nib_pair_magic(cg[w] >> (8 * s)), nib_pair_magic(cg8[w] >> (8 * s)),
                         nib_pair_magic(cg[w] >> (8 * s + 4)), nib_pair_magic(cg8[w] >> (8 * s + 4)),
                         xw[2 * s], xw[2 * s + 1]);
            }
        }
    }
    float xs0 = dx[0][0], xs1 = dx[0][1];
#pragma unroll
    for (int c2 = 1; c2 < CH; ++c2) xs0 += dx[c2][0], xs1 += dx[c2][1];
    // rows g (regs 0, 1) and g + 8 (regs 2, 3); tokens 2t (even regs), 2t + 1 (odd)
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            // per-warp staged scale (bf16 bits) and zero (0..15) of row g + 8h, group j
            const int si = (m * 16 + g + 8 * h) * ngw + j;
            const float z128 = __uint_as_float(0x43000000u | ((uint32_t)sm_z[si] << 16));   // 128 + z
            const float sc = __uint_as_float((uint32_t)sm_s[si] << 16);
            float v0 = d[m][0][2 * h], v1 = d[m][0][2 * h + 1];
#pragma unroll
            for (int c2 = 1; c2 < CH; ++c2) v0 += d[m][c2][2 * h], v1 += d[m][c2][2 * h + 1];
            acc[m][2 * h] = fmaf(sc, fmaf(-z128, xs0, v0), acc[m][2 * h]);
            acc[m][2 * h + 1] = fmaf(sc, fmaf(-z128, xs1, v1), acc[m][2 * h + 1]);
        }
    }
}

// ring bytes per warp: P stages x NMAT matrices x 2 row halves x 32 lanes x 16 B
template <int NMAT, int P>
constexpr int mma_gemv_ring_bytes() { return P * NMAT * 2 * 512; }
// staged scales (2 B) + zeros (1 B) per warp: NMAT x 16 rows x ngw groups
__host__ __device__ inline int mma_gemv_aux_bytes(int nmat, int ngw) { return (nmat * 16 * ngw * 3 + 15) & ~15; }

// One CTA per 16-row block; warp s streams groups [s*ngw, min((s+1)*ngw, NG)).
// NMAT = 2: h[r, n] = bf16(silu(x_r . W1[:, n]) * (x_r . W3[:, n]));
// NMAT = 1: out[r, n] += route_w[r] * (x_r . W2[:, n]).
// The code stream (the HBM bytes) runs P groups ahead through a lane-private
// cp.async ring in shared memory, so the depth costs no registers; scales /
// zeros and x run one group ahead in registers.
template <int NMAT, int P>
__global__ void __launch_bounds__(NMAT == 2 ? 64 : 256, NMAT == 2 ? 7 : 1) mma_gemv_kernel(const __nv_bfloat16* __restrict__ x, int R, W4Ptr wa,
                                                       W4Ptr wb, int K, int N, int ngw,
                                                       __nv_bfloat16* __restrict__ h,
                                                       const float* __restrict__ route_w, int route_stride,
                                                       float* __restrict__ out) {
    static_assert(P % 2 == 0, "aux / x are double-buffered by the parity of the unrolled stage index");
    extern __shared__ __align__(16) uint8_t gemv_smem[];
    __shared__ float red[NMAT == 2 ? 2 : 8][NMAT][4][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, S = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int NG = K >> 7;
    const int rowg = blockIdx.x * 16 + g;
    const int gbeg = warp * ngw;
    const int nsteps = max(0, min(ngw, NG - gbeg));
    // B columns of tokens >= R read row R - 1 (same addresses: a broadcast);
    // their D columns are never stored
    const int tok = g < R ? g : R - 1;
    GroupPtrs<NMAT> q;
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
        const W4Ptr W = (m == 0) ? wa : wb;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int row = rowg + 8 * hh;
            q.c[m][hh] = reinterpret_cast<const uint4*>(W.codes + (size_t)row * (K >> 3)) + gbeg * 4 + t;
        }
    }
    q.x = reinterpret_cast<const uint4*>(x + (size_t)tok * K) + gbeg * 16 + 4 * t;
    // lane-private ring: slot (stage p, matrix m, half h) at p*NMAT*1024 + (2m+h)*512 + lane*16
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(gemv_smem) +
                          (uint32_t)warp * mma_gemv_ring_bytes<NMAT, P>() + lane * 16u;
    const uint8_t* ring_ptr = gemv_smem + warp * mma_gemv_ring_bytes<NMAT, P>() + lane * 16;
    // the warp's scales (bf16) and zeros (0..15) for its 16 rows x ngw groups,
    // staged once behind the rings (no per-group scattered 2-byte loads)
    const int aux_bytes = mma_gemv_aux_bytes(NMAT, ngw);
    uint16_t* sm_s = reinterpret_cast<uint16_t*>(gemv_smem + S * mma_gemv_ring_bytes<NMAT, P>() + warp * aux_bytes);
    uint8_t* sm_z = reinterpret_cast<uint8_t*>(sm_s + NMAT * 16 * ngw);
    // programmatic dependent launch: let the next kernel (the down projection
    // after the SwiGLU GEMV) be scheduled as SMs free up; everything before
    // griddepcontrol.wait touches only weights, never the previous kernel's output
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int i = lane; i < NMAT * 16 * nsteps; i += 32) {
        const int m = i / (16 * nsteps), rem = i - m * 16 * nsteps, r = rem / nsteps, jj = rem - r * nsteps;
        const W4Ptr W = (m == 0) ? wa : wb;
        const int zi = (blockIdx.x * 16 + r) * NG + gbeg + jj;
        sm_s[(m * 16 + r) * ngw + jj] = __ldg(W.scales + zi);
        sm_z[(m * 16 + r) * ngw + jj] = (__ldg(W.zeros + (zi >> 1)) >> ((zi & 1) << 2)) & 15;
    }
    __syncwarp();

    float acc[NMAT][4];
#pragma unroll
    for (int m = 0; m < NMAT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (p < nsteps) issue_codes<NMAT>(ring + (uint32_t)p * NMAT * 1024u, q, p);
        cp_async_commit();                  // (possibly empty) group p
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");   // x (and out) come from the previous kernel
    uint4 xv[2][4];
    if (nsteps > 0) load_x(xv[0], q.x, 0);
    for (int s0 = 0; s0 < nsteps; s0 += P) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int j = s0 + p;
            if (j < nsteps) {
                if (j + 1 < nsteps) load_x(xv[(p + 1) & 1], q.x, j + 1);
                cp_async_wait<P - 1>();      // this lane's group j landed
                uint4 c[NMAT][2];
#pragma unroll
                for (int m = 0; m < NMAT; ++m)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
                        c[m][hh] = *reinterpret_cast<const uint4*>(ring_ptr + p * NMAT * 1024 + (m * 2 + hh) * 512);
                if (j + P < nsteps) issue_codes<NMAT>(ring + (uint32_t)p * NMAT * 1024u, q, j + P);
                cp_async_commit();
                mma_group<NMAT>(c, xv[p & 1], sm_s, sm_z, ngw, g, j, acc);
            }
        }
    }
    if (S > 1) {
#pragma unroll
        for (int m = 0; m < NMAT; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) red[warp][m][i][lane] = acc[m][i];
        __syncthreads();
        if (warp != 0) return;
#pragma unroll
        for (int m = 0; m < NMAT; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float v = red[0][m][i][lane];
                for (int w = 1; w < S; ++w) v += red[w][m][i][lane];
                acc[m][i] = v;
            }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = rowg + 8 * (i >> 1);
        const int tk = 2 * t + (i & 1);
        if (tk < R) {
            if constexpr (NMAT == 2) {
                const float av = acc[0][i], bv = acc[1][i];
                h[(size_t)tk * N + row] = __float2bfloat16_rn(av / (1.0f + expf(-av)) * bv);
            } else {
                float* o = out + (size_t)tk * N + row;
                *o = __fadd_rn(*o, __fmul_rn(route_w[(size_t)tk * route_stride], acc[0][i]));
            }
        }
    }
}

// Warps per CTA.  SwiGLU (NMAT = 2, N/16 = 896..1024 row blocks): 2 warps,
// so that all ~7 CTAs per SM are resident at once (one wave: no tail wave of
// a few row blocks).  Down (256..384 row blocks): up to 8 warps splitting K.
// Variant choice for G = 128 (measured on B200, scripts/kbench.py, one
// expert of 8x7B): at R = 1 the warp-per-row FHFMA GEMV (v2) streams the
// expert in 39.8 us against 43.9 us for the mma.sync GEMV, which is
// latency-bound at one token; the mma.sync GEMV carries up to 8 activation
// rows per pass at the cost of one (tokens sit on the mma N side), so it
// takes every R >= 2.  DS_K4_VARIANT=v2|mma forces one (A/B benchmarks).
inline bool k4_use_mma(int R) {
    static const char* v = getenv("DS_K4_VARIANT");
    if (v && v[0] == 'v') return false;
    if (v && v[0] == 'm') return true;
    return R >= 2;
}

inline int mma_gemv_warps(int NG, int nmat) {
    if (nmat == 2) return NG >= 2 ? 2 : 1;
    int S = (NG + 7) / 8;
    return S < 1 ? 1 : (S > 8 ? 8 : S);
}


__global__ void finalize_kernel(float* __restrict__ acc, const __nv_bfloat16* __restrict__ resid,
                                size_t n, __nv_bfloat16* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        out[i] = __float2bfloat16_rn(__fadd_rn(__bfloat162float(resid[i]), acc[i]));
        acc[i] = 0.f;
    }
}

W4Ptr to_ptr(const ds_w4_linear& l) {
    return W4Ptr{l.codes, static_cast<const uint16_t*>(l.scales), l.zeros};
}

int gemv_grid(const void* fn, size_t smem, int rows_needed) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGemvThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int wpc = kGemvThreads / 32;
    int grid = per_sm * num_sms();
    int need = (rows_needed + wpc - 1) / wpc;
    if (grid >= need) return need;
    // (shrinking the grid so every warp runs the same number of rows measured
    // slower on B200: 39.8 vs 37.7 us per 8x7B expert — the tail pass is cheap)
    return grid;
}

bool check_linear(const ds_w4_linear& l) { return l.codes && l.scales && l.zeros; }

}  // namespace
}  // namespace ds

using namespace ds;

extern "C" size_t ds_w4_expert_layout(int d, int ff, int G, size_t offsets[9]) {
    if (d <= 0 || ff <= 0 || G <= 0 || d % G || ff % G || G % 32) return 0;
    const size_t codes13 = (size_t)ff * d / 2, codes2 = (size_t)d * ff / 2;
    const size_t sc13 = (size_t)ff * (d / G) * 2, sc2 = (size_t)d * (ff / G) * 2;
    const size_t z13 = ((size_t)ff * (d / G) + 1) / 2, z2 = ((size_t)d * (ff / G) + 1) / 2;
    const size_t sizes[9] = {codes13, codes13, codes2, sc13, sc13, sc2, z13, z13, z2};
    size_t off = 0;
    for (int i = 0; i < 9; ++i) {
        if (offsets) offsets[i] = off;
        off = align_up(off + sizes[i]);
    }
    return off;
}

extern "C" int ds_w4_generate(uint64_t seed, int layer, int expert, int d, int ff, int G, void* blob,
                              void* stream) {
    size_t off[9];
    DS_CHECK_ARG(ds_w4_expert_layout(d, ff, G, off) > 0, "ds_w4_generate: bad shape d=%d ff=%d G=%d", d, ff, G);
    DS_CHECK_ARG(blob && ((uintptr_t)blob & 255) == 0, "ds_w4_generate: blob must be 256B aligned");
    DS_CHECK_ARG(layer >= 0 && expert >= 0 && expert < 64, "ds_w4_generate: bad layer/expert");
    cudaStream_t st = as_stream(stream);
    char* base = static_cast<char*>(blob);
    const int Ks[3] = {d, d, ff}, Ns[3] = {ff, ff, d};
    const int grid = 4 * num_sms();
    for (int m = 0; m < 3; ++m) {
        const size_t words = (size_t)Ns[m] * Ks[m] / 8;
        const size_t groups = (size_t)Ns[m] * (Ks[m] / G);
        gen_codes_kernel<<<grid, 256, 0, st>>>(stream_key(seed, layer, expert, m, 0), words,
                                               (uint32_t*)(base + off[m]));
        gen_scales_kernel<<<grid, 256, 0, st>>>(stream_key(seed, layer, expert, m, 2), groups, Ks[m],
                                                (uint16_t*)(base + off[3 + m]));
        gen_zeros_kernel<<<grid, 256, 0, st>>>(stream_key(seed, layer, expert, m, 1), (groups + 1) / 2,
                                               (uint8_t*)(base + off[6 + m]));
    }
    DS_LAUNCH_CHECK("ds_w4_generate");
    return DS_OK;
}

extern "C" size_t ds_w4_linear_layout(int K, int N, int G, size_t offsets[3]) {
    if (K <= 0 || N <= 0 || G <= 0 || K % G || G % 32 || K % 8) return 0;
    const size_t sizes[3] = {(size_t)N * K / 2, (size_t)N * (K / G) * 2, ((size_t)N * (K / G) + 1) / 2};
    size_t off = 0;
    for (int i = 0; i < 3; ++i) {
        if (offsets) offsets[i] = off;
        off = align_up(off + sizes[i]);
    }
    return off;
}

extern "C" int ds_w4_generate_linear(uint64_t seed, int layer, int tag, int matrix, int K, int N, int G, void* blob,
                                     void* stream) {
    size_t off[3];
    DS_CHECK_ARG(ds_w4_linear_layout(K, N, G, off) > 0, "ds_w4_generate_linear: bad shape K=%d N=%d G=%d", K, N, G);
    DS_CHECK_ARG(blob && ((uintptr_t)blob & 255) == 0, "ds_w4_generate_linear: blob must be 256B aligned");
    DS_CHECK_ARG(layer >= 0 && tag >= 0 && tag < 64 && matrix >= 0 && matrix < 4,
                 "ds_w4_generate_linear: bad layer/tag/matrix");
    cudaStream_t st = as_stream(stream);
    char* base = static_cast<char*>(blob);
    const int grid = 4 * num_sms();
    const size_t words = (size_t)N * K / 8, groups = (size_t)N * (K / G);
    gen_codes_kernel<<<grid, 256, 0, st>>>(stream_key(seed, layer, tag, matrix, 0), words, (uint32_t*)(base + off[0]));
    gen_scales_kernel<<<grid, 256, 0, st>>>(stream_key(seed, layer, tag, matrix, 2), groups, K,
                                            (uint16_t*)(base + off[1]));
    gen_zeros_kernel<<<grid, 256, 0, st>>>(stream_key(seed, layer, tag, matrix, 1), (groups + 1) / 2,
                                           (uint8_t*)(base + off[2]));
    DS_LAUNCH_CHECK("ds_w4_generate_linear");
    return DS_OK;
}

__device__ const float g_one_f32 = 1.0f;

// Plain W4 linear for a few rows (decode attention projections): y = x W^T
// through the decode down-GEMV (K4) with routing weight 1 into a zeroed y.
extern "C" int ds_w4_linear_gemv(const void* x, int R, const ds_w4_linear* w, int K, int N, int G, float* y,
                                 void* stream) {
    DS_CHECK_ARG(w && check_linear(*w) && x && y, "ds_w4_linear_gemv: NULL pointer");
    DS_CHECK_ARG(R >= 1 && R <= 64, "ds_w4_linear_gemv: 1 <= R <= 64");
    cudaStream_t st = as_stream(stream);
    static const float* one = nullptr;
    if (!one) {
        void* p = nullptr;
        cudaError_t e = cudaGetSymbolAddress(&p, g_one_f32);
        if (e != cudaSuccess) return cuda_status(e, "ds_w4_linear_gemv: constant");
        one = static_cast<const float*>(p);
    }
    cudaError_t e = cudaMemsetAsync(y, 0, (size_t)R * N * sizeof(float), st);
    if (e != cudaSuccess) return cuda_status(e, "ds_w4_linear_gemv: zero y");
    ds_w4_expert ex{};
    ex.w2 = *w;
    return ds_w4_down_gemv(x, R, &ex, N, K, G, one, 0, y, stream);
}

extern "C" int ds_w4_dequant(const ds_w4_linear* w, int K, int N, int G, void* out, void* stream) {
    DS_CHECK_ARG(w && check_linear(*w) && out, "ds_w4_dequant: NULL pointer");
    DS_CHECK_ARG(K > 0 && N > 0 && G > 0 && K % G == 0 && G % 8 == 0, "ds_w4_dequant: bad shape");
    dequant_kernel<<<4 * num_sms(), 256, 0, as_stream(stream)>>>(
        w->codes, (const uint16_t*)w->scales, w->zeros, K, N, G, (__nv_bfloat16*)out);
    DS_LAUNCH_CHECK("ds_w4_dequant");
    return DS_OK;
}

static int check_gemv_shape(int R, int d, int ff, int G) {
    DS_CHECK_ARG(R >= 0 && R <= 64, "w4 gemv: R must be in [0, 64]");
    DS_CHECK_ARG(d > 0 && ff > 0 && d % 128 == 0 && ff % 128 == 0 && (G == 64 || G == 128),
                 "w4 gemv: need d, ff multiples of 128 and G in {64,128}");
    return DS_OK;
}

template <int R, int G, int U, bool GUARD>
static int swiglu_launch_u(const __nv_bfloat16* x, const ds_w4_expert* e, int d, int ff, __nv_bfloat16* h,
                           cudaStream_t st) {
    if (first_use_on_device((const void*)swiglu_gemv_kernel<R, G, U, GUARD>)) {
        cudaFuncSetAttribute(swiglu_gemv_kernel<R, G, U, GUARD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
    }
    const size_t smem = (size_t)R * d * 2 + (size_t)R * (d / 32) * 4;
    const int grid = gemv_grid((const void*)swiglu_gemv_kernel<R, G, U, GUARD>, smem, ff);
    swiglu_gemv_kernel<R, G, U, GUARD><<<grid, kGemvThreads, smem, st>>>(x, to_ptr(e->w1), to_ptr(e->w3), d, ff, h);
    DS_LAUNCH_CHECK("ds_w4_swiglu_gemv");
    return DS_OK;
}

template <int R, int G, int U, bool GUARD>
static int down_launch_u(const __nv_bfloat16* h, const ds_w4_expert* e, int d, int ff, const float* rw, int rs,
                         float* acc, cudaStream_t st) {
    if (first_use_on_device((const void*)down_gemv_kernel<R, G, U, GUARD>))
        cudaFuncSetAttribute(down_gemv_kernel<R, G, U, GUARD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
    const size_t smem = (size_t)R * ff * 2 + (size_t)R * (ff / 32) * 4;
    const int grid = gemv_grid((const void*)down_gemv_kernel<R, G, U, GUARD>, smem, d);
    cudaLaunchConfig_t cfg = {};   // PDL: launch overlaps the SwiGLU GEMV's tail
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemvThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, down_gemv_kernel<R, G, U, GUARD>, h, to_ptr(e->w2), ff, d, rw, rs, acc);
    DS_LAUNCH_CHECK("ds_w4_down_gemv");
    return DS_OK;
}

// v5 (bulk-staged) launchers; return 1 when the shape has no staged
// instantiation (the caller falls back to v2).  DS_K4_VARIANT=v2|mma forces
// the older variants (A/B runs).
// one ticket slot per launch, shared by every instantiation (a SwiGLU GEMV and
// the PDL down GEMV that overlaps it must not share a counter)
inline unsigned k4s_next_slot() {
    static std::atomic<unsigned> seq{0};
    return seq.fetch_add(1, std::memory_order_relaxed) % k4s::kTicketSlots;
}

// v5 SwiGLU GEMV with the tensor cores (G = 128, R = 1): the same producer /
// ring / ticket structure with 16-row blocks; the 16 consumer warps take a
// block together and split K: warp w owns quantisation groups
// [w*GPR/16, (w+1)*GPR/16) of all 16 rows.  Per group,
// lane (g, t) dequantises code chunk t of rows g and g+8 straight into
// mma.m16n8k16 A fragments (v3's mapping: 8 mmas per matrix per group, the k
// permutation inside an mma applied to x as well), x (unswizzled in shared
// memory) gives the B fragments, and the group scale is factored out with a
// precomputed per-group sum of x:  s * (D - (128 + z) * sum_group x).  With
// one activation row every D column holds the same dot product.  The 16
// partial sums per row are reduced through shared memory in a fixed order
// (deterministic); 2.3x fewer issue slots per weight than the FHFMA
// consumer, which is issue-bound on the SwiGLU half.
template <int CPL>
__global__ void __launch_bounds__(k4s::kThreads, 1) staged_mma_swiglu_kernel(
    const __nv_bfloat16* __restrict__ x, W4Ptr wa, W4Ptr wb, int N, int S, __nv_bfloat16* __restrict__ hout,
    unsigned slot_id, unsigned long long* dbg) {
    using namespace ds::sm100;
    constexpr int NMAT = 2, G = 128, RB = 16;
    using Gm = k4s::Geo<NMAT, CPL, G, RB>;
    constexpr int K = Gm::K, GPR = Gm::GPR;
    constexpr int WPG = k4s::kConsumers;                    // warps per block (K split): one group
    constexpr int NG = k4s::kConsumers / WPG;               // consumer groups
    constexpr int GPW = GPR / WPG;                          // quantisation groups per warp
    constexpr int XB = (K * 2 + GPR * 4 + 127) & ~127;
    static_assert(GPR % WPG == 0, "K split must be whole groups");
    extern __shared__ __align__(128) uint8_t smem[];
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(smem);
    float* xgs = reinterpret_cast<float*>(smem + K * 2);   // sum of x per quantisation group
    uint8_t* stages = smem + XB;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)S * Gm::STAGE_B);
    uint64_t* empty = full + S;
    int* hdr = reinterpret_cast<int*>(empty + S);
    float* red = reinterpret_cast<float*>(hdr + ((S + 3) & ~3));   // [2 parity][NG][WPG][NMAT][16]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const W4Ptr W[2] = {wa, wb};
    if (threadIdx.x == 0) {
        if (dbg) {
            unsigned long long ts;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
            atomicMax(dbg + blockIdx.x * 8, ts);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], WPG);
        }
        fence_mbar_init();
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the down GEMV may launch early
    if (warp == k4s::kConsumers) {
        if (lane == 0) k4s_produce<NMAT, CPL, G, RB>(W, N, S, NG, stages, full, empty, hdr, slot_id, dbg);
        return;
    }
    {   // x -> shared memory (plain layout), then the per-group sums (one warp per group)
        constexpr int NT = 32 * k4s::kConsumers;
        constexpr int UNITS = K / 8;
        constexpr int PER = (UNITS + NT - 1) / NT;
        const uint4* xu = reinterpret_cast<const uint4*>(x);
        uint4 v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (threadIdx.x + j * NT < UNITS) v[j] = __ldg(xu + threadIdx.x + j * NT);
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (threadIdx.x + j * NT < UNITS) reinterpret_cast<uint4*>(smem)[threadIdx.x + j * NT] = v[j];
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        for (int j = warp; j < GPR; j += k4s::kConsumers) {
            const uint32_t* p = reinterpret_cast<const uint32_t*>(xs + 128 * j) + 2 * lane;
            float s_ = (bf16_lo(p[0]) + bf16_hi(p[0])) + (bf16_lo(p[1]) + bf16_hi(p[1]));
            s_ = warp_sum(s_);
            if (lane == 0) xgs[j] = s_;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    }
    const int grp = warp / WPG, wk = warp % WPG;
    const int g = lane >> 2, t = lane & 3;
    for (int s = grp, it = 0;; s += NG, ++it) {
        const int slot = s % S;
        mbar_wait(&full[slot], (s / S) & 1);
        const int tb = hdr[slot];
        if (tb < 0) break;                                  // end of this group's stream
        const int r0 = tb * RB;
        const uint8_t* base = stages + (size_t)slot * Gm::STAGE_B;
        const uint32_t zb0 = ((uint32_t)(r0 * GPR) >> 1) & ~15u;
        float acc[NMAT][2] = {};
#pragma unroll
        for (int jj = 0; jj < GPW; ++jj) {
            const int j = wk * GPW + jj;
            uint4 xv[4];
            const uint4* xp = reinterpret_cast<const uint4*>(xs + 128 * j + 32 * t);
#pragma unroll
            for (int w = 0; w < 4; ++w) xv[w] = xp[w];
            uint4 c[NMAT][2];
#pragma unroll
            for (int m = 0; m < NMAT; ++m)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
                    c[m][hh] = *reinterpret_cast<const uint4*>(base + m * Gm::MAT_B + (g + 8 * hh) * Gm::CODE_B +
                                                               (4 * j + t) * 16);
            float d[NMAT][4] = {};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint32_t xw[4] = {xv[w].x, xv[w].y, xv[w].z, xv[w].w};
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
#pragma unroll
                    for (int m = 0; m < NMAT; ++m) {
                        const uint32_t* cg = reinterpret_cast<const uint32_t*>(&c[m][0]);
                        const uint32_t* cg8 = reinterpret_cast<const uint32_t*>(&c[m][1]);
                        mma16816(d[m], nib_pair_magic(cg[w] >> (8 * s2)), nib_pair_magic(cg8[w] >> (8 * s2)),
                                 nib_pair_magic(cg[w] >> (8 * s2 + 4)), nib_pair_magic(cg8[w] >> (8 * s2 + 4)),
                                 xw[2 * s2], xw[2 * s2 + 1]);
                    }
                }
            }
            const float xg = xgs[j];
#pragma unroll
            for (int m = 0; m < NMAT; ++m) {
                const uint8_t* mb = base + m * Gm::MAT_B;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int row = g + 8 * hh;
                    const uint16_t sv = reinterpret_cast<const uint16_t*>(mb + RB * Gm::CODE_B + row * Gm::SC_B)[j];
                    const uint32_t zn = (uint32_t)((r0 + row) * GPR + j);
                    const uint32_t zq = ((uint32_t)mb[RB * (Gm::CODE_B + Gm::SC_B) + (zn >> 1) - zb0] >> ((zn & 1) << 2)) & 15u;
                    const float z128 = __uint_as_float(0x43000000u | (zq << 16));
                    const float sc = __uint_as_float((uint32_t)sv << 16);
                    acc[m][hh] = fmaf(sc, fmaf(-z128, xg, d[m][2 * hh]), acc[m][hh]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);           // the block's bytes are consumed
        float* rd = red + (size_t)((it & 1) * NG + grp) * WPG * NMAT * 16;
        if (t == 0) {
#pragma unroll
            for (int m = 0; m < NMAT; ++m) {
                rd[(wk * NMAT + m) * 16 + g] = acc[m][0];
                rd[(wk * NMAT + m) * 16 + g + 8] = acc[m][1];
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(2 + grp), "n"(32 * WPG) : "memory");
        if (wk == 0 && lane < 16) {
            float av = 0.f, bv = 0.f;
#pragma unroll
            for (int w = 0; w < WPG; ++w) {
                av += rd[(w * NMAT + 0) * 16 + lane];
                bv += rd[(w * NMAT + 1) * 16 + lane];
            }
            const int n = r0 + lane;
            if (n < N) hout[n] = __float2bfloat16_rn(av / (1.0f + expf(-av)) * bv);
        }
    }
}

template <int CPL>
static int staged_mma_launch(const __nv_bfloat16* x, W4Ptr a, W4Ptr b, int N, __nv_bfloat16* hout, cudaStream_t st) {
    using Gm = k4s::Geo<2, CPL, 128, 16>;
    constexpr int XB = (Gm::K * 2 + Gm::GPR * 4 + 127) & ~127;
    constexpr int RED = 2 * 1 * 16 * 2 * 16 * 4;            // [parity][NG = 1][WPG = 16][NMAT][16 rows]
    static int S = -1;
    static size_t smem = 0;
    if (S < 0) {
        int s_ = (k4s::kSmemBudget - XB - RED - 16) / (Gm::STAGE_B + 20);
        if (s_ > 8) s_ = 8;
        smem = (size_t)XB + (size_t)s_ * Gm::STAGE_B + 16 * (size_t)s_ + 4 * (size_t)((s_ + 3) & ~3) + RED;
        S = s_;
    }
    if (S >= 2 && first_use_on_device((const void*)staged_mma_swiglu_kernel<CPL>))
        cudaFuncSetAttribute(staged_mma_swiglu_kernel<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (S < 2) return 1;
    const int grid = N / 16 < num_sms() ? N / 16 : num_sms();
    static const bool want_dbg = getenv("DS_K4_TIMELINE") != nullptr;
    static unsigned long long* dbg = nullptr;
    if (want_dbg && !dbg) cudaMalloc(&dbg, 8 * 1024 * sizeof(unsigned long long));
    if (want_dbg) cudaMemsetAsync(dbg, 0, 8 * 1024 * sizeof(unsigned long long), st);
    staged_mma_swiglu_kernel<CPL><<<grid, k4s::kThreads, smem, st>>>(x, a, b, N, S, hout, k4s_next_slot(),
                                                                     want_dbg ? dbg : nullptr);
    DS_LAUNCH_CHECK("ds_w4_swiglu_gemv (staged mma)");
    if (want_dbg) {
        static unsigned long long h[8 * 1024];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, dbg, 8 * grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, t1 = 0, t3 = 0;
        for (int bi = 0; bi < grid; ++bi) {
            t0 = h[8 * bi] < t0 ? h[8 * bi] : t0;
            t3 = h[8 * bi + 3] > t3 ? h[8 * bi + 3] : t3;
            t1 = h[8 * bi + 1] > t1 ? h[8 * bi + 1] : t1;
        }
        fprintf(stderr, "K4 staged mma swiglu: last first-issue %.2f us, last producer done %.2f us\n",
                (t1 - t0) / 1e3, (t3 - t0) / 1e3);
    }
    return DS_OK;
}

// ------------------------------------------ K4 v6: one persistent launch per expert
// (R = 1, G = 128).  The SwiGLU GEMV (phase A: 16-row tiles of W1 and W3,
// the tensor-core consumer of staged_mma_swiglu_kernel) and the down GEMV
// (phase B: 8-row tiles of W2, 16 consumer warps as 8 rows x 2 K-halves, the
// FHFMA dot product with h read through L1) run in ONE cooperative launch
// with a grid barrier between them.  Tickets run over phase-A then phase-B
// tiles, so each producer streams W2 tiles into its ring as soon as phase A
// is handed out — the down projection's bytes land while the SwiGLU phase
// drains, and the second launch's ramp / first-byte latency disappears.
// The consumers cross the barrier (all h written) on their first phase-B
// stage, compute the per-32 sums of h once, and consume the staged W2 tiles.
namespace k4f {
constexpr int kConsumers = 16;
constexpr int kThreads = 32 * (kConsumers + 1);
constexpr int kSmemCap = 227 * 1024;

template <int KA, int KB, int RBA_, int RBB_>
struct Geo {
    static constexpr int RBA = RBA_, RBB = RBB_;            // phase-A / phase-B tile rows
    static constexpr int PARTS = kConsumers / RBB;          // phase B: K parts per row (one warp each)
    static constexpr int GPRA = KA / 128, CODEA = KA / 2, SCA = GPRA * 2;
    static constexpr int ZA = (RBA * GPRA / 2 + 32 + 15) & ~15;
    static constexpr int MATA = RBA * CODEA + RBA * SCA + ZA;
    static constexpr int STAGEA = 2 * MATA;
    static constexpr int GPRB = KB / 128, CODEB = KB / 2, SCB = GPRB * 2;
    static constexpr int ZB = (RBB * GPRB / 2 + 32 + 15) & ~15;
    static constexpr int STAGEB = RBB * CODEB + RBB * SCB + ZB;
    static constexpr int SLOT = ((STAGEA > STAGEB ? STAGEA : STAGEB) + 127) & ~127;
    static constexpr int NCHB = KB / 32;                       // 32-code chunks of a W2 row
    static constexpr int CPLB = NCHB / PARTS / 32;             // chunks per lane per K part
    static constexpr int XA = KA * 2 + GPRA * 4;               // phase A: x + per-group sums
    static constexpr int XREG = ((XA > NCHB * 4 ? XA : NCHB * 4) + 127) & ~127;   // phase B: per-32 sums of h
    // phase B keeps h (KB bf16 = 64 B per 32-chunk) in shared memory: the x
    // region after the per-chunk sums, then the tail of every ring slot (a
    // phase-B stage is smaller than a phase-A stage)
    static constexpr int HX_OFF = (NCHB * 4 + 127) & ~127;
    static constexpr int HX_CH = (XREG - HX_OFF) / 64;                  // chunks in the x region
    static constexpr int HT_OFF = (STAGEB + 127) & ~127;
    static constexpr int HT_CH = (SLOT - HT_OFF) / 64;                  // chunks per slot tail
    static constexpr int RED = 2 * kConsumers * 2 * 16 * 4 + 2 * kConsumers * 4;
    static constexpr int FIXED = XREG + RED + 64;
    static constexpr int stages() {
        int n = (kSmemCap - FIXED) / (SLOT + 24);
        return n > 6 ? 6 : n;
    }
    static constexpr size_t smem(int S) { return (size_t)FIXED + (size_t)S * (SLOT + 24); }
    static constexpr bool h_fits(int S) { return HX_CH + S * HT_CH >= NCHB; }
};
}  // namespace k4f

__device__ unsigned g_k4f_bar[k4s::kTicketSlots];
// diagnostics (DS_K4_V6_TIMELINE=1): per-CTA %globaltimer stamps of the last
// launch — entry, phase A consumed, grid barrier passed, h staged, exit
__device__ unsigned long long g_k4f_dbg[1024 * 8];
__device__ unsigned g_k4f_exit[k4s::kTicketSlots];
// always-on device-clock span of every v6 launch: first CTA entry -> last CTA
// exit on %globaltimer (entries kept as ~t so a zero-initialised atomicMax
// finds the earliest), accumulated over launches.  CUDA-event spans on the
// launching stream also contain the front end's event-timestamp cost, which
// grows from ~7 to ~29 us while the copy engine streams host memory
// (scripts/launchprobe.cu); this is the kernel's own duration beside them.
__device__ unsigned long long g_k4f_first[k4s::kTicketSlots];
__device__ unsigned long long g_k4f_span_ns, g_k4f_span_n;

template <int KA, int KB, int RBA, int RBB>
__global__ void __launch_bounds__(k4f::kThreads, 1) expert_fused_v6_kernel(
    const __nv_bfloat16* __restrict__ x, W4Ptr w1, W4Ptr w3, W4Ptr w2, int S, __nv_bfloat16* __restrict__ hout,
    const float* __restrict__ route_w, float* __restrict__ out, unsigned slot_id, int dbg) {
    using namespace ds::sm100;
    using Gm = k4f::Geo<KA, KB, RBA, RBB>;
    auto stamp = [&](int i) {
        if (dbg && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            g_k4f_dbg[blockIdx.x * 8 + i] = t;
        }
    };
    stamp(0);
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(g_k4f_first + slot_id, ~t);
    }
    constexpr int GPRA = Gm::GPRA, GPRB = Gm::GPRB;
    constexpr int TA = KB / Gm::RBA;                 // phase-A tiles: rows of W1 / W3 (N = ff = KB)
    constexpr int TB = KA / Gm::RBB;                 // phase-B tiles: rows of W2 (N = d = KA)
    constexpr int T = TA + TB;
    constexpr int GPW = GPRA / k4f::kConsumers;       // phase A: quantisation groups per warp
    static_assert(GPRA % k4f::kConsumers == 0, "phase A K split must be whole groups");
    static_assert((Gm::NCHB / Gm::PARTS) % 32 == 0, "phase B K parts must be whole lane chunks");
    static_assert(RBA == 16 || RBA == 8, "phase A tiles: 16 rows, or 8 (half-used m16 MMA) for wide K");
    extern __shared__ __align__(128) uint8_t smem[];
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(smem);
    float* xgs = reinterpret_cast<float*>(smem + KA * 2);          // phase A: sum of x per group
    float* hsum = reinterpret_cast<float*>(smem);                  // phase B: sum of h per 32-chunk (aliases x)
    float* red = reinterpret_cast<float*>(smem + Gm::XREG);        // [2][16 warps][2 mats][16 rows]
    float* redb = red + 2 * k4f::kConsumers * 2 * 16;              // [2][RBB rows][PARTS]
    uint8_t* stages = smem + Gm::FIXED;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)S * Gm::SLOT);
    uint64_t* empty = full + S;
    int* hdr = reinterpret_cast<int*>(empty + S);
    auto h_chunk = [&](int c) -> uint4* {       // 64-byte chunk c of h in shared memory (phase B)
        if (c < Gm::HX_CH) return reinterpret_cast<uint4*>(smem + Gm::HX_OFF + 64 * c);
        c -= Gm::HX_CH;
        const int sl = c / Gm::HT_CH;
        return reinterpret_cast<uint4*>(stages + (size_t)sl * Gm::SLOT + Gm::HT_OFF + 64 * (c - sl * Gm::HT_CH));
    };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], k4f::kConsumers);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == k4f::kConsumers) {                                 // producer
        if (lane != 0) return;
        unsigned* tk = g_k4s_ticket + slot_id;
        const uint64_t pol = l2_evict_first_policy();
        const int first = (int)atomicAdd(tk, (unsigned)S);
        int pending = -1;
        for (int s = 0;; ++s) {
            const int slot = s % S;
            if (s >= S) mbar_wait(&empty[slot], ((s / S) - 1) & 1);
            int t = s < S ? first + s : pending;
            if (s >= S - 1 && t < T) {
                pending = (int)atomicAdd(tk, 1u);
                if (pending >= TA && pending < T) {
                    // the next W2 tile is ours: pull it into L2 now, so its bulk copy (issued once a
                    // slot frees, typically after the phase barrier) hits L2
                    const int rp = (pending - TA) * Gm::RBB;
                    bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(w2.codes) + (size_t)rp * Gm::CODEB,
                                     Gm::RBB * Gm::CODEB);
                    bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(w2.scales) + (size_t)rp * Gm::SCB,
                                     Gm::RBB * Gm::SCB);
                }
            }
            if (t >= T || t < 0) {
                hdr[slot] = -1;
                mbar_arrive(&full[slot]);
                break;
            }
            hdr[slot] = t;
            uint8_t* dst = stages + (size_t)slot * Gm::SLOT;
            if (t < TA) {
                const int r0 = t * Gm::RBA;
                const uint32_t zb0 = ((uint32_t)(r0 * GPRA) >> 1) & ~15u;
                const uint32_t zb1 = (((uint32_t)((r0 + Gm::RBA) * GPRA) >> 1) + 15u) & ~15u;
                const uint32_t cb = Gm::RBA * Gm::CODEA, sb = Gm::RBA * Gm::SCA, zb = zb1 - zb0;
                mbar_expect_tx(&full[slot], 2 * (cb + sb + zb));
                const W4Ptr W[2] = {w1, w3};
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    uint8_t* md = dst + m * Gm::MATA;
                    bulk_load(md, reinterpret_cast<const uint8_t*>(W[m].codes) + (size_t)r0 * Gm::CODEA, cb,
                              &full[slot], pol);
                    bulk_load(md + cb, reinterpret_cast<const uint8_t*>(W[m].scales) + (size_t)r0 * Gm::SCA, sb,
                              &full[slot], pol);
                    bulk_load(md + cb + sb, W[m].zeros + zb0, zb, &full[slot], pol);
                }
            } else {
                const int r0 = (t - TA) * Gm::RBB;
                const uint32_t zb0 = ((uint32_t)(r0 * GPRB) >> 1) & ~15u;
                const uint32_t zb1 = (((uint32_t)((r0 + Gm::RBB) * GPRB) >> 1) + 15u) & ~15u;
                const uint32_t cb = Gm::RBB * Gm::CODEB, sb = Gm::RBB * Gm::SCB, zb = zb1 - zb0;
                mbar_expect_tx(&full[slot], cb + sb + zb);
                bulk_load(dst, reinterpret_cast<const uint8_t*>(w2.codes) + (size_t)r0 * Gm::CODEB, cb, &full[slot],
                          pol);
                bulk_load(dst + cb, reinterpret_cast<const uint8_t*>(w2.scales) + (size_t)r0 * Gm::SCB, sb,
                          &full[slot], pol);
                bulk_load(dst + cb + sb, w2.zeros + zb0, zb, &full[slot], pol);
            }
        }
        __threadfence();
        if (atomicAdd(g_k4s_done + slot_id, 1u) == gridDim.x - 1) {   // every ticket of the launch is taken
            atomicExch(tk, 0u);
            atomicExch(g_k4s_done + slot_id, 0u);
        }
        return;
    }

    {   // phase A input: x -> shared memory (plain layout) and per-group sums
        constexpr int NT = 32 * k4f::kConsumers;
        constexpr int UNITS = KA / 8;
        constexpr int PER = (UNITS + NT - 1) / NT;
        const uint4* xu = reinterpret_cast<const uint4*>(x);
        uint4 v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (threadIdx.x + j * NT < UNITS) v[j] = __ldg(xu + threadIdx.x + j * NT);
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (threadIdx.x + j * NT < UNITS) reinterpret_cast<uint4*>(smem)[threadIdx.x + j * NT] = v[j];
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        for (int j = warp; j < GPRA; j += k4f::kConsumers) {
            const uint32_t* p = reinterpret_cast<const uint32_t*>(xs + 128 * j) + 2 * lane;
            float s_ = (bf16_lo(p[0]) + bf16_hi(p[0])) + (bf16_lo(p[1]) + bf16_hi(p[1]));
            s_ = warp_sum(s_);
            if (lane == 0) xgs[j] = s_;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    }
    const int g = lane >> 2, tq = lane & 3;
    bool crossed = false;
    int ita = 0, itb = 0;
    for (int s = 0;; ++s) {
        const int slot = s % S;
        mbar_wait(&full[slot], (s / S) & 1);
        const int t = hdr[slot];
        const uint8_t* base = stages + (size_t)slot * Gm::SLOT;
        if (t >= 0 && t < TA) {                                    // ---- phase A: SwiGLU tile
            const int r0 = t * Gm::RBA;
            const uint32_t zb0 = ((uint32_t)(r0 * GPRA) >> 1) & ~15u;
            float acc[2][2] = {};
#pragma unroll
            for (int jj = 0; jj < GPW; ++jj) {
                const int j = warp * GPW + jj;
                uint4 xv[4];
                const uint4* xp = reinterpret_cast<const uint4*>(xs + 128 * j + 32 * tq);
#pragma unroll
                for (int w = 0; w < 4; ++w) xv[w] = xp[w];
                uint4 c[2][2];
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
                        c[m][hh] = (hh == 0 || RBA == 16)
                                       ? *reinterpret_cast<const uint4*>(base + m * Gm::MATA + (g + 8 * hh) * Gm::CODEA +
                                                                          (4 * j + tq) * 16)
                                       : make_uint4(0u, 0u, 0u, 0u);       // 8-row tile: MMA rows 8-15 unused
                float dd[2][4] = {};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const uint32_t xw[4] = {xv[w].x, xv[w].y, xv[w].z, xv[w].w};
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
#pragma unroll
                        for (int m = 0; m < 2; ++m) {
                            const uint32_t* cg = reinterpret_cast<const uint32_t*>(&c[m][0]);
                            const uint32_t* cg8 = reinterpret_cast<const uint32_t*>(&c[m][1]);
                            mma16816(dd[m], nib_pair_magic(cg[w] >> (8 * s2)), nib_pair_magic(cg8[w] >> (8 * s2)),
                                     nib_pair_magic(cg[w] >> (8 * s2 + 4)), nib_pair_magic(cg8[w] >> (8 * s2 + 4)),
                                     xw[2 * s2], xw[2 * s2 + 1]);
                        }
                    }
                }
                const float xg = xgs[j];
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const uint8_t* mb = base + m * Gm::MATA;
#pragma unroll
                    for (int hh = 0; hh < (RBA == 16 ? 2 : 1); ++hh) {
                        const int row = g + 8 * hh;
                        const uint16_t sv = reinterpret_cast<const uint16_t*>(mb + Gm::RBA * Gm::CODEA +
                                                                              row * Gm::SCA)[j];
                        const uint32_t zn = (uint32_t)((r0 + row) * GPRA + j);
                        const uint32_t zq = ((uint32_t)mb[Gm::RBA * (Gm::CODEA + Gm::SCA) + (zn >> 1) - zb0] >>
                                             ((zn & 1) << 2)) & 15u;
                        const float z128 = __uint_as_float(0x43000000u | (zq << 16));
                        const float sc = __uint_as_float((uint32_t)sv << 16);
                        acc[m][hh] = fmaf(sc, fmaf(-z128, xg, dd[m][2 * hh]), acc[m][hh]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            float* rd = red + (size_t)(ita & 1) * k4f::kConsumers * 2 * 16;
            if (tq == 0) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    rd[(warp * 2 + m) * 16 + g] = acc[m][0];
                    rd[(warp * 2 + m) * 16 + g + 8] = acc[m][1];
                }
            }
            asm volatile("bar.sync 2, %0;" ::"n"(32 * k4f::kConsumers) : "memory");
            if (warp == 0 && lane < RBA) {
                float av = 0.f, bv = 0.f;
#pragma unroll
                for (int w = 0; w < k4f::kConsumers; ++w) {
                    av += rd[(w * 2 + 0) * 16 + lane];
                    bv += rd[(w * 2 + 1) * 16 + lane];
                }
                hout[r0 + lane] = __float2bfloat16_rn(av / (1.0f + expf(-av)) * bv);
            }
            ++ita;
            continue;
        }
        if (!crossed) {                                            // ---- phase boundary (grid barrier)
            asm volatile("bar.sync 3, %0;" ::"n"(32 * k4f::kConsumers) : "memory");   // this CTA's h is written
            stamp(1);
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(g_k4f_bar + slot_id, 1u);
            }
            crossed = true;
            if (t < 0) break;
            if (threadIdx.x == 0) {
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(g_k4f_bar + slot_id));
                } while (v < gridDim.x);
            }
            stamp(2);
            asm volatile("bar.sync 3, %0;" ::"n"(32 * k4f::kConsumers) : "memory");
            for (int i = threadIdx.x; i < Gm::NCHB; i += 32 * k4f::kConsumers) {   // h -> smem, per-32 sums
                const uint4* hp = reinterpret_cast<const uint4*>(hout) + 4 * i;
                uint4 v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = __ldcg(hp + q);
                uint4* dst = h_chunk(i);
                float s_ = 0.f;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    dst[q ^ ((i >> 1) & 3)] = v[q];     // 8 consecutive chunks hit 8 distinct 16-B bank groups
                    const uint32_t vv[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) s_ += bf16_lo(vv[u]) + bf16_hi(vv[u]);
                }
                hsum[i] = s_;
            }
            asm volatile("bar.sync 3, %0;" ::"n"(32 * k4f::kConsumers) : "memory");
            stamp(3);
        }
        if (t < 0) break;
        {                                                          // ---- phase B: down tile
            const int r0 = (t - TA) * Gm::RBB;
            const int r = warp % Gm::RBB, hf = warp / Gm::RBB;      // row of the tile, K part
            const int n = r0 + r;
            const uint32_t zb0 = ((uint32_t)(r0 * GPRB) >> 1) & ~15u;
            const float o_prev = (hf == 0 && lane == 0) ? out[n] : 0.f;   // in flight during the dot product
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < Gm::CPLB; ++i) {
                const int c = hf * (Gm::NCHB / Gm::PARTS) + lane + 32 * i;
                const int gq = c >> 2;
                const uint4* hp = h_chunk(c);
                uint4 xv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) xv[q] = hp[q ^ ((c >> 1) & 3)];
                const float xsm = hsum[c];
                const uint4 c4 = *reinterpret_cast<const uint4*>(base + r * Gm::CODEB + c * 16);
                const uint16_t sv = reinterpret_cast<const uint16_t*>(base + Gm::RBB * Gm::CODEB + r * Gm::SCB)[gq];
                const uint32_t zn = (uint32_t)(n * GPRB + gq);
                const uint8_t zv = base[Gm::RBB * (Gm::CODEB + Gm::SCB) + (zn >> 1) - zb0];
                const uint32_t cw[4] = {c4.x, c4.y, c4.z, c4.w};
                float pp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const uint32_t xx[4] = {xv[ii].x, xv[ii].y, xv[ii].z, xv[ii].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t pr = nib_pair_magic(cw[ii] >> (4 * q));
                        fma_bf16_lo(pp[(q & 1) * 2], pr, xx[q]);
                        fma_bf16_hi(pp[(q & 1) * 2 + 1], pr, xx[q]);
                    }
                }
                const float z128 = __uint_as_float(0x43000000u | ((((uint32_t)zv >> ((zn & 1) << 2)) & 15u) << 16));
                const float sc = __uint_as_float((uint32_t)sv << 16);
                acc = fmaf(sc, ((pp[0] + pp[1]) + (pp[2] + pp[3])) - z128 * xsm, acc);
            }
            acc = warp_sum(acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            float* rb = redb + (itb & 1) * k4f::kConsumers;
            if (lane == 0) rb[r * Gm::PARTS + hf] = acc;
            asm volatile("bar.sync 4, %0;" ::"n"(32 * k4f::kConsumers) : "memory");
            if (hf == 0 && lane == 0) {
                float y = rb[r * Gm::PARTS];
#pragma unroll
                for (int q = 1; q < Gm::PARTS; ++q) y += rb[r * Gm::PARTS + q];   // fixed order
                out[n] = __fadd_rn(o_prev, __fmul_rn(route_w[0], y));
            }
            ++itb;
        }
    }
    // last CTA out resets the grid-barrier counter of this ticket slot
    asm volatile("bar.sync 3, %0;" ::"n"(32 * k4f::kConsumers) : "memory");
    stamp(4);
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(g_k4f_exit + slot_id, 1u) == gridDim.x - 1) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            const unsigned long long first = ~atomicExch(g_k4f_first + slot_id, 0ull);
            atomicAdd(&g_k4f_span_ns, t - first);
            atomicAdd(&g_k4f_span_n, 1ull);
            atomicExch(g_k4f_bar + slot_id, 0u);
            atomicExch(g_k4f_exit + slot_id, 0u);
        }
    }
}

template <int KA, int KB, int RBA, int RBB>
static int expert_v6_launch(const __nv_bfloat16* x, const ds_w4_expert* e, __nv_bfloat16* h, const float* rw,
                            float* acc, cudaStream_t st) {
    using Gm = k4f::Geo<KA, KB, RBA, RBB>;
    constexpr int S = Gm::stages();
    if constexpr (S < 2 || !Gm::h_fits(S)) {
        return 1;
    } else {
        const size_t smem = Gm::smem(S);
        if (first_use_on_device((const void*)expert_fused_v6_kernel<KA, KB, RBA, RBB>))
            cudaFuncSetAttribute(expert_fused_v6_kernel<KA, KB, RBA, RBB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(num_sms());
        cfg.blockDim = dim3(k4f::kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;     // the grid barrier needs every CTA resident
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        static const bool coop = !(getenv("DS_K4_V6_COOP") && getenv("DS_K4_V6_COOP")[0] == '0');   // A/B runs
        cfg.numAttrs = coop ? 1 : 0;
        const unsigned slot_id = k4s_next_slot();
        static const int dbg = getenv("DS_K4_V6_TIMELINE") ? 1 : 0;
        cudaError_t er = cudaLaunchKernelEx(&cfg, expert_fused_v6_kernel<KA, KB, RBA, RBB>, x, to_ptr(e->w1), to_ptr(e->w3),
                                            to_ptr(e->w2), S, h, rw, acc, slot_id, dbg);
        return er == cudaSuccess ? DS_OK : cuda_status(er, "ds_w4_expert_gemv (v6 fused)");
    }
}

// v6 for the shapes it is instantiated for; 1 = not applicable (caller uses v5)
static int expert_v6(const void* x, int R, const ds_w4_expert* e, int d, int ff, int G, void* h, const float* rw,
                     float* acc, cudaStream_t st) {
    static const bool on = !(getenv("DS_K4_V6") && getenv("DS_K4_V6")[0] == '0');
    if (!on || R != 1 || G != 128 || !e || !x || !h || !rw || !acc) return 1;
    if (!check_linear(e->w1) || !check_linear(e->w3) || !check_linear(e->w2)) return 1;
    const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
    __nv_bfloat16* hb = static_cast<__nv_bfloat16*>(h);
    if (d == 4096 && ff == 14336) return expert_v6_launch<4096, 14336, 16, 8>(xb, e, hb, rw, acc, st);   // 8x7B
    // 8x22B (d = 6144): a 16-row W1/W3 tile leaves two ring slots, and the 8-row
    // variant <6144, 16384, 8, 4> measured 55.7 us against 48.2 us for the v5
    // PDL pair (profiles/r2/k4_v6_22b.json) -> v5 stays there
    if (d == 6144 && ff == 16384 && getenv("DS_K4_V6_22B")) {
        if (getenv("DS_K4_V6_22B")[0] == '8') return expert_v6_launch<6144, 16384, 8, 4>(xb, e, hb, rw, acc, st);
        return expert_v6_launch<6144, 16384, 16, 8>(xb, e, hb, rw, acc, st);     // two ring slots
    }
    return 1;
}

inline bool k4_staged_enabled() {
    static const char* v = getenv("DS_K4_VARIANT");
    return !(v && (v[0] == 'v' || v[0] == 'm'));
}

template <int NMAT, int CPL, int G, int RB, bool SWIGLU>
static int staged_launch(const __nv_bfloat16* x, W4Ptr a, W4Ptr b, int N, __nv_bfloat16* hout, const float* rw,
                         float* out, cudaStream_t st) {
    using Gm = k4s::Geo<NMAT, CPL, G, RB>;
    static int S = -1;
    static size_t smem = 0;
    if (S < 0) {
        int s_ = (k4s::kSmemBudget - Gm::X_B) / (Gm::STAGE_B + 20);
        if (s_ > 8) s_ = 8;
        // ring depth a multiple of the consumer-group count: slot j then always
        // serves the same group, so a group never waits on a slot whose previous
        // phase (another group's stage, possibly still landing) is incomplete —
        // with mbarrier parity waits that phase would alias the awaited one
        s_ -= s_ % (k4s::kConsumers / RB);
        smem = (size_t)Gm::X_B + (size_t)s_ * Gm::STAGE_B + 20 * (size_t)s_;
        S = s_;
    }
    if (S >= 2 && first_use_on_device((const void*)staged_gemv_kernel<NMAT, CPL, G, RB, SWIGLU>))
        cudaFuncSetAttribute(staged_gemv_kernel<NMAT, CPL, G, RB, SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (S < 2 || S < k4s::kConsumers / RB) return 1;   // every consumer group needs its own slot
    static const int gcap = getenv("DS_K4S_GRID") ? atoi(getenv("DS_K4S_GRID")) : 0;   // A/B runs
    int grid = N < num_sms() ? N : num_sms();
    if (gcap > 0 && gcap < grid) grid = gcap;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(k4s::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];   // down: PDL launch, its first stages stream during the SwiGLU tail
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = SWIGLU ? 0 : 1;
    static const bool want_dbg = getenv("DS_K4_TIMELINE") != nullptr;
    static unsigned long long* dbg = nullptr;
    if (want_dbg && !dbg) cudaMalloc(&dbg, 8 * 1024 * sizeof(unsigned long long));
    if (want_dbg) cudaMemsetAsync(dbg, 0, 8 * 1024 * sizeof(unsigned long long), st);
    const unsigned slot_id = k4s_next_slot();
    cudaLaunchKernelEx(&cfg, staged_gemv_kernel<NMAT, CPL, G, RB, SWIGLU>, x, a, b, N, S, hout, rw, out, slot_id,
                       want_dbg ? dbg : nullptr);
    DS_LAUNCH_CHECK(SWIGLU ? "ds_w4_swiglu_gemv (staged)" : "ds_w4_down_gemv (staged)");
    if (want_dbg) {      // diagnostics only: per-CTA stamps (us from the earliest CTA entry)
        static unsigned long long h[8 * 1024];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, dbg, 8 * grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < grid; ++b) t0 = h[8 * b] < t0 ? h[8 * b] : t0;
        const char* names[6] = {"entry", "issued", "x_staged", "producer_done", "first_stage", "consumer_done"};
        fprintf(stderr, "K4 staged %s timeline (us, min/median/max over %d CTAs):", SWIGLU ? "swiglu" : "down", grid);
        for (int i = 0; i < 6; ++i) {
            double v[1024];
            int n = 0;
            for (int b = 0; b < grid; ++b)
                if (h[8 * b + i]) v[n++] = (h[8 * b + i] - t0) / 1e3;
            std::sort(v, v + n);
            if (n) fprintf(stderr, " %s %.2f/%.2f/%.2f", names[i], v[0], v[n / 2], v[n - 1]);
        }
        fprintf(stderr, " late:");
        for (int b = 0; b < grid; ++b)
            if (h[8 * b] - t0 > 2000) fprintf(stderr, " %d(%.1f)", b, (h[8 * b] - t0) / 1e3);
        fprintf(stderr, "\n");
    }
    return DS_OK;
}

template <int G>
static bool staged_shape_ok(int K, int N) {
    const int gpr = K / G;   // scale rows 16-B aligned, zero-nibble array a multiple of 16 B
    return K % 1024 == 0 && gpr % 8 == 0 && ((long long)N * gpr) % 32 == 0 && N > 0;
}

template <int G>
static int swiglu_staged(const __nv_bfloat16* x, const ds_w4_expert* e, int d, int ff, __nv_bfloat16* h,
                         cudaStream_t st) {
    if (!k4_staged_enabled() || !staged_shape_ok<G>(d, ff)) return 1;
    static const bool mma = !(getenv("DS_K4S_MMA") && getenv("DS_K4S_MMA")[0] == '0');   // A/B runs
    if constexpr (G == 128) {
        if (mma && ff % 16 == 0) {
            if (d / 1024 == 4) return staged_mma_launch<4>(x, to_ptr(e->w1), to_ptr(e->w3), ff, h, st);
            if (d / 1024 == 6) return staged_mma_launch<6>(x, to_ptr(e->w1), to_ptr(e->w3), ff, h, st);
        }
    }
    static const int rb = getenv("DS_K4S_RB_UP") ? atoi(getenv("DS_K4S_RB_UP")) : 8;   // A/B runs
#define DS_SW(CPL, RB) staged_launch<2, CPL, G, RB, true>(x, to_ptr(e->w1), to_ptr(e->w3), ff, h, nullptr, nullptr, st)
    switch (d / 1024) {
        case 4: return rb == 4 ? DS_SW(4, 4) : rb == 16 ? DS_SW(4, 16) : DS_SW(4, 8);
        case 6: return rb == 4 ? DS_SW(6, 4) : rb == 16 ? DS_SW(6, 16) : DS_SW(6, 8);
        default: return 1;
    }
#undef DS_SW
}

template <int G>
static int down_staged(const __nv_bfloat16* h, const ds_w4_expert* e, int d, int ff, const float* rw, float* acc,
                       cudaStream_t st) {
    if (!k4_staged_enabled() || !staged_shape_ok<G>(ff, d)) return 1;
    static const int rb = getenv("DS_K4S_RB_DOWN") ? atoi(getenv("DS_K4S_RB_DOWN")) : 4;   // A/B runs
    if (rb == 0) return 1;                                                                   // v2 down
#define DS_DN(CPL, RB) staged_launch<1, CPL, G, RB, false>(h, to_ptr(e->w2), to_ptr(e->w2), d, nullptr, rw, acc, st)
    switch (ff / 1024) {
        case 4: return DS_DN(4, 4);          // W4 attention projections (8x7B: K = 4096)
        case 6: return DS_DN(6, 4);          // (8x22B: K = 6144)
        case 14: return rb == 2 ? DS_DN(14, 2) : rb == 8 ? DS_DN(14, 8) : DS_DN(14, 4);
        case 16: return rb == 2 ? DS_DN(16, 2) : rb == 8 ? DS_DN(16, 8) : DS_DN(16, 4);
        default: return 1;
    }
#undef DS_DN
}

// batch size per lane U (16-byte loads in flight per matrix) chosen so that
// (K/32)/32 is a multiple of U: no predicates in the streaming loop
template <int R, int G>
static int swiglu_launch_g(const __nv_bfloat16* x, const ds_w4_expert* e, int d, int ff, __nv_bfloat16* h,
                           cudaStream_t st) {
    if constexpr (R == 1) {
        const int rc = swiglu_staged<G>(x, e, d, ff, h, st);
        if (rc <= 0) return rc;
    }
    const int per_lane = (d / 32) % 32 == 0 ? (d / 32) / 32 : 0;
    if (per_lane && per_lane % 4 == 0) return swiglu_launch_u<R, G, 4, false>(x, e, d, ff, h, st);
    if (per_lane && per_lane % 3 == 0) return swiglu_launch_u<R, G, 3, false>(x, e, d, ff, h, st);
    if (per_lane && per_lane % 2 == 0) return swiglu_launch_u<R, G, 2, false>(x, e, d, ff, h, st);
    return swiglu_launch_u<R, G, 2, true>(x, e, d, ff, h, st);
}

template <int R, int G>
static int down_launch_g(const __nv_bfloat16* h, const ds_w4_expert* e, int d, int ff, const float* rw, int rs,
                         float* acc, cudaStream_t st) {
    if constexpr (R == 1) {
        const int rc = down_staged<G>(h, e, d, ff, rw, acc, st);
        if (rc <= 0) return rc;
    }
    const int per_lane = (ff / 32) % 32 == 0 ? (ff / 32) / 32 : 0;
    if (per_lane && per_lane % 8 == 0) return down_launch_u<R, G, 8, false>(h, e, d, ff, rw, rs, acc, st);
    if (per_lane && per_lane % 7 == 0) return down_launch_u<R, G, 7, false>(h, e, d, ff, rw, rs, acc, st);
    if (per_lane && per_lane % 6 == 0) return down_launch_u<R, G, 6, false>(h, e, d, ff, rw, rs, acc, st);
    if (per_lane && per_lane % 4 == 0) return down_launch_u<R, G, 4, false>(h, e, d, ff, rw, rs, acc, st);
    return down_launch_u<R, G, 4, true>(h, e, d, ff, rw, rs, acc, st);
}

template <int R>
static int swiglu_launch(const __nv_bfloat16* x, const ds_w4_expert* e, int d, int ff, int G, __nv_bfloat16* h,
                         cudaStream_t st) {
    return G == 128 ? swiglu_launch_g<R, 128>(x, e, d, ff, h, st) : swiglu_launch_g<R, 64>(x, e, d, ff, h, st);
}

template <int R>
static int down_launch(const __nv_bfloat16* h, const ds_w4_expert* e, int d, int ff, int G, const float* rw,
                       int rs, float* acc, cudaStream_t st) {
    return G == 128 ? down_launch_g<R, 128>(h, e, d, ff, rw, rs, acc, st)
                    : down_launch_g<R, 64>(h, e, d, ff, rw, rs, acc, st);
}

extern "C" int ds_w4_swiglu_gemv(const void* x, int R, const ds_w4_expert* e, int d, int ff, int G, void* h,
                                 void* stream) {
    int rc = check_gemv_shape(R, d, ff, G);
    if (rc) return rc;
    DS_CHECK_ARG(e && check_linear(e->w1) && check_linear(e->w3) && x && h, "ds_w4_swiglu_gemv: NULL pointer");
    cudaStream_t st = as_stream(stream);
    const __nv_bfloat16* xb = (const __nv_bfloat16*)x;
    __nv_bfloat16* hb = (__nv_bfloat16*)h;
    if (G == 128 && k4_use_mma(R)) {
        constexpr int P = 6;
        const int NG = d / 128, S = mma_gemv_warps(NG, 2), ngw = (NG + S - 1) / S;
        const size_t smem = (size_t)S * (mma_gemv_ring_bytes<2, P>() + mma_gemv_aux_bytes(2, ngw));
        if (first_use_on_device((const void*)mma_gemv_kernel<2, P>))
            cudaFuncSetAttribute(mma_gemv_kernel<2, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int r0 = 0; r0 < R; r0 += kTok) {
            const int rr = R - r0 < kTok ? R - r0 : kTok;
            mma_gemv_kernel<2, P><<<ff / 16, 32 * S, smem, st>>>(xb + (size_t)r0 * d, rr, to_ptr(e->w1),
                                                                 to_ptr(e->w3), d, ff, ngw, hb + (size_t)r0 * ff,
                                                                 nullptr, 0, nullptr);
            DS_LAUNCH_CHECK("ds_w4_swiglu_gemv");
        }
        return DS_OK;
    }
    for (int r0 = 0; r0 < R;) {
        const int left = R - r0;
        if (left >= 4) { rc = swiglu_launch<4>(xb + (size_t)r0 * d, e, d, ff, G, hb + (size_t)r0 * ff, st); r0 += 4; }
        else if (left >= 2) { rc = swiglu_launch<2>(xb + (size_t)r0 * d, e, d, ff, G, hb + (size_t)r0 * ff, st); r0 += 2; }
        else { rc = swiglu_launch<1>(xb + (size_t)r0 * d, e, d, ff, G, hb + (size_t)r0 * ff, st); r0 += 1; }
        if (rc) return rc;
    }
    return DS_OK;
}

extern "C" int ds_w4_down_gemv(const void* h, int R, const ds_w4_expert* e, int d, int ff, int G,
                               const float* route_w, int route_stride, float* acc, void* stream) {
    int rc = check_gemv_shape(R, d, ff, G);
    if (rc) return rc;
    DS_CHECK_ARG(e && check_linear(e->w2) && h && route_w && acc, "ds_w4_down_gemv: NULL pointer");
    cudaStream_t st = as_stream(stream);
    const __nv_bfloat16* hb = (const __nv_bfloat16*)h;
    if (G == 128 && k4_use_mma(R)) {
        constexpr int P = 8;
        const int NG = ff / 128, S = mma_gemv_warps(NG, 1), ngw = (NG + S - 1) / S;
        const size_t smem = (size_t)S * (mma_gemv_ring_bytes<1, P>() + mma_gemv_aux_bytes(1, ngw));
        if (first_use_on_device((const void*)mma_gemv_kernel<1, P>))
            cudaFuncSetAttribute(mma_gemv_kernel<1, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int r0 = 0; r0 < R; r0 += kTok) {
            const int rr = R - r0 < kTok ? R - r0 : kTok;
            // PDL: the down GEMV's weight prologue overlaps the SwiGLU GEMV's tail
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(d / 16);
            cfg.blockDim = dim3(32 * S);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, mma_gemv_kernel<1, P>, hb + (size_t)r0 * ff, rr, to_ptr(e->w2), to_ptr(e->w2),
                               ff, d, ngw, (__nv_bfloat16*)nullptr, route_w + (size_t)r0 * route_stride,
                               route_stride, acc + (size_t)r0 * d);
            DS_LAUNCH_CHECK("ds_w4_down_gemv");
        }
        return DS_OK;
    }
    for (int r0 = 0; r0 < R;) {
        const int left = R - r0;
        const size_t ho = (size_t)r0 * ff, ao = (size_t)r0 * d;
        const float* rw = route_w + (size_t)r0 * route_stride;
        if (left >= 4) { rc = down_launch<4>(hb + ho, e, d, ff, G, rw, route_stride, acc + ao, st); r0 += 4; }
        else if (left >= 2) { rc = down_launch<2>(hb + ho, e, d, ff, G, rw, route_stride, acc + ao, st); r0 += 2; }
        else { rc = down_launch<1>(hb + ho, e, d, ff, G, rw, route_stride, acc + ao, st); r0 += 1; }
        if (rc) return rc;
    }
    return DS_OK;
}


extern "C" int ds_w4_expert_gemv(const void* x, int R, const ds_w4_expert* e, int d, int ff, int G, void* h,
                                 const float* route_w, int route_stride, float* acc, void* ev_start, void* ev_end,
                                 void* stream) {
    cudaStream_t st = as_stream(stream);
    // with a span requested, hold the stream until both launches are queued
    // (the span then excludes host submission latency; see gate_hold)
    const uint64_t key = (((1ull * 64 + (uint64_t)R) * 65536 + (uint64_t)d) * 65536 + (uint64_t)ff) * 256 + (uint64_t)G;
    const unsigned gate = (ev_start && gate_warm(key)) ? gate_hold(st) : 0;
    int rc = DS_OK;
    if (ev_start) {
        cudaError_t er = cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_start), st);
        if (er != cudaSuccess) rc = cuda_status(er, "ds_w4_expert_gemv: event");
    }
    if (!rc) rc = expert_v6(x, R, e, d, ff, G, h, route_w, acc, st);
    if (rc == 1) {        // no fused variant for this shape: the two-kernel path
        rc = ds_w4_swiglu_gemv(x, R, e, d, ff, G, h, stream);
        if (!rc) rc = ds_w4_down_gemv(h, R, e, d, ff, G, route_w, route_stride, acc, stream);
    }
    if (!rc && ev_end) {
        cudaError_t er = cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_end), st);
        if (er != cudaSuccess) rc = cuda_status(er, "ds_w4_expert_gemv: event");
    }
    gate_release(gate);                 // on every path: a held stream must never stay blocked
    return rc;
}

// ---------------------------------------------------------------------------
// K4 through a CUDA graph.  While the copy engine streams an expert over the
// host link (97 % of decode), every command the host submits reaches the GPU
// ~25-30 us late: the front end fetches the pushbuffer from host memory behind
// the copy engine's queued PCIe reads (profiles/r2/k4_ce_timeline.json: the v6
// kernel itself runs 28.0 -> 28.7 us beside the copy, its event span 47 ->
// 60 us).  An uploaded graph lives in device memory, so one graph launch
// carries [wait for the slot's ready event] -> ev_start -> K4 -> ev_end with
// no further host fetch between the data landing and the kernel starting.
// Graphs are cached per argument set (static decode buffers: 4-8 slots x k
// routing columns + pinned experts); the events are swapped per launch.
namespace {
struct K4GraphKey {
    const void* x; const void* h; const float* rw; const float* acc; ds_w4_expert e;
    int R, d, ff, G, rs; bool wait, evs; int dev;
    bool operator<(const K4GraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) < 0; }
};
struct K4Graph {
    cudaGraph_t graph = nullptr;      // kept: its node handles address the exec's nodes
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t wait = nullptr, start = nullptr, end = nullptr;
    // library-owned placeholder events: the nodes point at these between
    // launches, never at a caller's event that may since have been destroyed
    cudaEvent_t own[3] = {nullptr, nullptr, nullptr};
};

void k4g_destroy(K4Graph& g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    for (auto& e : g.own)
        if (e) cudaEventDestroy(e);
    g = K4Graph();
}
std::mutex g_k4g_mu;
std::map<K4GraphKey, K4Graph> g_k4g;
constexpr size_t kK4GraphCap = 1024;

void k4g_clear_locked() {
    for (auto& kv : g_k4g) k4g_destroy(kv.second);
    g_k4g.clear();
}

int k4g_capture(const K4GraphKey& k, cudaEvent_t wait_ev, cudaEvent_t e0, cudaEvent_t e1, cudaGraph_t* gout);

int k4g_build(const K4GraphKey& k, K4Graph* out) {
    for (auto& e : out->own)
        if (cudaEventCreate(&e) != cudaSuccess) {
            k4g_destroy(*out);
            return fail(DS_ERR_STATE, "ds_w4_expert_gemv_graph: placeholder events");
        }
    cudaGraph_t g = nullptr;
    int rc = k4g_capture(k, out->own[0], out->own[1], out->own[2], &g);
    if (rc) {
        k4g_destroy(*out);
        return rc;
    }
    cudaError_t er;

    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(g, nodes.data(), &n);
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        size_t n_dep = 0, n_out = 0;
        cudaGraphNodeGetDependencies(nd, nullptr, &n_dep);
        cudaGraphNodeGetDependentNodes(nd, nullptr, &n_out);
        if (getenv("DS_K4G_DEBUG"))
            fprintf(stderr, "[k4 graph] node %p type %d deps %zu dependents %zu\n", (void*)nd, (int)t, n_dep, n_out);
        if (t == cudaGraphNodeTypeWaitEvent) {
            out->wait = nd;
        } else if (t == cudaGraphNodeTypeEventRecord) {
            // the span's end is the record node nothing depends on
            (n_out == 0 ? out->end : out->start) = nd;
        }
    }
    out->graph = g;
    er = cudaGraphInstantiate(&out->exec, g, 0);
    if (er != cudaSuccess) {
        k4g_destroy(*out);
        return cuda_status(er, "ds_w4_expert_gemv_graph: instantiate");
    }
    if ((k.wait && !out->wait) || (k.evs && (!out->start || !out->end))) {
        k4g_destroy(*out);
        return fail(DS_ERR_STATE, "ds_w4_expert_gemv_graph: captured graph lacks its event nodes");
    }
    return DS_OK;
}
int k4g_capture(const K4GraphKey& k, cudaEvent_t wait_ev, cudaEvent_t e0, cudaEvent_t e1, cudaGraph_t* gout) {
    static thread_local cudaStream_t caps[64] = {};        // private capture stream per device (never runs work)
    cudaStream_t& cap = caps[k.dev & 63];
    if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess)
        return fail(DS_ERR_STATE, "ds_w4_expert_gemv_graph: capture stream");
    // relaxed: the link thread keeps issuing copies while this thread captures
    cudaError_t er = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
    if (er != cudaSuccess) return cuda_status(er, "ds_w4_expert_gemv_graph: begin capture");
    int rc = DS_OK;
    if (k.wait) er = cudaStreamWaitEvent(cap, wait_ev, cudaEventWaitExternal);
    if (er == cudaSuccess && k.evs) er = cudaEventRecordWithFlags(e0, cap, cudaEventRecordExternal);
    if (er != cudaSuccess) rc = cuda_status(er, "ds_w4_expert_gemv_graph: capture events");
    if (!rc) rc = expert_v6(k.x, k.R, &k.e, k.d, k.ff, k.G, const_cast<void*>(k.h), k.rw,
                            const_cast<float*>(k.acc), cap);
    if (rc == 1) {
        rc = ds_w4_swiglu_gemv(k.x, k.R, &k.e, k.d, k.ff, k.G, const_cast<void*>(k.h), cap);
        if (!rc) rc = ds_w4_down_gemv(k.h, k.R, &k.e, k.d, k.ff, k.G, k.rw, k.rs, const_cast<float*>(k.acc), cap);
    }
    if (!rc && k.evs) {
        er = cudaEventRecordWithFlags(e1, cap, cudaEventRecordExternal);
        if (er != cudaSuccess) rc = cuda_status(er, "ds_w4_expert_gemv_graph: capture events");
    }
    cudaGraph_t g = nullptr;
    er = cudaStreamEndCapture(cap, &g);
    if (!rc && er != cudaSuccess) rc = cuda_status(er, "ds_w4_expert_gemv_graph: end capture");
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    *gout = g;
    return DS_OK;
}
}  // namespace

extern "C" int ds_w4_expert_gemv_graph(const void* x, int R, const ds_w4_expert* e, int d, int ff, int G,
                                       void* h, const float* route_w, int route_stride, float* acc,
                                       void* wait_event, void* ev_start, void* ev_end, void* stream) {
    DS_CHECK_ARG(x && e && h && route_w && acc && R >= 1 && R <= 16, "ds_w4_expert_gemv_graph: bad arguments");
    DS_CHECK_ARG((ev_start == nullptr) == (ev_end == nullptr), "ds_w4_expert_gemv_graph: events come in pairs");
    cudaStream_t st = as_stream(stream);
    K4GraphKey k;
    std::memset(&k, 0, sizeof(k));                           // padding bytes take part in the key
    k.x = x; k.h = h; k.rw = route_w; k.acc = acc; k.e = *e;
    k.R = R; k.d = d; k.ff = ff; k.G = G; k.rs = route_stride;
    k.wait = wait_event != nullptr; k.evs = ev_start != nullptr;
    cudaGetDevice(&k.dev);
    auto w_ev = reinterpret_cast<cudaEvent_t>(wait_event);
    auto e0 = reinterpret_cast<cudaEvent_t>(ev_start), e1 = reinterpret_cast<cudaEvent_t>(ev_end);
    std::lock_guard<std::mutex> lk(g_k4g_mu);
    auto it = g_k4g.find(k);
    if (it == g_k4g.end()) {
        if (g_k4g.size() >= kK4GraphCap) k4g_clear_locked();
        K4Graph kg;
        int rc = k4g_build(k, &kg);
        if (rc) return rc;
        cudaError_t er = cudaGraphUpload(kg.exec, st);       // device-resident before its first launch
        if (er != cudaSuccess) {
            k4g_destroy(kg);
            return cuda_status(er, "ds_w4_expert_gemv_graph: upload");
        }
        it = g_k4g.emplace(k, kg).first;
    }
    K4Graph& kg = it->second;
    // point the nodes at this call's events, launch, point them back at the
    // placeholders (exec updates never affect a launch already submitted)
    auto set = [&](cudaEvent_t w, cudaEvent_t a, cudaEvent_t b) -> cudaError_t {
        cudaError_t er = cudaSuccess;
        if (k.wait) er = cudaGraphExecEventWaitNodeSetEvent(kg.exec, kg.wait, w);
        if (er == cudaSuccess && k.evs) er = cudaGraphExecEventRecordNodeSetEvent(kg.exec, kg.start, a);
        if (er == cudaSuccess && k.evs) er = cudaGraphExecEventRecordNodeSetEvent(kg.exec, kg.end, b);
        return er;
    };
    cudaError_t er = set(w_ev, e0, e1);
    if (er != cudaSuccess) return cuda_status(er, "ds_w4_expert_gemv_graph: set events");
    er = cudaGraphLaunch(kg.exec, st);
    cudaError_t er2 = set(kg.own[0], kg.own[1], kg.own[2]);
    if (er != cudaSuccess) return cuda_status(er, "ds_w4_expert_gemv_graph: launch");
    return er2 == cudaSuccess ? DS_OK : cuda_status(er2, "ds_w4_expert_gemv_graph: reset events");
}

extern "C" int ds_w4_graph_cache_clear(void) {
    std::lock_guard<std::mutex> lk(g_k4g_mu);
    k4g_clear_locked();
    return DS_OK;
}

extern "C" int ds_combine_finalize(float* acc, const void* resid, int R, int d, void* out,
                                   void* stream) {
    DS_CHECK_ARG(R >= 0 && d > 0, "ds_combine_finalize: bad shape");
    if (R == 0) return DS_OK;
    DS_CHECK_ARG(acc && resid && out, "ds_combine_finalize: NULL pointer");
    size_t n = (size_t)R * d;
    int grid = (int)((n + 255) / 256);
    if (grid > 4 * num_sms()) grid = 4 * num_sms();
    finalize_kernel<<<grid, 256, 0, as_stream(stream)>>>(acc, (const __nv_bfloat16*)resid, n,
                                                         (__nv_bfloat16*)out);
    DS_LAUNCH_CHECK("ds_combine_finalize");
    return DS_OK;
}

// Device-clock totals of every fused (v6) K4 launch since the library loaded:
// sum of (last CTA exit - first CTA entry) in ns and the launch count.
extern "C" int ds_k4_device_span(unsigned long long* ns, unsigned long long* n) {
    DS_CHECK_ARG(ns && n, "ds_k4_device_span: NULL pointer");
    cudaError_t e = cudaMemcpyFromSymbol(ns, g_k4f_span_ns, sizeof(*ns));
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(n, g_k4f_span_n, sizeof(*n));
    return cuda_status(e, "ds_k4_device_span");
}

// Diagnostics: the per-CTA stamps of the last v6 launch run with DS_K4_V6_TIMELINE=1
// ([n_ctas][8] u64 globaltimer ns; see expert_fused_v6_kernel).
extern "C" int ds_debug_k4v6_timeline(unsigned long long* out, int n_ctas) {
    DS_CHECK_ARG(out && n_ctas > 0 && n_ctas <= 1024, "ds_debug_k4v6_timeline: bad arguments");
    cudaError_t e = cudaMemcpyFromSymbol(out, g_k4f_dbg, (size_t)n_ctas * 8 * sizeof(unsigned long long));
    return cuda_status(e, "ds_debug_k4v6_timeline");
}
