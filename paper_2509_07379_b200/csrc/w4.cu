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

__device__ __forceinline__ void stage_x(const __nv_bfloat16* __restrict__ x, int R, int K,
                                        uint32_t* xs, float* xsum) {
    const int words = K / 2;
    const int units = words / 4;                        // 16-byte units per row
    const uint4* xu = reinterpret_cast<const uint4*>(x);
    for (int i = threadIdx.x; i < R * units; i += blockDim.x) {
        const int r = i / units, u = i - r * units;
        *reinterpret_cast<uint4*>(xs + r * words + swz_unit(u) * 4) = __ldg(xu + i);
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
    int grid = per_sm * num_sms();
    int need = (rows_needed + (kGemvThreads / 32) - 1) / (kGemvThreads / 32);
    return grid < need ? grid : need;
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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(swiglu_gemv_kernel<R, G, U, GUARD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(down_gemv_kernel<R, G, U, GUARD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
    }
    const size_t smem = (size_t)R * ff * 2 + (size_t)R * (ff / 32) * 4;
    const int grid = gemv_grid((const void*)down_gemv_kernel<R, G, U, GUARD>, smem, d);
    down_gemv_kernel<R, G, U, GUARD><<<grid, kGemvThreads, smem, st>>>(h, to_ptr(e->w2), ff, d, rw, rs, acc);
    DS_LAUNCH_CHECK("ds_w4_down_gemv");
    return DS_OK;
}

// batch size per lane U (16-byte loads in flight per matrix) chosen so that
// (K/32)/32 is a multiple of U: no predicates in the streaming loop
template <int R, int G>
static int swiglu_launch_g(const __nv_bfloat16* x, const ds_w4_expert* e, int d, int ff, __nv_bfloat16* h,
                           cudaStream_t st) {
    const int per_lane = (d / 32) % 32 == 0 ? (d / 32) / 32 : 0;
    if (per_lane && per_lane % 4 == 0) return swiglu_launch_u<R, G, 4, false>(x, e, d, ff, h, st);
    if (per_lane && per_lane % 3 == 0) return swiglu_launch_u<R, G, 3, false>(x, e, d, ff, h, st);
    if (per_lane && per_lane % 2 == 0) return swiglu_launch_u<R, G, 2, false>(x, e, d, ff, h, st);
    return swiglu_launch_u<R, G, 2, true>(x, e, d, ff, h, st);
}

template <int R, int G>
static int down_launch_g(const __nv_bfloat16* h, const ds_w4_expert* e, int d, int ff, const float* rw, int rs,
                         float* acc, cudaStream_t st) {
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
