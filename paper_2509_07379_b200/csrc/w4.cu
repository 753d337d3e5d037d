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
constexpr int kGemvThreads = 256;
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
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(x);
    for (int i = threadIdx.x; i < R * words; i += blockDim.x) {
        const int r = i / words, w = i - r * words;
        xs[r * words + swz_unit(w >> 2) * 4 + (w & 3)] = __ldg(xw + i);
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

// Partial dot of one lane's 32 codes against its x chunk: sum x*(128+q).
// xc = start of the (swizzled) chunk, sw = (chunk >> 1) & 3.
__device__ __forceinline__ float dot32(const uint4 c, const uint32_t* xc, int sw) {
    float acc = 0.f;
    const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xc + 4 * (i ^ sw));
        const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const uint32_t p = nib_pair_magic(cw[i] >> (4 * s));
            fma_bf16_lo(acc, p, xx[s]);
            fma_bf16_hi(acc, p, xx[s]);
        }
    }
    return acc;
}

__device__ __forceinline__ float group_term(const W4Ptr& m, int n, int gpr, int g, float part,
                                            float xsum) {
    const size_t zi = (size_t)n * gpr + g;
    const float z = (float)((__ldg(m.zeros + (zi >> 1)) >> ((zi & 1) * 4)) & 15);
    const float s = __uint_as_float((uint32_t)__ldg(m.scales + zi) << 16);
    return s * (part - (128.f + z) * xsum);
}

// h[r, n] = bf16( silu(x_r . W1[:, n]) * (x_r . W3[:, n]) )
__global__ void __launch_bounds__(kGemvThreads) swiglu_gemv_kernel(
    const __nv_bfloat16* __restrict__ x, int R, W4Ptr w1, W4Ptr w3, int K, int N, int G,
    __nv_bfloat16* __restrict__ h) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* xs = sm;                               // R * K/2 words
    float* xsum = reinterpret_cast<float*>(sm + R * K / 2);  // R * K/32
    stage_x(x, R, K, xs, xsum);
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int gpr = K / G;
    const int kwords = K / 8;
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += warps) {
        float a[kRMax], b[kRMax];
#pragma unroll
        for (int r = 0; r < kRMax; ++r) a[r] = b[r] = 0.f;
        const uint4* c1 = reinterpret_cast<const uint4*>(w1.codes + (size_t)n * kwords);
        const uint4* c3 = reinterpret_cast<const uint4*>(w3.codes + (size_t)n * kwords);
#pragma unroll 2
        for (int kk = lane * 32; kk < K; kk += 1024) {
            const uint4 v1 = ldg_nc_v4(c1 + (kk >> 5));
            const uint4 v3 = ldg_nc_v4(c3 + (kk >> 5));
            const int g = kk / G;
#pragma unroll
            for (int r = 0; r < kRMax; ++r) {
                if (r < R) {
                    const uint32_t* xc = xs + (size_t)r * (K / 2) + kk / 2;
                    const int sw = (kk >> 6) & 3;
                    const float xsm = xsum[r * (K / 32) + (kk >> 5)];
                    a[r] += group_term(w1, n, gpr, g, dot32(v1, xc, sw), xsm);
                    b[r] += group_term(w3, n, gpr, g, dot32(v3, xc, sw), xsm);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kRMax; ++r) {
            if (r < R) {
                const float av = warp_sum(a[r]);
                const float bv = warp_sum(b[r]);
                if (lane == r) {
                    const float sl = av / (1.0f + expf(-av));
                    h[(size_t)r * N + n] = __float2bfloat16_rn(sl * bv);
                }
            }
        }
    }
}

// acc[r, n] += route_w[r] * (h_r . W2[:, n])
__global__ void __launch_bounds__(kGemvThreads) down_gemv_kernel(
    const __nv_bfloat16* __restrict__ hin, int R, W4Ptr w2, int K, int N, int G,
    const float* __restrict__ route_w, int route_stride, float* __restrict__ acc) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* xs = sm;
    float* xsum = reinterpret_cast<float*>(sm + R * K / 2);
    stage_x(hin, R, K, xs, xsum);
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int gpr = K / G;
    const int kwords = K / 8;
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += warps) {
        float y[kRMax];
#pragma unroll
        for (int r = 0; r < kRMax; ++r) y[r] = 0.f;
        const uint4* c2 = reinterpret_cast<const uint4*>(w2.codes + (size_t)n * kwords);
#pragma unroll 4
        for (int kk = lane * 32; kk < K; kk += 1024) {
            const uint4 v = ldg_nc_v4(c2 + (kk >> 5));
            const int g = kk / G;
#pragma unroll
            for (int r = 0; r < kRMax; ++r) {
                if (r < R) {
                    const uint32_t* xc = xs + (size_t)r * (K / 2) + kk / 2;
                    y[r] += group_term(w2, n, gpr, g, dot32(v, xc, (kk >> 6) & 3),
                                       xsum[r * (K / 32) + (kk >> 5)]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kRMax; ++r) {
            if (r < R) {
                const float yv = warp_sum(y[r]);
                if (lane == r) {
                    float* o = acc + (size_t)r * N + n;
                    *o = __fadd_rn(*o, __fmul_rn(route_w[(size_t)r * route_stride], yv));
                }
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
    DS_CHECK_ARG(d > 0 && ff > 0 && d % 128 == 0 && ff % 128 == 0 && (G == 32 || G == 64 || G == 128),
                 "w4 gemv: need d, ff multiples of 128 and G in {32,64,128}");
    return DS_OK;
}

extern "C" int ds_w4_swiglu_gemv(const void* x, int R, const ds_w4_expert* e, int d, int ff, int G,
                                 void* h, void* stream) {
    int rc = check_gemv_shape(R, d, ff, G);
    if (rc) return rc;
    DS_CHECK_ARG(e && check_linear(e->w1) && check_linear(e->w3) && x && h, "ds_w4_swiglu_gemv: NULL pointer");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(swiglu_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr = true;
    }
    cudaStream_t st = as_stream(stream);
    for (int r0 = 0; r0 < R; r0 += kRMax) {
        const int rr = R - r0 < kRMax ? R - r0 : kRMax;
        const size_t smem = (size_t)rr * d * 2 + (size_t)rr * (d / 32) * 4;
        const int grid = gemv_grid((const void*)swiglu_gemv_kernel, smem, ff);
        swiglu_gemv_kernel<<<grid, kGemvThreads, smem, st>>>(
            (const __nv_bfloat16*)x + (size_t)r0 * d, rr, to_ptr(e->w1), to_ptr(e->w3), d, ff, G,
            (__nv_bfloat16*)h + (size_t)r0 * ff);
        DS_LAUNCH_CHECK("ds_w4_swiglu_gemv");
    }
    return DS_OK;
}

extern "C" int ds_w4_down_gemv(const void* h, int R, const ds_w4_expert* e, int d, int ff, int G,
                               const float* route_w, int route_stride, float* acc, void* stream) {
    int rc = check_gemv_shape(R, d, ff, G);
    if (rc) return rc;
    DS_CHECK_ARG(e && check_linear(e->w2) && h && route_w && acc, "ds_w4_down_gemv: NULL pointer");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(down_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr = true;
    }
    cudaStream_t st = as_stream(stream);
    for (int r0 = 0; r0 < R; r0 += kRMax) {
        const int rr = R - r0 < kRMax ? R - r0 : kRMax;
        const size_t smem = (size_t)rr * ff * 2 + (size_t)rr * (ff / 32) * 4;
        const int grid = gemv_grid((const void*)down_gemv_kernel, smem, d);
        down_gemv_kernel<<<grid, kGemvThreads, smem, st>>>(
            (const __nv_bfloat16*)h + (size_t)r0 * ff, rr, to_ptr(e->w2), ff, d, G,
            route_w + (size_t)r0 * route_stride, route_stride, acc + (size_t)r0 * d);
        DS_LAUNCH_CHECK("ds_w4_down_gemv");
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
