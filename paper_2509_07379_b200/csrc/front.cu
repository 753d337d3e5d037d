// Decode front (batch-1 token): the elementwise steps around the W4 q|k|v / o
// projections fused into three small kernels.
//
// Why: after layer l's last expert lands, the host link has nothing certain to
// move until layer l+1's gate result reaches the host (its misses are unknown
// until then); everything on the compute stream in between — K4, combine,
// attention(l+1), norm, K1 — is a window the link spends on speculative
// chunks (profiles/r2/decode_window).  The torch version of the front was
// ~40 kernels (107 us per layer inside one CUDA graph); these three replace
// ~30 of them.  Same arithmetic as model.py's torch ops (f32 math, one bf16
// rounding where torch rounds), reduction order aside.
//
//   ds_rmsnorm           out = bf16( (f32(x) * rsqrt(mean(x^2) + eps)) * f32(g) )
//   ds_rope_kv_decode    y (f32 q|k|v of one token) -> bf16 -> RoPE(q, k) at the
//                        device-resident position; q out, k / v written into the
//                        layer's KV cache at that position
//   ds_residual_rmsnorm  h1 = bf16( f32(h) + y );  a = rmsnorm(h1, g)
#include "ds_common.cuh"

namespace ds {
namespace {

constexpr int kFrontThreads = 512;

__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? red[l] : 0.f;
        v = warp_sum(v);
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    const float s = red[0];
    __syncthreads();
    return s;
}

// one CTA per row; d <= 8 * kFrontThreads, d % 8 == 0
__device__ void rms_row(const float* xf, int d, const __nv_bfloat16* __restrict__ g, float eps,
                        __nv_bfloat16* __restrict__ out, float* red) {
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss = __fmaf_rn(xf[i], xf[i], ss);
    const float mean = __fdiv_rn(block_sum(ss, red), (float)d);
    const float r = rsqrtf(__fadd_rn(mean, eps));
    for (int i = threadIdx.x; i < d; i += blockDim.x)
        out[i] = __float2bfloat16_rn(__fmul_rn(__fmul_rn(xf[i], r), __bfloat162float(g[i])));
}

__global__ void __launch_bounds__(kFrontThreads) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                                const __nv_bfloat16* __restrict__ g, int d,
                                                                float eps, __nv_bfloat16* __restrict__ out) {
    extern __shared__ float xs[];                     // [d] f32 row + 32 reduction slots
    float* red = xs + d;
    const __nv_bfloat16* xr = x + (size_t)blockIdx.x * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) xs[i] = __bfloat162float(xr[i]);
    __syncthreads();
    rms_row(xs, d, g, eps, out + (size_t)blockIdx.x * d, red);
}

__global__ void __launch_bounds__(kFrontThreads) residual_rmsnorm_kernel(
    const __nv_bfloat16* __restrict__ h, const float* __restrict__ y, const __nv_bfloat16* __restrict__ g, int d,
    float eps, __nv_bfloat16* __restrict__ h1, __nv_bfloat16* __restrict__ a) {
    extern __shared__ float xs[];
    float* red = xs + d;
    const size_t o = (size_t)blockIdx.x * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const __nv_bfloat16 v = __float2bfloat16_rn(__fadd_rn(__bfloat162float(h[o + i]), y[o + i]));
        h1[o + i] = v;
        xs[i] = __bfloat162float(v);
    }
    __syncthreads();
    rms_row(xs, d, g, eps, a + o, red);
}

// y: [nh + 2 nkv][hd] f32 of one token; cos / sin: [max_seq][hd] f32 tables;
// kc / vc: this layer's cache [nkv][max_seq][hd] bf16.  torch order:
// q = bf16(y); out = bf16( f32(q) * cos + rot(f32(q)) * sin ), rot = [-x2, x1].
__global__ void rope_kv_decode_kernel(const float* __restrict__ y, int nh, int nkv, int hd,
                                      const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                      const long long* __restrict__ pos_p, int max_seq,
                                      __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ kc,
                                      __nv_bfloat16* __restrict__ vc) {
    const long long pos = *pos_p;
    const float* c = cos_t + pos * hd;
    const float* s = sin_t + pos * hd;
    const int half = hd / 2;
    const int n_rot = (nh + nkv) * hd;
    const int total = n_rot + nkv * hd;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        if (i < n_rot) {
            const int head = i / hd, j = i - head * hd;
            const float x = __bfloat162float(__float2bfloat16_rn(y[i]));
            const int pj = j < half ? j + half : j - half;
            const float xp = __bfloat162float(__float2bfloat16_rn(y[head * hd + pj]));
            const float rot = j < half ? -xp : xp;
            const __nv_bfloat16 r = __float2bfloat16_rn(__fadd_rn(__fmul_rn(x, c[j]), __fmul_rn(rot, s[j])));
            if (head < nh) q[i] = r;
            else kc[((size_t)(head - nh) * max_seq + pos) * hd + j] = r;
        } else {
            const int t = i - n_rot, head = t / hd, j = t - head * hd;
            vc[((size_t)head * max_seq + pos) * hd + j] = __float2bfloat16_rn(y[i]);
        }
    }
}

}  // namespace
}  // namespace ds

using namespace ds;

extern "C" int ds_rmsnorm(const void* x, int R, int d, const void* gamma, float eps, void* out, void* stream) {
    DS_CHECK_ARG(x && gamma && out && R >= 0 && d > 0 && d % 8 == 0 && d <= 16384, "ds_rmsnorm: bad arguments");
    if (R == 0) return DS_OK;
    const size_t smem = (size_t)(d + 32) * sizeof(float);
    rmsnorm_kernel<<<R, kFrontThreads, smem, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma), d, eps,
        static_cast<__nv_bfloat16*>(out));
    DS_LAUNCH_CHECK("ds_rmsnorm");
    return DS_OK;
}

extern "C" int ds_residual_rmsnorm(const void* h, const float* y, int R, int d, const void* gamma, float eps,
                                   void* h1, void* a, void* stream) {
    DS_CHECK_ARG(h && y && gamma && h1 && a && R >= 0 && d > 0 && d % 8 == 0 && d <= 16384,
                 "ds_residual_rmsnorm: bad arguments");
    if (R == 0) return DS_OK;
    const size_t smem = (size_t)(d + 32) * sizeof(float);
    residual_rmsnorm_kernel<<<R, kFrontThreads, smem, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16*>(h), y, static_cast<const __nv_bfloat16*>(gamma), d, eps,
        static_cast<__nv_bfloat16*>(h1), static_cast<__nv_bfloat16*>(a));
    DS_LAUNCH_CHECK("ds_residual_rmsnorm");
    return DS_OK;
}

extern "C" int ds_rope_kv_decode(const float* y, int nh, int nkv, int hd, const float* cos_t, const float* sin_t,
                                 const long long* pos, int max_seq, void* q, void* k_cache, void* v_cache,
                                 void* stream) {
    DS_CHECK_ARG(y && cos_t && sin_t && pos && q && k_cache && v_cache && nh > 0 && nkv > 0 && hd > 0 &&
                     hd % 2 == 0 && max_seq > 0,
                 "ds_rope_kv_decode: bad arguments");
    const int total = (nh + 2 * nkv) * hd;
    rope_kv_decode_kernel<<<(total + 255) / 256, 256, 0, as_stream(stream)>>>(
        y, nh, nkv, hd, cos_t, sin_t, pos, max_seq, static_cast<__nv_bfloat16*>(q),
        static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache));
    DS_LAUNCH_CHECK("ds_rope_kv_decode");
    return DS_OK;
}
