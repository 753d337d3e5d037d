// K1 gate top-k, K2 permute / unpermute-combine, K7 cache check, and the
// online routing histogram.
//
// The reference has no gate: routing appears only as sampled paths
// (trace.py:178-242).  The gate follows HF MixtralTopKRouter semantics
// (transformers 5.5.0, modeling_mixtral.py:109-116: logits = x W_g^T,
// softmax, top-k, renormalise) with two B200-build contracts that make the
// expert indices bit-exact against oracle/routing_ref.py:
//   * logits are accumulated in float64 in a FIXED order independent of the
//     launch shape: thread q of 256 sums 8-element vectors v = q, q+256, ...
//     (bf16*bf16 products are exact in f64), then a pairwise tree
//     P[q] += P[q+off], off = 128..1;
//   * top-k on the f64 logits with ties to the lower index, emitted sorted
//     ascending — the reference's tie rule (predictor.py:419-421) and its
//     trace format (sorted k-tuples, trace.py:39-58).
#include "ds_common.cuh"

namespace ds {
namespace {

constexpr int kGateThreads = 256;
constexpr int kGateMaxM = 16;

__global__ void __launch_bounds__(kGateThreads) gate_topk_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, int T, int d, int M,
    int k, int32_t* __restrict__ idx, float* __restrict__ w, double* __restrict__ logits,
    int32_t* __restrict__ counts, int32_t* __restrict__ hist, int hist_stride, int layer) {
    __shared__ double part[kGateMaxM][kGateThreads];
    const int t = blockIdx.x;
    const int q = threadIdx.x;
    double acc[kGateMaxM];
#pragma unroll
    for (int e = 0; e < kGateMaxM; ++e) acc[e] = 0.0;
    const int nvec = d / 8;
    const uint4* xv = reinterpret_cast<const uint4*>(x + (size_t)t * d);
    for (int v = q; v < nvec; v += kGateThreads) {
        // all M weight vectors and x issued before any math (predicated on
        // e < M rather than a break, which would serialise the loads)
        uint4 xr = __ldg(xv + v);
        uint4 wr[kGateMaxM];
#pragma unroll
        for (int e = 0; e < kGateMaxM; ++e)
            if (e < M) wr[e] = __ldg(reinterpret_cast<const uint4*>(wg + (size_t)e * d) + v);
        const uint32_t xs[4] = {xr.x, xr.y, xr.z, xr.w};
#pragma unroll
        for (int e = 0; e < kGateMaxM; ++e) {
            if (e < M) {
                const uint32_t ws[4] = {wr[e].x, wr[e].y, wr[e].z, wr[e].w};
                double a = acc[e];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a = fma((double)bf16_lo(xs[i]), (double)bf16_lo(ws[i]), a);
                    a = fma((double)bf16_hi(xs[i]), (double)bf16_hi(ws[i]), a);
                }
                acc[e] = a;
            }
        }
    }
    for (int e = 0; e < M; ++e) part[e][q] = acc[e];
    __syncthreads();
    for (int off = kGateThreads / 2; off > 0; off >>= 1) {
        if (q < off)
            for (int e = 0; e < M; ++e) part[e][q] = __dadd_rn(part[e][q], part[e][q + off]);
        __syncthreads();
    }
    if (q != 0) return;
    double lg[kGateMaxM];
    for (int e = 0; e < M; ++e) lg[e] = part[e][0];
    if (logits)
        for (int e = 0; e < M; ++e) logits[(size_t)t * M + e] = lg[e];
    uint32_t taken = 0;
    double top = 0.0;
    for (int r = 0; r < k; ++r) {
        int best = -1;
        for (int e = 0; e < M; ++e) {
            if (taken >> e & 1u) continue;
            if (best < 0 || lg[e] > lg[best]) best = e;
        }
        if (r == 0) top = lg[best];
        taken |= 1u << best;
    }
    // renormalised softmax over the selected set, f64, ascending order
    double ex[kGateMaxM];
    double den = 0.0;
    int j = 0;
    for (int e = 0; e < M; ++e) {
        if (!(taken >> e & 1u)) continue;
        ex[j] = exp(__dsub_rn(lg[e], top));
        den = __dadd_rn(den, ex[j]);
        ++j;
    }
    j = 0;
    for (int e = 0; e < M; ++e) {
        if (!(taken >> e & 1u)) continue;
        idx[(size_t)t * k + j] = e;
        w[(size_t)t * k + j] = (float)__ddiv_rn(ex[j], den);
        if (counts) atomicAdd(counts + e, 1);
        if (hist) hist[(size_t)t * hist_stride + (size_t)layer * k + j] = e + 1;
        ++j;
    }
}

// Stable counting sort of T*k pairs by expert (one CTA, chunks of 1024).
constexpr int kPermThreads = 1024;

__global__ void __launch_bounds__(kPermThreads) permute_index_kernel(
    const int32_t* __restrict__ idx, int n, int M, int k, int32_t* __restrict__ offsets,
    int32_t* __restrict__ pos, int32_t* __restrict__ src_token) {
    __shared__ int cnt[DS_MAX_EXPERTS];
    __shared__ int base[DS_MAX_EXPERTS];
    __shared__ int wcnt[kPermThreads / 32][DS_MAX_EXPERTS];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < M) cnt[tid] = 0;
    __syncthreads();
    for (int p = tid; p < n; p += kPermThreads) atomicAdd(&cnt[idx[p]], 1);
    __syncthreads();
    if (tid == 0) {
        int s = 0;
        for (int e = 0; e < M; ++e) {
            base[e] = s;
            offsets[e] = s;
            s += cnt[e];
        }
        offsets[M] = s;
    }
    __syncthreads();
    for (int c0 = 0; c0 < n; c0 += kPermThreads) {
        const int p = c0 + tid;
        const int e = p < n ? idx[p] : -1;
        const unsigned same = __match_any_sync(0xffffffffu, e);
        const int rank = __popc(same & ((1u << lane) - 1u));
        for (int i = lane; i < M; i += 32) wcnt[wid][i] = 0;
        __syncwarp();
        if (e >= 0 && rank == 0) wcnt[wid][e] = __popc(same);
        __syncthreads();
        if (e >= 0) {
            int before = 0;
            for (int w2 = 0; w2 < wid; ++w2) before += wcnt[w2][e];
            const int r = base[e] + before + rank;
            pos[p] = r;
            src_token[r] = p / k;
        }
        __syncthreads();
        if (tid < M) {
            int tot = 0;
            for (int w2 = 0; w2 < kPermThreads / 32; ++w2) tot += wcnt[w2][tid];
            base[tid] += tot;
        }
        __syncthreads();
    }
}

// one warp per grouped row: xperm[r] = x[src_token[r]]
__global__ void gather_rows_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ src,
                                   int rows, int vec_per_row, uint4* __restrict__ xperm) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const uint4* s = x + (size_t)src[warp] * vec_per_row;
    uint4* dst = xperm + (size_t)warp * vec_per_row;
    for (int i = lane; i < vec_per_row; i += 32) dst[i] = __ldg(s + i);
}

__global__ void unpermute_combine_kernel(const float* __restrict__ y, const int32_t* __restrict__ pos,
                                         const float* __restrict__ w, const __nv_bfloat16* __restrict__ resid,
                                         int T, int d, int k, __nv_bfloat16* __restrict__ out) {
    const int t = blockIdx.x;
    for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < k; ++j) {
            const float wj = w[(size_t)t * k + j];
            const float4 v = *reinterpret_cast<const float4*>(y + (size_t)pos[(size_t)t * k + j] * d + c);
            acc[0] = __fadd_rn(acc[0], __fmul_rn(wj, v.x));
            acc[1] = __fadd_rn(acc[1], __fmul_rn(wj, v.y));
            acc[2] = __fadd_rn(acc[2], __fmul_rn(wj, v.z));
            acc[3] = __fadd_rn(acc[3], __fmul_rn(wj, v.w));
        }
        const __nv_bfloat16* rr = resid + (size_t)t * d + c;
        __nv_bfloat16* o = out + (size_t)t * d + c;
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = __float2bfloat16_rn(__fadd_rn(__bfloat162float(rr[i]), acc[i]));
    }
}

// Expert-parallel partial combine: out[t] = sum_j [expert(t,j) owned] w[t,j] y[pos[t,j]]
// (f32, j order) — the per-rank term of the all-reduce.
__global__ void unpermute_partial_kernel(const float* __restrict__ y, const int32_t* __restrict__ pos,
                                         const float* __restrict__ w, const int32_t* __restrict__ idx,
                                         unsigned long long owned, int T, int d, int k, float* __restrict__ out) {
    const int t = blockIdx.x;
    for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < k; ++j) {
            if (!((owned >> idx[(size_t)t * k + j]) & 1ull)) continue;
            const float wj = w[(size_t)t * k + j];
            const float4 v = *reinterpret_cast<const float4*>(y + (size_t)pos[(size_t)t * k + j] * d + c);
            acc[0] = __fadd_rn(acc[0], __fmul_rn(wj, v.x));
            acc[1] = __fadd_rn(acc[1], __fmul_rn(wj, v.y));
            acc[2] = __fadd_rn(acc[2], __fmul_rn(wj, v.z));
            acc[3] = __fadd_rn(acc[3], __fmul_rn(wj, v.w));
        }
        *reinterpret_cast<float4*>(out + (size_t)t * d + c) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
}

__global__ void cache_check_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ pred,
                                   int T, int k, int32_t* __restrict__ miss) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    int m = 0;
    for (int j = 0; j < k; ++j) {
        bool hit = false;
        for (int i = 0; i < k; ++i) hit |= (idx[(size_t)t * k + j] == pred[(size_t)t * k + i]);
        if (!hit) m |= 1 << j;
    }
    miss[t] = m;
}

__global__ void route_histogram_kernel(const int32_t* __restrict__ paths, int N, int L, int M, int k,
                                       unsigned long long* __restrict__ pop,
                                       unsigned long long* __restrict__ aff) {
    const size_t n_items = (size_t)N * L;
    for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < n_items;
         it += (size_t)gridDim.x * blockDim.x) {
        const int l = (int)(it % L);
        const int32_t* sel = paths + it * k;
        for (int j = 0; j < k; ++j) atomicAdd(pop + (size_t)l * M + sel[j], 1ull);
        if (l + 1 < L) {
            const int32_t* nxt = sel + k;
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b)
                    atomicAdd(aff + ((size_t)l * M + sel[a]) * M + nxt[b], 1ull);
        }
    }
}

}  // namespace
}  // namespace ds

using namespace ds;

extern "C" int ds_gate_topk(const void* x, const void* wg, int T, int d, int M, int k, int32_t* idx,
                            float* w, double* logits, int32_t* counts, int32_t* hist,
                            int hist_stride, int layer, void* stream) {
    DS_CHECK_ARG(T >= 0 && d > 0 && d % 8 == 0, "ds_gate_topk: d must be a positive multiple of 8");
    DS_CHECK_ARG(M >= 2 && M <= kGateMaxM && k >= 1 && k < M, "ds_gate_topk: need 1<=k<M<=%d", kGateMaxM);
    DS_CHECK_ARG(T == 0 || (x && wg && idx && w), "ds_gate_topk: NULL pointer");
    DS_CHECK_ARG(((uintptr_t)x & 15) == 0 && ((uintptr_t)wg & 15) == 0, "ds_gate_topk: 16B alignment");
    if (T == 0) return DS_OK;
    gate_topk_kernel<<<T, kGateThreads, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)x, (const __nv_bfloat16*)wg, T, d, M, k, idx, w, logits, counts, hist,
        hist_stride, layer);
    DS_LAUNCH_CHECK("ds_gate_topk");
    return DS_OK;
}

extern "C" int ds_permute(const int32_t* idx, const void* x, int T, int d, int M, int k,
                          int32_t* offsets, int32_t* pos, int32_t* src_token, void* xperm,
                          void* stream) {
    DS_CHECK_ARG(T >= 0 && M >= 1 && M <= DS_MAX_EXPERTS && k >= 1, "ds_permute: bad shape");
    DS_CHECK_ARG(offsets && (T == 0 || (idx && pos && src_token)), "ds_permute: NULL pointer");
    cudaStream_t st = as_stream(stream);
    permute_index_kernel<<<1, kPermThreads, 0, st>>>(idx, T * k, M, k, offsets, pos, src_token);
    DS_LAUNCH_CHECK("ds_permute: index");
    if (xperm && T > 0) {
        DS_CHECK_ARG(x && d % 8 == 0, "ds_permute: gather needs x and d % 8 == 0");
        int rows = T * k;
        gather_rows_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(
            (const uint4*)x, src_token, rows, d / 8, (uint4*)xperm);
        DS_LAUNCH_CHECK("ds_permute: gather");
    }
    return DS_OK;
}

extern "C" int ds_unpermute_combine(const float* y, const int32_t* pos, const float* w,
                                    const void* resid, int T, int d, int k, void* out,
                                    void* stream) {
    DS_CHECK_ARG(T >= 0 && d % 4 == 0 && k >= 1, "ds_unpermute_combine: bad shape");
    if (T == 0) return DS_OK;
    DS_CHECK_ARG(y && pos && w && resid && out, "ds_unpermute_combine: NULL pointer");
    unpermute_combine_kernel<<<T, 256, 0, as_stream(stream)>>>(
        y, pos, w, (const __nv_bfloat16*)resid, T, d, k, (__nv_bfloat16*)out);
    DS_LAUNCH_CHECK("ds_unpermute_combine");
    return DS_OK;
}

extern "C" int ds_unpermute_partial(const float* y, const int32_t* pos, const float* w, const int32_t* idx,
                                    uint64_t owned_mask, int T, int d, int k, float* out, void* stream) {
    DS_CHECK_ARG(T >= 0 && d % 4 == 0 && k >= 1, "ds_unpermute_partial: bad shape");
    if (T == 0) return DS_OK;
    DS_CHECK_ARG(y && pos && w && idx && out, "ds_unpermute_partial: NULL pointer");
    unpermute_partial_kernel<<<T, 256, 0, as_stream(stream)>>>(y, pos, w, idx, owned_mask, T, d, k, out);
    DS_LAUNCH_CHECK("ds_unpermute_partial");
    return DS_OK;
}

extern "C" int ds_cache_check(const int32_t* idx, const int32_t* pred, int T, int k,
                              int32_t* miss_mask, void* stream) {
    DS_CHECK_ARG(T >= 0 && k >= 1 && k <= 30, "ds_cache_check: bad shape");
    if (T == 0) return DS_OK;
    cache_check_kernel<<<(T + 127) / 128, 128, 0, as_stream(stream)>>>(idx, pred, T, k, miss_mask);
    DS_LAUNCH_CHECK("ds_cache_check");
    return DS_OK;
}

extern "C" int ds_route_histogram(const int32_t* paths, int N, int L, int M, int k,
                                  int64_t* pop_counts, int64_t* aff_counts, void* stream) {
    DS_CHECK_ARG(N >= 0 && L >= 2 && M >= 2 && k >= 1 && k < M, "ds_route_histogram: bad shape");
    if (N == 0) return DS_OK;
    DS_CHECK_ARG(paths && pop_counts && aff_counts, "ds_route_histogram: NULL pointer");
    size_t items = (size_t)N * L;
    int blocks = (int)((items + 255) / 256);
    if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
    route_histogram_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
        paths, N, L, M, k, (unsigned long long*)pop_counts, (unsigned long long*)aff_counts);
    DS_LAUNCH_CHECK("ds_route_histogram");
    return DS_OK;
}
