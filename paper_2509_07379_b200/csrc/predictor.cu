// K5 — fused State Constructor + ExpertMLP eval forward + top-k, float64.
//
// Reference semantics (/root/reference/pkg/src/duoserve/predictor.py):
//   features   :53-106  x = [hist/M (L*k, idx+1, 0-pad for layers >= l) ||
//                            pop[l] || mean_j aff[l-1][E_{l-1,j}] (or concat) ||
//                            l/(L-1)]
//   forward    :197-232 6x [Z = A@W_i + b_i; zhat = (Z-mu)*(1/sqrt(var+1e-5));
//                           H = gamma*zhat + beta; ReLU] -> A@W_6 + b_6 -> sigmoid
//   sigmoid    :132-138 piecewise stable
//   topk       :419-421 stable argsort(-p)[:k], returned sorted
// Elementwise steps use explicitly rounded __d*_rn ops in the reference's
// order (no FMA contraction); only the dot-product summation order differs
// from BLAS, so probabilities agree to ~1e-15 and the predicted SETS are
// bit-exact except at |p_k - p_{k+1}| below that (tests log the margin).
//
// Two launch shapes:
//   B <= 8  : one cooperative persistent kernel (grid = #SMs) with a
//             software grid barrier between layers — the decode path
//             (one token, one target layer), ~all SMs stream the 23.8 MB of
//             weights from L2/HBM once per call.
//   B >  8  : per-layer 64x64 register-tiled f64 GEMM with the BN/ReLU or
//             sigmoid epilogue fused, then a top-k kernel — the batched
//             evaluate / PrecomputedPredictor path.
#include "ds_common.cuh"

#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace ds {
namespace {

constexpr double kBnEps = 1e-5;
constexpr int kFusedMaxB = 8;
constexpr int kFusedThreads = 256;

struct LayerPtrs {
    int in, out, ld;  // ld = padded row stride of Wt (even)
    size_t w, b, mu, istd, gamma, beta;  // offsets in doubles (mu.. only hidden)
};

struct MlpPlan {
    int n_layers;
    LayerPtrs layer[DS_MAX_HIDDEN + 1];
    size_t packed;
    size_t container;
    int max_width;
};

bool make_plan(const ds_mlp_desc* d, MlpPlan* p) {
    if (!d || d->n_hidden < 0 || d->n_hidden > DS_MAX_HIDDEN || d->input_dim < 1 ||
        d->output_dim < 1 || d->output_dim > DS_MAX_EXPERTS)
        return false;
    int dims[DS_MAX_HIDDEN + 2];
    dims[0] = d->input_dim;
    for (int i = 0; i < d->n_hidden; ++i) {
        if (d->hidden[i] < 1) return false;
        dims[i + 1] = d->hidden[i];
    }
    dims[d->n_hidden + 1] = d->output_dim;
    p->n_layers = d->n_hidden + 1;
    size_t off = 0, cont = 0;
    p->max_width = 0;
    for (int i = 0; i < p->n_layers; ++i) {
        LayerPtrs& L = p->layer[i];
        L.in = dims[i];
        L.out = dims[i + 1];
        L.ld = (L.in + 1) & ~1;
        L.w = off;  off += (size_t)L.out * L.ld;
        L.b = off;  off += L.out;
        if (i < d->n_hidden) {
            L.mu = off;    off += L.out;
            L.istd = off;  off += L.out;
            L.gamma = off; off += L.out;
            L.beta = off;  off += L.out;
        } else {
            L.mu = L.istd = L.gamma = L.beta = 0;
        }
        off = (off + 1) & ~size_t(1);
        cont += (size_t)L.in * L.out + L.out;
        if (L.in > p->max_width) p->max_width = L.in;
        if (L.out > p->max_width) p->max_width = L.out;
    }
    for (int i = 0; i < d->n_hidden; ++i) cont += 4 * (size_t)dims[i + 1];
    p->packed = off;
    p->container = cont;
    return true;
}

// ---------------------------------------------------------------- packing
__global__ void transpose_kernel(const double* __restrict__ W, int in, int out, int ld,
                                 double* __restrict__ Wt) {
    __shared__ double tile[32][33];
    int a0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int a = a0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (a < in && j < out) ? W[(size_t)a * out + j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int j = j0 + r, a = a0 + threadIdx.x;
        if (j < out && a < ld) Wt[(size_t)j * ld + a] = (a < in) ? tile[threadIdx.x][r] : 0.0;
    }
}

// bias copy + BN folding: istd = 1/sqrt(var + eps) exactly as numpy does it
// (np.sqrt and the division are correctly rounded in both).
__global__ void pack_vectors_kernel(const double* __restrict__ b, const double* __restrict__ gamma,
                                    const double* __restrict__ beta, const double* __restrict__ mean,
                                    const double* __restrict__ var, int out, int hidden,
                                    double* __restrict__ pb, double* __restrict__ pmu,
                                    double* __restrict__ pistd, double* __restrict__ pgamma,
                                    double* __restrict__ pbeta) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= out) return;
    pb[j] = b[j];
    if (hidden) {
        pmu[j] = mean[j];
        pistd[j] = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var[j], kBnEps)));
        pgamma[j] = gamma[j];
        pbeta[j] = beta[j];
    }
}

// ------------------------------------------------------------- epilogues
__device__ __forceinline__ double sigmoid_ref(double z) {
    if (z >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-z)));
    double ez = exp(z);
    return __ddiv_rn(ez, __dadd_rn(1.0, ez));
}

__device__ __forceinline__ double hidden_epilogue(double dot, const double* P, const LayerPtrs& L,
                                                  int j) {
    double z = __dadd_rn(dot, P[L.b + j]);
    double zhat = __dmul_rn(__dsub_rn(z, P[L.mu + j]), P[L.istd + j]);
    double h = __dadd_rn(__dmul_rn(P[L.gamma + j], zhat), P[L.beta + j]);
    return h > 0.0 ? h : 0.0;
}

// k largest with ties to the lower index, emitted ascending (predictor.py:419-421)
__device__ void topk_row(const double* p, int M, int k, int32_t* out) {
    uint64_t taken = 0;
    int sel[DS_MAX_EXPERTS];
    for (int r = 0; r < k; ++r) {
        int best = -1;
        double bv = 0.0;
        for (int i = 0; i < M; ++i) {
            if (taken >> i & 1ull) continue;
            if (best < 0 || p[i] > bv) { best = i; bv = p[i]; }
        }
        taken |= 1ull << best;
        sel[r] = best;
    }
    int w = 0;
    for (int i = 0; i < M && w < k; ++i)
        if (taken >> i & 1ull) out[w++] = i;
    (void)sel;
}

// -------------------------------------------------------- feature builder
struct StateArgs {
    const int32_t* hist;
    const int32_t* target;
    const double* pop;
    const double* aff;
    int L, M, k, mode, d_in;
};

__device__ double feature_value(const StateArgs& s, int b, int f) {
    const int l = s.target[b];
    const int Lk = s.L * s.k;
    const int32_t* h = s.hist + (size_t)b * Lk;
    if (f < Lk) {
        int v = (f < l * s.k) ? h[f] : 0;
        return __ddiv_rn((double)v, (double)s.M);
    }
    f -= Lk;
    if (f < s.M) return s.pop[(size_t)l * s.M + f];
    f -= s.M;
    const double* A = s.aff + (size_t)(l - 1) * s.M * s.M;
    const int32_t* prev = h + (l - 1) * s.k;
    if (s.mode == 0) {
        if (f < s.M) {
            double acc = A[(size_t)(prev[0] - 1) * s.M + f];
            for (int j = 1; j < s.k; ++j) acc = __dadd_rn(acc, A[(size_t)(prev[j] - 1) * s.M + f]);
            return __ddiv_rn(acc, (double)s.k);
        }
        f -= s.M;
    } else {
        if (f < s.k * s.M) return A[(size_t)(prev[f / s.M] - 1) * s.M + (f % s.M)];
        f -= s.k * s.M;
    }
    return __ddiv_rn((double)l, (double)(s.L - 1));
}

__global__ void features_kernel(StateArgs s, int B, double* __restrict__ X) {
    size_t n = (size_t)B * s.d_in;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        int b = (int)(i / s.d_in), f = (int)(i % s.d_in);
        X[i] = feature_value(s, b, f);
    }
}

// -------------------------------------------------------- fused (B <= 8)
struct FusedArgs {
    unsigned long long* dbg;   // optional per-layer globaltimer stamps (DS_K5_TIMELINE), CTA 0
    MlpPlan plan;
    const double* P;
    StateArgs s;
    const double* X;  // raw features (non-null => skip the State Constructor)
    int B, topk;
    double* act0;
    double* act1;
    unsigned* barrier;
    int32_t* topk_out;
    double* probs_out;
};

// Grid barrier: the CTA's writes are ordered before the arrival by the
// __syncthreads + a gpu-scope RELEASE add (no full __threadfence, which also
// invalidates L1), and the spin is an ACQUIRE load; the next layer reads the
// activations with ld.global.cg (L2), so nothing stale is served from L1.
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// BMAX: compile-time bound on the batch (1 for the decode path: no predicated
// dead lanes of the batch loop in the streaming inner product)
template <int BMAX>
__global__ void __launch_bounds__(kFusedThreads, 1) mlp_fused_kernel(FusedArgs a) {
    extern __shared__ __align__(16) double smem[];  // [B][max_width]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps_cta = blockDim.x >> 5;
    const int gwarp = blockIdx.x * nwarps_cta + warp;
    const int nwarps = gridDim.x * nwarps_cta;
    const int B = a.B;
    unsigned phase = 0;

    // State Constructor: every CTA builds the (tiny: B x d_in, 81 for 8x7B)
    // feature rows straight into its shared-memory A stage, so no grid
    // barrier (and no global round trip) precedes the first layer
    const bool fused_features = (a.X == nullptr);
    const double* in_act = a.X;
    double* out_act = a.act1;

    auto stamp = [&](int slot) {
        if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.dbg[slot] = t;
        }
    };
    stamp(0);
    for (int li = 0; li < a.plan.n_layers; ++li) {
        const LayerPtrs& L = a.plan.layer[li];
        const bool last = (li == a.plan.n_layers - 1);
        if (last && blockIdx.x != 0) break;  // output layer: CTA 0 alone
        stamp(1 + 3 * li);
        // stage A (B x in) in shared memory, L2-coherent loads
        if (li == 0 && fused_features) {
            for (int i = threadIdx.x; i < B * L.in; i += blockDim.x) {
                int b = i / L.in, c = i % L.in;
                smem[b * L.ld + c] = feature_value(a.s, b, c);
            }
        } else {
            // batched: 8 independent L2 loads per thread in flight, then the stores
            constexpr int SU = 8;
            for (int i0 = threadIdx.x; i0 < B * L.in; i0 += blockDim.x * SU) {
                double v[SU];
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < B * L.in) v[u] = __ldcg(in_act + i);   // [B][in] rows are contiguous
                }
#pragma unroll
                for (int u = 0; u < SU; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < B * L.in) {
                        const int b = i / L.in, c = i - b * L.in;
                        smem[b * L.ld + c] = v[u];
                    }
                }
            }
        }
        if (L.in & 1)
            for (int b = threadIdx.x; b < B; b += blockDim.x) smem[b * L.ld + L.in] = 0.0;
        __syncthreads();
        stamp(2 + 3 * li);
        const double* W = a.P + L.w;
        const int wstart = last ? warp : gwarp;
        const int wstride = last ? nwarps_cta : nwarps;
        for (int j = wstart; j < L.out; j += wstride) {
            double acc[BMAX];
#pragma unroll
            for (int b = 0; b < BMAX; ++b) acc[b] = 0.0;
            const double2* wrow = reinterpret_cast<const double2*>(W + (size_t)j * L.ld);
            const int n2 = L.ld >> 1;                   // double2 per row (ld is even)
            // batches of U independent 16-byte loads per lane issued before any
            // math (a runtime trip count otherwise leaves one load in flight);
            // each lane still accumulates its elements in increasing c
            constexpr int U = 8;
            for (int c0 = lane; c0 < n2; c0 += 32 * U) {
                double2 w2[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (c0 + 32 * u < n2) w2[u] = __ldg(wrow + c0 + 32 * u);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (c0 + 32 * u < n2) {
                        const int c = 2 * (c0 + 32 * u);
#pragma unroll
                        for (int b = 0; b < BMAX; ++b) {
                            if (b < B) {
                                double2 x2 = *reinterpret_cast<const double2*>(smem + b * L.ld + c);
                                acc[b] = fma(w2[u].x, x2.x, acc[b]);
                                acc[b] = fma(w2[u].y, x2.y, acc[b]);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < BMAX; ++b) {
                if (b < B) {
                    double v = acc[b];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    acc[b] = v;
                }
            }
            if (lane < B) {
                double dot = 0.0;
#pragma unroll
                for (int b = 0; b < BMAX; ++b)
                    if (b == lane) dot = acc[b];
                double r;
                if (!last) {
                    r = hidden_epilogue(dot, a.P, L, j);
                    out_act[(size_t)lane * L.out + j] = r;
                } else {
                    r = sigmoid_ref(__dadd_rn(dot, a.P[L.b + j]));
                    out_act[(size_t)lane * L.out + j] = r;
                }
            }
        }
        stamp(3 + 3 * li);
        if (!last) {
            grid_barrier(a.barrier, ++phase * gridDim.x);
            in_act = out_act;
            out_act = (out_act == a.act1) ? a.act0 : a.act1;
        } else {
            __syncthreads();
            __threadfence_block();
            const int M = L.out;
            for (int b = threadIdx.x; b < B; b += blockDim.x) {
                const double* p = out_act + (size_t)b * M;
                double row[DS_MAX_EXPERTS];
                for (int i = 0; i < M; ++i) row[i] = __ldcg(p + i);
                if (a.probs_out)
                    for (int i = 0; i < M; ++i) a.probs_out[(size_t)b * M + i] = row[i];
                if (a.topk > 0) topk_row(row, M, a.topk, a.topk_out + (size_t)b * a.topk);
            }
        }
    }
}

// ------------------------------------------------------ tiled (B > 8)
constexpr int TB = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) mlp_layer_tiled_kernel(const double* __restrict__ A, int B,
                                                              const double* __restrict__ P,
                                                              LayerPtrs L, int last,
                                                              double* __restrict__ C) {
    __shared__ double As[TK][TB + 1];
    __shared__ double Ws[TK][TN + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.x * TB, n0 = blockIdx.y * TN;
    const double* W = P + L.w;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < L.in; k0 += TK) {
        for (int i = threadIdx.x; i < TB * TK; i += 256) {
            int r = i / TK, kk = i % TK;
            int m = m0 + r, k = k0 + kk;
            As[kk][r] = (m < B && k < L.in) ? A[(size_t)m * L.in + k] : 0.0;
            int n = n0 + r;
            Ws[kk][r] = (n < L.out && k < L.in) ? W[(size_t)n * L.ld + k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            double av[4], wv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) wv[j] = Ws[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], wv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int m = m0 + ty + 16 * i;
        if (m >= B) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int n = n0 + tx + 16 * j;
            if (n >= L.out) continue;
            double r = last ? sigmoid_ref(__dadd_rn(acc[i][j], P[L.b + n]))
                            : hidden_epilogue(acc[i][j], P, L, n);
            C[(size_t)m * L.out + n] = r;
        }
    }
}

__global__ void topk_kernel(const double* __restrict__ probs, int B, int M, int k,
                            int32_t* __restrict__ out, double* __restrict__ probs_out) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double row[DS_MAX_EXPERTS];
    for (int i = 0; i < M; ++i) row[i] = probs[(size_t)b * M + i];
    if (probs_out)
        for (int i = 0; i < M; ++i) probs_out[(size_t)b * M + i] = row[i];
    if (k > 0) topk_row(row, M, k, out + (size_t)b * k);
}

int run_forward(const ds_mlp_desc* d, const double* packed, const StateArgs* s, const double* X,
                int B, int topk, int32_t* topk_out, double* probs_out, void* ws, size_t ws_bytes,
                cudaStream_t st) {
    MlpPlan plan;
    DS_CHECK_ARG(make_plan(d, &plan), "ds_predictor: invalid mlp descriptor");
    DS_CHECK_ARG(packed != nullptr, "ds_predictor: packed weights are NULL");
    DS_CHECK_ARG(B >= 0, "ds_predictor: B must be >= 0");
    DS_CHECK_ARG(topk >= 0 && topk <= d->output_dim, "ds_predictor: topk must be in [0, M]");
    DS_CHECK_ARG(topk == 0 || topk_out != nullptr, "ds_predictor: topk_out is NULL");
    if (B == 0) return DS_OK;
    size_t need = ds_mlp_workspace_bytes(d, B);
    if (ws_bytes < need || ws == nullptr)
        return fail(DS_ERR_WORKSPACE, "ds_predictor: workspace %zu < %zu bytes", ws_bytes, need);
    char* base = static_cast<char*>(ws);
    unsigned* barrier = reinterpret_cast<unsigned*>(base);
    double* act0 = reinterpret_cast<double*>(base + 256);
    double* act1 = act0 + (size_t)B * plan.max_width;

    if (B <= kFusedMaxB) {
        FusedArgs a;
        static unsigned long long* dbg = nullptr;
        static const bool want_dbg = getenv("DS_K5_TIMELINE") != nullptr;
        if (want_dbg && !dbg) cudaMalloc(&dbg, 64 * sizeof(unsigned long long));
        a.dbg = want_dbg ? dbg : nullptr;
        a.plan = plan;
        a.P = packed;
        if (s) a.s = *s; else memset(&a.s, 0, sizeof(a.s));
        a.X = X;
        a.B = B;
        a.topk = topk;
        a.act0 = act0;
        a.act1 = act1;
        a.barrier = barrier;
        a.topk_out = topk_out;
        a.probs_out = probs_out;
        int max_ld = 0;
        for (int i = 0; i < plan.n_layers; ++i) max_ld = plan.layer[i].ld > max_ld ? plan.layer[i].ld : max_ld;
        size_t smem = (size_t)B * max_ld * sizeof(double);
        const void* fn = B == 1 ? (const void*)mlp_fused_kernel<1> : (const void*)mlp_fused_kernel<kFusedMaxB>;
        if (first_use_on_device((const void*)mlp_fused_kernel<1>)) {
            cudaFuncSetAttribute(mlp_fused_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaFuncSetAttribute(mlp_fused_kernel<kFusedMaxB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024);
        }
        if (smem > 200 * 1024) return fail(DS_ERR_UNSUPPORTED, "ds_predictor: layer too wide");
        // CTAs of the persistent kernel (one per SM by default); DS_K5_CTAS caps it
        // (A/B: fewer SMs leave room for the decode GEMV it overlaps with)
        static const int cap = getenv("DS_K5_CTAS") ? atoi(getenv("DS_K5_CTAS")) : 0;
        int grid = num_sms();
        if (cap > 0 && cap < grid) grid = cap;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFusedThreads, smem);
        if (per_sm < 1) return fail(DS_ERR_UNSUPPORTED, "ds_predictor: fused kernel cannot be resident");
        cudaError_t e = cudaMemsetAsync(barrier, 0, sizeof(unsigned), st);
        if (e != cudaSuccess) return cuda_status(e, "ds_predictor: memset");
        void* args[] = {&a};
        e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kFusedThreads), args, smem, st);
        if (want_dbg && e == cudaSuccess) {                  // diagnostics only: per-layer stamps (ns)
            unsigned long long h[64];
            cudaStreamSynchronize(st);
            cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
            fprintf(stderr, "K5 timeline (us from start):");
            for (int i = 1; i <= 3 * plan.n_layers; ++i) fprintf(stderr, " %.2f", (h[i] - h[0]) / 1e3);
            fprintf(stderr, "\n");
        }
        return cuda_status(e, "ds_predictor: fused launch");
    }

    const double* cur = X;
    if (!X) {
        int blocks = (int)(((size_t)B * plan.layer[0].in + 255) / 256);
        if (blocks > 4096) blocks = 4096;
        features_kernel<<<blocks, 256, 0, st>>>(*s, B, act0);
        DS_LAUNCH_CHECK("ds_predictor: features");
        cur = act0;
    }
    double* out = act1;
    for (int li = 0; li < plan.n_layers; ++li) {
        const LayerPtrs& L = plan.layer[li];
        dim3 grid((B + TB - 1) / TB, (L.out + TN - 1) / TN);
        mlp_layer_tiled_kernel<<<grid, 256, 0, st>>>(cur, B, packed, L, li == plan.n_layers - 1, out);
        DS_LAUNCH_CHECK("ds_predictor: tiled layer");
        cur = out;
        out = (out == act1) ? act0 : act1;
    }
    topk_kernel<<<(B + 127) / 128, 128, 0, st>>>(cur, B, d->output_dim, topk, topk_out, probs_out);
    DS_LAUNCH_CHECK("ds_predictor: topk");
    return DS_OK;
}

}  // namespace
}  // namespace ds

using namespace ds;

extern "C" size_t ds_mlp_container_doubles(const ds_mlp_desc* d) {
    MlpPlan p;
    return make_plan(d, &p) ? p.container : 0;
}

extern "C" size_t ds_mlp_packed_doubles(const ds_mlp_desc* d) {
    MlpPlan p;
    return make_plan(d, &p) ? p.packed : 0;
}

extern "C" size_t ds_mlp_workspace_bytes(const ds_mlp_desc* d, int B) {
    MlpPlan p;
    if (!make_plan(d, &p) || B < 0) return 0;
    int w = p.max_width > d->input_dim ? p.max_width : d->input_dim;
    return 256 + 2 * (size_t)(B > 0 ? B : 1) * w * sizeof(double);
}

extern "C" int ds_mlp_pack(const ds_mlp_desc* d, const double* container, double* packed,
                           void* stream) {
    MlpPlan p;
    DS_CHECK_ARG(make_plan(d, &p), "ds_mlp_pack: invalid mlp descriptor");
    DS_CHECK_ARG(container && packed, "ds_mlp_pack: NULL pointer");
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(packed, 0, p.packed * sizeof(double), st);
    if (e != cudaSuccess) return cuda_status(e, "ds_mlp_pack: memset");
    // container offsets: W_i, b_i for all layers, then per hidden gamma,beta,mean,var
    size_t off = 0;
    std::vector<size_t> woff(p.n_layers), boff(p.n_layers);
    for (int i = 0; i < p.n_layers; ++i) {
        woff[i] = off; off += (size_t)p.layer[i].in * p.layer[i].out;
        boff[i] = off; off += p.layer[i].out;
    }
    for (int i = 0; i < p.n_layers; ++i) {
        const LayerPtrs& L = p.layer[i];
        dim3 tg((L.out + 31) / 32, (L.ld + 31) / 32);
        transpose_kernel<<<tg, dim3(32, 8), 0, st>>>(container + woff[i], L.in, L.out, L.ld, packed + L.w);
        DS_LAUNCH_CHECK("ds_mlp_pack: transpose");
        const bool hidden = i < d->n_hidden;
        const double *g = nullptr, *be = nullptr, *mu = nullptr, *var = nullptr;
        if (hidden) {
            g = container + off; off += L.out;
            be = container + off; off += L.out;
            mu = container + off; off += L.out;
            var = container + off; off += L.out;
        }
        pack_vectors_kernel<<<(L.out + 255) / 256, 256, 0, st>>>(
            container + boff[i], g, be, mu, var, L.out, hidden, packed + L.b,
            hidden ? packed + L.mu : nullptr, hidden ? packed + L.istd : nullptr,
            hidden ? packed + L.gamma : nullptr, hidden ? packed + L.beta : nullptr);
        DS_LAUNCH_CHECK("ds_mlp_pack: vectors");
    }
    return DS_OK;
}

extern "C" int ds_predictor_forward(const ds_mlp_desc* d, const double* packed, const int32_t* hist,
                                    const int32_t* target_layer, const double* pop, const double* aff,
                                    int L, int M, int k, int affinity_mode, int B, int topk,
                                    int32_t* topk_out, double* probs_out, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    DS_CHECK_ARG(d != nullptr, "ds_predictor_forward: NULL descriptor");
    DS_CHECK_ARG(L >= 2 && M >= 2 && M <= DS_MAX_EXPERTS && k >= 1 && k < M,
                 "ds_predictor_forward: bad shape L=%d M=%d k=%d", L, M, k);
    DS_CHECK_ARG(affinity_mode == 0 || affinity_mode == 1, "ds_predictor_forward: affinity_mode");
    int want = L * k + M + (affinity_mode == 0 ? M : k * M) + 1;
    DS_CHECK_ARG(d->input_dim == want,
                 "ds_predictor_forward: input_dim %d != feature length %d", d->input_dim, want);
    DS_CHECK_ARG(d->output_dim == M, "ds_predictor_forward: output_dim %d != M %d", d->output_dim, M);
    DS_CHECK_ARG(B == 0 || (hist && target_layer && pop && aff), "ds_predictor_forward: NULL input");
    StateArgs s{hist, target_layer, pop, aff, L, M, k, affinity_mode, want};
    return run_forward(d, packed, &s, nullptr, B, topk, topk_out, probs_out, workspace,
                       workspace_bytes, as_stream(stream));
}

extern "C" int ds_mlp_forward_features(const ds_mlp_desc* d, const double* packed, const double* X,
                                       int B, int topk, int32_t* topk_out, double* probs_out,
                                       void* workspace, size_t workspace_bytes, void* stream) {
    DS_CHECK_ARG(d != nullptr, "ds_mlp_forward_features: NULL descriptor");
    DS_CHECK_ARG(B == 0 || X != nullptr, "ds_mlp_forward_features: NULL X");
    return run_forward(d, packed, nullptr, X, B, topk, topk_out, probs_out, workspace,
                       workspace_bytes, as_stream(stream));
}
