/*
 * duoserve_b200.h — C-ABI of libduoserve_sm100.so, the B200 (sm_100a) hot path
 * of DuoServe-MoE (arXiv 2509.07379).
 *
 * The reference (/root/reference/pkg/src/duoserve) is pure Python/NumPy and
 * has no FFI; its plug-in surface is duck-typed Python.  Each entry point
 * below names the reference function (file:line) whose computation it
 * replaces; INTEGRATION.md shows the ctypes binding the reference-side
 * maintainer would add.  The Python package paper_2509_07379_b200 is that
 * binding plus the host mirror of the reference API.
 *
 * Conventions (every function):
 *   - plain pointers and sizes only; device pointers are caller-owned
 *     (allocated by the caller, e.g. as torch tensors), "stream" is a
 *     cudaStream_t passed as void*; no entry point allocates device memory
 *     (the diagnostic DS_K4_TIMELINE switch excepted; the driver-managed
 *     executables of ds_w4_expert_gemv_graph's graph cache are released by
 *     ds_w4_graph_cache_clear);
 *   - return 0 on success, a positive cudaError_t on a CUDA failure, or a
 *     negative DS_ERR_* on invalid arguments; ds_last_error() returns the
 *     calling thread's last message;
 *   - asynchronous with respect to the host unless stated otherwise;
 *   - no CPU fallback: without a usable sm_100 device every compute entry
 *     point fails with a CUDA error.
 */
#ifndef DUOSERVE_B200_H
#define DUOSERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define DS_ABI_VERSION 1

#define DS_OK 0
#define DS_ERR_ARG (-1)        /* invalid argument / shape                  */
#define DS_ERR_UNSUPPORTED (-2)/* shape outside the kernels' supported range */
#define DS_ERR_WORKSPACE (-3)  /* workspace too small                       */
#define DS_ERR_STATE (-4)      /* object in the wrong state                 */

#define DS_MAX_HIDDEN 8        /* ExpertMLP hidden layers (reference: 6)    */
#define DS_MAX_EXPERTS 64

int ds_abi_version(void);
const char *ds_last_error(void);
/* Number of SMs of the current device and whether it is sm_100 (1/0).  */
int ds_device_info(int *num_sms, int *is_sm100);

/* ========================================================================
 * K5 — fused State Constructor + ExpertMLP (eval) + top-k, float64.
 * Replaces: construct_input + StateVector.as_features (predictor.py:53-106),
 *           ExpertMLP.forward(train=False) / _forward_full (predictor.py:191-232),
 *           _sigmoid (predictor.py:132-138), topk_indices (predictor.py:419-421);
 *           i.e. MLPPredictor.predict (predictor.py:435-438) for B=1 and
 *           PrecomputedPredictor.from_net (predictor.py:492-507) batched.
 * ===================================================================== */
typedef struct {
    int input_dim;             /* L*k + M + (M | k*M) + 1                    */
    int output_dim;            /* M                                          */
    int n_hidden;              /* <= DS_MAX_HIDDEN                           */
    int hidden[DS_MAX_HIDDEN]; /* widths, e.g. 2048,1024,512,256,128,64      */
} ds_mlp_desc;

/* doubles in the reference container's data section (predictor.py:577-587):
 * W0,b0,...,W_n,b_n then gamma_i,beta_i,run_mean_i,run_var_i per hidden i. */
size_t ds_mlp_container_doubles(const ds_mlp_desc *d);
/* doubles of the packed device layout (W transposed to [out,in], BN folded
 * into (mu, 1/sqrt(var+eps), gamma, beta)).                                */
size_t ds_mlp_packed_doubles(const ds_mlp_desc *d);
/* container (device copy of the raw <f8 data) -> packed (device).          */
int ds_mlp_pack(const ds_mlp_desc *d, const double *container, double *packed, void *stream);
size_t ds_mlp_workspace_bytes(const ds_mlp_desc *d, int B);

/* State-Constructor path: row b predicts layer target_layer[b] in [1, L).
 *   hist   [B, L*k] int32: expert index + 1 of layers < target (sorted per
 *          layer, as the gate emits), anything at positions >= target*k is
 *          ignored (masked in-kernel, matching the reference's zero pad);
 *   pop    [L, M] f64; aff [L-1, M, M] f64 (device tables);
 *   affinity_mode 0 = pool (mean of the k rows), 1 = concat.
 * Outputs: topk_out [B, topk] int32 ascending; probs_out [B, M] or NULL.   */
int ds_predictor_forward(const ds_mlp_desc *d, const double *packed, const int32_t *hist,
                         const int32_t *target_layer, const double *pop, const double *aff,
                         int L, int M, int k, int affinity_mode, int B, int topk,
                         int32_t *topk_out, double *probs_out, void *workspace,
                         size_t workspace_bytes, void *stream);
/* Raw-features path (ExpertMLP.forward on given X [B, input_dim]).  topk may
 * be 0 (no top-k output).                                                  */
int ds_mlp_forward_features(const ds_mlp_desc *d, const double *packed, const double *X, int B,
                            int topk, int32_t *topk_out, double *probs_out, void *workspace,
                            size_t workspace_bytes, void *stream);

/* ========================================================================
 * K1 / K2 / K7 — routing.  The reference has no gate (its routing is
 * sampled, trace.py:178-242); semantics follow HF MixtralTopKRouter
 * (transformers 5.5.0 modeling_mixtral.py:109-116) with the reference's
 * top-k tie rule (predictor.py:419-421) and a fixed float64 accumulation
 * order that oracle/ reproduces bit-for-bit.
 * ===================================================================== */
/* x [T, d] bf16, wg [M, d] bf16.  Outputs: idx [T, k] int32 ascending,
 * w [T, k] f32 (renormalised softmax of the selected logits), logits [T, M]
 * f64 (or NULL), counts [M] int32 (+= selections; caller zeroes), and,
 * when hist != NULL, hist[t*hist_stride + layer*k + j] = idx+1 (the State
 * Constructor history, predictor.py:96-98, written on device).            */
int ds_gate_topk(const void *x, const void *wg, int T, int d, int M, int k, int32_t *idx,
                 float *w, double *logits, int32_t *counts, int32_t *hist, int hist_stride,
                 int layer, void *stream);
/* Group the T*k (token, slot) pairs by expert, stable in token order
 * ("groups the tokens by their assigned experts").
 * Outputs: offsets [M+1], pos [T*k] (row of pair (t,j) in the grouped
 * buffer), src_token [T*k] (token of each grouped row); when xperm != NULL
 * also gathers rows: xperm[pos[t*k+j]] = x[t] (bf16 [T*k, d]).            */
int ds_permute(const int32_t *idx, const void *x, int T, int d, int M, int k, int32_t *offsets,
               int32_t *pos, int32_t *src_token, void *xperm, void *stream);
/* out[t] = bf16( resid[t] + sum_j w[t,j] * y[pos[t*k+j]] ), sum in f32 in j
 * order ("unpacks the results").  y is f32 [T*k, d].        */
int ds_unpermute_combine(const float *y, const int32_t *pos, const float *w, const void *resid,
                         int T, int d, int k, void *out, void *stream);
/* Expert-parallel combine term: out[t] (f32) = sum_j [owned_mask bit idx[t,j]]
 * w[t,j] * y[pos[t*k+j]]; all-reduced across ranks then finalised with
 * ds_combine_finalize (bit-identical to ds_unpermute_combine for k = 2).     */
int ds_unpermute_partial(const float *y, const int32_t *pos, const float *w, const int32_t *idx,
                         uint64_t owned_mask, int T, int d, int k, float *out, void *stream);
/* K7: per token, hits/misses of gate set vs the resident prediction
 * (SPEC.md:386 sync point 1).  pred, idx [T,k]; miss_mask [T] bit j set
 * when idx[t,j] not in pred[t,:].                                          */
int ds_cache_check(const int32_t *idx, const int32_t *pred, int T, int k, int32_t *miss_mask,
                   void *stream);
/* Online statistics (stats.py:52-71 counts): pop_counts [L,M] += 1 per
 * selection, aff_counts [L-1,M,M] += 1 per (i at l, j at l+1); paths
 * [N, L, k] int32.  Integer, order-independent => bit-exact.              */
int ds_route_histogram(const int32_t *paths, int N, int L, int M, int k, int64_t *pop_counts,
                       int64_t *aff_counts, void *stream);

/* ========================================================================
 * K3 / K4 — W4 (AWQ-style, group G) SwiGLU expert FFN.
 * No reference code (PAPER.md:188,192 uses vLLM AWQ ops); dequant is
 * w = bf16_rn((q - z) * s).  Device format per linear with
 * input K, output N:  codes u32 [N, K/8] (nibble j of word w holds
 * k = 8w + {0,2,4,6,1,3,5,7}[j]), scales bf16 [N, K/G], zeros u4 [N*K/G]
 * (nibble n*K/G+g, low nibble first).
 * ===================================================================== */
typedef struct {
    const uint32_t *codes;
    const void *scales;        /* bf16 */
    const uint8_t *zeros;
} ds_w4_linear;

typedef struct {
    ds_w4_linear w1;           /* gate proj, K=d,  N=ff */
    ds_w4_linear w3;           /* up proj,   K=d,  N=ff */
    ds_w4_linear w2;           /* down proj, K=ff, N=d  */
} ds_w4_expert;

/* Byte offsets of the sections of one expert blob (the unit of H2D copy);
 * offsets[9] = {c1,c3,c2,s1,s3,s2,z1,z3,z2}; returns total bytes.          */
size_t ds_w4_expert_layout(int d, int ff, int G, size_t offsets[9]);
/* Counter-based random init of expert (layer, expert) into a device blob:
 * codes, zeros ~ U{0..15}; scales = bf16_rn((0.5+u)/(8 sqrt(K))).
 * oracle/w4_ref.py regenerates identical bytes on the CPU.                 */
int ds_w4_generate(uint64_t seed, int layer, int expert, int d, int ff, int G, void *blob,
                   void *stream);
/* Dequantise one linear to bf16 [N, K] (test/inspection path).            */
int ds_w4_dequant(const ds_w4_linear *w, int K, int N, int G, void *out, void *stream);
/* Decode GEMV (K4), rows R <= 16: h = bf16( silu(x W1) * (x W3) ) [R, ff];
 * then acc[R, d] (f32) += route_w[r] * (h W2).                             */
int ds_w4_swiglu_gemv(const void *x, int R, const ds_w4_expert *e, int d, int ff, int G, void *h,
                      void *stream);
int ds_w4_down_gemv(const void *h, int R, const ds_w4_expert *e, int d, int ff, int G,
                    const float *route_w, int route_stride, float *acc, void *stream);
/* One expert's decode FFN in one call: ds_w4_swiglu_gemv then
 * ds_w4_down_gemv (the down GEMV launched as a programmatic dependent of the
 * SwiGLU GEMV).  ev_start / ev_end (cudaEvent_t, may be NULL) are recorded on
 * `stream` immediately around the two launches: the kernel-time span a
 * profiler reads without host latency in it.                              */
int ds_w4_expert_gemv(const void *x, int R, const ds_w4_expert *e, int d, int ff, int G, void *h,
                      const float *route_w, int route_stride, float *acc, void *ev_start, void *ev_end,
                      void *stream);
/* The same expert FFN as ONE launch of a cached, device-uploaded CUDA graph:
 * [stream waits wait_event (the slot's ready event; may be NULL)] ->
 * ev_start -> K4 -> ev_end.  While the copy engine streams experts, commands
 * submitted from the host reach the GPU ~25-30 us late (the front end fetches
 * them over the busy host link); inside an uploaded graph the wait, the span
 * events and the launches run from device memory.  Graphs are keyed by every
 * argument except the three events (swapped per launch); R <= 16.
 * Replaces the per-expert FFN call of the reference's decode loop
 * ("vLLM AWQ operators"; SPEC.md:383-391 decode compute).     */
int ds_w4_expert_gemv_graph(const void *x, int R, const ds_w4_expert *e, int d, int ff, int G, void *h,
                            const float *route_w, int route_stride, float *acc, void *wait_event,
                            void *ev_start, void *ev_end, void *stream);
/* Destroy every cached K4 graph (their static buffers are being freed).    */
int ds_w4_graph_cache_clear(void);
/* Device-clock (%globaltimer) totals of every fused K4 launch so far: the sum
 * of first-CTA-entry -> last-CTA-exit in ns and the launch count (synchronous
 * read; the profiler's in-loop kernel duration beside its CUDA-event spans). */
int ds_k4_device_span(unsigned long long *ns, unsigned long long *n);
/* The same for K3: every grouped FFN call given span events (GEMM1's first
 * CTA entry -> a one-thread kernel queued right after the call's last one). */
int ds_k3_device_span(unsigned long long *ns, unsigned long long *n);
/* ------------------------------------------------------------------------
 * Decode front of one token (the non-MoE steps between two MoE layers; no
 * reference counterpart — the reference has no forward pass — but they sit
 * in the decode window before sync point 1).  bf16 in / out,
 * f32 math.
 * -------------------------------------------------------------------- */
/* out[R, d] = bf16( (f32(x) * rsqrt(mean(x^2) + eps)) * f32(gamma) )        */
int ds_rmsnorm(const void *x, int R, int d, const void *gamma, float eps, void *out, void *stream);
/* h1 = bf16( f32(h) + y ) (y f32, the o projection); a = rmsnorm(h1, gamma) */
int ds_residual_rmsnorm(const void *h, const float *y, int R, int d, const void *gamma, float eps, void *h1,
                        void *a, void *stream);
/* One token's f32 q|k|v row y[(nh + 2 nkv) * hd] -> bf16 -> RoPE(q, k) with
 * the cos / sin tables [max_seq, hd] (f32) at the device-resident position
 * *pos; q[nh, hd] out; k, v written into the layer's cache [nkv, max_seq, hd]. */
int ds_rope_kv_decode(const float *y, int nh, int nkv, int hd, const float *cos_t, const float *sin_t,
                      const long long *pos, int max_seq, void *q, void *k_cache, void *v_cache, void *stream);
/* ------------------------------------------------------------------------
 * Plain W4 linears: the non-MoE projections (attention q|k|v and o) kept
 * resident in HBM in the same W4 format, so the non-MoE weights fit the
 * paper's W4 model budget ("2.15 GB"; SPEC.md:392-398 peak
 * memory).  One blob per linear: codes | scales | zeros, each 256-B aligned.
 * -------------------------------------------------------------------- */
size_t ds_w4_linear_layout(int K, int N, int G, size_t offsets[3]);
/* Counter-based init of one linear (tag < 64 names the matrix family; the
 * experts use tags 0..M-1 via ds_w4_generate).                            */
int ds_w4_generate_linear(uint64_t seed, int layer, int tag, int matrix, int K, int N, int G, void *blob,
                          void *stream);
/* y[R, N] (f32, overwritten) = x[R, K] (bf16) W^T for R <= 64 rows: the K4
 * decode GEMV with routing weight 1 (exact (q - z) s products).           */
int ds_w4_linear_gemv(const void *x, int R, const ds_w4_linear *w, int K, int N, int G, float *y,
                      void *stream);
/* Same for many rows on the tcgen05 GEMM (K3's down-projection kernel,
 * bf16_rn((q - z) s) weights); workspace for the split-K partials.        */
size_t ds_w4_linear_workspace(int rows, int K, int N);
int ds_w4_linear_gemm(const void *x, int rows, const ds_w4_linear *w, int K, int N, int G, float *y,
                      void *workspace, size_t workspace_bytes, void *stream);
/* out[r] = bf16(resid[r] + acc[r]) and acc zeroed for the next layer.      */
int ds_combine_finalize(float *acc, const void *resid, int R, int d, void *out, void *stream);
/* Prefill grouped FFN (K3): for experts e in [0,E) (E <= 16): rows
 * [offsets[e], offsets[e+1]) of xperm [*, d] bf16 through experts[e];
 * y f32 [offsets[E], d] (un-weighted expert outputs).  h is bf16
 * [offsets[E], ff] scratch.  offsets and experts are HOST arrays (the host
 * scheduler knows the grouping; weights are device pointers, e.g. cache
 * slots).  tcgen05.mma (kind::f16, f32 accumulators in TMEM, BM=128 weight
 * rows x BN=128 token rows), activation tiles by TMA (SWIZZLE_128B), W4
 * dequantised into UMMA SWIZZLE_128B shared-memory tiles.  Split-K partials
 * of the down projection are reduced in a fixed order (deterministic).     */
size_t ds_w4_grouped_ffn_workspace(int total_rows, int d, int ff);
int ds_w4_grouped_ffn(const void *xperm, const int32_t *offsets, int E, const ds_w4_expert *experts,
                      int d, int ff, int G, void *h, float *y, void *workspace,
                      size_t workspace_bytes, void *stream);
/* Same, with cudaEvent_t ev_start / ev_end (may be NULL) recorded on `stream`
 * right before the first and after the last launch (host-side tensor-map
 * preparation excluded): the kernel-time span a profiler reads.           */
int ds_w4_grouped_ffn_ev(const void *xperm, const int32_t *offsets, int E, const ds_w4_expert *experts,
                         int d, int ff, int G, void *h, float *y, void *workspace,
                         size_t workspace_bytes, void *ev_start, void *ev_end, void *stream);
/* Same over arbitrary row segments of xperm / h / y: expert i owns rows
 * [row_start[i], row_start[i] + rows[i]) (host arrays; segments need not be
 * contiguous — e.g. the HBM-resident pinned experts of a layer in one launch);
 * rows outside every segment are not written.  The workspace is sized for
 * max_i(row_start[i] + rows[i]) rows.                                       */
size_t ds_w4_grouped_ffn_seg_workspace(const int32_t *row_start, const int32_t *rows, int E, int d, int ff,
                                       int G);
int ds_w4_grouped_ffn_seg_ev(const void *xperm, const int32_t *row_start, const int32_t *rows, int E,
                             const ds_w4_expert *experts, int d, int ff, int G, void *h, float *y,
                             void *workspace, size_t workspace_bytes, void *ev_start, void *ev_end,
                             void *stream);

/* ========================================================================
 * K6 — host->device expert link (copy engine), native scheduler thread.
 * Replaces the paper's communication stream (SPEC's single
 * serial link).  Transfers are issued in `chunk_bytes` pieces,
 * at most `depth` queued on `copy_stream`; before the first chunk the stream
 * waits `wait_event`, after the last `done_event` is recorded (both raw
 * cudaEvent_t, may be NULL).  ds_link_cancel drops the chunks not yet issued
 * (a prefetch proven wrong at sync point 1).
 * ===================================================================== */
typedef struct ds_link ds_link;
int ds_link_create(void *copy_stream, size_t chunk_bytes, int depth, ds_link **out);
int ds_link_destroy(ds_link *link);
int ds_link_submit(ds_link *link, void *dst, const void *src, size_t bytes, void *wait_event,
                   void *done_event, uint64_t *ticket);
/* Speculative transfer (a predicted prefetch) issued in `chunk_bytes` pieces so a
 * cancellation leaves little in flight; ds_link_promote switches a confirmed one
 * back to the link's default chunk size. */
int ds_link_submit_chunked(ds_link *link, void *dst, const void *src, size_t bytes, size_t chunk_bytes,
                           void *wait_event, void *done_event, uint64_t *ticket);
int ds_link_promote(ds_link *link, uint64_t ticket);
int ds_link_cancel(ds_link *link, uint64_t ticket, size_t *bytes_issued);
/* Block until every chunk of `ticket` is issued (its done_event recorded) or it was cancelled. */
int ds_link_wait_issued(ds_link *link, uint64_t ticket);
int ds_link_idle(ds_link *link);
int ds_link_stats(ds_link *link, uint64_t *bytes_issued, uint64_t *bytes_wasted, uint64_t *chunks);
int ds_link_reset_stats(ds_link *link);
/* Trace mode (measurement only): a timing event pair around every chunk.
 * ds_link_trace_read returns the copy-busy intervals [start_ms, end_ms] of the
 * chunks issued since the last read, relative to `ref_event` (a timing
 * cudaEvent_t recorded earlier on the same device), for the copy/compute
 * overlap fraction. */
int ds_link_trace(ds_link *link, int enable);
int ds_link_trace_read(ds_link *link, void *ref_event, float *start_ms, float *end_ms, size_t max_spans,
                       size_t *n_out);

/* L2 residency for one stream's kernels: a persisting access-policy window
 * over [base, base + bytes) (the predictor's f64 weights, so the streaming
 * expert kernels do not evict them between calls); raises the device's
 * persisting set-aside as needed. */
int ds_l2_persist_window(void *stream, const void *base, size_t bytes, float hit_ratio);

/* Diagnostics: per-CTA %globaltimer stamps (ns; [n_ctas][8]: entry, phase A
 * consumed, grid barrier passed, h staged, exit) of the last fused K4 v6
 * launch made with DS_K4_V6_TIMELINE=1 in the environment. */
int ds_debug_k4v6_timeline(unsigned long long *out, int n_ctas);
/* Same for K3 with DS_K3_TIMELINE=1 (nmat 2: GEMM1, 1: GEMM2): entry, scales
 * staged, first MMA issued, last MMA issued, accumulators ready, exit. */
int ds_debug_k3_timeline(unsigned long long *out, int nmat, int n_ctas);

/* SM-driven host->HBM copy: `ctas` CTAs stream `bytes` from mapped pinned host
 * memory (cudaHostAlloc / cudaHostRegister, UVA) over PCIe with 16-byte loads
 * and streaming stores into `dst` on `stream`.  An alternative to the copy
 * engine for the expert link (PAPER.md:177-188 prescribes only "a dedicated
 * communication stream"); 16-byte aligned pointers and size. */
int ds_h2d_sm_copy(void *dst, const void *src_host, size_t bytes, int ctas, void *stream);
/* Same contract, moved by TMA bulk copies (one thread per CTA, a shared-memory
 * ring of 32 KB chunks): a few CTAs keep the PCIe reads in flight. */
int ds_h2d_tma_copy(void *dst, const void *src_host, size_t bytes, int ctas, void *stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* DUOSERVE_B200_H */
