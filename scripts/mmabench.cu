// tcgen05.mma issue-rate microbenchmark (B200): one CTA per SM, one thread
// issues back-to-back kind::f16 MMAs (M = 128, N = TN, K = 16) from shared
// memory operands (SWIZZLE_128B K-major, contents irrelevant) into TMEM, then
// commits and waits.  Reports MACs / cycle / SM and the implied dense bf16
// TFLOP/s across all SMs: the ceiling the K3 MMA issuer can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2509_07379_b200/csrc -o scripts/mmabench scripts/mmabench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace ds::sm100;

template <int TN, bool A_TMEM, int COMMITS = 0>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* a_tile = smem;                 // 128 rows x 128 B
    uint8_t* b_tile = smem + 128 * 128;     // TN rows x 128 B
    __shared__ uint64_t done;
    __shared__ uint64_t sink[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    constexpr uint32_t COLS = A_TMEM ? 512 : (TN < 32 ? 32 : TN);
    if (warp == 0) tmem_alloc<COLS>(&tslot);
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        mbar_init(&sink[0], 1);
        mbar_init(&sink[1], 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, TN);
        const uint64_t ad = umma_desc_sw128(smem_u32(a_tile));
        const uint64_t bd = umma_desc_sw128(smem_u32(b_tile));
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if constexpr (A_TMEM)
                    mma_bf16_ts(tmem, tmem + 256 + kk * 8, bd + 2 * kk, idesc, (i | kk) != 0);
                else
                    mma_bf16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (i | kk) != 0);
            }
            // COMMITS per 4 MMAs (the K3 issuer commits twice per k-tile)
            if (COMMITS >= 1) mma_commit(&sink[0]);
            if (COMMITS >= 2) mma_commit(&sink[1]);
        }
        mma_commit(&done);
        mbar_wait(&done, 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<COLS>(tmem);
    }
}

template <int TN, bool A_TMEM, int COMMITS = 0>
void run(int sms, unsigned long long* d_cycles) {
    const int iters = 4096;
    const size_t smem = 128 * 128 + TN * 128 + 1024;
    cudaFuncSetAttribute(mma_rate<TN, A_TMEM, COMMITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mma_rate<TN, A_TMEM, COMMITS><<<sms, 128, smem>>>(16, d_cycles);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_rate<TN, A_TMEM, COMMITS><<<sms, 128, smem>>>(iters, d_cycles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d_cycles, sizeof(cyc), cudaMemcpyDeviceToHost);
    const double macs = 128.0 * TN * 16 * 4 * iters;         // per CTA
    printf("commits/4mma %d  M128 N%-3d A_%s: %.1f cycles per MMA (clock64), %.0f MAC/clk/SM, %.0f TFLOP/s over %d SMs (events) [%s]\n",
           COMMITS, TN, A_TMEM ? "tmem" : "smem", (double)cyc / (4.0 * iters), macs / (double)cyc,
           2.0 * macs * sms / (ms * 1e-3) / 1e12, sms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d = nullptr;
    cudaMalloc(&d, sizeof(unsigned long long));
    run<64, false>(sms, d);
    run<128, false>(sms, d);
    run<256, false>(sms, d);
    run<128, true>(sms, d);
    run<256, true>(sms, d);
    run<128, true, 1>(sms, d);
    run<128, true, 2>(sms, d);
    run<128, false, 2>(sms, d);
    return 0;
}
