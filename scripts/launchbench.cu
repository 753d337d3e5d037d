// Launch overhead floor for K4-sized grids: event-timed empty kernels with
// 148 CTAs x 544 threads, without / with ~218 KB dynamic shared memory, and
// cooperative.  nvcc -gencode arch=compute_100a,code=sm_100a -o launchbench launchbench.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) *p = 1; }
int main() {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
    int smem = 218 * 1024;
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int mode = 0; mode < 4; ++mode) {
        std::vector<float> ts;
        for (int i = 0; i < 60; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(n);
            cfg.blockDim = dim3(mode == 3 ? 128 : 544);
            cfg.dynamicSmemBytes = (mode >= 1 && mode != 3) ? smem : 0;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            cfg.attrs = at;
            cfg.numAttrs = mode == 2 ? 1 : 0;
            cudaEventRecord(a, s);
            cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
            cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (i >= 10) ts.push_back(ms * 1e3f / 2);
        }
        std::sort(ts.begin(), ts.end());
        const char* names[4] = {"544 thr, no smem", "544 thr, 218 KB smem", "544 thr, 218 KB, cooperative",
                                "128 thr, no smem"};
        printf("%-32s median %.2f us per launch (2 back to back)\n", names[mode], ts[ts.size() / 2]);
    }
    return 0;
}
