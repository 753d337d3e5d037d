// Probe: kernel-to-kernel launch gaps on a compute stream, idle vs while the
// copy engine streams pinned host memory into HBM (the decode link's load).
// Each tiny kernel stamps %globaltimer at entry; gaps = consecutive entry
// differences.  Eager launches vs the same chain captured in one graph, plus
// event-record overhead (event pair around one tiny kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/launchprobe scripts/launchprobe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void stamp(unsigned long long* out, int i) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        out[i] = t;
    }
}

static double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0 : v[v.size() / 2];
}

int main() {
    const size_t bytes = 512ull << 20;
    void *h, *dst;
    cudaMallocHost(&h, bytes);
    cudaMalloc(&dst, bytes);
    unsigned long long* ts;
    cudaMalloc(&ts, 4096 * 8);
    cudaStream_t cs, st, cap;
    cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    const int N = 64;
    cudaGraph_t g;
    cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < N; ++i) stamp<<<148, 128, 0, cap>>>(ts, i);
    cudaStreamEndCapture(cap, &g);
    cudaGraphExec_t x;
    cudaGraphInstantiate(&x, g, 0);
    cudaGraphUpload(x, st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEvent_t n0;
    cudaEventCreateWithFlags(&n0, cudaEventDisableTiming);
    for (int load = 0; load < 2; ++load) {
        for (int mode = 0; mode < 5; ++mode) {
            std::vector<double> gaps, spans;
            for (int rep = 0; rep < 5; ++rep) {
                cudaDeviceSynchronize();
                if (load) {
                    cudaMemcpyAsync(dst, h, bytes, cudaMemcpyHostToDevice, cs);   // ~9 ms of link traffic
                    stamp<<<1, 32, 0, st>>>(ts, 4000);                        // spin the compute stream briefly
                    cudaStreamSynchronize(st);
                    for (volatile int s = 0; s < 200000; ++s) {}
                }
                if (mode == 0) {
                    for (int i = 0; i < N; ++i) stamp<<<148, 128, 0, st>>>(ts, i);
                } else if (mode == 1) {
                    cudaGraphLaunch(x, st);
                } else if (mode == 3 || mode == 4) {
                    // chain of tiny kernels with a non-timing event record (3) or
                    // record + wait on it (4) between consecutive kernels
                    for (int i = 0; i < N; ++i) {
                        stamp<<<148, 128, 0, st>>>(ts, i);
                        cudaEventRecord(n0, st);
                        if (mode == 4) cudaStreamWaitEvent(st, n0, 0);
                    }
                } else {
                    for (int i = 0; i < 16; ++i) {
                        cudaEventRecord(e0, st);
                        stamp<<<148, 128, 0, st>>>(ts, i);
                        cudaEventRecord(e1, st);
                        cudaEventSynchronize(e1);
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        spans.push_back(ms * 1e3);
                    }
                }
                cudaStreamSynchronize(st);
                if (mode != 2) {
                    unsigned long long hts[N];
                    cudaMemcpy(hts, ts, N * 8, cudaMemcpyDeviceToHost);
                    for (int i = 1; i < N; ++i) gaps.push_back((hts[i] - hts[i - 1]) / 1e3);
                }
                cudaDeviceSynchronize();
            }
            const char* names[] = {"eager chain", "graph chain", "event pair", "+nt record", "+nt rec+wait"};
            if (mode != 2)
                printf("%s %-12s kernel-to-kernel gap median %.2f us max %.2f\n", load ? "LOAD" : "idle", names[mode],
                       median(gaps), *std::max_element(gaps.begin(), gaps.end()));
            else
                printf("%s %-12s span median %.2f us max %.2f\n", load ? "LOAD" : "idle", names[mode], median(spans),
                       *std::max_element(spans.begin(), spans.end()));
        }
    }
    return 0;
}
