// Probe: which CUDA-graph event-node operations work on this driver?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/graphprobe scripts/graphprobe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k(int* p) { if (threadIdx.x == 0) atomicAdd(p, 1); }

#define P(x) do { cudaError_t e = (x); printf("%-60s %s\n", #x, cudaGetErrorString(e)); } while (0)

int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaStream_t cap, st;
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t w0, w1, a0, a1, b0, b1;
    for (cudaEvent_t* e : {&w0, &w1, &a0, &a1, &b0, &b1}) cudaEventCreate(e);
    cudaEventRecord(w0, st);
    cudaEventRecord(w1, st);
    cudaStreamSynchronize(st);

    // 1. captured external nodes
    cudaGraph_t g;
    P(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
    P(cudaStreamWaitEvent(cap, w0, cudaEventWaitExternal));
    P(cudaEventRecordWithFlags(a0, cap, cudaEventRecordExternal));
    k<<<1, 32, 0, cap>>>(d);
    P(cudaEventRecordWithFlags(a1, cap, cudaEventRecordExternal));
    P(cudaStreamEndCapture(cap, &g));
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(g, nodes.data(), &n);
    cudaGraphNode_t wn = nullptr, r0 = nullptr, r1 = nullptr;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        printf("node type %d\n", (int)t);
        if (t == cudaGraphNodeTypeWaitEvent) wn = nd;
        if (t == cudaGraphNodeTypeEventRecord) {
            cudaEvent_t ev;
            cudaGraphEventRecordNodeGetEvent(nd, &ev);
            (ev == a0 ? r0 : r1) = nd;
        }
    }
    cudaGraphExec_t x;
    P(cudaGraphInstantiate(&x, g, 0));
    P(cudaGraphUpload(x, st));
    P(cudaGraphLaunch(x, st));
    P(cudaStreamSynchronize(st));
    P(cudaGraphExecEventWaitNodeSetEvent(x, wn, w1));
    P(cudaGraphExecEventRecordNodeSetEvent(x, r0, b0));
    P(cudaGraphExecEventRecordNodeSetEvent(x, r1, b1));
    P(cudaGraphLaunch(x, st));
    P(cudaStreamSynchronize(st));
    float ms = -1;
    P(cudaEventElapsedTime(&ms, b0, b1));
    printf("span b0->b1 %.3f us\n", ms * 1e3);

    // 2. explicitly built nodes
    cudaGraph_t g2;
    cudaGraphCreate(&g2, 0);
    cudaGraphNode_t n0, n1, n2, n3;
    P(cudaGraphAddEventWaitNode(&n0, g2, nullptr, 0, w0));
    P(cudaGraphAddEventRecordNode(&n1, g2, &n0, 1, a0));
    cudaKernelNodeParams kp = {};
    void* args[] = {&d};
    kp.func = (void*)k;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(32);
    kp.kernelParams = args;
    P(cudaGraphAddKernelNode(&n2, g2, &n1, 1, &kp));
    P(cudaGraphAddEventRecordNode(&n3, g2, &n2, 1, a1));
    cudaGraphExec_t x2;
    P(cudaGraphInstantiate(&x2, g2, 0));
    P(cudaGraphExecEventWaitNodeSetEvent(x2, n0, w1));
    P(cudaGraphExecEventRecordNodeSetEvent(x2, n1, b0));
    P(cudaGraphExecEventRecordNodeSetEvent(x2, n3, b1));
    P(cudaGraphLaunch(x2, st));
    P(cudaStreamSynchronize(st));
    P(cudaEventElapsedTime(&ms, b0, b1));
    printf("span b0->b1 %.3f us\n", ms * 1e3);
    // 3. whole-graph update as the alternative
    cudaGraph_t g3;
    P(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
    P(cudaStreamWaitEvent(cap, w1, cudaEventWaitExternal));
    P(cudaEventRecordWithFlags(b0, cap, cudaEventRecordExternal));
    k<<<1, 32, 0, cap>>>(d);
    P(cudaEventRecordWithFlags(b1, cap, cudaEventRecordExternal));
    P(cudaStreamEndCapture(cap, &g3));
    cudaGraphExecUpdateResultInfo info;
    P(cudaGraphExecUpdate(x, g3, &info));
    printf("update result %d\n", (int)info.result);
    P(cudaGraphLaunch(x, st));
    P(cudaStreamSynchronize(st));
    // 4. cooperative kernel between captured event nodes
    for (int variant = 0; variant < 2; ++variant) {
        cudaGraph_t g4;
        P(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
        P(cudaStreamWaitEvent(cap, w0, cudaEventWaitExternal));
        P(cudaEventRecordWithFlags(a0, cap, cudaEventRecordExternal));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(544);
        cfg.stream = cap;
        cudaLaunchAttribute at[1];
        if (variant == 0) {
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
        } else {
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            k<<<1, 32, 0, cap>>>(d);
        }
        cfg.attrs = at;
        cfg.numAttrs = 1;
        P(cudaLaunchKernelEx(&cfg, k, d));
        P(cudaEventRecordWithFlags(a1, cap, cudaEventRecordExternal));
        P(cudaStreamEndCapture(cap, &g4));
        cudaGraphGetNodes(g4, nullptr, &n);
        nodes.resize(n);
        cudaGraphGetNodes(g4, nodes.data(), &n);
        wn = r0 = r1 = nullptr;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(nd, &t);
            printf("variant %d node type %d\n", variant, (int)t);
            if (t == cudaGraphNodeTypeWaitEvent) wn = nd;
            if (t == cudaGraphNodeTypeEventRecord) {
                cudaEvent_t ev;
                cudaGraphEventRecordNodeGetEvent(nd, &ev);
                (ev == a0 ? r0 : r1) = nd;
            }
        }
        cudaGraphExec_t x4;
        P(cudaGraphInstantiate(&x4, g4, 0));
        P(cudaGraphUpload(x4, st));
        P(cudaGraphLaunch(x4, st));
        P(cudaGraphExecEventWaitNodeSetEvent(x4, wn, w1));
        P(cudaGraphExecEventRecordNodeSetEvent(x4, r0, b0));
        P(cudaGraphExecEventRecordNodeSetEvent(x4, r1, b1));
        P(cudaGraphLaunch(x4, st));
        P(cudaStreamSynchronize(st));
        P(cudaEventElapsedTime(&ms, b0, b1));
        printf("variant %d span %.3f us\n", variant, ms * 1e3);
    }
    return 0;
}
