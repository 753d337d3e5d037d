// Shared helpers for the sm_100a kernels of libduoserve_sm100.so.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/duoserve_b200.h"

namespace ds {

// ---- error plumbing (thread-local last message, int status codes) -------
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

inline int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return DS_OK;
    return fail((int)e, "%s: %s", what, cudaGetErrorString(e));
}

#define DS_CHECK_ARG(cond, ...)                        \
    do {                                               \
        if (!(cond)) return ::ds::fail(DS_ERR_ARG, __VA_ARGS__); \
    } while (0)

#define DS_LAUNCH_CHECK(what) \
    do { cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) return ::ds::cuda_status(_e, what); } while (0)

int num_sms();

// True the first time `key` (a kernel's address) is seen on the current
// device: per-device one-time setup such as cudaFuncSetAttribute, which is a
// per-device property (a process may drive several GPUs).
bool first_use_on_device(const void* key);

// ---- launch gate (measurement hygiene for CUDA-event kernel spans) -------
// A span [ev_start, ev_end] recorded on an idle stream around host-side
// launches also contains the host's submission latency (the start event fires
// as soon as it is recorded, the kernel only once the host has submitted it).
// gate_hold() makes the stream wait (cuStreamWaitValue32 on a device word)
// until gate_release() — issued after every launch of the span is queued —
// so the span covers device execution only.  Returns 0 when the stream memory
// operations are unavailable (then the span is recorded ungated).
// Between hold and release the caller must not make a synchronous CUDA call
// (cudaMemcpy, cudaMemset, cudaMalloc, ...): on the legacy default stream it
// would wait for the held work and never return.  DS_LAUNCH_GATE=0 disables
// the gate (A/B runs).
unsigned gate_hold(cudaStream_t st);
void gate_release(unsigned seq);
// true once a call path `key` has run before: its kernels are then loaded
// (CUDA lazy loading may synchronise the context on a kernel's first use,
// which would deadlock against a held stream — the first call is not gated)
bool gate_warm(uint64_t key);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- counter-based generator (splitmix64 finaliser) ---------------------
// Shared bit-for-bit with oracle/w4_ref.py.
__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// stream key for (seed, layer, expert, matrix, kind)
__host__ __device__ inline uint64_t stream_key(uint64_t seed, int layer, int expert, int matrix,
                                               int kind) {
    uint64_t tag = ((((uint64_t)layer * 64u + (uint64_t)expert) * 4u + (uint64_t)matrix) * 4u +
                    (uint64_t)kind);
    return mix64(seed ^ mix64(tag));
}

__host__ __device__ inline uint64_t draw(uint64_t key, uint64_t counter) {
    return mix64(key + counter * 0xD1B54A32D192ED03ull);
}

// ---- bf16 bit helpers -----------------------------------------------------
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
    __nv_bfloat16 b = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t*>(&b);
}

// Mixed-precision FMA (sm_100: FHFMA.BF16): acc(f32) += a(bf16) * b(bf16),
// selecting 16-bit halves of packed registers without conversion.
__device__ __forceinline__ void fma_bf16_lo(float& acc, uint32_t a, uint32_t b) {
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc) : "h"((uint16_t)(a & 0xFFFF)), "h"((uint16_t)(b & 0xFFFF)));
}
__device__ __forceinline__ void fma_bf16_hi(float& acc, uint32_t a, uint32_t b) {
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc) : "h"((uint16_t)(a >> 16)), "h"((uint16_t)(b >> 16)));
}

// int4 nibble pairs -> packed bf16x2 {128+q_lo, 128+q_hi} via the exponent
// trick: 0x4300 is bf16 128.0 and its 7 mantissa bits hold q exactly.
__device__ __forceinline__ uint32_t nib_pair_magic(uint32_t v) {
    uint32_t r;
    asm("lop3.b32 %0, %1, 0x000F000F, 0x43004300, 0xEA;" : "=r"(r) : "r"(v));  // (v & m) | c
    return r;
}

// Codes order within a u32 word: nibble j holds k = 8w + kPerm[j].
// So (v >> 4i) & 0x000F000F = {q[2i], q[2i+1]} for i = 0..3.
//   kPerm = {0, 2, 4, 6, 1, 3, 5, 7}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

}  // namespace ds
