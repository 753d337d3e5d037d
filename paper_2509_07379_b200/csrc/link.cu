// K6 — the host->device expert link: a native scheduler thread that feeds the
// copy engine in chunks.
//
// experts stream from the pinned "CPU expert cache" to the
// GPU expert cache on a dedicated communication stream.  The decode schedule
// needs two things a plain cudaMemcpyAsync queue cannot give:
//   * just-in-time issue — at most `depth` chunks are queued on the copy
//     engine, so a prefetch that the gate proves wrong (sync point 1,
//     PAPER.md:185) can be cancelled after its in-flight chunks instead of
//     holding the link for the whole 91.5 MB expert;
//   * continuity — the queue is topped up by this thread, not by the Python
//     thread that is busy launching attention/gate kernels, so the link never
//     drains while the host is launching work.
// Per transfer: the copy stream first waits `wait_event` (the slot's last
// compute), then the chunks are issued, then `done_event` is recorded (the
// slot's ready event, waited on by the compute stream).
#include "ds_common.cuh"
#include "sm100.cuh"

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <memory>
#include <unordered_map>
#include <vector>

namespace ds {
namespace {

struct Xfer {
    uint64_t ticket;
    char* dst;
    const char* src;
    size_t bytes;
    size_t next = 0;        // bytes already issued
    size_t chunk = 0;       // chunk size of this transfer (speculative transfers use small chunks)
    cudaEvent_t wait_ev;
    cudaEvent_t done_ev;
    bool cancelled = false;
    bool issued = false;
};

}  // namespace
}  // namespace ds

struct ds_link {
    cudaStream_t stream;
    size_t chunk;
    int depth;
    int device;
    std::mutex mu;
    std::condition_variable cv;       // wakes the worker
    std::condition_variable cv_done;  // wakes waiters
    std::deque<std::shared_ptr<ds::Xfer>> pending;
    std::unordered_map<uint64_t, std::shared_ptr<ds::Xfer>> live;
    std::deque<cudaEvent_t> inflight;
    std::vector<cudaEvent_t> pool;
    uint64_t next_ticket = 1;
    uint64_t bytes_issued = 0, bytes_wasted = 0, chunks = 0;
    // trace mode: a timing event pair around every transfer's run of chunks
    // (copy-busy intervals for the copy/compute overlap fraction); off by
    // default.  One pair per transfer, not per chunk: while the copy engine
    // streams host memory a timing event costs ~22 us of stream time
    // (profiles/r2/graph_k4), so per-chunk events would stall the very link
    // they measure.  The open span of the transfer being issued:
    bool trace = false;
    const void* trace_x = nullptr;
    cudaEvent_t trace_t0 = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans;
    std::vector<cudaEvent_t> tpool;
    int error = 0;
    bool stop = false;
    std::thread worker;
};

namespace ds {
namespace {

cudaEvent_t take_event(ds_link* L) {
    if (!L->pool.empty()) {
        cudaEvent_t e = L->pool.back();
        L->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
}

cudaEvent_t take_timing_event(ds_link* L) {
    if (!L->tpool.empty()) {
        cudaEvent_t e = L->tpool.back();
        L->tpool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Close the open trace span after the chunks issued so far.  L->mu held.
void trace_close_locked(ds_link* L) {
    if (!L->trace_x) return;
    cudaEvent_t t1 = take_timing_event(L);
    cudaEventRecord(t1, L->stream);
    L->spans.emplace_back(L->trace_t0, t1);
    L->trace_x = nullptr;
    L->trace_t0 = nullptr;
}

// Issue as many chunks as the depth allows.  Called with L->mu held.
void issue_locked(ds_link* L) {
    while (!L->inflight.empty() && cudaEventQuery(L->inflight.front()) == cudaSuccess) {
        L->pool.push_back(L->inflight.front());
        L->inflight.pop_front();
    }
    while (!L->pending.empty() && (int)L->inflight.size() < L->depth) {
        auto x = L->pending.front();
        if (x->next == 0 && x->wait_ev) cudaStreamWaitEvent(L->stream, x->wait_ev, 0);
        const size_t n = std::min(x->chunk ? x->chunk : L->chunk, x->bytes - x->next);
        if (L->trace && L->trace_x != x.get()) {
            trace_close_locked(L);                    // the previous transfer (e.g. a cancelled one) ends here
            L->trace_t0 = take_timing_event(L);
            cudaEventRecord(L->trace_t0, L->stream);
            L->trace_x = x.get();
        }
        cudaError_t e = cudaMemcpyAsync(x->dst + x->next, x->src + x->next, n, cudaMemcpyHostToDevice, L->stream);
        if (e != cudaSuccess) L->error = (int)e;
        cudaEvent_t ev = take_event(L);
        cudaEventRecord(ev, L->stream);
        L->inflight.push_back(ev);
        x->next += n;
        L->bytes_issued += n;
        L->chunks++;
        if (x->next >= x->bytes) {
            if (L->trace) trace_close_locked(L);
            if (x->done_ev) cudaEventRecord(x->done_ev, L->stream);
            x->issued = true;
            L->pending.pop_front();
            L->live.erase(x->ticket);
            L->cv_done.notify_all();
        }
    }
}

void worker_loop(ds_link* L) {
    cudaSetDevice(L->device);
    std::unique_lock<std::mutex> lk(L->mu);
    while (!L->stop) {
        issue_locked(L);
        if (L->pending.empty()) {
            L->cv.wait_for(lk, std::chrono::microseconds(200));
        } else {
            // queue full: spin (yielding) on the oldest chunk without holding the
            // lock — sleep_for() has ~50 us timer slack, longer than a 4 MB chunk
            lk.unlock();
            const auto t0 = std::chrono::steady_clock::now();
            while (std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(2))
                std::this_thread::yield();
            lk.lock();
        }
    }
}

}  // namespace
}  // namespace ds

using namespace ds;

extern "C" int ds_link_create(void* copy_stream, size_t chunk_bytes, int depth, ds_link** out) {
    DS_CHECK_ARG(out && chunk_bytes >= 4096 && depth >= 1 && depth <= 64, "ds_link_create: bad arguments");
    ds_link* L = new ds_link();
    L->stream = as_stream(copy_stream);
    L->chunk = chunk_bytes;
    L->depth = depth;
    cudaGetDevice(&L->device);
    L->worker = std::thread(worker_loop, L);
    *out = L;
    return DS_OK;
}

extern "C" int ds_link_destroy(ds_link* L) {
    if (!L) return DS_OK;
    {
        std::lock_guard<std::mutex> g(L->mu);
        L->stop = true;
    }
    L->cv.notify_all();
    L->worker.join();
    cudaStreamSynchronize(L->stream);
    for (auto e : L->inflight) cudaEventDestroy(e);
    for (auto e : L->pool) cudaEventDestroy(e);
    for (auto& sp : L->spans) {
        cudaEventDestroy(sp.first);
        cudaEventDestroy(sp.second);
    }
    for (auto e : L->tpool) cudaEventDestroy(e);
    if (L->trace_t0) cudaEventDestroy(L->trace_t0);
    delete L;
    return DS_OK;
}

extern "C" int ds_link_submit(ds_link* L, void* dst, const void* src, size_t bytes, void* wait_event,
                              void* done_event, uint64_t* ticket) {
    DS_CHECK_ARG(L && dst && src && bytes > 0 && ticket, "ds_link_submit: bad arguments");
    auto x = std::make_shared<Xfer>();
    x->dst = static_cast<char*>(dst);
    x->src = static_cast<const char*>(src);
    x->bytes = bytes;
    x->wait_ev = static_cast<cudaEvent_t>(wait_event);
    x->done_ev = static_cast<cudaEvent_t>(done_event);
    {
        std::lock_guard<std::mutex> g(L->mu);
        x->ticket = L->next_ticket++;
        L->pending.push_back(x);
        L->live[x->ticket] = x;
        *ticket = x->ticket;
        issue_locked(L);
    }
    L->cv.notify_one();
    return DS_OK;
}

extern "C" int ds_link_submit_chunked(ds_link* L, void* dst, const void* src, size_t bytes, size_t chunk_bytes,
                                      void* wait_event, void* done_event, uint64_t* ticket) {
    DS_CHECK_ARG(L && dst && src && bytes > 0 && ticket && chunk_bytes >= 4096, "ds_link_submit_chunked: bad arguments");
    auto x = std::make_shared<Xfer>();
    x->dst = static_cast<char*>(dst);
    x->src = static_cast<const char*>(src);
    x->bytes = bytes;
    x->chunk = chunk_bytes;
    x->wait_ev = static_cast<cudaEvent_t>(wait_event);
    x->done_ev = static_cast<cudaEvent_t>(done_event);
    {
        std::lock_guard<std::mutex> g(L->mu);
        x->ticket = L->next_ticket++;
        L->pending.push_back(x);
        L->live[x->ticket] = x;
        *ticket = x->ticket;
        issue_locked(L);
    }
    L->cv.notify_one();
    return DS_OK;
}

// A speculative transfer the gate confirmed: finish it with the link's
// default (large) chunks.
extern "C" int ds_link_promote(ds_link* L, uint64_t ticket) {
    DS_CHECK_ARG(L, "ds_link_promote: NULL link");
    std::lock_guard<std::mutex> g(L->mu);
    auto it = L->live.find(ticket);
    if (it != L->live.end()) it->second->chunk = 0;
    return DS_OK;
}

extern "C" int ds_link_cancel(ds_link* L, uint64_t ticket, size_t* bytes_issued) {
    DS_CHECK_ARG(L, "ds_link_cancel: NULL link");
    std::lock_guard<std::mutex> g(L->mu);
    auto it = L->live.find(ticket);
    size_t done = 0;
    if (it != L->live.end()) {
        auto x = it->second;
        done = x->next;
        x->cancelled = true;
        // its trace span ends after the chunks already in flight (recorded now,
        // not when the next transfer starts: the link may idle in between)
        if (L->trace && L->trace_x == x.get()) trace_close_locked(L);
        L->bytes_wasted += x->next;
        for (auto p = L->pending.begin(); p != L->pending.end(); ++p)
            if ((*p)->ticket == ticket) {
                L->pending.erase(p);
                break;
            }
        L->live.erase(it);
        L->cv_done.notify_all();
    }
    if (bytes_issued) *bytes_issued = done;
    return DS_OK;
}

extern "C" int ds_link_wait_issued(ds_link* L, uint64_t ticket) {
    DS_CHECK_ARG(L, "ds_link_wait_issued: NULL link");
    std::unique_lock<std::mutex> lk(L->mu);
    L->cv.notify_one();
    L->cv_done.wait(lk, [&] { return L->live.find(ticket) == L->live.end(); });
    if (L->error) return fail(L->error, "ds_link: cudaMemcpyAsync failed: %s", cudaGetErrorString((cudaError_t)L->error));
    return DS_OK;
}

extern "C" int ds_link_idle(ds_link* L) {
    if (!L) return 1;
    std::lock_guard<std::mutex> g(L->mu);
    return L->pending.empty() ? 1 : 0;
}

extern "C" int ds_link_stats(ds_link* L, uint64_t* issued, uint64_t* wasted, uint64_t* chunks) {
    DS_CHECK_ARG(L, "ds_link_stats: NULL link");
    std::lock_guard<std::mutex> g(L->mu);
    if (issued) *issued = L->bytes_issued;
    if (wasted) *wasted = L->bytes_wasted;
    if (chunks) *chunks = L->chunks;
    return DS_OK;
}

extern "C" int ds_link_reset_stats(ds_link* L) {
    DS_CHECK_ARG(L, "ds_link_reset_stats: NULL link");
    std::lock_guard<std::mutex> g(L->mu);
    L->bytes_issued = L->bytes_wasted = L->chunks = 0;
    return DS_OK;
}

extern "C" int ds_link_trace(ds_link* L, int enable) {
    DS_CHECK_ARG(L, "ds_link_trace: NULL link");
    std::lock_guard<std::mutex> g(L->mu);
    if (!enable) trace_close_locked(L);
    L->trace = enable != 0;
    return DS_OK;
}

// Copy-busy intervals of the chunks issued since the last read, in ms relative
// to `ref_event` (a timing event recorded before them on any stream of the
// device).  Synchronises on the last chunk; returns the spans' events to the
// pool.  *n_out = number of spans written (<= max_spans; the rest are dropped).
extern "C" int ds_link_trace_read(ds_link* L, void* ref_event, float* start_ms, float* end_ms, size_t max_spans,
                                  size_t* n_out) {
    DS_CHECK_ARG(L && ref_event && n_out, "ds_link_trace_read: bad arguments");
    std::lock_guard<std::mutex> g(L->mu);
    trace_close_locked(L);                            // a transfer cut short by a cancellation
    cudaEvent_t ref = static_cast<cudaEvent_t>(ref_event);
    size_t n = 0;
    int err = 0;
    if (!L->spans.empty()) cudaEventSynchronize(L->spans.back().second);
    for (auto& sp : L->spans) {
        if (n < max_spans && start_ms && end_ms) {
            float a = 0.f, b = 0.f;
            cudaError_t e1 = cudaEventElapsedTime(&a, ref, sp.first);
            cudaError_t e2 = cudaEventElapsedTime(&b, ref, sp.second);
            if (e1 != cudaSuccess || e2 != cudaSuccess) err = (int)(e1 != cudaSuccess ? e1 : e2);
            start_ms[n] = a;
            end_ms[n] = b;
            ++n;
        }
        L->tpool.push_back(sp.first);
        L->tpool.push_back(sp.second);
    }
    L->spans.clear();
    *n_out = n;
    if (err) return fail(err, "ds_link_trace_read: cudaEventElapsedTime failed: %s", cudaGetErrorString((cudaError_t)err));
    return DS_OK;
}

// ---------------------------------------------------------------------------
// SM-driven host->HBM copy (experiment: an alternative to the copy engine for
// the expert link).  Pinned host memory is mapped into the device's address
// space (UVA), so a kernel can stream it over PCIe with ordinary loads.  Each
// thread keeps U 16-byte loads in flight; stores to HBM are streaming (.cs).
namespace ds_zc {
constexpr int kZcThreads = 256;
constexpr int kZcU = 8;

__global__ void __launch_bounds__(kZcThreads) zc_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                             size_t n16) {
    const size_t stride = (size_t)gridDim.x * kZcThreads * kZcU;
    for (size_t base = (size_t)blockIdx.x * kZcThreads * kZcU + threadIdx.x; base < n16; base += stride) {
        uint4 v[kZcU];
#pragma unroll
        for (int u = 0; u < kZcU; ++u) {
            const size_t i = base + (size_t)u * kZcThreads;
            if (i < n16) {
                const uint4* p = src + i;
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
            }
        }
#pragma unroll
        for (int u = 0; u < kZcU; ++u) {
            const size_t i = base + (size_t)u * kZcThreads;
            if (i < n16) __stcs(dst + i, v[u]);
        }
    }
}
}  // namespace ds_zc

extern "C" int ds_h2d_sm_copy(void* dst, const void* src_host, size_t bytes, int ctas, void* stream) {
    DS_CHECK_ARG(dst && src_host, "ds_h2d_sm_copy: NULL pointer");
    DS_CHECK_ARG(bytes % 16 == 0 && ((uintptr_t)dst & 15) == 0 && ((uintptr_t)src_host & 15) == 0,
                 "ds_h2d_sm_copy: pointers and size must be 16-byte aligned");
    DS_CHECK_ARG(ctas > 0 && ctas <= 4096, "ds_h2d_sm_copy: ctas=%d", ctas);
    void* dsrc = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dsrc, const_cast<void*>(src_host), 0);
    if (e != cudaSuccess) return cuda_status(e, "ds_h2d_sm_copy: source is not mapped pinned host memory");
    if (bytes == 0) return DS_OK;
    ds_zc::zc_copy_kernel<<<ctas, ds_zc::kZcThreads, 0, ds::as_stream(stream)>>>(static_cast<uint4*>(dst),
                                                                  static_cast<const uint4*>(dsrc), bytes / 16);
    DS_LAUNCH_CHECK("ds_h2d_sm_copy");
    return DS_OK;
}

// TMA-driven host->HBM copy: one thread per CTA streams CH-byte chunks from
// mapped pinned host memory into a shared-memory ring with cp.async.bulk
// (mbarrier transaction counts) and writes each back to HBM with a bulk
// shared->global store, so a handful of SMs (no per-byte instructions) keep
// ~ring-size bytes of PCIe reads in flight.
namespace ds_zc {
constexpr int kTmaChunk = 32 * 1024;
constexpr int kTmaSlots = 6;

__global__ void __launch_bounds__(32) tma_copy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                      size_t bytes) {
    using namespace ds::sm100;
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ __align__(8) uint64_t full[kTmaSlots];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < kTmaSlots; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
    const size_t nchunks = (bytes + kTmaChunk - 1) / kTmaChunk;
    size_t issued = 0, done = 0;
    // chunk j of this CTA = global chunk blockIdx.x + j * gridDim.x
    auto chunk_of = [&](size_t j) { return (size_t)blockIdx.x + j * gridDim.x; };
    size_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    while (done < mine) {
        while (issued < mine && issued - done < (size_t)kTmaSlots) {
            const int slot = (int)(issued % kTmaSlots);
            if (issued >= (size_t)kTmaSlots) {
                // the slot's previous store must have finished reading shared memory
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaSlots - 1) : "memory");
            }
            const size_t c = chunk_of(issued);
            const uint32_t n = (uint32_t)min((size_t)kTmaChunk, bytes - c * kTmaChunk);
            mbar_expect_tx(&full[slot], n);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(ring + (size_t)slot * kTmaChunk)),
                "l"(reinterpret_cast<uint64_t>(src + c * kTmaChunk)), "r"(n), "r"(smem_u32(&full[slot]))
                : "memory");
            ++issued;
        }
        const int slot = (int)(done % kTmaSlots);
        mbar_wait(&full[slot], (uint32_t)((done / kTmaSlots) & 1));
        const size_t c = chunk_of(done);
        const uint32_t n = (uint32_t)min((size_t)kTmaChunk, bytes - c * kTmaChunk);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<uint64_t>(dst + c * kTmaChunk)),
                     "r"(smem_u32(ring + (size_t)slot * kTmaChunk)), "r"(n)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        ++done;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
}  // namespace ds_zc

extern "C" int ds_h2d_tma_copy(void* dst, const void* src_host, size_t bytes, int ctas, void* stream) {
    DS_CHECK_ARG(dst && src_host, "ds_h2d_tma_copy: NULL pointer");
    DS_CHECK_ARG(bytes % 16 == 0 && ((uintptr_t)dst & 15) == 0 && ((uintptr_t)src_host & 15) == 0,
                 "ds_h2d_tma_copy: pointers and size must be 16-byte aligned");
    DS_CHECK_ARG(ctas > 0 && ctas <= 1024, "ds_h2d_tma_copy: ctas=%d", ctas);
    void* dsrc = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dsrc, const_cast<void*>(src_host), 0);
    if (e != cudaSuccess) return cuda_status(e, "ds_h2d_tma_copy: source is not mapped pinned host memory");
    if (bytes == 0) return DS_OK;
    const int smem = ds_zc::kTmaChunk * ds_zc::kTmaSlots;
    if (ds::first_use_on_device((const void*)ds_zc::tma_copy_kernel))
        cudaFuncSetAttribute(ds_zc::tma_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    ds_zc::tma_copy_kernel<<<ctas, 32, smem, ds::as_stream(stream)>>>(static_cast<uint8_t*>(dst),
                                                                      static_cast<const uint8_t*>(dsrc), bytes);
    DS_LAUNCH_CHECK("ds_h2d_tma_copy");
    return DS_OK;
}
