// Host -> device uploads from pageable memory at the PCIe rate.
//
// A caller of the drop-in API hands over plain numpy arrays (pageable
// memory).  cudaMemcpyAsync from pageable memory goes through the driver's
// own small bounce buffer and runs far below the link rate, so large uploads
// are staged here instead: a per-thread ring of page-locked chunks, each
// filled by several host threads in parallel (the host copy is the slow leg)
// while the DMA of the previous chunk runs.  Page-locked sources and small
// copies go straight to cudaMemcpyAsync.  When the call returns the source
// may be reused (the ring's chunks are owned by the library; a page-locked
// source is waited for), as with a plain pageable cudaMemcpy.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "b2sr_internal.cuh"

namespace b2sr {

namespace {

constexpr size_t kChunk = 32u << 20;  // bytes per staging chunk
constexpr int kRing = 3;              // chunks in flight per host thread
constexpr size_t kDirect = 4u << 20;  // below this, plain cudaMemcpyAsync

struct Ring {
    int device = -1;
    void *buf[kRing] = {};
    cudaEvent_t done[kRing] = {};

    ~Ring() {
        for (int k = 0; k < kRing; k++) {
            if (done[k]) cudaEventDestroy(done[k]);
            if (buf[k]) cudaFreeHost(buf[k]);
        }
    }
    void init(int dev) {
        if (device == dev) return;
        this->~Ring();
        for (int k = 0; k < kRing; k++) {
            buf[k] = nullptr;
            done[k] = nullptr;
        }
        for (int k = 0; k < kRing; k++) {
            CK(cudaHostAlloc(&buf[k], kChunk, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
        }
        device = dev;
    }
};

Ring &ring() {
    static thread_local Ring r;
    return r;
}

int copy_threads() {
    static int t = [] {
        const char *e = getenv("B2SR_H2D_THREADS");
        int v = e ? atoi(e) : 0;
        // 16-core GPU host, 1 GB upload: 8 / 12 / 16 threads gave 34.8 / 38.3 / 29.5 GB/s
        if (v <= 0) v = std::min(12, std::max(1, (int)std::thread::hardware_concurrency() * 3 / 4));
        return v;
    }();
    return t;
}

bool page_locked(const void *p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

void parallel_memcpy(void *dst, const void *src, size_t len, int threads) {
    const size_t grain = 1u << 20;
    int t = (int)std::min<size_t>(threads, (len + grain - 1) / grain);
    if (t <= 1) {
        memcpy(dst, src, len);
        return;
    }
    const size_t part = (len / t + 63) & ~(size_t)63;
    std::vector<std::thread> pool;
    pool.reserve(t - 1);
    for (int i = 1; i < t; i++) {
        size_t b = std::min(len, (size_t)i * part), e = std::min(len, b + part);
        if (e > b)
            pool.emplace_back([=] { memcpy((char *)dst + b, (const char *)src + b, e - b); });
    }
    memcpy(dst, src, std::min(len, part));
    for (auto &th : pool) th.join();
}

}  // namespace

void h2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    if (page_locked(src)) {  // DMA straight from the caller's buffer; wait so it may be reused
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    if (bytes < kDirect) {  // pageable: the driver copies it out before returning
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    Ring &r = ring();
    r.init(dev);
    const int threads = copy_threads();
    int k = 0;
    for (size_t off = 0; off < bytes; off += kChunk, k = (k + 1) % kRing) {
        const size_t len = std::min(kChunk, bytes - off);
        CK(cudaEventSynchronize(r.done[k]));  // the chunk's previous DMA has drained
        parallel_memcpy(r.buf[k], (const char *)src + off, len, threads);
        CK(cudaMemcpyAsync((char *)dst + off, r.buf[k], len, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(r.done[k], s));
    }
}

}  // namespace b2sr

extern "C" int b2sr_h2d(void *d_dst, const void *h_src, uint64_t bytes, void *stream) {
    API_BEGIN
    b2sr::h2d(d_dst, h_src, bytes, (cudaStream_t)stream);
    API_END
}
