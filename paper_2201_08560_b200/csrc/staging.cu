// Host -> device uploads from pageable memory at the PCIe rate.
//
// A caller of the drop-in API hands over plain numpy arrays (pageable
// memory).  cudaMemcpyAsync from pageable memory goes through the driver's
// own small bounce buffer and runs far below the link rate (11 GB/s on the
// B200 box), and pinning the caller's pages in place costs more than it saves
// (cudaHostRegister of 1 GB: 146 ms, tools/h2d_probe.py).  Large uploads are
// staged instead: the upload is cut into 16 MB chunks and T host threads own
// every T-th chunk, each with two page-locked slots of a per-device pool --
// copy the chunk into a free slot, queue its DMA on the caller's stream,
// record the slot's event, move on -- so T host copies run while the DMA
// engine drains the queue.  (The first version re-created its copy threads
// for every 32 MB chunk and waited for them before each DMA: 34 GB/s.)
// Page-locked sources and small copies go straight to cudaMemcpyAsync.  When
// the call returns the source may be reused (the slots are owned by the
// library; a page-locked source is waited for), as with a plain pageable
// cudaMemcpy.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "b2sr_internal.cuh"

namespace b2sr {

namespace {

constexpr size_t kChunk = 16u << 20;  // bytes per staging chunk
constexpr size_t kDirect = 4u << 20;  // below this, plain cudaMemcpyAsync

int copy_threads() {
    static int t = [] {
        const char *e = getenv("B2SR_H2D_THREADS");
        int v = e ? atoi(e) : 0;
        if (v <= 0) v = std::min(12, std::max(1, (int)std::thread::hardware_concurrency() * 3 / 4));
        return v;
    }();
    return t;
}

// two page-locked slots per copy thread, allocated once per device
struct StagePool {
    std::mutex mu;  // one staged upload per device at a time
    int threads = 0;
    std::vector<void *> buf;
    std::vector<cudaEvent_t> done;

    void init(int nthreads) {
        if (threads) return;
        for (int k = 0; k < 2 * nthreads; k++) {
            void *p = nullptr;
            cudaEvent_t e = nullptr;
            CK(cudaHostAlloc(&p, kChunk, cudaHostAllocPortable));
            buf.push_back(p);
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            done.push_back(e);
        }
        threads = nthreads;
    }
};

StagePool &pool(int dev) {
    static std::mutex mu;
    static std::map<int, StagePool *> pools;  // process lifetime (freed by the driver at exit)
    std::lock_guard<std::mutex> lk(mu);
    StagePool *&p = pools[dev];
    if (!p) p = new StagePool();
    return *p;
}

bool page_locked(const void *p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

}  // namespace

// The staged loop: src_bytes of pageable input in chunks of kChunk * IN /
// OUT source bytes, each turned into <= kChunk staged bytes by `fill(slot,
// src_chunk, len) -> staged bytes` and DMA'd to dst + chunk * (kChunk).
template <class Fill>
static void staged(void *dst, const void *src, size_t src_bytes, size_t src_chunk, size_t dst_chunk, Fill fill,
                   cudaStream_t s) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    StagePool &P = pool(dev);
    std::lock_guard<std::mutex> lk(P.mu);
    P.init(copy_threads());
    const size_t nchunks = (src_bytes + src_chunk - 1) / src_chunk;
    const int T = (int)std::min<size_t>(P.threads, nchunks);
    std::vector<std::exception_ptr> err(T);
    std::vector<std::string> msg(T);  // the error text is thread-local: carry it to the caller's thread
    auto worker = [&](int i) {
        try {
            CK(cudaSetDevice(dev));
            size_t round = 0;
            for (size_t c = i; c < nchunks; c += T, round++) {
                const int slot = i + P.threads * (int)(round & 1);
                const size_t off = c * src_chunk, len = std::min(src_chunk, src_bytes - off);
                CK(cudaEventSynchronize(P.done[slot]));  // the slot's previous DMA has drained
                const size_t out = fill(P.buf[slot], (const char *)src + off, len);
                CK(cudaMemcpyAsync((char *)dst + c * dst_chunk, P.buf[slot], out, cudaMemcpyHostToDevice, s));
                CK(cudaEventRecord(P.done[slot], s));
            }
        } catch (...) {
            err[i] = std::current_exception();
            msg[i] = b2sr_last_error();
        }
    };
    std::vector<std::thread> pool_threads;
    pool_threads.reserve(T - 1);
    for (int i = 1; i < T; i++) pool_threads.emplace_back(worker, i);
    worker(0);
    for (auto &th : pool_threads) th.join();
    for (int i = 0; i < T; i++)
        if (err[i]) {
            set_error(B2SR_ECUDA, "%s", msg[i].c_str());
            std::rethrow_exception(err[i]);
        }
}

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
    staged(dst, src, bytes, kChunk, kChunk,
           [](void *slot, const char *from, size_t len) {
               memcpy(slot, from, len);
               return len;
           },
           s);
}

// d = 4 bit tiles: four row bytes of which only the low nibbles may be set
// (formats.py:289).  The upload packs them to 16 bits per tile on the host
// (inside the copy the staging threads do anyway) and widens them again on
// the device: 512 -> 256 MB over PCIe at R-MAT s22.  A tile with a high
// nibble set (a FormatError the device check must report, with the
// reference's message) makes the caller fall back to the plain copy.
__global__ void k_unpack_nibbles(uint64_t T, const uint16_t *__restrict__ in, uint32_t *__restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = in[t];
        out[t] = (p & 0xFu) | ((p & 0xF0u) << 4) | ((p & 0xF00u) << 8) | ((p & 0xF000u) << 12);
    }
}

bool h2d_tiles4(void *d_tiles, const void *h_tiles, uint64_t T, cudaStream_t s) {
    const size_t bytes = T * 4;
    if (bytes < 4 * kDirect || page_locked(h_tiles)) return false;
    Buf<uint16_t> packed(T, s);
    std::atomic<bool> high{false};
    staged(packed.p, h_tiles, bytes, 2 * kChunk, kChunk,
           [&](void *slot, const char *from, size_t len) {
               const uint32_t *w = reinterpret_cast<const uint32_t *>(from);
               uint16_t *o = static_cast<uint16_t *>(slot);
               const size_t n = len / 4;
               uint32_t hi = 0;
               for (size_t i = 0; i < n; i++) {
                   const uint32_t v = w[i];
                   hi |= v;
                   o[i] = (uint16_t)((v & 0xFu) | ((v >> 4) & 0xF0u) | ((v >> 8) & 0xF00u) | ((v >> 12) & 0xF000u));
               }
               if (hi & 0xF0F0F0F0u) high.store(true, std::memory_order_relaxed);
               return n * 2;
           },
           s);
    if (high.load()) return false;  // the stream drains `packed` before its memory is reused
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((T + 255) / 256, (uint64_t)num_sms() * 16));
    LAUNCH(k_unpack_nibbles, g, 256, 0, s, T, packed.p, static_cast<uint32_t *>(d_tiles));
    return true;
}

}  // namespace b2sr

extern "C" int b2sr_h2d(void *d_dst, const void *h_src, uint64_t bytes, void *stream) {
    API_BEGIN
    b2sr::h2d(d_dst, h_src, bytes, (cudaStream_t)stream);
    API_END
}
