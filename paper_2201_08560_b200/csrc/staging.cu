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
        // 16-core GPU host, R-MAT s22 B2SR-4 host matrix (1.03 GB, tiles packed):
        // 4 / 8 / 12 / 16 threads: 46.5 / 30.2 / 27.7 / 22.9 ms (tools/upload_probe.py)
        if (v <= 0) v = std::min(16, std::max(1, (int)std::thread::hardware_concurrency()));
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

// One staged upload: a list of jobs (dst, pageable src, bytes, kind), cut
// into chunks that fill at most one kChunk slot; T host threads take every
// T-th chunk of the whole list, so several arrays stream without a join
// between them.  kind COPY: memcpy; kind PACK4: d = 4 bit tiles, four row
// bytes -> 16 bits (only the low nibbles may be set, formats.py:289).
enum { COPY = 0, PACK4 = 1, PACKB = 2 };
struct Job {
    void *dst;
    const void *src;
    size_t bytes;  // source bytes
    int kind;
    int bits = 0;  // PACKB: bits per u32 value (the column range of tile_col_ind)
};

// PACKB: n u32 values (n a multiple of 32, or the tail) packed at `bits` bits
// each: group g of 32 values -> words [g*bits, (g+1)*bits).  Returns the OR of
// the values' bits above `bits` (non-zero: a value does not fit -- the caller
// re-sends plainly so the device check reports it).
template <int BITS>
static uint32_t pack_bits_t(const uint32_t *in, size_t n, uint32_t *out) {
    constexpr uint32_t LIM = BITS == 32 ? 0u : ~0u << BITS;
    uint32_t over = 0;
    size_t g = 0;
    for (; g + 32 <= n; g += 32) {  // whole groups: every shift is a constant
        const uint32_t *v = in + g;
        uint32_t *o = out + (g / 32) * BITS;
        uint64_t acc = 0;
        int fill = 0, w = 0;
        for (int k = 0; k < 32; k++) {
            over |= v[k] & LIM;
            acc |= (uint64_t)v[k] << fill;
            fill += BITS;
            if (fill >= 32) {
                o[w++] = (uint32_t)acc;
                acc >>= 32;
                fill -= 32;
            }
        }
    }
    if (g < n) {  // the tail group
        uint32_t *o = out + (g / 32) * BITS;
        uint64_t acc = 0;
        int fill = 0, w = 0;
        for (size_t k = g; k < n; k++) {
            over |= in[k] & LIM;
            acc |= (uint64_t)in[k] << fill;
            fill += BITS;
            if (fill >= 32) {
                o[w++] = (uint32_t)acc;
                acc >>= 32;
                fill -= 32;
            }
        }
        if (fill > 0) o[w] = (uint32_t)acc;
    }
    return over;
}

// PACKB: n u32 values packed at `bits` bits each, group g of 32 values in
// words [g*bits, (g+1)*bits).  Returns the OR of the values' bits above `bits`
// (non-zero: a value does not fit -- the caller re-sends plainly so the device
// check reports it).
static uint32_t pack_bits(const uint32_t *in, size_t n, int bits, uint32_t *out) {
    switch (bits) {
#define PB(B) case B: return pack_bits_t<B>(in, n, out);
        PB(1) PB(2) PB(3) PB(4) PB(5) PB(6) PB(7) PB(8) PB(9) PB(10) PB(11) PB(12)
        PB(13) PB(14) PB(15) PB(16) PB(17) PB(18) PB(19) PB(20) PB(21) PB(22) PB(23) PB(24)
#undef PB
        default: return ~0u;  // not packed (the caller only asks for <= 24)
    }
}

static void staged(const std::vector<Job> &jobs, bool *high, cudaStream_t s) {
    struct Chunk {
        int job;
        size_t off;  // source offset
        size_t len;  // source bytes
    };
    std::vector<Chunk> chunks;
    for (int j = 0; j < (int)jobs.size(); j++) {
        // source bytes per chunk: the staged output fills at most one kChunk slot
        size_t step = kChunk;
        if (jobs[j].kind == PACK4) step = 2 * kChunk;
        if (jobs[j].kind == PACKB) step = (kChunk * 32 / jobs[j].bits) / 128 * 128;  // whole 32-value groups
        for (size_t off = 0; off < jobs[j].bytes; off += step)
            chunks.push_back({j, off, std::min(step, jobs[j].bytes - off)});
    }
    if (chunks.empty()) return;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    StagePool &P = pool(dev);
    std::lock_guard<std::mutex> lk(P.mu);
    P.init(copy_threads());
    const size_t nchunks = chunks.size();
    const int T = (int)std::min<size_t>(P.threads, nchunks);
    std::atomic<bool> hi{false};
    std::vector<std::exception_ptr> err(T);
    std::vector<std::string> msg(T);  // the error text is thread-local: carry it to the caller's thread
    auto worker = [&](int i) {
        try {
            CK(cudaSetDevice(dev));
            size_t round = 0;
            for (size_t c = i; c < nchunks; c += T, round++) {
                const int slot = i + P.threads * (int)(round & 1);
                const Chunk &ch = chunks[c];
                const Job &jb = jobs[ch.job];
                const char *from = (const char *)jb.src + ch.off;
                CK(cudaEventSynchronize(P.done[slot]));  // the slot's previous DMA has drained
                size_t out = ch.len, doff = ch.off;
                if (jb.kind == COPY) {
                    memcpy(P.buf[slot], from, ch.len);
                } else if (jb.kind == PACKB) {
                    const size_t n = ch.len / 4;
                    if (pack_bits(reinterpret_cast<const uint32_t *>(from), n, jb.bits, static_cast<uint32_t *>(P.buf[slot])))
                        hi.store(true, std::memory_order_relaxed);
                    out = ((n + 31) / 32) * (size_t)jb.bits * 4;  // whole groups (the tail group padded)
                    doff = (ch.off / 4 / 32) * (size_t)jb.bits * 4;
                } else {
                    const uint32_t *w = reinterpret_cast<const uint32_t *>(from);
                    uint16_t *o = static_cast<uint16_t *>(P.buf[slot]);
                    const size_t n = ch.len / 4;
                    uint32_t h = 0;
                    for (size_t k = 0; k < n; k++) {
                        const uint32_t v = w[k];
                        h |= v;
                        o[k] = (uint16_t)((v & 0xFu) | ((v >> 4) & 0xF0u) | ((v >> 8) & 0xF00u) | ((v >> 12) & 0xF000u));
                    }
                    if (h & 0xF0F0F0F0u) hi.store(true, std::memory_order_relaxed);
                    out = n * 2;
                    doff = ch.off / 2;
                }
                CK(cudaMemcpyAsync((char *)jb.dst + doff, P.buf[slot], out, cudaMemcpyHostToDevice, s));
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
    if (high) *high = hi.load();
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
    staged({{dst, src, bytes, COPY}}, nullptr, s);
}

// d = 4 bit tiles travel nibble-packed: 512 -> 256 MB over PCIe at R-MAT s22,
// widened again on the device.  A tile with a high nibble set (a FormatError
// the device check reports with the reference's message) is re-sent plainly.
__global__ void k_unpack_nibbles(uint64_t T, const uint16_t *__restrict__ in, uint32_t *__restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = in[t];
        out[t] = (p & 0xFu) | ((p & 0xF0u) << 4) | ((p & 0xF00u) << 8) | ((p & 0xF000u) << 12);
    }
}

// tile_col_ind travels at ceil(log2 ntr) bits per value (20 instead of 32 at
// R-MAT s22 d=4): group g of 32 values in words [g*bits, (g+1)*bits)
__global__ void k_unpack_bits(uint64_t T, int bits, const uint32_t *__restrict__ in, uint32_t *__restrict__ out) {
    const uint32_t mask = bits == 32 ? 0xFFFFFFFFu : (1u << bits) - 1u;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bit = (t >> 5) * (uint64_t)bits * 32 + (t & 31) * (uint64_t)bits;
        const uint64_t wi = bit >> 5;
        const uint32_t sh = (uint32_t)(bit & 31);
        uint64_t v = in[wi];
        if (sh + bits > 32) v |= (uint64_t)in[wi + 1] << 32;
        out[t] = (uint32_t)(v >> sh) & mask;
    }
}

// the three arrays of a host B2SR matrix in one staged upload
void upload_b2sr(b2sr_matrix *m, const uint32_t *h_trp, const uint32_t *h_tci, const void *h_tiles, cudaStream_t s) {
    const size_t trp_b = ((size_t)m->ntr + 1) * 4, tci_b = m->num_tiles * 4;
    const size_t tile_b = m->num_tiles * (size_t)m->dim * word_bytes(m->dim);
    const bool pinned = page_locked(h_tci);
    if (pinned || tci_b + tile_b < 4 * kDirect) {
        h2d(m->trp, h_trp, trp_b, s);
        h2d(m->tci, h_tci, tci_b, s);
        h2d(m->tiles, h_tiles, tile_b, s);
        return;
    }
    // B2SR_H2D_PACK (A/B): default tiles packed; "all": tiles and columns (bit-packed
    // tile_col_ind measured no faster on the box -- 22.3-27.0 vs 22.8-23.4 ms for
    // the s22 host matrix: the packing loop costs what the smaller DMA saves);
    // 0: plain copies (26.5-26.8 ms)
    const int pack_mode = [] {  // read per upload (tests switch it)
        const char *e = getenv("B2SR_H2D_PACK");
        return !e ? 2 : (e[0] == '0' ? 0 : (e[0] == 'a' ? 1 : 2));
    }();
    const bool pack_on = pack_mode != 0;
    const bool pack = pack_on && m->dim == 4 && !page_locked(h_tiles);  // B2SR_H2D_PACK=0: plain copy (A/B)
    // columns of a full matrix are < ntr: ceil(log2 ntr) bits each (a row block's too)
    const uint32_t ncols = tile_rows(m->n, m->dim);
    int cb = 1;
    while (cb < 32 && ((uint64_t)(ncols - 1) >> cb)) cb++;
    const bool packc = pack_mode == 1 && cb <= 24;
    const uint64_t T = m->num_tiles;
    Buf<uint16_t> packed(pack ? T : 1, s);
    Buf<uint32_t> packedc(packc ? ((T + 31) / 32) * cb + 1 : 1, s);
    std::vector<Job> jobs;
    if (trp_b < kDirect) CK(cudaMemcpyAsync(m->trp, h_trp, trp_b, cudaMemcpyHostToDevice, s));
    else jobs.push_back({m->trp, h_trp, trp_b, COPY});
    if (packc) jobs.push_back({packedc.p, h_tci, tci_b, PACKB, cb});
    else jobs.push_back({m->tci, h_tci, tci_b, COPY});
    if (pack) jobs.push_back({packed.p, h_tiles, tile_b, PACK4});
    else if (page_locked(h_tiles)) h2d(m->tiles, h_tiles, tile_b, s);
    else jobs.push_back({m->tiles, h_tiles, tile_b, COPY});
    bool high = false;  // a value did not fit its packed width: re-send plainly (the stream
    staged(jobs, &high, s);  // drains the packed buffers before their memory is reused)
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((T + 255) / 256, (uint64_t)num_sms() * 16));
    if (high) {
        if (packc) h2d(m->tci, h_tci, tci_b, s);
        if (pack) h2d(m->tiles, h_tiles, tile_b, s);
        return;
    }
    if (packc) LAUNCH(k_unpack_bits, g, 256, 0, s, T, cb, packedc.p, m->tci);
    if (pack) LAUNCH(k_unpack_nibbles, g, 256, 0, s, T, packed.p, static_cast<uint32_t *>(m->tiles));
}

}  // namespace b2sr

extern "C" int b2sr_h2d(void *d_dst, const void *h_src, uint64_t bytes, void *stream) {
    API_BEGIN
    b2sr::h2d(d_dst, h_src, bytes, (cudaStream_t)stream);
    API_END
}
