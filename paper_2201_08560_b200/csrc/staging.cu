// Host -> device uploads from pageable memory at the PCIe rate.
//
// A caller of the drop-in API hands over plain numpy arrays (pageable
// memory).  cudaMemcpyAsync from pageable memory goes through the driver's
// own small bounce buffer and runs far below the link rate (11 GB/s on the
// B200 box), and pinning the caller's pages in place costs more than it saves
// (cudaHostRegister of 1 GB: 146 ms, tools/h2d_probe.py).  Large uploads are
// staged instead: the upload is cut into chunks of <= 16 MB staged output and
// T host threads take the next free chunk, each with two page-locked slots of
// a per-device pool --
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

#if defined(__x86_64__) && !defined(__CUDA_ARCH__)
#include <immintrin.h>
#define B2SR_NT_STAGING 1
#endif

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
// into chunks that fill at most one kChunk slot; T host threads take the
// next chunk of the whole list, so several arrays stream without a join
// between them.  kind COPY: memcpy; kind PACK4: d = 4 bit tiles, four row
// bytes -> 16 bits (only the low nibbles may be set, formats.py:289).
enum { COPY = 0, PACK4 = 1, PACKB = 2, SPLIT = 3 };
struct Job {
    void *dst;
    const void *src;
    size_t bytes;  // source bytes
    int kind;
    int bits = 0;  // PACKB / SPLIT: bits per u32 value (the column range of tile_col_ind)
    void *dst2 = nullptr;  // SPLIT: the high parts
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

#ifdef B2SR_NT_STAGING
// The staging slots are written once and only read by the DMA engine:
// streaming (non-temporal) stores skip the read-for-ownership a plain store
// pays on every slot line, a third of the host-memory traffic of a packed
// chunk (B2SR_H2D_NT=0: plain memcpy / scalar pack, A/B).
static bool nt_enabled() {
    static const bool on = [] {
        const char *e = getenv("B2SR_H2D_NT");
        return !(e && e[0] == '0');
    }();
    return on;
}

// dst 16-byte aligned (a slot), src any alignment
static void copy_nt(void *dst, const void *src, size_t n) {
    __m128i *d = static_cast<__m128i *>(dst);
    const __m128i *q = static_cast<const __m128i *>(src);
    size_t k = 0, v = n / 16;
    for (; k + 4 <= v; k += 4) {
        const __m128i a = _mm_loadu_si128(q + k), b = _mm_loadu_si128(q + k + 1);
        const __m128i c = _mm_loadu_si128(q + k + 2), e = _mm_loadu_si128(q + k + 3);
        _mm_stream_si128(d + k, a);
        _mm_stream_si128(d + k + 1, b);
        _mm_stream_si128(d + k + 2, c);
        _mm_stream_si128(d + k + 3, e);
    }
    for (; k < v; k++) _mm_stream_si128(d + k, _mm_loadu_si128(q + k));
    if (n % 16) memcpy(static_cast<char *>(dst) + v * 16, static_cast<const char *>(src) + v * 16, n % 16);
}

// PACK4 with SSSE3: per u32 of four row bytes, maddubs by (1, 16) gives
// (b0 | b1 << 4, b2 | b3 << 4) as two 16-bit lanes <= 255, packus keeps their
// low bytes: the u16 b0 | b1 << 4 | b2 << 8 | b3 << 12.  Returns the OR of the
// inputs (the caller checks the high nibbles).
__attribute__((target("ssse3"))) static uint32_t pack4_nt(const uint32_t *w, size_t n, uint16_t *o) {
    const __m128i K = _mm_set1_epi16(0x1001);  // bytes (1, 16)
    __m128i h = _mm_setzero_si128();
    size_t k = 0;
    for (; k + 8 <= n; k += 8) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + k));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + k + 4));
        h = _mm_or_si128(h, _mm_or_si128(a, b));
        _mm_stream_si128(reinterpret_cast<__m128i *>(o + k), _mm_packus_epi16(_mm_maddubs_epi16(a, K), _mm_maddubs_epi16(b, K)));
    }
    uint32_t hs[4];
    _mm_storeu_si128(reinterpret_cast<__m128i *>(hs), h);
    uint32_t hv = hs[0] | hs[1] | hs[2] | hs[3];
    for (; k < n; k++) {
        const uint32_t v = w[k];
        hv |= v;
        o[k] = (uint16_t)((v & 0xFu) | ((v >> 4) & 0xF0u) | ((v >> 8) & 0xF00u) | ((v >> 12) & 0xF000u));
    }
    return hv;
}

// SPLIT (bits <= 24): each u32 value -> its low 16 bits (u16 stream, streaming
// stores) + its bits 16..bits-1 (bits <= 20: a nibble per value, two per byte;
// else a byte per value).  Returns the OR of the values (the caller checks the
// bits above `bits`).
__attribute__((target("ssse3"))) static uint32_t split_nt(const uint32_t *w, size_t n, bool nib, uint16_t *lo,
                                                          uint8_t *hi) {
    const __m128i SLO = _mm_setr_epi8(0, 1, 4, 5, 8, 9, 12, 13, -1, -1, -1, -1, -1, -1, -1, -1);
    const __m128i SHI = _mm_setr_epi8(2, 6, 10, 14, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1);
    const __m128i K = _mm_set1_epi16(0x1001);
    __m128i acc = _mm_setzero_si128();
    size_t k = 0;
    for (; k + 8 <= n; k += 8) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + k));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + k + 4));
        acc = _mm_or_si128(acc, _mm_or_si128(a, b));
        _mm_stream_si128(reinterpret_cast<__m128i *>(lo + k),
                         _mm_unpacklo_epi64(_mm_shuffle_epi8(a, SLO), _mm_shuffle_epi8(b, SLO)));
        const __m128i h8 = _mm_unpacklo_epi32(_mm_shuffle_epi8(a, SHI), _mm_shuffle_epi8(b, SHI));  // 8 bytes
        if (nib) {
            const __m128i p = _mm_packus_epi16(_mm_maddubs_epi16(h8, K), _mm_setzero_si128());  // 4 bytes
            const uint32_t v = (uint32_t)_mm_cvtsi128_si32(p);
            memcpy(hi + k / 2, &v, 4);
        } else {
            _mm_storel_epi64(reinterpret_cast<__m128i *>(hi + k), h8);
        }
    }
    uint32_t as[4];
    _mm_storeu_si128(reinterpret_cast<__m128i *>(as), acc);
    uint32_t o = as[0] | as[1] | as[2] | as[3];
    for (; k < n; k++) {  // the tail (k even here: nibble pairs start fresh)
        const uint32_t v = w[k];
        o |= v;
        lo[k] = (uint16_t)v;
        const uint8_t h = (uint8_t)(v >> 16);
        if (!nib) hi[k] = h;
        else if (k & 1) hi[k / 2] |= (uint8_t)((h & 0xF) << 4);
        else hi[k / 2] = (uint8_t)(h & 0xF);
    }
    return o;
}
#endif

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
        if (jobs[j].kind == SPLIT) step = ((kChunk - 64) / 3 * 4) / 64 * 64;  // <= 3 output bytes per value + padding
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
    std::atomic<size_t> next{0};  // chunks are taken in list order by whichever thread is free
    std::vector<std::exception_ptr> err(T);
    std::vector<std::string> msg(T);  // the error text is thread-local: carry it to the caller's thread
    auto worker = [&](int i) {
        try {
            CK(cudaSetDevice(dev));
            size_t round = 0;
            for (size_t c; (c = next.fetch_add(1, std::memory_order_relaxed)) < nchunks; round++) {
                const int slot = i + P.threads * (int)(round & 1);
                const Chunk &ch = chunks[c];
                const Job &jb = jobs[ch.job];
                const char *from = (const char *)jb.src + ch.off;
                CK(cudaEventSynchronize(P.done[slot]));  // the slot's previous DMA has drained
                size_t out = ch.len, doff = ch.off;
                if (jb.kind == COPY) {
#ifdef B2SR_NT_STAGING
                    if (nt_enabled()) copy_nt(P.buf[slot], from, ch.len);
                    else
#endif
                        memcpy(P.buf[slot], from, ch.len);
#ifdef B2SR_NT_STAGING
                } else if (jb.kind == SPLIT) {
                    const size_t n = ch.len / 4, v0 = ch.off / 4;
                    const bool nib = jb.bits <= 20;
                    uint16_t *lo = static_cast<uint16_t *>(P.buf[slot]);
                    uint8_t *hp = static_cast<uint8_t *>(P.buf[slot]) + ((n * 2 + 63) & ~size_t(63));
                    if (split_nt(reinterpret_cast<const uint32_t *>(from), n, nib, lo, hp) >> jb.bits)
                        hi.store(true, std::memory_order_relaxed);
                    _mm_sfence();
                    CK(cudaMemcpyAsync((uint16_t *)jb.dst + v0, lo, n * 2, cudaMemcpyHostToDevice, s));
                    if (jb.bits > 16)
                        CK(cudaMemcpyAsync((uint8_t *)jb.dst2 + (nib ? v0 / 2 : v0), hp, nib ? (n + 1) / 2 : n,
                                           cudaMemcpyHostToDevice, s));
                    CK(cudaEventRecord(P.done[slot], s));
                    continue;
#endif
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
#ifdef B2SR_NT_STAGING
                    if (nt_enabled()) h = pack4_nt(w, n, o);
                    else
#endif
                        for (size_t k = 0; k < n; k++) {
                            const uint32_t v = w[k];
                            h |= v;
                            o[k] = (uint16_t)((v & 0xFu) | ((v >> 4) & 0xF0u) | ((v >> 8) & 0xF00u) | ((v >> 12) & 0xF000u));
                        }
                    if (h & 0xF0F0F0F0u) hi.store(true, std::memory_order_relaxed);
                    out = n * 2;
                    doff = ch.off / 2;
                }
#ifdef B2SR_NT_STAGING
                _mm_sfence();  // the streaming stores are weakly ordered: drain them before the DMA reads the slot
#endif
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

// SPLIT columns: low 16 bits + bits 16.. as a nibble (hb <= 4) or a byte
__global__ void k_unpack_split(uint64_t T, int hb, const uint16_t *__restrict__ lo, const uint8_t *__restrict__ hi,
                               uint32_t *__restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = 0;
        if (hb > 4) h = hi[t];
        else if (hb > 0) h = (hi[t >> 1] >> ((t & 1) * 4)) & 0xFu;
        out[t] = (uint32_t)lo[t] | (h << 16);
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
    // B2SR_H2D_PACK (A/B): default tiles packed and tile_col_ind split into a u16
    // stream + 4 or 8 high bits (SIMD, streaming stores); "tiles": tiles only;
    // "all": tiles and columns bit-packed by a scalar loop (no faster than
    // "tiles": 22.3-27.0 vs 22.8-23.4 ms for the s22 host matrix, the loop
    // costs what the smaller DMA saves); 0: plain copies (26.5-26.8 ms)
    const int pack_mode = [] {  // read per upload (tests switch it)
        const char *e = getenv("B2SR_H2D_PACK");
        return !e ? 3 : (e[0] == '0' ? 0 : (e[0] == 'a' ? 1 : (e[0] == 't' ? 2 : 3)));
    }();
    const bool pack_on = pack_mode != 0;
    const bool pack = pack_on && m->dim == 4 && !page_locked(h_tiles);  // B2SR_H2D_PACK=0: plain copy (A/B)
    // columns of a full matrix are < ntr: ceil(log2 ntr) bits each (a row block's too)
    const uint32_t ncols = tile_rows(m->n, m->dim);
    int cb = 1;
    while (cb < 32 && ((uint64_t)(ncols - 1) >> cb)) cb++;
    const bool packc = pack_mode == 1 && cb <= 24;
#ifdef B2SR_NT_STAGING
    const bool split = pack_mode == 3 && cb <= 24 && nt_enabled();
#else
    const bool split = false;
#endif
    const int hb = cb > 16 ? cb - 16 : 0;  // high bits per column: 0, a nibble (<= 4) or a byte
    const uint64_t T = m->num_tiles;
    Buf<uint16_t> packed(pack ? T : 1, s);
    Buf<uint32_t> packedc(packc ? ((T + 31) / 32) * cb + 1 : 1, s);
    Buf<uint16_t> slo(split ? T : 1, s);
    Buf<uint8_t> shi(split && hb ? (hb <= 4 ? (T + 1) / 2 : T) : 1, s);
    std::vector<Job> jobs;
    if (trp_b < kDirect) CK(cudaMemcpyAsync(m->trp, h_trp, trp_b, cudaMemcpyHostToDevice, s));
    else jobs.push_back({m->trp, h_trp, trp_b, COPY});
    if (packc) jobs.push_back({packedc.p, h_tci, tci_b, PACKB, cb});
    else if (split) jobs.push_back({slo.p, h_tci, tci_b, SPLIT, std::max(cb, 16), shi.p});
    else jobs.push_back({m->tci, h_tci, tci_b, COPY});
    if (pack) jobs.push_back({packed.p, h_tiles, tile_b, PACK4});
    else if (page_locked(h_tiles)) h2d(m->tiles, h_tiles, tile_b, s);
    else jobs.push_back({m->tiles, h_tiles, tile_b, COPY});
    bool high = false;  // a value did not fit its packed width: re-send plainly (the stream
    staged(jobs, &high, s);  // drains the packed buffers before their memory is reused)
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((T + 255) / 256, (uint64_t)num_sms() * 16));
    if (high) {
        if (packc || split) h2d(m->tci, h_tci, tci_b, s);
        if (pack) h2d(m->tiles, h_tiles, tile_b, s);
        return;
    }
    if (packc) LAUNCH(k_unpack_bits, g, 256, 0, s, T, cb, packedc.p, m->tci);
    if (split) LAUNCH(k_unpack_split, g, 256, 0, s, T, hb, slo.p, shi.p, m->tci);
    if (pack) LAUNCH(k_unpack_nibbles, g, 256, 0, s, T, packed.p, static_cast<uint32_t *>(m->tiles));
}

}  // namespace b2sr

extern "C" int b2sr_h2d(void *d_dst, const void *h_src, uint64_t bytes, void *stream) {
    API_BEGIN
    b2sr::h2d(d_dst, h_src, bytes, (cudaStream_t)stream);
    API_END
}
