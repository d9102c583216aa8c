// Hot-column x cache for the bit-vector SpMV kernels (K4 bbb, BFS pull).
//
// On R-MAT the x gather, not the tile stream, bounds K4 at d <= 8: every tile
// needs one random byte of x, and a 32-lane gather of random bytes costs the
// L1 ~32 wavefronts (B300_MICROARCH.md "L1tex wavefront queue", ~1 cyc/wf),
// so 128 M tiles at s22 d=4 keep every SM's L1 busy for ~0.6 ms -- 4x the
// HBM time of the stream.  Column popularity is skewed (s22 d=4: the top 192 K
// of 1 M tile columns carry 85 % of the tiles), so the x words of the most
// referenced tile columns are staged in shared memory, where a random 32-lane
// byte gather costs a few bank cycles instead.
//
// Plan (built once per matrix, cached, immutable like the matrix):
//   cols[S]   the S tile columns with the most tiles (ties: lower column)
//   tci2[T]   per tile: its slot (< S) when the column is hot, else S + column
// Per call, k_hot_fill gathers hx[i] = x[cols[i]] (S words, a few us) and the
// kernels copy hx into shared memory before streaming the tiles.  When the
// whole x fits (S = number of tile columns), cols is the identity and tci2 is
// the matrix's own tci.  Nothing about the tiles or their order changes, so
// the outputs are exactly those of the plain kernels.
#include <map>
#include <mutex>
#include <unordered_map>

#include "bmv_common.cuh"

namespace b2sr {

struct HotPlan {
    uint32_t S = 0;             // hot slots (== column tile-rows when identity)
    bool identity = false;
    uint32_t *cols = nullptr;   // S tile columns (null when identity)
    uint32_t *tci2 = nullptr;   // T remapped column indices (m->tci when identity)
};

void free_hot(void *p) {
    HotPlan *h = static_cast<HotPlan *>(p);
    if (!h) return;
    dfree(h->cols, nullptr);
    if (!h->identity) dfree(h->tci2, nullptr);
    delete h;
}

__global__ void k_hot_col_hist(uint64_t T, const uint32_t *__restrict__ tci, uint32_t *__restrict__ cnt) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + tci[t], 1u);
}

// key = ~count so an ascending stable sort puts popular columns first
__global__ void k_hot_keys(uint32_t nc, const uint32_t *__restrict__ cnt, uint32_t *__restrict__ key,
                           uint32_t *__restrict__ col) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        key[c] = ~cnt[c];
        col[c] = c;
    }
}

__global__ void k_hot_slots(uint32_t S, const uint32_t *__restrict__ sorted_cols, uint32_t *__restrict__ cols,
                            uint32_t *__restrict__ slot_of) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
        uint32_t c = sorted_cols[i];
        cols[i] = c;
        slot_of[c] = i;
    }
}

__global__ void k_hot_remap(uint64_t T, uint32_t S, const uint32_t *__restrict__ tci,
                            const uint32_t *__restrict__ slot_of, uint32_t *__restrict__ tci2) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = tci[t], sl = slot_of[c];
        tci2[t] = sl != 0xFFFFFFFFu ? sl : S + c;
    }
}

static unsigned hgrid(uint64_t work) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)num_sms() * 16));
}

HotView hot_view(b2sr_matrix *m, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (!m->hot) {
        const uint32_t nc = tile_rows(m->n, m->dim);  // column tile space is global for row blocks
        const uint32_t wb = (uint32_t)word_bytes((int)m->dim);
        const char *e = getenv("B2SR_HOT_BYTES");     // parity tests force the remapped path on small graphs
        uint32_t budget = e ? (uint32_t)atoi(e) : HOT_SMEM_BYTES;
        uint32_t cap = (m->dim == 4 && HOT_NIBBLES) ? budget * 2 : budget / wb;  // d=4: two 4-bit words per byte
        HotPlan *h = new HotPlan();
        try {
            if (nc <= cap) {
                h->identity = true;
                h->S = nc;
                h->tci2 = m->tci;
            } else {
                h->S = cap;
                Buf<uint32_t> cnt(nc, s), key(nc, s), col(nc, s), slot_of(nc, s);
                CK(cudaMemsetAsync(cnt.p, 0, (size_t)nc * 4, s));
                if (m->num_tiles) LAUNCH(k_hot_col_hist, hgrid(m->num_tiles), 256, 0, s, m->num_tiles, m->tci, cnt.p);
                LAUNCH(k_hot_keys, hgrid(nc), 256, 0, s, nc, cnt.p, key.p, col.p);
                uint32_t *ko, *vo;
                Buf<uint32_t> kalt, valt;
                radix_sort_pairs_u32(key.p, col.p, nc, 32, s, &ko, &vo, &kalt, &valt);
                Buf<uint32_t> cols(h->S, s);
                CK(cudaMemsetAsync(slot_of.p, 0xFF, (size_t)nc * 4, s));
                LAUNCH(k_hot_slots, hgrid(h->S), 256, 0, s, h->S, vo, cols.p, slot_of.p);
                Buf<uint32_t> tci2(std::max<uint64_t>(m->num_tiles, 1), s);
                if (m->num_tiles)
                    LAUNCH(k_hot_remap, hgrid(m->num_tiles), 256, 0, s, m->num_tiles, h->S, m->tci, slot_of.p, tci2.p);
                h->cols = cols.release();
                h->tci2 = tci2.release();
                CK(cudaStreamSynchronize(s));  // scratch buffers die here
            }
        } catch (...) {
            free_hot(h);
            throw;
        }
        m->hot = h;
    }
    HotPlan *h = static_cast<HotPlan *>(m->hot);
    return HotView{h->S, h->cols, h->tci2};
}

template <typename W>
__global__ void k_hot_fill(uint32_t S, const uint32_t *__restrict__ cols, const W *__restrict__ x, W *__restrict__ hx) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
        hx[i] = x[cols ? cols[i] : i];
}

// d=4: slot pair (2i, 2i+1) shares byte i (low nibble = even slot)
__global__ void k_hot_fill4(uint32_t S, const uint32_t *__restrict__ cols, const uint8_t *__restrict__ x,
                            uint8_t *__restrict__ hx) {
    const uint32_t nb = (S + 1) / 2;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
        uint32_t a = 2 * i, b = 2 * i + 1;
        uint32_t lo = x[cols ? cols[a] : a] & 0xFu;
        uint32_t hi = b < S ? (x[cols ? cols[b] : b] & 0xFu) : 0u;
        hx[i] = (uint8_t)(lo | (hi << 4));
    }
}

static size_t hot_used_bytes(const HotView &hv, int dim) {
    return (dim == 4 && HOT_NIBBLES) ? ((size_t)hv.S + 1) / 2 : (size_t)hv.S * word_bytes(dim);
}

size_t hot_fill_bytes(const HotView &hv, int dim) { return (hot_used_bytes(hv, dim) + 15) / 16 * 16; }

void hot_fill(const HotView &hv, int dim, const void *x, void *hx, cudaStream_t s) {
    size_t b = hot_fill_bytes(hv, dim);
    size_t used = hot_used_bytes(hv, dim);
    if (b > used) CK(cudaMemsetAsync(static_cast<char *>(hx) + used, 0, b - used, s));
    unsigned g = hgrid(hv.S);
    if (dim == 4 && HOT_NIBBLES) {
        LAUNCH(k_hot_fill4, g, 256, 0, s, hv.S, hv.cols, (const uint8_t *)x, (uint8_t *)hx);
        return;
    }
    switch (word_bytes(dim)) {
        case 1: LAUNCH(k_hot_fill<uint8_t>, g, 256, 0, s, hv.S, hv.cols, (const uint8_t *)x, (uint8_t *)hx); break;
        case 2: LAUNCH(k_hot_fill<uint16_t>, g, 256, 0, s, hv.S, hv.cols, (const uint16_t *)x, (uint16_t *)hx); break;
        default: LAUNCH(k_hot_fill<uint32_t>, g, 256, 0, s, hv.S, hv.cols, (const uint32_t *)x, (uint32_t *)hx); break;
    }
}

void hot_smem_attr_raw(const void *kernel, size_t bytes) {
    static std::mutex mu;
    // (device, kernel) -> dynamic smem limit already set: the attribute is per
    // device context, so a second GPU in the same process sets its own
    static std::map<std::pair<int, const void *>, size_t> set;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t &cur = set[{dev, kernel}];
    if (bytes <= cur) return;
    size_t b = std::max<size_t>(bytes, HOT_SMEM_BYTES + 16);
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b));
    cur = b;
}

bool hot_enabled(int dim) {
    const char *e = getenv("B2SR_HOT");  // B2SR_HOT=0: plain L1/L2 gathers (A/B)
    if (e && e[0] == '0') return false;
    return dim <= 8;
}

}  // namespace b2sr
