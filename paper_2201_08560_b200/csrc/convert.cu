// K1/K2: CSR -> B2SR conversion on the device (replaces formats.py:444-464).
//
// The reference sorts all tile keys (r//d)*ntr + c//d with np.unique and ORs
// the bits in with np.bitwise_or.at.  Here a tile row I owns the contiguous
// col_ind segment of its d CSR rows, each already sorted, so its distinct
// tile columns are the d-way merge of the d runs of c//d:
//   * a group of d lanes takes one tile row (lane r = bit-row r), 32/d tile
//     rows per warp;
//   * each step the group min-reduces the current tile column (redux.sync
//     at d=32, shfl_xor below), the lanes sitting on that column consume
//     their run and build their row word, and one tile is emitted;
//   * K1 runs the loop counting tiles -> exclusive scan -> tile_row_ptr;
//     K2 re-runs it writing tile_col_ind and the bit rows.
// (Staging each warp's runs in shared memory first -- coalesced loads, merge
// steps on shared memory -- measured no faster at d = 4 (10.6 ms at s22 either
// way) and 8-10x slower at d = 16/32 (a third of the resident warps), so the
// merge reads its runs from global memory.)
// Long tile rows (hubs) are split into column ranges of ~CONV_CHUNK entries
// so no group walks a hub alone; the split points are found by binary
// search and the ranges' counts are scanned in order, so the layout is
// exactly the reference's (row-major tiles, ascending columns).
#include "b2sr_internal.cuh"

namespace b2sr {

constexpr uint32_t CONV_CHUNK = 1024;  // CSR entries per work item (target)
constexpr uint32_t INF32 = 0xFFFFFFFFu;

struct ConvItem {
    uint32_t row;   // tile row
    uint32_t klo;   // first tile column of this range
    uint32_t khi;   // one past the last tile column
    uint32_t pad;
};

// one item per tile row with <= whole entries, else ceil(e / chunk) column ranges
__global__ void k_conv_chunks(uint32_t n, uint32_t d, uint32_t ntr, const uint32_t *row_ptr, uint32_t *pcount,
                              uint32_t whole, uint32_t chunk) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= ntr) return;
    uint64_t r0 = (uint64_t)I * d, r1 = min((uint64_t)n, r0 + d);
    uint32_t e = row_ptr[r1] - row_ptr[r0];
    uint32_t p = e <= whole ? 1u : (e + chunk - 1) / chunk;
    pcount[I] = p ? p : 1u;
}

__global__ void k_conv_items(uint32_t ntr, const uint64_t *pofs, ConvItem *items) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= ntr) return;
    uint64_t b = pofs[I];
    uint32_t P = (uint32_t)(pofs[I + 1] - b);
    for (uint32_t j = 0; j < P; j++) {
        ConvItem it;
        it.row = I;
        it.klo = (uint32_t)((uint64_t)j * ntr / P);
        it.khi = (uint32_t)((uint64_t)(j + 1) * ntr / P);
        it.pad = 0;
        items[b + j] = it;
    }
}

template <int D>
__device__ __forceinline__ uint32_t group_min(uint32_t v) {
    if constexpr (D == 32) {
        return __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int o = D / 2; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o, D));
        return v;
    }
}

template <int D, bool PACK>
__global__ void __launch_bounds__(256) k_conv(const ConvItem *__restrict__ items, uint32_t n_items, uint32_t n,
                                              const uint32_t *__restrict__ row_ptr,
                                              const uint32_t *__restrict__ col_ind, const uint64_t *__restrict__ iofs,
                                              uint32_t *__restrict__ cnt, uint32_t *__restrict__ tci,
                                              typename WordT<D>::T *__restrict__ tiles,
                                              const uint32_t *__restrict__ order, const uint8_t *__restrict__ only,
                                              uint64_t *__restrict__ toff) {
    constexpr uint32_t GPW = 32 / D;  // groups (items) per warp
    const uint32_t lane = lane_id(), r = lane % D;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t wb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wb * GPW < n_items; wb += warps) {
        const uint32_t slot = wb * GPW + lane / D;
        bool valid = slot < n_items;
        uint32_t item = valid ? (order ? order[slot] : slot) : slot;
        if (valid && only && !only[item]) valid = false;  // the warp merge did this item
        ConvItem it = valid ? items[item] : ConvItem{0, 0, 0, 0};
        uint64_t row = (uint64_t)it.row * D + r;
        uint32_t p = 0, end = 0, rs = 0;
        if (valid && row < n) {
            p = rs = row_ptr[row];
            end = row_ptr[row + 1];
            if (it.klo > 0) {  // split range: first entry with c >= klo*D
                uint32_t key = it.klo * (uint32_t)D, a = p, b = end;
                while (a < b) {
                    uint32_t mid = (a + b) >> 1;
                    if (col_ind[mid] < key) a = mid + 1; else b = mid;
                }
                p = a;
            }
        }
        uint32_t c = 0, cur = INF32;
        if (p < end) {
            c = col_ind[p];
            if (c / D < it.khi) cur = c / D;
        }
        uint64_t t = 0;
        if (PACK && toff) {  // fused: the item's tiles go to its first CSR entry's slot of the staging arrays
            uint32_t skip = p - rs;
#pragma unroll
            for (int o = D / 2; o; o >>= 1) skip += __shfl_xor_sync(0xffffffffu, skip, o, D);
            t = (uint64_t)__shfl_sync(0xffffffffu, rs, 0, D) + skip;
        } else if (PACK && valid) {
            t = iofs[item];
        }
        const uint64_t t0 = t;
        uint32_t count = 0;
        while (__any_sync(0xffffffffu, cur != INF32)) {
            uint32_t K = group_min<D>(cur);
            uint32_t word = 0;
            while (cur == K && K != INF32) {  // consume this lane's run inside tile column K
                word |= 1u << (c % D);
                ++p;
                cur = INF32;
                if (p < end) {
                    c = col_ind[p];
                    uint32_t k = c / D;
                    if (k < it.khi) cur = k;
                }
            }
            if (K != INF32) {
                if constexpr (PACK) {
                    tiles[t * D + r] = (typename WordT<D>::T)word;
                    if (r == 0) tci[t] = K;
                }
                ++t;
                ++count;
            }
        }
        if (valid && r == 0 && (!PACK || toff)) {
            cnt[item] = count;
            if (PACK) toff[item] = t0;
        }
    }
}

// ------------------------------------------------------------ warp merge (d = 4, 8)
// One warp per item of <= CM_CAP CSR entries.  The item's d runs (one per
// bit-row, each sorted by column) are staged in shared memory as u32 values
// v = c << S | r (S = log2 d; needs n <= 2^(32-S)), then merged pairwise in
// S levels -- each element finds its place in the merged pair with one binary
// search of the partner run (values are distinct: no ties) -- which sorts
// the item by (c, r), hence by tile column k = c >> S.  A ballot over "k
// differs from the previous element" numbers the tiles; K1 counts them, K2
// writes tile_col_ind at the first element of each tile and ORs every
// element's bit into a shared-memory tile buffer that is then stored with
// coalesced 32-bit stores.  Per element that is S searches of a ~30-entry run
// instead of the per-step group min of the lock-step merge, whose warps loop
// until their longest of 8 tile rows is done (ncu, s22 d=4: 2.13 G warp
// instructions per pass).  Items over CM_CAP entries (hub rows cut into column
// ranges that came out long) go to the lock-step merge above.
constexpr uint32_t CM_CAP = 512;

template <int D>
struct ConvMerge {
    static constexpr uint32_t S = D == 4 ? 2 : 3;
    static constexpr uint32_t NW = D == 4 ? 8 : 4;        // warps per CTA (32 KB static shared memory)
    static constexpr uint32_t TW = D == 4 ? 1 : 2;        // u32 words per tile
    static constexpr uint32_t TBUF = D == 4 ? 0 : 2 * CM_CAP;  // d = 8: separate tile buffer
};

template <int D, bool PACK>
__global__ void __launch_bounds__(ConvMerge<D>::NW * 32) k_conv_merge(
    const ConvItem *__restrict__ items, uint32_t n_items, uint32_t n, const uint32_t *__restrict__ row_ptr,
    const uint32_t *__restrict__ col_ind, const uint64_t *__restrict__ iofs, uint32_t *__restrict__ cnt,
    uint32_t *__restrict__ tci, uint32_t *__restrict__ tiles32, uint8_t *__restrict__ big,
    uint64_t *__restrict__ toff) {
    using CMt = ConvMerge<D>;
    constexpr uint32_t S = CMt::S, NW = CMt::NW, TW = CMt::TW;
    __shared__ uint32_t buf[NW][2][CM_CAP];
    __shared__ uint32_t tbuf[NW][CMt::TBUF ? CMt::TBUF : 1];
    __shared__ uint32_t soff[NW][D + 1];
    __shared__ uint32_t sst[NW][D];
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t *off = soff[wid], *st = sst[wid];
    for (uint32_t item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < n_items; item += warps) {
        const ConvItem it = items[item];
        // run r = bit-row r of tile row it.row, restricted to tile columns [klo, khi)
        uint32_t p0 = 0, p1 = 0, rs = 0;
        if (lane < (uint32_t)D) {
            const uint64_t row = (uint64_t)it.row * D + lane;
            if (row < n) {
                p0 = rs = row_ptr[row];
                p1 = row_ptr[row + 1];
                if (it.klo > 0) {
                    uint32_t a = p0, b = p1;
                    const uint32_t key = it.klo * (uint32_t)D;
                    while (a < b) { const uint32_t m = (a + b) >> 1; if (__ldg(col_ind + m) < key) a = m + 1; else b = m; }
                    p0 = a;
                }
                if ((uint64_t)it.khi * D < n) {
                    uint32_t a = p0, b = p1;
                    const uint32_t key = it.khi * (uint32_t)D;
                    while (a < b) { const uint32_t m = (a + b) >> 1; if (__ldg(col_ind + m) < key) a = m + 1; else b = m; }
                    p1 = a;
                }
            }
        }
        const uint32_t len = p1 - p0;
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < D; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        const uint32_t E = __shfl_sync(0xffffffffu, incl, D - 1);
        if (E > CM_CAP) {  // the lock-step merge takes it
            if ((!PACK || toff) && lane == 0) big[item] = 1;
            continue;
        }
        // fused mode: this item's tiles go to the slot of its first CSR entry
        // (an item has at most as many tiles as entries, so the items' slot
        // ranges of the staging arrays are disjoint)
        const uint64_t tslot = toff ? (uint64_t)__shfl_sync(0xffffffffu, rs, 0) +
                                          __reduce_add_sync(0xffffffffu, p0 - rs)
                                    : 0;
        __syncwarp();  // the previous item's readers of off/st are done
        if (lane < (uint32_t)D) {
            off[lane + 1] = incl;
            st[lane] = p0;
        }
        if (lane == 0) off[0] = 0;
        __syncwarp();
        // stage: element i of run r (CSR index st[r] + i - off[r]) -> c << S | r
        uint32_t *X = buf[wid][0], *Y = buf[wid][1];
        for (uint32_t i0 = 0; i0 < E; i0 += 128) {  // four loads in flight per lane
            uint32_t v[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t i = i0 + j * 32 + lane;
                uint32_t r = 0;
#pragma unroll
                for (int q = 1; q < D; q++) r += off[q] <= i;
                v[j] = i < E ? (__ldg(col_ind + st[r] + (i - off[r])) << S) | r : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t i = i0 + j * 32 + lane;
                if (i < E) X[i] = v[j];
            }
        }
        __syncwarp();
        // S pairwise merge levels: level l merges runs of 2^l bit-rows in pairs
#pragma unroll
        for (uint32_t l = 0; l < S; l++) {
            for (uint32_t i = lane; i < E; i += 32) {
                const uint32_t v = X[i];
                // the value carries its bit-row r, and the level-l run holding
                // element i is the one of runs [j << l, (j + 1) << l), j = r >> l
                const uint32_t j = (v & (D - 1)) >> l;       // level-l run of element i
                const uint32_t a = off[j << l];              // its start
                const uint32_t pj = j ^ 1u;                  // partner run
                const uint32_t pa = off[pj << l], pb = off[min((pj + 1) << l, (uint32_t)D)];
                const uint32_t ms = off[(j & ~1u) << l];     // merged run start
                uint32_t lo = pa, hi = pb;
                while (lo < hi) { const uint32_t m = (lo + hi) >> 1; if (X[m] < v) lo = m + 1; else hi = m; }
                Y[ms + (i - a) + (lo - pa)] = v;
            }
            __syncwarp();
            uint32_t *t = X; X = Y; Y = t;
        }
        // X: sorted by (c, r).  Tiles = runs of equal k = v >> 2S.
        if constexpr (PACK) {
            uint32_t *T = CMt::TBUF ? tbuf[wid] : Y;
            for (uint32_t q = lane; q < E * TW; q += 32) T[q] = 0;
            __syncwarp();
            const uint64_t tb = toff ? tslot : iofs[item];
            uint32_t run = 0;
            for (uint32_t base = 0; base < E; base += 32) {
                const uint32_t i = base + lane;
                const uint32_t v = i < E ? X[i] : 0u;
                const uint32_t k = v >> (2 * S);
                const bool first = i < E && (i == 0 || (X[i - 1] >> (2 * S)) != k);
                const uint32_t fm = __ballot_sync(0xffffffffu, first);
                const uint32_t t = run + __popc(fm & lt_mask) + (first ? 1u : 0u) - 1u;  // tile of element i
                if (i < E) {
                    const uint32_t r = v & (D - 1), c = (v >> S) & (D - 1);
                    if (first) tci[tb + t] = k;
                    // tile word: row r in byte r (d = 8: two u32 words per tile)
                    atomicOr(T + t * TW + (r >> 2), 1u << (8 * (r & 3) + c));
                }
                run += __popc(fm);
            }
            __syncwarp();
            uint32_t *dst = tiles32 + tb * TW;
            for (uint32_t q = lane; q < run * TW; q += 32) dst[q] = T[q];
            if (toff && lane == 0) {
                cnt[item] = run;
                toff[item] = tb;
            }
        } else {
            uint32_t run = 0;
            for (uint32_t base = 0; base < E; base += 32) {
                const uint32_t i = base + lane;
                const bool first = i < E && (i == 0 || (X[i - 1] >> (2 * S)) != (X[i] >> (2 * S)));
                run += __popc(__ballot_sync(0xffffffffu, first));
            }
            if (lane == 0) cnt[item] = run;
        }
    }
}

__global__ void k_conv_trp(uint32_t ntr, const uint64_t *pofs, const uint64_t *iofs, uint32_t *trp) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I <= ntr) trp[I] = (uint32_t)iofs[pofs[I]];
}

template <int D>
static void conv_launch(bool pack, const ConvItem *items, uint32_t n_items, uint32_t n, const uint32_t *row_ptr,
                        const uint32_t *col_ind, const uint64_t *iofs, uint32_t *cnt, uint32_t *tci, void *tiles,
                        cudaStream_t s, const uint32_t *order, const uint8_t *only, uint64_t *toff) {
    constexpr uint32_t GPW = 32 / D;
    uint64_t warps = (n_items + GPW - 1) / GPW;
    uint64_t blocks = (warps + 7) / 8;
    uint64_t cap = (uint64_t)num_sms() * 8;  // 8 CTAs x 8 warps per SM, grid-stride beyond
    unsigned g = (unsigned)(blocks < cap ? blocks : cap);
    if (pack)
        LAUNCH((k_conv<D, true>), g, 256, 0, s, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci,
               (typename WordT<D>::T *)tiles, order, only, toff);
    else
        LAUNCH((k_conv<D, false>), g, 256, 0, s, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci,
               (typename WordT<D>::T *)tiles, order, only, nullptr);
}

static void conv_dispatch(uint32_t d, bool pack, const ConvItem *items, uint32_t n_items, uint32_t n,
                          const uint32_t *row_ptr, const uint32_t *col_ind, const uint64_t *iofs, uint32_t *cnt,
                          uint32_t *tci, void *tiles, cudaStream_t s, const uint32_t *order = nullptr,
                          const uint8_t *only = nullptr, uint64_t *toff = nullptr) {
    switch (d) {
        case 4: conv_launch<4>(pack, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci, tiles, s, order, only, toff); break;
        case 8: conv_launch<8>(pack, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci, tiles, s, order, only, toff); break;
        case 16: conv_launch<16>(pack, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci, tiles, s, order, only, toff); break;
        default: conv_launch<32>(pack, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci, tiles, s, order, only, toff); break;
    }
}

// K1 for the warp-merge items: the tile count of an item is the number of
// DISTINCT tile columns among its entries, which needs no sorted order: each
// warp inserts its item's tile columns into a 1024-slot shared-memory hash set
// (linear probing, atomicCAS) and counts the successful inserts.  Entries of
// one run with the same tile column as their predecessor are skipped first
// (runs are sorted).  About a dozen instructions per entry instead of the
// log2 d merge levels (K2 still merges: it needs the order).
constexpr uint32_t CH_SLOTS = 1024;  // >= 2 * CM_CAP: load factor <= 1/2

template <int D>
__global__ void __launch_bounds__(256) k_conv_count_hash(const ConvItem *__restrict__ items, uint32_t n_items, uint32_t n,
                                                        const uint32_t *__restrict__ row_ptr,
                                                        const uint32_t *__restrict__ col_ind, uint32_t *__restrict__ cnt,
                                                        uint8_t *__restrict__ big) {
    constexpr uint32_t S = D == 4 ? 2 : 3;
    __shared__ uint32_t hset[8][CH_SLOTS];
    __shared__ uint32_t soff[8][D + 1];
    __shared__ uint32_t sst[8][D];
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    uint32_t *H = hset[wid], *off = soff[wid], *st = sst[wid];
    for (uint32_t q = lane; q < CH_SLOTS; q += 32) H[q] = 0;
    for (uint32_t item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < n_items; item += warps) {
        const ConvItem it = items[item];
        uint32_t p0 = 0, p1 = 0;
        if (lane < (uint32_t)D) {
            const uint64_t row = (uint64_t)it.row * D + lane;
            if (row < n) {
                p0 = row_ptr[row];
                p1 = row_ptr[row + 1];
                if (it.klo > 0) {
                    uint32_t a = p0, b = p1;
                    const uint32_t key = it.klo * (uint32_t)D;
                    while (a < b) { const uint32_t m = (a + b) >> 1; if (__ldg(col_ind + m) < key) a = m + 1; else b = m; }
                    p0 = a;
                }
                if ((uint64_t)it.khi * D < n) {
                    uint32_t a = p0, b = p1;
                    const uint32_t key = it.khi * (uint32_t)D;
                    while (a < b) { const uint32_t m = (a + b) >> 1; if (__ldg(col_ind + m) < key) a = m + 1; else b = m; }
                    p1 = a;
                }
            }
        }
        const uint32_t len = p1 - p0;
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < D; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        const uint32_t E = __shfl_sync(0xffffffffu, incl, D - 1);
        if (E > CM_CAP) {  // the lock-step merge takes it
            if (lane == 0) big[item] = 1;
            continue;
        }
        __syncwarp();
        if (lane < (uint32_t)D) {
            off[lane + 1] = incl;
            st[lane] = p0;
        }
        if (lane == 0) off[0] = 0;
        __syncwarp();
        uint32_t count = 0;
        for (uint32_t i = lane; i < E; i += 32) {
            uint32_t r = 0;
#pragma unroll
            for (int q = 1; q < D; q++) r += off[q] <= i;
            const uint32_t g = st[r] + (i - off[r]);
            const uint32_t k = __ldg(col_ind + g) >> S;
            if (i > off[r] && (__ldg(col_ind + g - 1) >> S) == k) continue;  // same tile as the run's previous entry
            uint32_t h = (k * 0x9E3779B1u) >> (32 - 10);
            for (;;) {
                const uint32_t old = atomicCAS(H + h, 0u, k + 1);
                if (old == 0) { count++; break; }
                if (old == k + 1) break;
                h = (h + 1) & (CH_SLOTS - 1);
            }
        }
        count = __reduce_add_sync(0xffffffffu, count);
        __syncwarp();
        for (uint32_t q = lane; q < CH_SLOTS; q += 32) H[q] = 0;
        if (lane == 0) cnt[item] = count;
    }
}

template <int D>
static void merge_launch(bool pack, const ConvItem *items, uint32_t n_items, uint32_t n, const uint32_t *row_ptr,
                         const uint32_t *col_ind, const uint64_t *iofs, uint32_t *cnt, uint32_t *tci, void *tiles,
                         uint8_t *big, cudaStream_t s, uint64_t *toff = nullptr) {
    constexpr uint32_t NW = ConvMerge<D>::NW;
    int per_sm = 1;
    if (pack) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conv_merge<D, true>, NW * 32, 0));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conv_merge<D, false>, NW * 32, 0));
    const unsigned g = (unsigned)std::min<uint64_t>(((uint64_t)n_items + NW - 1) / NW,
                                                    (uint64_t)num_sms() * std::max(per_sm, 1));
    if (pack)
        LAUNCH((k_conv_merge<D, true>), g, NW * 32, 0, s, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci,
               (uint32_t *)tiles, big, toff);
    else
        LAUNCH((k_conv_merge<D, false>), g, NW * 32, 0, s, items, n_items, n, row_ptr, col_ind, iofs, cnt, tci,
               (uint32_t *)tiles, big, nullptr);
}

// warp merge for d = 4, 8 (B2SR_CONV_MERGE=0: lock-step merge only, A/B)
static bool conv_merge_enabled(uint32_t n, uint32_t d) {
    const char *e = getenv("B2SR_CONV_MERGE");
    if (e && e[0] == '0') return false;
    return (d == 4 && n <= (1u << 30)) || (d == 8 && n <= (1u << 29));
}

// Optionally, items sorted by their (estimated) CSR entry count, so the GPW items a warp
// merges in lock-step have similar lengths: the warp loops until its LONGEST
// item is done, and on R-MAT a random group of 8 tile rows (d = 4) is
// dominated by one long row (ncu, s22 d=4: 2.13 G warp instructions for the
// count pass, issue-bound).  Output offsets follow the items' own order, so
// the layout does not depend on the processing order.
__global__ void k_conv_item_len(uint32_t n_items, uint32_t n, uint32_t d, const ConvItem *__restrict__ items,
                                const uint32_t *__restrict__ row_ptr, const uint64_t *__restrict__ pofs,
                                uint32_t *__restrict__ key, uint32_t *__restrict__ val) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += gridDim.x * blockDim.x) {
        const ConvItem it = items[i];
        const uint64_t r0 = (uint64_t)it.row * d, r1 = min((uint64_t)n, r0 + d);
        const uint32_t e = row_ptr[r1] - row_ptr[r0];
        const uint32_t P = (uint32_t)(pofs[it.row + 1] - pofs[it.row]);
        key[i] = min(0xFFFFu, e / P);
        val[i] = i;
    }
}

// Measured slower (s22 d=4: 8.6 vs 6.3 ms): the sort costs more than the
// imbalance it removes, and neighbouring tile rows no longer share cache
// lines.  Off by default; B2SR_CONV_SORT=1 enables it (A/B).
static bool conv_sorted() {
    const char *e = getenv("B2SR_CONV_SORT");
    return e && e[0] == '1';
}

// fused conversion, last step: each item's tiles move from the slot of its
// first CSR entry in the staging arrays to their place in the matrix (a warp
// per item, coalesced 4-byte copies; tiles are TW u32 words)
template <int TW>
__global__ void __launch_bounds__(256) k_conv_compact(uint32_t n_items, const uint64_t *__restrict__ toff,
                                                      const uint64_t *__restrict__ iofs,
                                                      const uint32_t *__restrict__ stci,
                                                      const uint32_t *__restrict__ stiles, uint32_t *__restrict__ tci,
                                                      uint32_t *__restrict__ tiles) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < n_items; item += warps) {
        const uint64_t src = toff[item], dst = iofs[item];
        const uint32_t c = (uint32_t)(iofs[item + 1] - dst);
        // all loads of a 128-tile step in flight before the stores (a plain
        // strided loop waited one DRAM round trip per 32 tiles: 0.67 ms at s22)
        for (uint32_t base = 0; base < c; base += 128) {
            uint32_t a[4], b[4 * TW];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t q = base + j * 32 + lane;
                if (q < c) a[j] = stci[src + q];
            }
#pragma unroll
            for (int j = 0; j < 4 * TW; j++) {
                const uint32_t q = base * TW + j * 32 + lane;
                if (q < c * TW) b[j] = stiles[src * TW + q];
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t q = base + j * 32 + lane;
                if (q < c) tci[dst + q] = a[j];
            }
#pragma unroll
            for (int j = 0; j < 4 * TW; j++) {
                const uint32_t q = base * TW + j * 32 + lane;
                if (q < c * TW) tiles[dst * TW + q] = b[j];
            }
        }
    }
}

// B2SR_CONV_FUSED=0 (A/B): count pass, then pack straight into the matrix
static bool conv_fused_enabled() {
    const char *e = getenv("B2SR_CONV_FUSED");
    return !(e && e[0] == '0');
}

b2sr_matrix *csr_to_b2sr_device(uint32_t n, uint32_t d, const uint32_t *row_ptr, const uint32_t *col_ind,
                                cudaStream_t s) {
    uint32_t ntr = tile_rows(n, d);
    Buf<uint32_t> pcount(ntr, s);
    Buf<uint64_t> pofs((size_t)ntr + 1, s);
    const bool merge = conv_merge_enabled(n, d);
    // warp merge: whole tile rows up to CM_CAP entries, longer ones in ranges of ~CM_CAP/2
    LAUNCH(k_conv_chunks, (ntr + 255) / 256, 256, 0, s, n, d, ntr, row_ptr, pcount.p, merge ? CM_CAP : CONV_CHUNK,
           merge ? CM_CAP / 2 : CONV_CHUNK);
    exclusive_scan_u32_to_u64(pcount.p, pofs.p, ntr, s);
    uint64_t n_items64 = read_scalar(pofs.p + ntr, s);
    if (n_items64 > 0xFFFFFFFFull) B2SR_THROW(B2SR_EINVAL, "too many conversion work items");
    uint32_t n_items = (uint32_t)n_items64;
    Buf<ConvItem> items(n_items, s);
    LAUNCH(k_conv_items, (ntr + 255) / 256, 256, 0, s, ntr, pofs.p, items.p);
    Buf<uint32_t> order_k, order_v, kalt, valt;
    uint32_t *order = nullptr;
    if (conv_sorted() && n_items > 1) {
        order_k = Buf<uint32_t>(n_items, s);
        order_v = Buf<uint32_t>(n_items, s);
        LAUNCH(k_conv_item_len, (unsigned)std::min<uint64_t>((n_items + 255) / 256, (uint64_t)num_sms() * 8), 256, 0, s,
               n_items, n, d, items.p, row_ptr, pofs.p, order_k.p, order_v.p);
        uint32_t *ko = nullptr, *vo = nullptr;
        radix_sort_pairs_u32(order_k.p, order_v.p, n_items, 16, s, &ko, &vo, &kalt, &valt);
        order = vo;
    }
    Buf<uint32_t> cnt(n_items, s);
    Buf<uint64_t> iofs((size_t)n_items + 1, s);
    Buf<uint8_t> big;
    // d = 16 too (lock-step merge only): its count pass is a whole second
    // merge, the staging costs 36 bytes per CSR entry (bounded below); at
    // d = 32 (132 bytes per entry) moving the staged tiles costs what it saves
    const uint64_t nnz = (merge || d == 16) && conv_fused_enabled() && !order ? read_scalar(row_ptr + n, s) : 0;
    const uint32_t TWc = d == 4 ? 1 : d == 8 ? 2 : 8;  // u32 words per tile
    if ((merge || (d == 16 && nnz * (4 + 4 * TWc) <= (24ull << 30))) && conv_fused_enabled() && !order) {
        // one merge pass: pack every item into staging arrays at the slot of its
        // first CSR entry (tiles <= entries), counting its tiles; scan; move
        // the items' tiles into the matrix.  Replaces the count pass.
        const uint32_t TW = TWc;
        Buf<uint32_t> stci(std::max<uint64_t>(nnz, 1), s), stiles(std::max<uint64_t>(nnz, 1) * TW, s);
        Buf<uint64_t> toff(std::max<uint32_t>(n_items, 1), s);
        if (merge) {
            big = Buf<uint8_t>(std::max<uint32_t>(n_items, 1), s);
            CK(cudaMemsetAsync(big.p, 0, n_items, s));
            if (d == 4) merge_launch<4>(true, items.p, n_items, n, row_ptr, col_ind, nullptr, cnt.p, stci.p, stiles.p, big.p, s, toff.p);
            else merge_launch<8>(true, items.p, n_items, n, row_ptr, col_ind, nullptr, cnt.p, stci.p, stiles.p, big.p, s, toff.p);
        }
        conv_dispatch(d, true, items.p, n_items, n, row_ptr, col_ind, nullptr, cnt.p, stci.p, stiles.p, s, nullptr,
                      merge ? big.p : nullptr, toff.p);
        exclusive_scan_u32_to_u64(cnt.p, iofs.p, n_items, s);
        uint64_t T = read_scalar(iofs.p + n_items, s);
        if (T > 0xFFFFFFFFull) B2SR_THROW(B2SR_EFORMAT, "tile count exceeds 32-bit index range");
        b2sr_matrix *m = new_matrix(n, d, ntr, T, s);
        try {
            LAUNCH(k_conv_trp, (ntr + 256) / 256, 256, 0, s, ntr, pofs.p, iofs.p, m->trp);
            if (T) {
                const unsigned g = (unsigned)std::min<uint64_t>(((uint64_t)n_items + 7) / 8, (uint64_t)num_sms() * 8);
                if (d == 4) LAUNCH(k_conv_compact<1>, g, 256, 0, s, n_items, toff.p, iofs.p, stci.p, stiles.p, m->tci, (uint32_t *)m->tiles);
                else if (d == 8) LAUNCH(k_conv_compact<2>, g, 256, 0, s, n_items, toff.p, iofs.p, stci.p, stiles.p, m->tci, (uint32_t *)m->tiles);
                else LAUNCH(k_conv_compact<8>, g, 256, 0, s, n_items, toff.p, iofs.p, stci.p, stiles.p, m->tci, (uint32_t *)m->tiles);
            }
        } catch (...) {
            free_matrix(m);
            throw;
        }
        return m;
    }
    if (merge) {
        big = Buf<uint8_t>(std::max<uint32_t>(n_items, 1), s);
        CK(cudaMemsetAsync(big.p, 0, n_items, s));
        // K1: distinct tile columns counted through a shared-memory hash set
        // (B2SR_CONV_COUNT=merge: the merge kernel's count pass, A/B)
        const char *ce = getenv("B2SR_CONV_COUNT");
        if (ce && ce[0] == 'm') {
            if (d == 4) merge_launch<4>(false, items.p, n_items, n, row_ptr, col_ind, nullptr, cnt.p, nullptr, nullptr, big.p, s);
            else merge_launch<8>(false, items.p, n_items, n, row_ptr, col_ind, nullptr, cnt.p, nullptr, nullptr, big.p, s);
        } else {
            const unsigned g = (unsigned)std::min<uint64_t>(((uint64_t)n_items + 7) / 8, (uint64_t)num_sms() * 6);
            if (d == 4) LAUNCH(k_conv_count_hash<4>, g, 256, 0, s, items.p, n_items, n, row_ptr, col_ind, cnt.p, big.p);
            else LAUNCH(k_conv_count_hash<8>, g, 256, 0, s, items.p, n_items, n, row_ptr, col_ind, cnt.p, big.p);
        }
    }
    conv_dispatch(d, false, items.p, n_items, n, row_ptr, col_ind, nullptr, cnt.p, nullptr, nullptr, s, order,
                  merge ? big.p : nullptr);
    exclusive_scan_u32_to_u64(cnt.p, iofs.p, n_items, s);
    uint64_t T = read_scalar(iofs.p + n_items, s);
    if (T > 0xFFFFFFFFull) B2SR_THROW(B2SR_EFORMAT, "tile count exceeds 32-bit index range");
    b2sr_matrix *m = new_matrix(n, d, ntr, T, s);
    try {
        LAUNCH(k_conv_trp, (ntr + 256) / 256, 256, 0, s, ntr, pofs.p, iofs.p, m->trp);
        if (T && merge) {
            if (d == 4) merge_launch<4>(true, items.p, n_items, n, row_ptr, col_ind, iofs.p, nullptr, m->tci, m->tiles, big.p, s);
            else merge_launch<8>(true, items.p, n_items, n, row_ptr, col_ind, iofs.p, nullptr, m->tci, m->tiles, big.p, s);
        }
        if (T) conv_dispatch(d, true, items.p, n_items, n, row_ptr, col_ind, iofs.p, nullptr, m->tci, m->tiles, s, order,
                             merge ? big.p : nullptr);
    } catch (...) {
        free_matrix(m);
        throw;
    }
    return m;
}

// ------------------------------------------------------------ sampling profiler
// sample_profile (profile.py:73-127): the tiles that the sampled tile rows
// would store at width d, counted by the K1 merge loop over just those rows
// (same chunked work items, so hub rows are split), plus their CSR entries.
__global__ void k_prof_chunks(uint32_t n, uint32_t d, const uint32_t *rows, uint32_t m, const uint32_t *row_ptr,
                              uint32_t *pcount, unsigned long long *nnz) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e = 0;
    if (i < m) {
        uint64_t r0 = (uint64_t)rows[i] * d, r1 = min((uint64_t)n, r0 + d);
        e = row_ptr[r1] - row_ptr[r0];
        uint32_t p = (e + CONV_CHUNK - 1) / CONV_CHUNK;
        pcount[i] = p ? p : 1u;
    }
    e = __reduce_add_sync(0xffffffffu, e);  // distinct rows: the sum is <= nnz < 2^32
    if (lane_id() == 0 && e) atomicAdd(nnz, (unsigned long long)e);
}

__global__ void k_prof_items(uint32_t ntr, const uint32_t *rows, uint32_t m, const uint64_t *pofs, ConvItem *items) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    uint64_t b = pofs[i];
    uint32_t P = (uint32_t)(pofs[i + 1] - b);
    for (uint32_t j = 0; j < P; j++)
        items[b + j] = ConvItem{rows[i], (uint32_t)((uint64_t)j * ntr / P), (uint32_t)((uint64_t)(j + 1) * ntr / P), 0};
}

__global__ void k_sum_u32(uint32_t n, const uint32_t *v, unsigned long long *out) {
    unsigned long long acc = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += v[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0 && acc) atomicAdd(out, acc);
}

}  // namespace b2sr

using namespace b2sr;

extern "C" int b2sr_profile_rows(uint32_t n, uint32_t dim, const uint32_t *d_row_ptr, const uint32_t *d_col_ind,
                                 const uint32_t *d_rows, uint32_t m, uint64_t *tiles, uint64_t *nnz, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (dim != 4 && dim != 8 && dim != 16 && dim != 32) B2SR_THROW(B2SR_EINVAL, "tile dim must be 4/8/16/32");
    *tiles = 0;
    *nnz = 0;
    if (n == 0 || m == 0) return B2SR_OK;
    const uint32_t ntr = tile_rows(n, dim);
    Buf<uint32_t> pcount(m, s);
    Buf<uint64_t> pofs((size_t)m + 1, s);
    Buf<unsigned long long> acc(2, s);
    CK(cudaMemsetAsync(acc.p, 0, 16, s));
    LAUNCH(k_prof_chunks, (m + 255) / 256, 256, 0, s, n, dim, d_rows, m, d_row_ptr, pcount.p, acc.p + 1);
    exclusive_scan_u32_to_u64(pcount.p, pofs.p, m, s);
    uint64_t n_items64 = read_scalar(pofs.p + m, s);
    if (n_items64 > 0xFFFFFFFFull) B2SR_THROW(B2SR_EINVAL, "too many profiling work items");
    const uint32_t n_items = (uint32_t)n_items64;
    Buf<ConvItem> items(n_items, s);
    LAUNCH(k_prof_items, (m + 255) / 256, 256, 0, s, ntr, d_rows, m, pofs.p, items.p);
    Buf<uint32_t> cnt(n_items, s);
    conv_dispatch(dim, false, items.p, n_items, n, d_row_ptr, d_col_ind, nullptr, cnt.p, nullptr, nullptr, s);
    unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_items + 255) / 256, (uint64_t)num_sms() * 8));
    LAUNCH(k_sum_u32, g, 256, 0, s, n_items, cnt.p, acc.p);
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *tiles = h[0];
    *nnz = h[1];
    API_END
}

extern "C" int b2sr_from_csr(uint32_t n, uint32_t dim, const uint32_t *d_row_ptr, const uint32_t *d_col_ind,
                             uint64_t nnz, void *stream, b2sr_matrix **out) {
    API_BEGIN
    (void)nnz;
    if (dim != 4 && dim != 8 && dim != 16 && dim != 32) B2SR_THROW(B2SR_EINVAL, "tile dim must be 4/8/16/32");
    if (n == 0) B2SR_THROW(B2SR_EFORMAT, "cannot tile an empty matrix");
    *out = csr_to_b2sr_device(n, dim, d_row_ptr, d_col_ind, (cudaStream_t)stream);
    API_END
}
