// K3 tile transpose (formats.py:477-489), b2sr_to_csr (formats.py:467-474),
// diagonal drop in tile form (algorithms.py:96-101, 111).
//
// Transpose = stable radix sort of (tile column, tile id) + a gather that
// bit-transposes each tile in registers (Hacker's-Delight block swaps, one
// thread per tile, 16-byte loads/stores of whole tiles).  The reference
// unpacks every tile into a (T, d, d) uint64 temporary (~16*d^2 bytes per
// tile); here the working set is 16 bytes of indices per tile.
#include <type_traits>

#include "b2sr_internal.cuh"

namespace b2sr {

// In-register transpose of a D x D bit tile, row r = a[r], LSB = column 0.
template <int D>
__device__ __forceinline__ void bit_transpose(uint32_t (&a)[D]) {
    uint32_t m = (D == 32) ? 0x0000FFFFu : (D == 16) ? 0x00FFu : (D == 8) ? 0x0Fu : 0x3u;
#pragma unroll
    for (int j = D / 2; j; j >>= 1) {
#pragma unroll
        for (int k = 0; k < D; k = (k + j + 1) & ~j) {
            uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k] ^= t << j;
            a[k + j] ^= t;
        }
        m ^= m << (j / 2);
    }
}

template <int D>
__device__ __forceinline__ void load_tile(const void *tiles, size_t t, uint32_t (&a)[D]) {
    if constexpr (D == 32) {
        const uint4 *p = reinterpret_cast<const uint4 *>(tiles) + t * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            uint4 v = __ldg(p + i);
            a[4 * i] = v.x; a[4 * i + 1] = v.y; a[4 * i + 2] = v.z; a[4 * i + 3] = v.w;
        }
    } else if constexpr (D == 16) {
        const uint4 *p = reinterpret_cast<const uint4 *>(tiles) + t * 2;
#pragma unroll
        for (int i = 0; i < 2; i++) {
            uint4 v = __ldg(p + i);
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; k++) { a[8 * i + 2 * k] = w[k] & 0xFFFFu; a[8 * i + 2 * k + 1] = w[k] >> 16; }
        }
    } else if constexpr (D == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2 *>(tiles) + t);
#pragma unroll
        for (int k = 0; k < 4; k++) { a[k] = (v.x >> (8 * k)) & 0xFFu; a[4 + k] = (v.y >> (8 * k)) & 0xFFu; }
    } else {
        uint32_t v = __ldg(reinterpret_cast<const uint32_t *>(tiles) + t);
#pragma unroll
        for (int k = 0; k < 4; k++) a[k] = (v >> (8 * k)) & 0xFFu;
    }
}

template <int D>
__device__ __forceinline__ void store_tile(void *tiles, size_t t, const uint32_t (&a)[D]) {
    if constexpr (D == 32) {
        uint4 *p = reinterpret_cast<uint4 *>(tiles) + t * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) p[i] = make_uint4(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]);
    } else if constexpr (D == 16) {
        uint4 *p = reinterpret_cast<uint4 *>(tiles) + t * 2;
#pragma unroll
        for (int i = 0; i < 2; i++)
            p[i] = make_uint4(a[8 * i] | (a[8 * i + 1] << 16), a[8 * i + 2] | (a[8 * i + 3] << 16),
                              a[8 * i + 4] | (a[8 * i + 5] << 16), a[8 * i + 6] | (a[8 * i + 7] << 16));
    } else if constexpr (D == 8) {
        uint2 v;
        v.x = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
        v.y = a[4] | (a[5] << 8) | (a[6] << 16) | (a[7] << 24);
        reinterpret_cast<uint2 *>(tiles)[t] = v;
    } else {
        reinterpret_cast<uint32_t *>(tiles)[t] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
    }
}


__global__ void k_u64_to_u32(const uint64_t *in, uint32_t *out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// one warp per tile row: rowid[t] = I for t in [trp[I], trp[I+1])
__global__ void k_row_ids(uint32_t ntr, const uint32_t *trp, uint32_t *rowid) {
    uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < ntr; I += warps)
        for (uint32_t t = trp[I] + lane_id(); t < trp[I + 1]; t += 32) rowid[t] = I;
}

__global__ void k_iota(uint32_t *v, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

template <int D>
__global__ void __launch_bounds__(256) k_transpose_gather(uint64_t T, const uint32_t *__restrict__ order,
                                                          const uint32_t *__restrict__ rowid,
                                                          const void *__restrict__ tiles, uint32_t *__restrict__ tci_out,
                                                          void *__restrict__ tiles_out) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < T; p += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t t = order[p];
        tci_out[p] = rowid[t];
        uint32_t a[D];
        load_tile<D>(tiles, t, a);
        bit_transpose<D>(a);
        store_tile<D>(tiles_out, p, a);
    }
}

// d=4 fast path: a 4x4 tile is 16 bits of payload, so (column | row | tile)
// fits one 64-bit key and a stable radix sort over the column bits carries
// every tile to its transposed position -- no random gathers afterwards.
// (a warp per tile row without the row-id array measured 2.8 vs 0.7 ms at s22:
// a hub row of ~10^5 tiles serialises on one warp)
__global__ void k_pack4(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                        const uint32_t *__restrict__ tiles, int cb, uint64_t *__restrict__ keys) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = tiles[t];  // four row bytes, low nibbles
        const uint32_t nib = (w & 0xFu) | ((w >> 4) & 0xF0u) | ((w >> 8) & 0xF00u) | ((w >> 12) & 0xF000u);
        keys[t] = (uint64_t)tci[t] | ((uint64_t)rowid[t] << cb) | ((uint64_t)nib << (2 * cb));
    }
}

// k_pack4 without the row-id array: a CTA packs PK_TILES consecutive tiles and
// recovers their rows from tile_row_ptr in shared memory.  Q(x) = #{r in
// [1, ntr] : trp[r] <= x} is the row of tile x; the rows that start inside the
// CTA's range are r in (Q(t0), Q(t0 + PK_TILES - 1)], each adds one at its
// start position, and an inclusive scan over the positions gives every tile's
// row (empty rows add at the same position: no special case).  Saves the row-id
// pass (a 4-byte write and read per tile).
constexpr int PK_THREADS = 256, PK_PER = 8, PK_TILES = PK_THREADS * PK_PER;
static_assert(PK_TILES == RADIX_TILE, "the first digit's counts are per radix tile");

__global__ void k_pack4_bounds(uint64_t T, uint32_t ntr, const uint32_t *__restrict__ trp, uint32_t nb,
                               uint32_t *__restrict__ q) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const uint64_t t0 = (uint64_t)b * PK_TILES, te = min(T - 1, t0 + PK_TILES - 1);
    for (int k = 0; k < 2; k++) {
        const uint64_t x = k ? te : t0;
        uint32_t lo = 1, hi = ntr + 1;  // first r in [1, ntr] with trp[r] > x
        while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            if (trp[m] <= x) lo = m + 1; else hi = m;
        }
        q[2 * b + k] = lo - 1;
    }
}

// D = 4: key = column | row << cb | 16-bit tile << 2 cb; D = 8: key = column |
// row << cb and the 8-byte tile goes to vals
template <int D>
__global__ void __launch_bounds__(PK_THREADS) k_pack_rows(uint64_t T, const uint32_t *__restrict__ trp,
                                                          const uint32_t *__restrict__ q,
                                                          const uint32_t *__restrict__ tci,
                                                          const void *__restrict__ tiles_, int cb,
                                                          uint64_t *__restrict__ keys, uint64_t *__restrict__ vals,
                                                          uint32_t *__restrict__ counts0, uint32_t dm0) {
    // D >= 16: no tile payload -- vals (u32) take the tile id, the tile is
    // gathered after the sort (one 32 / 128-byte read per tile)
    using TW = typename std::conditional<D == 4, uint32_t, uint64_t>::type;  // one tile (D = 4, 8)
    const TW *__restrict__ tiles = static_cast<const TW *>(tiles_);
    constexpr bool IDS = D >= 16;
    __shared__ uint32_t cnt[PK_TILES];
    __shared__ uint32_t hist[256];  // the first radix pass's digit counts of this tile
    __shared__ uint32_t wsum[PK_THREADS / 32];
    const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
    const uint64_t t0 = (uint64_t)blockIdx.x * PK_TILES;
    for (int j = 0; j < PK_PER; j++) cnt[j * PK_THREADS + tid] = 0;
    hist[tid] = 0;
    // this CTA's tiles: loads issued before the row recovery
    uint32_t c[PK_PER];
    TW v[PK_PER];
    const uint64_t tb = t0 + tid * PK_PER;
    if (tb + PK_PER <= T) {  // 32-byte aligned: 16-byte loads
        const uint4 c0 = reinterpret_cast<const uint4 *>(tci + tb)[0], c1 = reinterpret_cast<const uint4 *>(tci + tb)[1];
        c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w; c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
        if constexpr (IDS) {
#pragma unroll
            for (int j = 0; j < PK_PER; j++) v[j] = 0;
        } else if constexpr (D == 4) {
            const uint4 v0 = reinterpret_cast<const uint4 *>(tiles + tb)[0], v1 = reinterpret_cast<const uint4 *>(tiles + tb)[1];
            v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w; v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
        } else {
#pragma unroll
            for (int j = 0; j < PK_PER / 2; j++) {
                const ulonglong2 x = reinterpret_cast<const ulonglong2 *>(tiles + tb)[j];
                v[2 * j] = x.x;
                v[2 * j + 1] = x.y;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < PK_PER; j++) {
            const uint64_t t = tb + j;
            c[j] = t < T ? tci[t] : 0u;
            v[j] = (t < T && !IDS) ? tiles[t] : (TW)0;
        }
    }
    __syncthreads();
    const uint32_t qa = q[2 * blockIdx.x], qb = q[2 * blockIdx.x + 1];
    for (uint32_t r = qa + 1 + tid; r <= qb; r += PK_THREADS) atomicAdd(&cnt[trp[r] - t0], 1u);
    __syncthreads();
    // inclusive scan over the positions: thread tid owns positions [tid*8, tid*8+8)
    uint32_t loc[PK_PER], run = 0;
#pragma unroll
    for (int j = 0; j < PK_PER; j++) {
        run += cnt[tid * PK_PER + j];
        loc[j] = run;
    }
    uint32_t inc = run;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t off = inc - run;
    for (uint32_t ww = 0; ww < w; ww++) off += wsum[ww];
#pragma unroll
    for (int j = 0; j < PK_PER; j++)
        if (tb + j < T) atomicAdd(&hist[c[j] & dm0], 1u);
    uint64_t k[PK_PER];
#pragma unroll
    for (int j = 0; j < PK_PER; j++) {
        const uint32_t row = qa + off + loc[j];
        k[j] = (uint64_t)c[j] | ((uint64_t)row << cb);
        if constexpr (D == 4) {
            const uint32_t x = v[j];
            const uint32_t nib = (x & 0xFu) | ((x >> 4) & 0xF0u) | ((x >> 8) & 0xF00u) | ((x >> 12) & 0xF000u);
            k[j] |= (uint64_t)nib << (2 * cb);
        }
    }
    if (tb + PK_PER <= T) {
        ulonglong2 *o = reinterpret_cast<ulonglong2 *>(keys + tb);
#pragma unroll
        for (int j = 0; j < PK_PER / 2; j++) o[j] = make_ulonglong2(k[2 * j], k[2 * j + 1]);
        if constexpr (D == 8) {
            ulonglong2 *ov = reinterpret_cast<ulonglong2 *>(vals + tb);
#pragma unroll
            for (int j = 0; j < PK_PER / 2; j++) ov[j] = make_ulonglong2(v[2 * j], v[2 * j + 1]);
        } else if constexpr (IDS) {
            uint4 *ov = reinterpret_cast<uint4 *>(reinterpret_cast<uint32_t *>(vals) + tb);
            const uint32_t t32 = (uint32_t)tb;
            ov[0] = make_uint4(t32, t32 + 1, t32 + 2, t32 + 3);
            ov[1] = make_uint4(t32 + 4, t32 + 5, t32 + 6, t32 + 7);
        }
    } else {
#pragma unroll
        for (int j = 0; j < PK_PER; j++)
            if (tb + j < T) {
                keys[tb + j] = k[j];
                if constexpr (D == 8) vals[tb + j] = v[j];
                if constexpr (IDS) reinterpret_cast<uint32_t *>(vals)[tb + j] = (uint32_t)(tb + j);
            }
    }
    __syncthreads();
    counts0[(size_t)tid * gridDim.x + blockIdx.x] = hist[tid];
}

static bool tr8_sort_enabled() {  // B2SR_TR8=gather: (column, tile id) sort + random gathers (A/B)
    const char *e = getenv("B2SR_TR8");
    return !(e && !strcmp(e, "gather"));
}

static bool pack_rows_enabled() {  // B2SR_TR_PACK=rowid: the row-id array + k_pack4 (A/B)
    const char *e = getenv("B2SR_TR_PACK");
    return !(e && !strcmp(e, "rowid"));
}

// tile_row_ptr of the transpose from the column-sorted keys: position p starts
// every column in (column of p-1, column of p]; the last position closes the
// columns up to ntr (replaces a column histogram of T global atomics + scan)
template <typename K>
__device__ __forceinline__ void trp_bounds(uint64_t p, uint64_t T, K key, K prev, K mask, uint32_t ntr,
                                           uint32_t *__restrict__ trp_out) {
    const uint32_t c = (uint32_t)(key & mask);
    const uint32_t c0 = p ? (uint32_t)(prev & mask) + 1u : 0u;
    for (uint32_t q = c0; q <= c; q++) trp_out[q] = (uint32_t)p;
    if (p + 1 == T)
        for (uint32_t q = c + 1; q <= ntr; q++) trp_out[q] = (uint32_t)T;
}

// d >= 16 after a (column | row, tile id) sort: the row comes with the key,
// only the tile is gathered
template <int D>
__global__ void __launch_bounds__(256) k_transpose_gather_ids(uint64_t T, const uint64_t *__restrict__ keys,
                                                              const uint32_t *__restrict__ ids, int cb, uint32_t ntr,
                                                              const void *__restrict__ tiles,
                                                              uint32_t *__restrict__ trp_out,
                                                              uint32_t *__restrict__ tci_out,
                                                              void *__restrict__ tiles_out) {
    const uint64_t mask = (1ull << cb) - 1;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < T; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[p];
        const uint32_t t = ids[p];
        uint32_t a[D];
        load_tile<D>(tiles, t, a);
        trp_bounds<uint64_t>(p, T, k, p ? keys[p - 1] : 0ull, mask, ntr, trp_out);
        tci_out[p] = (uint32_t)((k >> cb) & mask);
        bit_transpose<D>(a);
        store_tile<D>(tiles_out, p, a);
    }
}

__global__ void k_trp_sorted(uint64_t T, const uint32_t *__restrict__ cols, uint32_t ntr, uint32_t *__restrict__ trp_out) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < T; p += (uint64_t)gridDim.x * blockDim.x)
        trp_bounds<uint32_t>(p, T, cols[p], p ? cols[p - 1] : 0u, 0xFFFFFFFFu, ntr, trp_out);
}

__global__ void k_unpack4(uint64_t T, const uint64_t *__restrict__ keys, int cb, uint32_t ntr,
                          uint32_t *__restrict__ trp_out, uint32_t *__restrict__ tci_out,
                          uint32_t *__restrict__ tiles_out) {
    const uint64_t mask = (1ull << cb) - 1;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < T; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[p];
        trp_bounds<uint64_t>(p, T, k, p ? keys[p - 1] : 0ull, mask, ntr, trp_out);
        tci_out[p] = (uint32_t)((k >> cb) & mask);  // the source row is the transposed column
        uint32_t nib = (uint32_t)(k >> (2 * cb));
        uint32_t a[4] = {nib & 0xFu, (nib >> 4) & 0xFu, (nib >> 8) & 0xFu, (nib >> 12) & 0xFu};
        bit_transpose<4>(a);
        tiles_out[p] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
    }
}

// ------------------------------------------------------------ two-level transpose (d = 4, 8)
// A stable counting sort of the tiles by column in two levels, the column cut
// into a high digit (HB bits: <= 2048 buckets) and a low digit (LB bits: <=
// 2048 columns per bucket):
//   A  each of G CTAs histograms the high digit over its contiguous tile range;
//      one scan gives every (bucket, CTA) its output start;
//   B  the same CTAs walk their ranges in sub-tiles of TR_SUB tiles in order:
//      tile rows are recovered from tile_row_ptr in shared memory (row starts
//      counted per sub-tile position, one block scan), elements (column | row
//      | tile) are ranked stably by high digit (__match_any_sync, per-warp
//      counters), staged by digit and written to their bucket with coalesced
//      runs -- the bucket then holds its elements in input (row-major) order;
//   C  one CTA per bucket: per-warp low-digit counts over its segment, one
//      scan over the bucket's columns (which is also tile_row_ptr of the
//      transpose), then each warp places its segment stably (match_any again)
//      and stores the row as the new tile column and the bit-transposed tile.
// HBM traffic: tci read twice, tiles once, 8 (d=4) / 16 (d=8) bytes per tile
// written and read twice -- against the three 8-bit LSD passes (each a
// histogram read plus a read and a write of 8-byte keys) plus pack and unpack
// passes and a column histogram of global atomics.
void hot_smem_attr_raw(const void *kernel, size_t bytes);  // hot.cu: opt-in dynamic shared memory

constexpr int TR_THREADS = 256, TR_WARPS = TR_THREADS / 32;
constexpr int TR_SUB = 2048, TR_PER = TR_SUB / TR_THREADS;  // tiles per sub-tile / per thread
constexpr int TR_MAXB = 2048;                                 // digit range

template <int D> struct TrElem;
template <> struct TrElem<4> {  // col | row << cb | 16-bit nibble tile << 2cb
    static constexpr bool PAY = false;
};
template <> struct TrElem<8> {  // key col | row << cb, payload: the 8-byte tile
    static constexpr bool PAY = true;
};

__device__ __forceinline__ uint32_t nib16(uint32_t w) {
    return (w & 0xFu) | ((w >> 4) & 0xF0u) | ((w >> 8) & 0xF00u) | ((w >> 12) & 0xF000u);
}

__global__ void __launch_bounds__(TR_THREADS) k_tr_hist(uint64_t T, uint32_t G, const uint32_t *__restrict__ tci,
                                                        int lb, uint32_t nb, uint32_t *__restrict__ hcnt) {
    __shared__ uint32_t h[TR_MAXB];
    for (uint32_t b = threadIdx.x; b < nb; b += TR_THREADS) h[b] = 0;
    __syncthreads();
    const uint64_t t0 = T * blockIdx.x / G, t1 = T * (blockIdx.x + 1) / G;
    for (uint64_t t = t0 + threadIdx.x; t < t1; t += TR_THREADS) atomicAdd(&h[__ldg(tci + t) >> lb], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += TR_THREADS) hcnt[(size_t)b * G + blockIdx.x] = h[b];
}

// largest r in [0, ntr) with trp[r] <= t
__device__ __forceinline__ uint32_t tr_row_of(const uint32_t *__restrict__ trp, uint32_t ntr, uint64_t t) {
    uint32_t lo = 0, hi = ntr - 1;
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo + 1) / 2;
        if (trp[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <int D>
__global__ void __launch_bounds__(TR_THREADS) k_tr_scatter(uint64_t T, uint32_t G, uint32_t ntr,
                                                           const uint32_t *__restrict__ trp,
                                                           const uint32_t *__restrict__ tci,
                                                           const void *__restrict__ tiles, int cb, int lb, uint32_t nb,
                                                           const uint64_t *__restrict__ hofs,
                                                           unsigned long long *__restrict__ ekey,
                                                           unsigned long long *__restrict__ epay) {
    extern __shared__ __align__(16) unsigned char tr_smem[];
    unsigned long long *skey = reinterpret_cast<unsigned long long *>(tr_smem);      // TR_SUB
    unsigned long long *spay = skey + TR_SUB;                                         // TR_SUB (d = 8)
    unsigned long long *pos = spay + (TrElem<D>::PAY ? TR_SUB : 0);                  // nb: next output slot
    uint32_t *rowc = reinterpret_cast<uint32_t *>(pos + nb);                          // TR_SUB + 1
    uint32_t *dbase = rowc + TR_SUB + 1;                                              // nb
    uint16_t *wc = reinterpret_cast<uint16_t *>(dbase + nb);                          // TR_WARPS * nb
    __shared__ uint32_t wsum[TR_WARPS];
    __shared__ uint32_t s_flag, s_row;
    const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5, lt = (1u << lane) - 1u;
    const uint64_t t_begin = T * blockIdx.x / G, t_end = T * (blockIdx.x + 1) / G;
    for (uint32_t b = tid; b < nb; b += TR_THREADS) pos[b] = hofs[(size_t)b * G + blockIdx.x];
    if (tid == 0) s_row = t_begin < t_end ? tr_row_of(trp, ntr, t_begin) : 0u;
    __syncthreads();
    uint32_t rcur = s_row;
    for (uint64_t t0 = t_begin; t0 < t_end; t0 += TR_SUB) {
        const uint32_t cnt = (uint32_t)min((uint64_t)TR_SUB, t_end - t0);
        // rows: rowc[p] = number of tile rows after rcur starting at or before t0 + p
        for (uint32_t q = tid; q <= TR_SUB; q += TR_THREADS) rowc[q] = 0;
        for (uint32_t b = tid; b < TR_WARPS * nb; b += TR_THREADS) wc[b] = 0;
        __syncthreads();
        for (uint32_t r = rcur + 1;; r += TR_THREADS) {
            bool more = false;
            const uint32_t rr = r + tid;
            if (rr < ntr) {
                const uint32_t st = __ldg(trp + rr);
                if (st <= t0 + cnt) {
                    atomicAdd(&rowc[st - t0], 1u);
                    more = true;
                }
            }
            if (!__syncthreads_or(more)) break;
        }
        // inclusive scan of rowc[0..TR_SUB] (TR_SUB + 1 entries; the last one only feeds the next rcur)
        {
            uint32_t v[TR_PER], run = 0;
#pragma unroll
            for (int k = 0; k < TR_PER; k++) { run += rowc[tid * TR_PER + k]; v[k] = run; }
            uint32_t incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            if (lane == 31) wsum[w] = incl;
            const uint32_t last = rowc[TR_SUB];
            __syncthreads();
            uint32_t off = incl - run;
            for (uint32_t u = 0; u < w; u++) off += wsum[u];
#pragma unroll
            for (int k = 0; k < TR_PER; k++) rowc[tid * TR_PER + k] = v[k] + off;
            if (tid == TR_THREADS - 1) s_flag = v[TR_PER - 1] + off + last;
            __syncthreads();
        }
        // elements of this thread (warp w: tiles [w*256, w*256+256) in rounds of 32), stable digit rank
        unsigned long long key[TR_PER], pay[TR_PER];
        uint32_t rank[TR_PER], dig[TR_PER];
#pragma unroll
        for (int j = 0; j < TR_PER; j++) {
            const uint32_t p = w * (TR_SUB / TR_WARPS) + j * 32 + lane;
            const bool ok = p < cnt;
            uint32_t dg = TR_MAXB;  // no element
            key[j] = 0;
            pay[j] = 0;
            if (ok) {
                const uint64_t t = t0 + p;
                const uint32_t col = __ldg(tci + t), row = rcur + rowc[p];
                dg = col >> lb;
                key[j] = (unsigned long long)col | ((unsigned long long)row << cb);
                if constexpr (D == 4) key[j] |= (unsigned long long)nib16(__ldg(reinterpret_cast<const uint32_t *>(tiles) + t)) << (2 * cb);
                else pay[j] = __ldg(reinterpret_cast<const unsigned long long *>(tiles) + t);
            }
            dig[j] = dg;
            const uint32_t peers = __match_any_sync(0xffffffffu, dg);
            const uint32_t before = dg < TR_MAXB ? wc[w * nb + dg] : 0u;
            rank[j] = before + __popc(peers & lt);
            __syncwarp();
            if (dg < TR_MAXB && lane == (uint32_t)(__ffs(peers) - 1)) wc[w * nb + dg] = (uint16_t)(before + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        // per digit: warp prefix (in place) and the CTA-local run start
        for (uint32_t b = tid; b < nb; b += TR_THREADS) {
            uint32_t run = 0;
#pragma unroll
            for (int u = 0; u < TR_WARPS; u++) {
                const uint32_t c = wc[u * nb + b];
                wc[u * nb + b] = (uint16_t)run;
                run += c;
            }
            dbase[b] = run;  // digit total, scanned below
        }
        __syncthreads();
        if (w == 0) {  // exclusive scan of the nb digit totals (one warp)
            uint32_t carry = 0;
            for (uint32_t b0 = 0; b0 < nb; b0 += 32) {
                const uint32_t b = b0 + lane;
                const uint32_t v = b < nb ? dbase[b] : 0u;
                uint32_t incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (uint32_t)o) incl += y;
                }
                if (b < nb) dbase[b] = carry + incl - v;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < TR_PER; j++)
            if (dig[j] < TR_MAXB) {
                const uint32_t lp = dbase[dig[j]] + wc[w * nb + dig[j]] + rank[j];
                skey[lp] = key[j];
                if constexpr (TrElem<D>::PAY) spay[lp] = pay[j];
            }
        __syncthreads();
        for (uint32_t lp = tid; lp < cnt; lp += TR_THREADS) {
            const unsigned long long k = skey[lp];
            const uint32_t dg = (uint32_t)(k & ((1ull << cb) - 1)) >> lb;
            const unsigned long long o = pos[dg] + (lp - dbase[dg]);
            ekey[o] = k;
            if constexpr (TrElem<D>::PAY) epay[o] = spay[lp];
        }
        __syncthreads();
        for (uint32_t b = tid; b < nb; b += TR_THREADS) {  // advance each digit by its count in this sub-tile
            const uint32_t nxt = b + 1 < nb ? dbase[b + 1] : cnt;
            pos[b] += nxt - dbase[b];
        }
        rcur += s_flag;
        __syncthreads();
    }
}

template <int D>
__global__ void __launch_bounds__(TR_THREADS) k_tr_bucket(uint32_t ntr, int cb, int lb, uint32_t G,
                                                          const uint64_t *__restrict__ hofs, uint64_t T,
                                                          const unsigned long long *__restrict__ ekey,
                                                          const unsigned long long *__restrict__ epay,
                                                          uint32_t *__restrict__ trp_out, uint32_t *__restrict__ tci_out,
                                                          void *__restrict__ tiles_out) {
    extern __shared__ __align__(16) unsigned char tr_smem[];
    const uint32_t nl = 1u << lb;
    uint32_t *wc = reinterpret_cast<uint32_t *>(tr_smem);  // TR_WARPS * nl
    uint32_t *cs = wc + TR_WARPS * nl;                       // nl
    const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5, lt = (1u << lane) - 1u;
    const uint32_t b = blockIdx.x;
    const uint64_t bs = hofs[(size_t)b * G], be = hofs[(size_t)(b + 1) * G];
    const uint64_t s0 = bs + (be - bs) * w / TR_WARPS, s1 = bs + (be - bs) * (w + 1) / TR_WARPS;
    const uint32_t lm = nl - 1;
    for (uint32_t q = tid; q < TR_WARPS * nl; q += TR_THREADS) wc[q] = 0;
    __syncthreads();
    for (uint64_t e = s0 + lane; e < s1; e += 32) atomicAdd(&wc[w * nl + ((uint32_t)ekey[e] & lm)], 1u);
    __syncthreads();
    for (uint32_t c = tid; c < nl; c += TR_THREADS) {
        uint32_t run = 0;
#pragma unroll
        for (int u = 0; u < TR_WARPS; u++) {
            const uint32_t v = wc[u * nl + c];
            wc[u * nl + c] = run;
            run += v;
        }
        cs[c] = run;
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the column totals -> tile_row_ptr of the transpose
        uint32_t carry = 0;
        for (uint32_t c0 = 0; c0 < nl; c0 += 32) {
            const uint32_t c = c0 + lane;
            const uint32_t v = c < nl ? cs[c] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            if (c < nl) {
                cs[c] = carry + incl - v;
                const uint64_t col = ((uint64_t)b << lb) + c;
                if (col < ntr) trp_out[col] = (uint32_t)(bs + carry + incl - v);
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (b == gridDim.x - 1 && lane == 0) trp_out[ntr] = (uint32_t)T;
    }
    __syncthreads();
    const unsigned long long cm = (1ull << cb) - 1;
    for (uint64_t e0 = s0; e0 < s1; e0 += 32) {  // warp-uniform: stable placement in order
        const uint64_t e = e0 + lane;
        const bool ok = e < s1;
        unsigned long long k = ok ? ekey[e] : 0ull;
        const uint32_t c = ok ? ((uint32_t)k & lm) : nl;
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        const uint32_t before = ok ? wc[w * nl + c] : 0u;
        __syncwarp();
        if (ok && lane == (uint32_t)(__ffs(peers) - 1)) wc[w * nl + c] = before + __popc(peers);
        __syncwarp();
        if (ok) {
            const uint64_t o = bs + cs[c] + before + __popc(peers & lt);
            tci_out[o] = (uint32_t)((k >> cb) & cm);  // the source row is the new column
            if constexpr (D == 4) {
                const uint32_t nib = (uint32_t)(k >> (2 * cb));
                uint32_t a[4] = {nib & 0xFu, (nib >> 4) & 0xFu, (nib >> 8) & 0xFu, (nib >> 12) & 0xFu};
                bit_transpose<4>(a);
                reinterpret_cast<uint32_t *>(tiles_out)[o] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
            } else {
                const unsigned long long v = epay[e];
                uint32_t a[8];
#pragma unroll
                for (int r = 0; r < 8; r++) a[r] = (uint32_t)(v >> (8 * r)) & 0xFFu;
                bit_transpose<8>(a);
                unsigned long long outv = 0;
#pragma unroll
                for (int r = 0; r < 8; r++) outv |= (unsigned long long)a[r] << (8 * r);
                reinterpret_cast<unsigned long long *>(tiles_out)[o] = outv;
            }
        }
    }
}

// Measured slower than the LSD path (s22: d=4 10.2 vs 7.0 ms, d=8 12.5 vs 11.5
// ms): the bucket pass writes 4-byte outputs scattered over its bucket's
// 1 MB range, and with ~700 buckets in flight the partially written sectors
// leave L2 before they fill (ncu: k_tr_bucket at 18 % issue, long-scoreboard
// bound).  Kept as an A/B path: B2SR_TRANSPOSE=two.
static bool tr2_enabled() {
    const char *e = getenv("B2SR_TRANSPOSE");
    return e && e[0] == 't';
}

// returns false when the two-level path does not apply (d >= 16, > 22 column bits)
template <int D>
static bool transpose_two_level(const b2sr_matrix *m, b2sr_matrix *o, int cb, cudaStream_t s) {
    if (cb > 22 || !tr2_enabled()) return false;
    const uint64_t T = m->num_tiles;
    const uint32_t ntr = m->ntr;
    const int lb = cb / 2, hb = cb - lb;
    const uint32_t nb = 1u << hb, nl = 1u << lb;
    const uint32_t G = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)num_sms() * 2, (T + TR_SUB - 1) / TR_SUB));
    Buf<uint32_t> hcnt((size_t)nb * G, s);
    Buf<uint64_t> hofs((size_t)nb * G + 1, s);
    LAUNCH(k_tr_hist, G, TR_THREADS, 0, s, T, G, m->tci, lb, nb, hcnt.p);
    exclusive_scan_u32_to_u64(hcnt.p, hofs.p, (size_t)nb * G, s);
    Buf<unsigned long long> ekey(T, s), epay(TrElem<D>::PAY ? T : 1, s);
    const size_t smem_b = (size_t)TR_SUB * 8 * (TrElem<D>::PAY ? 2 : 1) + (size_t)nb * 8 + (TR_SUB + 1) * 4 +
                          (size_t)nb * 4 + (size_t)TR_WARPS * nb * 2 + 16;
    hot_smem_attr_raw(reinterpret_cast<const void *>(k_tr_scatter<D>), smem_b);
    LAUNCH(k_tr_scatter<D>, G, TR_THREADS, smem_b, s, T, G, ntr, m->trp, m->tci, m->tiles, cb, lb, nb, hofs.p, ekey.p,
           epay.p);
    const size_t smem_c = (size_t)TR_WARPS * nl * 4 + (size_t)nl * 4;
    hot_smem_attr_raw(reinterpret_cast<const void *>(k_tr_bucket<D>), smem_c);
    LAUNCH(k_tr_bucket<D>, nb, TR_THREADS, smem_c, s, ntr, cb, lb, G, hofs.p, T, ekey.p, epay.p, o->trp, o->tci,
           o->tiles);
    return true;
}

void launch_row_ids(const b2sr_matrix *m, uint32_t *rowid, cudaStream_t s) {
    uint64_t b = ((uint64_t)m->ntr * 32 + 255) / 256, cap = (uint64_t)num_sms() * 16;
    LAUNCH(k_row_ids, (unsigned)std::max<uint64_t>(1, std::min(b, cap)), 256, 0, s, m->ntr, m->trp, rowid);
}

static int bits_for(uint32_t maxval) {
    int b = 0;
    while (b < 32 && (maxval >> b)) b++;
    return b;
}

static unsigned grid_for(uint64_t work, unsigned per = 256) {
    uint64_t b = (work + per - 1) / per, cap = (uint64_t)num_sms() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

b2sr_matrix *transpose_device(const b2sr_matrix *m, cudaStream_t s) {
    if (m->row0 != 0 || m->ntr != tile_rows(m->n, m->dim))
        B2SR_THROW(B2SR_EINVAL, "transpose needs a full matrix, not a row block");
    uint32_t ntr = m->ntr;
    uint64_t T = m->num_tiles;
    b2sr_matrix *o = new_matrix(m->n, m->dim, ntr, T, s);
    try {
        const int cb0 = std::max(1, bits_for(ntr - 1));  // >= 1: the packed fields must not overlap
        if (T && ((m->dim == 4 && transpose_two_level<4>(m, o, cb0, s)) ||
                  (m->dim == 8 && transpose_two_level<8>(m, o, cb0, s))))
            return o;
        const int cb = cb0;
        if (!T) {
            CK(cudaMemsetAsync(o->trp, 0, ((size_t)ntr + 1) * 4, s));
        } else if (m->dim == 4 && 2 * cb + 16 <= 64) {
            Buf<uint64_t> keys(T, s), kalt;
            Buf<uint32_t> counts0;
            if (pack_rows_enabled()) {
                const uint32_t nb = (uint32_t)((T + PK_TILES - 1) / PK_TILES);
                Buf<uint32_t> q(2 * (size_t)nb, s);
                counts0 = Buf<uint32_t>((size_t)nb * 256, s);
                LAUNCH(k_pack4_bounds, (nb + 255) / 256, 256, 0, s, T, ntr, m->trp, nb, q.p);
                LAUNCH(k_pack_rows<4>, nb, PK_THREADS, 0, s, T, m->trp, q.p, m->tci, m->tiles, cb, keys.p, nullptr,
                       counts0.p, cb >= 8 ? 0xFFu : (1u << cb) - 1u);
            } else {
                Buf<uint32_t> rowid(T, s);
                LAUNCH(k_row_ids, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, m->trp, rowid.p);
                LAUNCH(k_pack4, grid_for(T), 256, 0, s, T, rowid.p, m->tci, (const uint32_t *)m->tiles, cb, keys.p);
            }
            const char *ue = getenv("B2SR_TR_UNPACK");  // 0: sorted keys + k_unpack4 (A/B)
            if (ue && ue[0] == '0') {
                uint64_t *ks = nullptr;
                radix_sort_keys_u64(keys.p, T, cb, s, &ks, &kalt);
                LAUNCH(k_unpack4, grid_for(T), 256, 0, s, T, ks, cb, ntr, o->trp, o->tci, (uint32_t *)o->tiles);
            } else {  // the last sort pass writes the transpose (sort.cu, Unpack4)
                radix_sort_unpack4(keys.p, T, cb, ntr, o->trp, o->tci, (uint32_t *)o->tiles, s,
                                   counts0.p ? counts0.p : nullptr);
            }
        } else if (m->dim == 8 && 2 * cb <= 64 && tr8_sort_enabled()) {
            // (column | row) keys carrying the 8-byte tile: the last pass writes
            // the transpose, no random gathers of tiles and row ids
            const uint32_t nb = (uint32_t)((T + PK_TILES - 1) / PK_TILES);
            Buf<uint64_t> keys(T, s), vals(T, s);
            Buf<uint32_t> q(2 * (size_t)nb, s), counts0((size_t)nb * 256, s);
            LAUNCH(k_pack4_bounds, (nb + 255) / 256, 256, 0, s, T, ntr, m->trp, nb, q.p);
            LAUNCH(k_pack_rows<8>, nb, PK_THREADS, 0, s, T, m->trp, q.p, m->tci, m->tiles, cb, keys.p, vals.p, counts0.p,
                   cb >= 8 ? 0xFFu : (1u << cb) - 1u);
            radix_sort_unpack8(keys.p, vals.p, T, cb, ntr, o->trp, o->tci, static_cast<uint64_t *>(o->tiles), s, counts0.p);
        } else if (m->dim >= 16 && tr8_sort_enabled()) {
            // (column | row, tile id): the row travels with the key, only the
            // 32 / 128-byte tile is gathered afterwards (no row-id array)
            const uint32_t nb = (uint32_t)((T + PK_TILES - 1) / PK_TILES);
            Buf<uint64_t> keys(T, s), kalt;
            Buf<uint32_t> ids(T, s), valt, q(2 * (size_t)nb, s), counts0((size_t)nb * 256, s);
            LAUNCH(k_pack4_bounds, (nb + 255) / 256, 256, 0, s, T, ntr, m->trp, nb, q.p);
            LAUNCH(k_pack_rows<16>, nb, PK_THREADS, 0, s, T, m->trp, q.p, m->tci, m->tiles, cb, keys.p,
                   reinterpret_cast<uint64_t *>(ids.p), counts0.p, cb >= 8 ? 0xFFu : (1u << cb) - 1u);
            uint64_t *ks = nullptr;
            uint32_t *vs = nullptr;
            radix_sort_ids(keys.p, ids.p, T, cb, s, counts0.p, &kalt, &valt, &ks, &vs);
            const unsigned g = grid_for(T);
            if (m->dim == 16)
                LAUNCH(k_transpose_gather_ids<16>, g, 256, 0, s, T, ks, vs, cb, ntr, m->tiles, o->trp, o->tci, o->tiles);
            else
                LAUNCH(k_transpose_gather_ids<32>, g, 256, 0, s, T, ks, vs, cb, ntr, m->tiles, o->trp, o->tci, o->tiles);
        } else {
            Buf<uint32_t> keys(T, s), vals(T, s), rowid(T, s), kalt, valt;
            CK(cudaMemcpyAsync(keys.p, m->tci, T * 4, cudaMemcpyDeviceToDevice, s));
            LAUNCH(k_iota, grid_for(T), 256, 0, s, vals.p, T);
            LAUNCH(k_row_ids, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, m->trp, rowid.p);
            uint32_t *ks = nullptr, *vs = nullptr;
            radix_sort_pairs_u32(keys.p, vals.p, T, bits_for(ntr - 1), s, &ks, &vs, &kalt, &valt);
            LAUNCH(k_trp_sorted, grid_for(T), 256, 0, s, T, ks, ntr, o->trp);
            unsigned g = grid_for(T);
            switch (m->dim) {
                case 4: LAUNCH(k_transpose_gather<4>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
                case 8: LAUNCH(k_transpose_gather<8>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
                case 16: LAUNCH(k_transpose_gather<16>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
                default: LAUNCH(k_transpose_gather<32>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
            }
        }
    } catch (...) {
        free_matrix(o);
        throw;
    }
    return o;
}

// ------------------------------------------------------------ b2sr -> csr
template <int D>
__global__ void k_row_degrees(uint64_t T, const uint32_t *__restrict__ rowid, const typename WordT<D>::T *__restrict__ tiles,
                              uint32_t *__restrict__ deg) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t I = rowid[t];
#pragma unroll
        for (int r = 0; r < D; r++) {
            uint32_t c = __popc((uint32_t)tiles[t * D + r]);
            if (c) atomicAdd(deg + (size_t)I * D + r, c);
        }
    }
}

// group of D lanes per tile row, lane = bit-row, columns emitted in order
template <int D>
__global__ void k_csr_fill(uint32_t ntr, uint32_t n, const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                           const typename WordT<D>::T *__restrict__ tiles, const uint32_t *__restrict__ row_ptr,
                           uint32_t *__restrict__ col_ind) {
    constexpr uint32_t GPW = 32 / D;
    const uint32_t lane = lane_id(), r = lane % D;
    const uint32_t groups = ((gridDim.x * blockDim.x) >> 5) * GPW;
    for (uint32_t I = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * GPW + lane / D; I < ntr; I += groups) {
        uint64_t row = (uint64_t)I * D + r;
        if (row >= n) continue;
        uint32_t pos = row_ptr[row];
        for (uint32_t t = trp[I]; t < trp[I + 1]; t++) {
            uint32_t w = tiles[(size_t)t * D + r];
            uint32_t base = tci[t] * D;
            while (w) {
                col_ind[pos++] = base + (__ffs(w) - 1);
                w &= w - 1;
            }
        }
    }
}

// ------------------------------------------------------------ diagonal drop
template <int D>
__global__ void k_diag_flags(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                             const typename WordT<D>::T *__restrict__ tiles, uint32_t *__restrict__ keep) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t k = 1;
        if (rowid[t] == tci[t]) {
            uint32_t o = 0;
#pragma unroll
            for (int r = 0; r < D; r++) o |= (uint32_t)tiles[t * D + r] & ~(1u << r);
            k = o != 0;
        }
        keep[t] = k;
    }
}

template <int D>
__global__ void k_diag_compact(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                               const typename WordT<D>::T *__restrict__ tiles, const uint32_t *__restrict__ keep,
                               const uint64_t *__restrict__ ofs, uint32_t *__restrict__ tci_out,
                               typename WordT<D>::T *__restrict__ tiles_out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        if (!keep[t]) continue;
        uint64_t o = ofs[t];
        bool diag = rowid[t] == tci[t];
        tci_out[o] = tci[t];
#pragma unroll
        for (int r = 0; r < D; r++) {
            uint32_t w = tiles[t * D + r];
            if (diag) w &= ~(1u << r);
            tiles_out[o * D + r] = (typename WordT<D>::T)w;
        }
    }
}

__global__ void k_diag_trp(uint32_t ntr, const uint32_t *trp, const uint64_t *ofs, uint32_t *trp_out) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I <= ntr) trp_out[I] = (uint32_t)ofs[trp[I]];
}

template <int D>
static b2sr_matrix *drop_diag_impl(const b2sr_matrix *m, cudaStream_t s) {
    using W = typename WordT<D>::T;
    uint64_t T = m->num_tiles;
    Buf<uint32_t> rowid(T, s), keep(T, s);
    Buf<uint64_t> ofs(T + 1, s);
    LAUNCH(k_row_ids, grid_for((uint64_t)m->ntr * 32), 256, 0, s, m->ntr, m->trp, rowid.p);
    LAUNCH(k_diag_flags<D>, grid_for(T), 256, 0, s, T, rowid.p, m->tci, (const W *)m->tiles, keep.p);
    exclusive_scan_u32_to_u64(keep.p, ofs.p, T, s);
    uint64_t T2 = read_scalar(ofs.p + T, s);
    b2sr_matrix *o = new_matrix(m->n, m->dim, m->ntr, T2, s);
    try {
        LAUNCH(k_diag_trp, (m->ntr + 256) / 256, 256, 0, s, m->ntr, m->trp, ofs.p, o->trp);
        LAUNCH(k_diag_compact<D>, grid_for(T), 256, 0, s, T, rowid.p, m->tci, (const W *)m->tiles, keep.p, ofs.p,
               o->tci, (W *)o->tiles);
    } catch (...) {
        free_matrix(o);
        throw;
    }
    return o;
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_transpose(const b2sr_matrix *m, void *stream, b2sr_matrix **out) {
    API_BEGIN
    *out = transpose_device(m, (cudaStream_t)stream);
    API_END
}

int b2sr_to_csr_rowptr(const b2sr_matrix *m, uint32_t *d_row_ptr, uint64_t *nnz, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (m->row0 != 0) B2SR_THROW(B2SR_EINVAL, "b2sr_to_csr needs a full matrix");
    uint64_t T = m->num_tiles;
    size_t rows = (size_t)m->ntr * m->dim;
    Buf<uint32_t> deg(rows, s), rowid(T, s);
    Buf<uint64_t> ofs((size_t)m->n + 1, s);
    CK(cudaMemsetAsync(deg.p, 0, rows * 4, s));
    if (T) {
        LAUNCH(k_row_ids, grid_for((uint64_t)m->ntr * 32), 256, 0, s, m->ntr, m->trp, rowid.p);
        unsigned g = grid_for(T);
        switch (m->dim) {
            case 4: LAUNCH(k_row_degrees<4>, g, 256, 0, s, T, rowid.p, (const uint8_t *)m->tiles, deg.p); break;
            case 8: LAUNCH(k_row_degrees<8>, g, 256, 0, s, T, rowid.p, (const uint8_t *)m->tiles, deg.p); break;
            case 16: LAUNCH(k_row_degrees<16>, g, 256, 0, s, T, rowid.p, (const uint16_t *)m->tiles, deg.p); break;
            default: LAUNCH(k_row_degrees<32>, g, 256, 0, s, T, rowid.p, (const uint32_t *)m->tiles, deg.p); break;
        }
    }
    exclusive_scan_u32_to_u64(deg.p, ofs.p, m->n, s);
    uint64_t total = read_scalar(ofs.p + m->n, s);
    if (total > 0xFFFFFFFFull) B2SR_THROW(B2SR_EFORMAT, "nnz exceeds the 32-bit CSR index range");
    LAUNCH(k_u64_to_u32, grid_for((uint64_t)m->n + 1), 256, 0, s, ofs.p, d_row_ptr, (size_t)m->n + 1);
    *nnz = total;
    API_END
}

int b2sr_to_csr_fill(const b2sr_matrix *m, const uint32_t *d_row_ptr, uint32_t *d_col_ind, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (!m->num_tiles) return B2SR_OK;
    uint32_t gpw = 32 / m->dim;
    unsigned g = grid_for(((uint64_t)m->ntr + gpw - 1) / gpw * 32);
    switch (m->dim) {
        case 4: LAUNCH(k_csr_fill<4>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint8_t *)m->tiles, d_row_ptr, d_col_ind); break;
        case 8: LAUNCH(k_csr_fill<8>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint8_t *)m->tiles, d_row_ptr, d_col_ind); break;
        case 16: LAUNCH(k_csr_fill<16>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint16_t *)m->tiles, d_row_ptr, d_col_ind); break;
        default: LAUNCH(k_csr_fill<32>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint32_t *)m->tiles, d_row_ptr, d_col_ind); break;
    }
    API_END
}

int b2sr_drop_diagonal(const b2sr_matrix *m, void *stream, b2sr_matrix **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (m->row0 != 0) B2SR_THROW(B2SR_EINVAL, "drop_diagonal needs a full matrix");
    switch (m->dim) {
        case 4: *out = drop_diag_impl<4>(m, s); break;
        case 8: *out = drop_diag_impl<8>(m, s); break;
        case 16: *out = drop_diag_impl<16>(m, s); break;
        default: *out = drop_diag_impl<32>(m, s); break;
    }
    API_END
}

}  // extern "C"
