// Stable LSD radix sort (8-bit digits) used by the tile transpose (stable
// sort by tile column, formats.py:485 lexsort) and by COO -> CSR
// (formats.py:176-179 argsort/unique).
//
// Per pass: (1) per-CTA digit histograms, digit-major; (2) exclusive scan;
// (3) scatter with an in-CTA stable rank: each warp walks its 512 keys in 16
// rounds of 32, ranks equal digits with ballots (multi-split), keeps warp-private
// digit counters in shared memory, then warps are offset by a per-digit
// prefix.  Order = (CTA, warp, round, lane) = input order, so it is stable.
#include "b2sr_internal.cuh"

namespace b2sr {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 8;   // 16: 122 registers, 2 CTAs per SM
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;  // 2048 keys per CTA
static_assert(RS_TILE == RADIX_TILE, "k_pack4_rows counts the first digit over the same tiles");

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K *__restrict__ keys, size_t n, int sh, uint32_t dm,
                                                        uint32_t *__restrict__ counts, uint32_t nblocks) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    size_t base = (size_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int j = 0; j < RS_ROUNDS; j++) {
        size_t i = base + (size_t)j * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(uint32_t)(keys[i] >> sh) & dm], 1u);
    }
    __syncthreads();
    counts[(size_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// The d = 4 transpose's last pass writes the transposed matrix itself instead
// of the sorted keys (key = column | row << cb | 16-bit tile << 2 cb): the row
// as the new tile column, the bit-transposed tile, and tile_row_ptr -- a
// column's first element inside its CTA digit run fills (previous column,
// column] (empty columns included); an element that opens a CTA digit run
// does not know its predecessor and takes atomicMin on its own column; the
// columns left unset are closed by a suffix minimum afterwards.
struct Unpack4 {
    uint32_t *trp, *tci, *tiles;
    int cb;
};

__device__ __forceinline__ uint32_t tr4x4(uint32_t x) {  // 4x4 bit transpose, rows -> bytes
    uint32_t t = (x ^ (x >> 3)) & 0x0A0Au;
    x ^= t ^ (t << 3);
    t = (x ^ (x >> 6)) & 0x00CCu;
    x ^= t ^ (t << 6);
    return (x & 0xFu) | ((x & 0xF0u) << 4) | ((x & 0xF00u) << 8) | ((x & 0xF000u) << 12);
}

__device__ __forceinline__ uint64_t tr8x8(uint64_t x) {  // 8x8 bit transpose, rows in bytes
    uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x ^= t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x ^= t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x ^= t ^ (t << 28);
    return x;
}

// V = uint64_t carries the d = 8 tile through the passes (UNPACK: the last
// pass writes the transpose from key (column | row) and value (tile))
template <typename K, bool VALS, bool UNPACK = false, typename V = uint32_t>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const K *__restrict__ kin, const V *__restrict__ vin,
                                                           K *__restrict__ kout, V *__restrict__ vout,
                                                           size_t n, int sh, uint32_t dm,
                                                           const uint64_t *__restrict__ offs, uint32_t nblocks,
                                                           Unpack4 up = {}) {
    __shared__ uint32_t wc[RS_WARPS][256];
    __shared__ uint32_t dbase[256];            // CTA-local start of each digit run
    __shared__ K skey[RS_TILE];                // keys re-ordered by digit inside the CTA
    __shared__ V sval[VALS ? RS_TILE : 1];
    __shared__ uint64_t goff[256];             // this CTA's global start of each digit run
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
    for (int b = threadIdx.x; b < RS_WARPS * 256; b += RS_THREADS) (&wc[0][0])[b] = 0;
    // once per CTA instead of one dependent global load per key in the write loop
    for (int b = threadIdx.x; b < 256; b += RS_THREADS) goff[b] = offs[(size_t)b * nblocks + blockIdx.x];
    __syncthreads();
    size_t base = (size_t)blockIdx.x * RS_TILE + (size_t)w * (32 * RS_ROUNDS);
    K key[RS_ROUNDS];
    V val[RS_ROUNDS];
    uint32_t rank[RS_ROUNDS];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ROUNDS; j++) {
        size_t i = base + (size_t)j * 32 + lane;
        bool ok = i < n;
        key[j] = ok ? kin[i] : (K)0;
        if constexpr (VALS) val[j] = ok ? vin[i] : (V)0;
        uint32_t dg = ok ? ((uint32_t)(key[j] >> sh) & dm) : 256u;  // 256 = no item
        // lanes with the same digit: nine ballots (8 digit bits + the no-item
        // flag) instead of __match_any_sync (MATCH.ANY is a slow, multi-pass
        // instruction; this is the classic multi-split ranking)
        uint32_t peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 9; b++) {
            const bool bit = (dg >> b) & 1u;
            const uint32_t bb = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bb : ~bb;
        }
        uint32_t leader = __ffs(peers) - 1;
        uint32_t before = dg < 256 ? wc[w][dg] : 0u;
        rank[j] = before + __popc(peers & lt);
        __syncwarp();
        if (dg < 256 && lane == leader) wc[w][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {  // exclusive prefix over warps per digit, then over digits (CTA-local run starts)
        uint32_t d = threadIdx.x, run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ww++) {
            uint32_t c = wc[ww][d];
            wc[ww][d] = run;
            run += c;
        }
        // block-wide exclusive scan of the 256 digit totals (one per thread)
        uint32_t inc = run;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        __shared__ uint32_t wsum[RS_WARPS];
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        uint32_t off = 0;
        for (uint32_t ww = 0; ww < w; ww++) off += wsum[ww];
        dbase[d] = off + inc - run;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_ROUNDS; j++) {  // stage in digit order inside the CTA
        size_t i = base + (size_t)j * 32 + lane;
        if (i < n) {
            uint32_t dg = (uint32_t)(key[j] >> sh) & dm;
            uint32_t lp = dbase[dg] + wc[w][dg] + rank[j];
            skey[lp] = key[j];
            if constexpr (VALS) sval[lp] = val[j];
        }
    }
    __syncthreads();
    // consecutive threads write consecutive slots of each digit run: coalesced
    uint32_t count = (uint32_t)min((size_t)RS_TILE, n - (size_t)blockIdx.x * RS_TILE);
    for (uint32_t lp = threadIdx.x; lp < count; lp += RS_THREADS) {
        K k = skey[lp];
        uint32_t dg = (uint32_t)(k >> sh) & dm;
        size_t pos = goff[dg] + (lp - dbase[dg]);
        if constexpr (UNPACK) {
            const uint64_t cm = (1ull << up.cb) - 1;
            const uint32_t col = (uint32_t)(k & cm);
            up.tci[pos] = (uint32_t)((k >> up.cb) & cm);  // the source row is the transposed column
            if constexpr (sizeof(V) == 8) reinterpret_cast<uint64_t *>(up.tiles)[pos] = tr8x8((uint64_t)sval[lp]);
            else up.tiles[pos] = tr4x4((uint32_t)(k >> (2 * up.cb)) & 0xFFFFu);
            if (lp == dbase[dg]) {
                atomicMin(up.trp + col, (uint32_t)pos);
            } else {
                const uint32_t pc = (uint32_t)(skey[lp - 1] & cm);
                for (uint32_t q = pc + 1; q <= col; q++) up.trp[q] = (uint32_t)pos;
            }
        } else {
            kout[pos] = k;
            if constexpr (VALS) vout[pos] = sval[lp];
        }
    }
}

// tile_row_ptr[q] = min over c >= q of the marks (unset = ~0; the last entry
// is set to `last` here): block minima, an exclusive suffix minimum over the
// blocks (one CTA), then a block-local suffix minimum
constexpr int SM_TILE = 1024;
__global__ void __launch_bounds__(SM_TILE) k_sufmin_blocks(uint32_t m, uint32_t *__restrict__ a, uint32_t last,
                                                           uint32_t *__restrict__ bmin) {
    const uint32_t i = blockIdx.x * SM_TILE + threadIdx.x;
    uint32_t v = 0xFFFFFFFFu;
    if (i + 1 == m) a[i] = v = last;
    else if (i < m) v = a[i];
    v = __reduce_min_sync(0xffffffffu, v);
    __shared__ uint32_t w[SM_TILE / 32];
    if (lane_id() == 0) w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = __reduce_min_sync(0xffffffffu, w[threadIdx.x]);
        if (threadIdx.x == 0) bmin[blockIdx.x] = v;
    }
}

// block-wide inclusive suffix minimum of one value per thread
__device__ __forceinline__ uint32_t block_sufmin(uint32_t v, uint32_t *w) {
    const uint32_t lane = lane_id(), wi = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = min(v, y);
    }
    if (lane == 0) w[wi] = v;
    __syncthreads();
    uint32_t rest = 0xFFFFFFFFu;
    for (uint32_t ww = wi + 1; ww < SM_TILE / 32; ww++) rest = min(rest, w[ww]);
    __syncthreads();
    return min(v, rest);
}

__global__ void __launch_bounds__(SM_TILE) k_sufmin_scan(uint32_t nb, uint32_t *__restrict__ bmin) {
    __shared__ uint32_t w[SM_TILE / 32];
    uint32_t carry = 0xFFFFFFFFu;  // minimum of the blocks after this chunk
    for (int64_t c0 = ((int64_t)(nb - 1) / SM_TILE) * SM_TILE; c0 >= 0; c0 -= SM_TILE) {
        const uint32_t i = (uint32_t)c0 + threadIdx.x;
        const uint32_t v = i < nb ? bmin[i] : 0xFFFFFFFFu;
        const uint32_t inc = min(block_sufmin(v, w), carry);
        // exclusive: the minimum strictly after block i
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, inc, 1);
        __shared__ uint32_t first[SM_TILE / 32];
        if (lane_id() == 0) first[threadIdx.x >> 5] = inc;
        __syncthreads();
        uint32_t ex = lane_id() < 31 ? nxt : ((threadIdx.x >> 5) + 1 < SM_TILE / 32 ? first[(threadIdx.x >> 5) + 1] : carry);
        const uint32_t c_new = first[0];
        __syncthreads();
        if (i < nb) bmin[i] = ex;
        carry = c_new;
    }
}

__global__ void __launch_bounds__(SM_TILE) k_sufmin_apply(uint32_t m, uint32_t *__restrict__ a,
                                                          const uint32_t *__restrict__ after) {
    __shared__ uint32_t w[SM_TILE / 32];
    const uint32_t i = blockIdx.x * SM_TILE + threadIdx.x;
    const uint32_t v = i < m ? a[i] : 0xFFFFFFFFu;
    const uint32_t r = min(block_sufmin(v, w), after[blockIdx.x]);
    if (i < m) a[i] = r;
}

template <typename K, bool VALS>
static void rs_passes(K *ka, uint32_t *va, K *kb, uint32_t *vb, size_t n, int bits, cudaStream_t s, K **kres,
                      uint32_t **vres) {
    uint32_t nblocks = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
    Buf<uint32_t> counts((size_t)nblocks * 256, s);
    Buf<uint64_t> offs((size_t)nblocks * 256 + 1, s);
    K *kin = ka, *kout = kb;
    uint32_t *vin = va, *vout = vb;
    for (int sh = 0; sh < bits; sh += 8) {
        // the last digit covers only the remaining key bits: bits above `bits`
        // may carry payload (the d=4 transpose packs row and tile there)
        const uint32_t dm = bits - sh >= 8 ? 0xFFu : (1u << (bits - sh)) - 1u;
        LAUNCH(k_rs_hist<K>, nblocks, RS_THREADS, 0, s, kin, n, sh, dm, counts.p, nblocks);
        exclusive_scan_u32_to_u64(counts.p, offs.p, (size_t)nblocks * 256, s);
        LAUNCH((k_rs_scatter<K, VALS>), nblocks, RS_THREADS, 0, s, kin, vin, kout, vout, n, sh, dm, offs.p, nblocks,
               Unpack4{});
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    *kres = kin;
    if (vres) *vres = vin;
}

size_t radix_sort_pairs_u32(uint32_t *keys, uint32_t *vals, size_t n, int bits, cudaStream_t s, uint32_t **keys_out,
                            uint32_t **vals_out, Buf<uint32_t> *kalt, Buf<uint32_t> *valt) {
    *kalt = Buf<uint32_t>(n, s);
    *valt = Buf<uint32_t>(n, s);
    if (n == 0 || bits <= 0) {
        *keys_out = keys;
        *vals_out = vals;
        return n;
    }
    rs_passes<uint32_t, true>(keys, vals, kalt->p, valt->p, n, bits, s, keys_out, vals_out);
    return n;
}

// The d = 4 transpose: LSD passes over the column bits, the last one writing
// the transposed matrix (Unpack4 above).  trp has ntr + 1 entries.
void radix_sort_unpack4(uint64_t *keys, size_t n, int bits, uint32_t ntr, uint32_t *trp, uint32_t *tci,
                        uint32_t *tiles, cudaStream_t s, const uint32_t *counts0) {
    Buf<uint64_t> kalt(n, s);
    const uint32_t nblocks = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
    Buf<uint32_t> counts((size_t)nblocks * 256, s);
    Buf<uint64_t> offs((size_t)nblocks * 256 + 1, s);
    CK(cudaMemsetAsync(trp, 0xFF, ((size_t)ntr + 1) * 4, s));
    uint64_t *kin = keys, *kout = kalt.p;
    for (int sh = 0; sh < bits; sh += 8) {
        const uint32_t dm = bits - sh >= 8 ? 0xFFu : (1u << (bits - sh)) - 1u;
        if (sh == 0 && counts0) {
            exclusive_scan_u32_to_u64(counts0, offs.p, (size_t)nblocks * 256, s);
        } else {
            LAUNCH(k_rs_hist<uint64_t>, nblocks, RS_THREADS, 0, s, kin, n, sh, dm, counts.p, nblocks);
            exclusive_scan_u32_to_u64(counts.p, offs.p, (size_t)nblocks * 256, s);
        }
        if (sh + 8 >= bits) {
            LAUNCH((k_rs_scatter<uint64_t, false, true, uint32_t>), nblocks, RS_THREADS, 0, s, kin, (const uint32_t *)nullptr, kout, (uint32_t *)nullptr, n, sh,
                   dm, offs.p, nblocks, Unpack4{trp, tci, tiles, bits});
        } else {
            LAUNCH((k_rs_scatter<uint64_t, false, false, uint32_t>), nblocks, RS_THREADS, 0, s, kin, (const uint32_t *)nullptr, kout, (uint32_t *)nullptr, n, sh, dm,
                   offs.p, nblocks, Unpack4{});
            std::swap(kin, kout);
        }
    }
    const uint32_t m = ntr + 1, nb = (m + SM_TILE - 1) / SM_TILE;
    Buf<uint32_t> bmin(nb, s);
    LAUNCH(k_sufmin_blocks, nb, SM_TILE, 0, s, m, trp, (uint32_t)n, bmin.p);
    LAUNCH(k_sufmin_scan, 1, SM_TILE, 0, s, nb, bmin.p);
    LAUNCH(k_sufmin_apply, nb, SM_TILE, 0, s, m, trp, bmin.p);
}

// The d = 8 transpose: (column | row) keys with the 8-byte tile as the value,
// the last pass writing the transpose (no random tile / row-id gathers).
void radix_sort_unpack8(uint64_t *keys, uint64_t *vals, size_t n, int bits, uint32_t ntr, uint32_t *trp, uint32_t *tci,
                        uint64_t *tiles, cudaStream_t s, const uint32_t *counts0) {
    Buf<uint64_t> kalt(n, s), valt(n, s);
    const uint32_t nblocks = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
    Buf<uint32_t> counts((size_t)nblocks * 256, s);
    Buf<uint64_t> offs((size_t)nblocks * 256 + 1, s);
    CK(cudaMemsetAsync(trp, 0xFF, ((size_t)ntr + 1) * 4, s));
    uint64_t *kin = keys, *kout = kalt.p, *vin = vals, *vout = valt.p;
    for (int sh = 0; sh < bits; sh += 8) {
        const uint32_t dm = bits - sh >= 8 ? 0xFFu : (1u << (bits - sh)) - 1u;
        if (sh == 0 && counts0) {
            exclusive_scan_u32_to_u64(counts0, offs.p, (size_t)nblocks * 256, s);
        } else {
            LAUNCH(k_rs_hist<uint64_t>, nblocks, RS_THREADS, 0, s, kin, n, sh, dm, counts.p, nblocks);
            exclusive_scan_u32_to_u64(counts.p, offs.p, (size_t)nblocks * 256, s);
        }
        if (sh + 8 >= bits) {
            LAUNCH((k_rs_scatter<uint64_t, true, true, uint64_t>), nblocks, RS_THREADS, 0, s, kin, vin, kout, vout, n, sh,
                   dm, offs.p, nblocks, Unpack4{trp, tci, reinterpret_cast<uint32_t *>(tiles), bits});
        } else {
            LAUNCH((k_rs_scatter<uint64_t, true, false, uint64_t>), nblocks, RS_THREADS, 0, s, kin, vin, kout, vout, n,
                   sh, dm, offs.p, nblocks, Unpack4{});
            std::swap(kin, kout);
            std::swap(vin, vout);
        }
    }
    const uint32_t m = ntr + 1, nb = (m + SM_TILE - 1) / SM_TILE;
    Buf<uint32_t> bmin(nb, s);
    LAUNCH(k_sufmin_blocks, nb, SM_TILE, 0, s, m, trp, (uint32_t)n, bmin.p);
    LAUNCH(k_sufmin_scan, 1, SM_TILE, 0, s, nb, bmin.p);
    LAUNCH(k_sufmin_apply, nb, SM_TILE, 0, s, m, trp, bmin.p);
}

// (u64 key, u32 value) passes over the low `bits` of the key; counts0, when
// given, holds the first pass's per-tile digit counts
void radix_sort_ids(uint64_t *keys, uint32_t *vals, size_t n, int bits, cudaStream_t s, const uint32_t *counts0,
                    Buf<uint64_t> *kalt, Buf<uint32_t> *valt, uint64_t **kres, uint32_t **vres) {
    *kalt = Buf<uint64_t>(n, s);
    *valt = Buf<uint32_t>(n, s);
    const uint32_t nblocks = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
    Buf<uint32_t> counts((size_t)nblocks * 256, s);
    Buf<uint64_t> offs((size_t)nblocks * 256 + 1, s);
    uint64_t *kin = keys, *kout = kalt->p;
    uint32_t *vin = vals, *vout = valt->p;
    for (int sh = 0; sh < bits; sh += 8) {
        const uint32_t dm = bits - sh >= 8 ? 0xFFu : (1u << (bits - sh)) - 1u;
        if (sh == 0 && counts0) {
            exclusive_scan_u32_to_u64(counts0, offs.p, (size_t)nblocks * 256, s);
        } else {
            LAUNCH(k_rs_hist<uint64_t>, nblocks, RS_THREADS, 0, s, kin, n, sh, dm, counts.p, nblocks);
            exclusive_scan_u32_to_u64(counts.p, offs.p, (size_t)nblocks * 256, s);
        }
        LAUNCH((k_rs_scatter<uint64_t, true, false, uint32_t>), nblocks, RS_THREADS, 0, s, kin, vin, kout, vout, n, sh,
               dm, offs.p, nblocks, Unpack4{});
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    *kres = kin;
    *vres = vin;
}

void radix_sort_keys_u64(uint64_t *keys, size_t n, int bits, cudaStream_t s, uint64_t **keys_out,
                         Buf<uint64_t> *kalt) {
    *kalt = Buf<uint64_t>(n, s);
    if (n == 0 || bits <= 0) {
        *keys_out = keys;
        return;
    }
    rs_passes<uint64_t, false>(keys, nullptr, kalt->p, nullptr, n, bits, s, keys_out, nullptr);
}

}  // namespace b2sr
