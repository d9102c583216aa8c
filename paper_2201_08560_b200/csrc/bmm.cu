// K7/K8: bin-SpGEMM reductions (replaces kernels.py:271-367).
//
// bmm_bin_bin_sum: sum_ij (A B)_ij = sum_k colsum_A(k) * rowdeg_B(k)
// = sum over A's set bits (i,k) of rowdeg_B(k): K5 for rowdeg_B, then one
// coalesced pass over A's tile bytes (the reference's per-pair colpop*rowpop sum
// regrouped by k; integer arithmetic, so the regrouping is exact).
//
// bmm_bin_bin_sum_masked with B supplied transposed (Bt): for every stored
// mask tile (I,J) the tile columns of A's row I and Bt's row J are
// intersected, and each common K contributes, for every mask bit (r,c),
// popc(A_IK[r] & Bt_JK[c]) == sum_k A[i,k] B[k,j] inside the tile pair.
// One warp per mask tile: lanes take 32 entries of the shorter tile row and
// binary-search them in the longer one; AND+POPC on the integer pipe (b1
// MMA has no native sm_100a path -- SURVEY.md §0).  Triangle counting is
// the instance A = Bt = M = L (transpose(transpose(L)) == L).
#include "b2sr_internal.cuh"

namespace b2sr {

// sum(A B) = 1^T A (B 1) = sum over the set bits (i, k) of A of rowdeg_B(k).
// rowdeg_B = K5 bbf of B with x = all ones.  The gather streams A's tile
// array as raw 16-byte lane loads (512 B per warp, coalesced whatever the
// width); every 32-bit word lies inside one tile, whose column K gives the
// D row degrees the word's bits index.
template <int D>
__device__ __forceinline__ unsigned long long sum_word(uint32_t w, const uint32_t *__restrict__ tci,
                                                       uint64_t byte, const double *__restrict__ rowdeg) {
    constexpr uint32_t TB = D * (D == 32 ? 4 : (D == 16 ? 2 : 1));  // tile bytes
    constexpr uint32_t CM = D == 32 ? 31u : (D == 16 ? 15u : 7u);   // bit -> column within the tile
    unsigned long long acc = 0;
    if (w) {
        const double *x = rowdeg + (size_t)__ldg(tci + byte / TB) * D;
        do {
            acc += (unsigned long long)__ldg(x + ((__ffs(w) - 1) & CM));
            w &= w - 1;
        } while (w);
    }
    return acc;
}

template <int D>
__global__ void __launch_bounds__(256) k_bmm_sum_gather(uint64_t nbytes, const uint32_t *__restrict__ tci,
                                                        const uint8_t *__restrict__ tiles,
                                                        const double *__restrict__ rowdeg,
                                                        unsigned long long *__restrict__ out) {
    unsigned long long acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 16;
    for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; b < nbytes; b += stride) {
        if (b + 16 <= nbytes) {
            const uint4 v = ld_stream128(tiles + b);
            acc += sum_word<D>(v.x, tci, b, rowdeg) + sum_word<D>(v.y, tci, b + 4, rowdeg) +
                   sum_word<D>(v.z, tci, b + 8, rowdeg) + sum_word<D>(v.w, tci, b + 12, rowdeg);
        } else {
            for (uint64_t o = b; o < nbytes; o += 4)
                acc += sum_word<D>(*reinterpret_cast<const uint32_t *>(tiles + o), tci, o, rowdeg);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0 && acc) atomicAdd(out, acc);
}

static unsigned grid_for(uint64_t work) {
    uint64_t b = (work + 255) / 256, cap = (uint64_t)num_sms() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

static void row_ids(const b2sr_matrix *m, uint32_t *rowid, cudaStream_t s) { launch_row_ids(m, rowid, s); }

template <int D>
static void bmm_sum_gather(const b2sr_matrix *a, const double *rowdeg, unsigned long long *acc, cudaStream_t s) {
    const uint64_t nbytes = a->num_tiles * (uint64_t)D * word_bytes(D);
    if (nbytes)
        LAUNCH(k_bmm_sum_gather<D>, grid_for((nbytes + 15) / 16), 256, 0, s, nbytes, a->tci,
               (const uint8_t *)a->tiles, rowdeg, acc);
}

// ------------------------------------------------------------ masked
// lower_bound of `key` in v[lo, hi)
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *__restrict__ v, uint32_t lo, uint32_t hi, uint32_t key) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(v + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ------------------------------------------------------------ chunked items
// A mask tile whose two tile rows are both long (hub x hub) would pin one
// warp for milliseconds; split every mask tile into chunks of TC_CHUNK
// entries of its shorter tile row so such pairs spread over many warps
// (64 / 128 / 256 / 1024 / 2048 / 8192: s20 35.0 / 28.8 / 26.4 / 26.0 / 26.0 /
// 26.1 ms; s26 -, 6.81, 5.90, 5.39, 5.35, 5.43 s -- fewer, larger items win
// until the hub pairs stop spreading).  B2SR_TC_CHUNK overrides (A/B).
constexpr uint32_t TC_CHUNK = 2048;

__global__ void k_tc_item_counts(uint64_t TM, const uint32_t *__restrict__ m_rowid, const uint32_t *__restrict__ m_tci,
                                 uint32_t m_row0, const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ b_trp,
                                 uint32_t chunk, uint32_t *__restrict__ cnt, uint32_t hashed_max,
                                 const uint32_t *__restrict__ m_trp) {
    for (uint64_t mt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; mt < TM; mt += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t i = m_rowid[mt], I = i + m_row0, J = m_tci[mt];
        uint32_t la = a_trp[I + 1] - a_trp[I], lb = b_trp[J + 1] - b_trp[J];
        uint32_t sh = min(la, lb);
        // rows the row-hash kernel takes (A row and mask row both <= hashed_max) get no items here
        const bool hashed = la <= hashed_max && m_trp[i + 1] - m_trp[i] <= hashed_max;
        cnt[mt] = la && lb && !hashed ? (sh + chunk - 1) / chunk : 0;
    }
}

__global__ void k_tc_item_fill(uint64_t TM, const uint32_t *__restrict__ cnt, const uint64_t *__restrict__ ofs,
                               uint2 *__restrict__ items) {
    for (uint64_t mt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; mt < TM; mt += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t o = ofs[mt];
        for (uint32_t j = 0; j < cnt[mt]; j++) items[o + j] = make_uint2((uint32_t)mt, j);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_bmm_masked_items(uint64_t n_items, const uint2 *__restrict__ items,
                                                          const uint32_t *__restrict__ m_rowid,
                                                          const uint32_t *__restrict__ m_tci,
                                                          const typename WordT<D>::T *__restrict__ m_tiles,
                                                          const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci,
                                                          const typename WordT<D>::T *__restrict__ a_tiles,
                                                          const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
                                                          const typename WordT<D>::T *__restrict__ b_tiles,
                                                          uint32_t m_row0, unsigned long long *__restrict__ out,
                                                          unsigned long long *__restrict__ work, uint32_t chunk) {
    const uint32_t lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0, units = 0;
    for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        uint2 it = items[w];
        uint64_t mt = it.x;
        uint32_t I = m_rowid[mt] + m_row0, J = m_tci[mt];
        uint32_t mword = lane < (uint32_t)D ? (uint32_t)m_tiles[mt * D + lane] : 0u;
        uint32_t rows_used = __ballot_sync(0xffffffffu, mword != 0);
        uint32_t a0 = a_trp[I], a1 = a_trp[I + 1], b0 = b_trp[J], b1 = b_trp[J + 1];
        bool a_short = (a1 - a0) <= (b1 - b0);
        uint32_t s0 = a_short ? a0 : b0, s1 = a_short ? a1 : b1;
        uint32_t l0 = a_short ? b0 : a0, l1 = a_short ? b1 : a1;
        const uint32_t *stci = a_short ? a_tci : b_tci;
        const uint32_t *ltci = a_short ? b_tci : a_tci;
        uint32_t c0 = s0 + it.y * chunk, c1 = min(s1, c0 + chunk);
        // narrow the long row to the chunk's value range once per warp
        uint32_t first = __ldg(stci + c0), last = __ldg(stci + c1 - 1);
        uint32_t lo = lower_bound_u32(ltci, l0, l1, first);
        uint32_t hi = lower_bound_u32(ltci, lo, l1, last + 1);
        if (lo == hi || rows_used == 0) continue;
        for (uint32_t base = c0; base < c1; base += 32) {
            uint32_t si = base + lane;
            uint32_t ta = 0, tb = 0;
            bool hit = false;
            if (si < c1) {
                uint32_t K = __ldg(stci + si);
                uint32_t li = lower_bound_u32(ltci, lo, hi, K);
                if (li < hi && __ldg(ltci + li) == K) {
                    hit = true;
                    ta = a_short ? si : li;
                    tb = a_short ? li : si;
                }
            }
            if (!__ballot_sync(0xffffffffu, hit)) continue;
            uint32_t ru = rows_used;
            while (ru) {  // warp-uniform loop over non-empty mask rows
                int r = __ffs(ru) - 1;
                ru &= ru - 1;
                uint32_t mw = __shfl_sync(0xffffffffu, mword, r);
                if (hit) {
                    uint32_t aw = a_tiles[(size_t)ta * D + r];
                    if (work) units += aw ? __popc(mw) : 0u;  // AND+POPC units
                    while (aw && mw) {
                        int c = __ffs(mw) - 1;
                        mw &= mw - 1;
                        acc += __popc(aw & (uint32_t)b_tiles[(size_t)tb * D + c]);
                    }
                }
            }
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
    if (work) {
        for (int o = 16; o; o >>= 1) units += __shfl_xor_sync(0xffffffffu, units, o);
        if (lane == 0 && units) atomicAdd(work, units);
    }
}

// ------------------------------------------------------------ row-hash items
// Mask rows whose A row is short enough (<= TCH_MAX tiles): one warp per mask
// row I stages A's row I once as an open-addressing table in shared memory
// (tile column -> position; load factor <= 1/2), then for every mask tile
// (I, J) streams Bt's row J with coalesced loads and probes the table -- O(1)
// per entry instead of a binary search of the longer row per entry of the
// shorter one (s20 d=4: 2.5 G searched entries x ~8 dependent steps).  Hits
// do the AND+POPC of the pair's tiles exactly as below; the sum over common K
// is order-free integer arithmetic.  Longer A rows keep the chunked
// binary-search items.
constexpr uint32_t TCH_SLOTS = 1024;             // per warp
constexpr uint32_t TCH_MAX = TCH_SLOTS / 2;      // longest A row staged
constexpr uint32_t TCH_WARPS = 8;

__device__ __forceinline__ uint32_t tch_hash(uint32_t k, uint32_t shift) { return (k * 0x9E3779B1u) >> shift; }

template <int D>
__device__ __forceinline__ uint64_t tile_bits(const typename WordT<D>::T *__restrict__ tiles, size_t t) {
    // D <= 8: the whole tile in one load (row r in byte r; d = 4 keeps the high nibble clear)
    if constexpr (D == 4) return __ldg(reinterpret_cast<const uint32_t *>(tiles) + t);
    else return __ldg(reinterpret_cast<const unsigned long long *>(tiles) + t);
}

template <int D>
__global__ void __launch_bounds__(TCH_WARPS * 32) k_tc_rowhash(
    uint32_t m_ntr, uint32_t m_row0, const uint32_t *__restrict__ m_trp, const uint32_t *__restrict__ m_tci,
    const typename WordT<D>::T *__restrict__ m_tiles, const uint32_t *__restrict__ a_trp,
    const uint32_t *__restrict__ a_tci, const typename WordT<D>::T *__restrict__ a_tiles,
    const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
    const typename WordT<D>::T *__restrict__ b_tiles, const uint2 *__restrict__ hitems, uint32_t n_hitems,
    uint32_t *__restrict__ next_item, unsigned long long *__restrict__ out, unsigned long long *__restrict__ work) {
    __shared__ uint32_t keys[TCH_WARPS][TCH_SLOTS];
    __shared__ uint16_t posn[TCH_WARPS][TCH_SLOTS];
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t *kt = keys[wid];
    uint16_t *pt = posn[wid];
    unsigned long long acc = 0, units = 0;
    for (;;) {
        uint32_t w = 0;
        if (lane == 0) w = atomicAdd(next_item, 1u);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= n_hitems) break;
        const uint2 hit_item = hitems[w];
        const uint32_t i = hit_item.x, part = hit_item.y & 0xFFFFu, parts = hit_item.y >> 16;
        uint32_t m0 = __ldg(m_trp + i), m1 = __ldg(m_trp + i + 1);
        const uint32_t I = m_row0 + i, a0 = __ldg(a_trp + I), la = __ldg(a_trp + I + 1) - a0;
        if (parts > 1) {  // this item's share of the row's mask tiles: equal Bt-row entry counts
            const uint32_t nj = m1 - m0;  // <= TCH_MAX
            uint32_t lens[TCH_MAX / 32], run = 0;
#pragma unroll
            for (int k = 0; k < (int)(TCH_MAX / 32); k++) {
                const uint32_t j = k * 32 + lane;
                uint32_t l = 0;
                if (j < nj) {
                    const uint32_t J = __ldg(m_tci + m0 + j);
                    l = __ldg(b_trp + J + 1) - __ldg(b_trp + J);
                }
                uint32_t incl = l;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (uint32_t)o) incl += y;
                }
                lens[k] = run + incl - l;  // exclusive prefix of j
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            const unsigned long long tot = run;
            const uint32_t lo_t = (uint32_t)(tot * part / parts), hi_t = (uint32_t)(tot * (part + 1) / parts);
            uint32_t jlo = 0, jhi = 0;
#pragma unroll
            for (int k = 0; k < (int)(TCH_MAX / 32); k++) {
                const uint32_t j = k * 32 + lane;
                jlo += __popc(__ballot_sync(0xffffffffu, j < nj && lens[k] < lo_t));
                jhi += __popc(__ballot_sync(0xffffffffu, j < nj && lens[k] < hi_t));
            }
            if (part + 1 == parts) jhi = nj;
            if (part == 0) jlo = 0;
            m1 = m0 + jhi;
            m0 = m0 + jlo;
            if (m0 >= m1) continue;
        }
        const uint32_t lg = max(5u, 32u - __clz(2 * la - 1));  // slots = 2^lg >= 2*la
        const uint32_t S = 1u << lg, shift = 32 - lg;
        for (uint32_t q = lane; q < S; q += 32) kt[q] = 0;
        __syncwarp();
        for (uint32_t q = lane; q < la; q += 32) {
            const uint32_t K = __ldg(a_tci + a0 + q);
            uint32_t h = tch_hash(K, shift);
            while (atomicCAS(kt + h, 0u, K + 1) != 0u) h = (h + 1) & (S - 1);
            pt[h] = (uint16_t)q;
        }
        __syncwarp();
        for (uint32_t mt = m0; mt < m1; mt++) {
            const uint32_t J = __ldg(m_tci + mt);
            const uint32_t b0 = __ldg(b_trp + J), b1 = __ldg(b_trp + J + 1);
            if (b0 == b1) continue;
            uint64_t mbits = 0;
            uint32_t mword = 0, rows_used = 0;
            if constexpr (D <= 8) {
                mbits = tile_bits<D>(m_tiles, mt);
            } else {
                mword = lane < (uint32_t)D ? (uint32_t)m_tiles[(size_t)mt * D + lane] : 0u;
                rows_used = __ballot_sync(0xffffffffu, mword != 0);
            }
            for (uint32_t base = b0; base < b1; base += 32) {
                const uint32_t t = base + lane;
                uint32_t ta = 0xFFFFFFFFu;
                if (t < b1) {
                    const uint32_t K = __ldg(b_tci + t);
                    uint32_t h = tch_hash(K, shift);
                    for (;;) {
                        const uint32_t k = kt[h];
                        if (k == K + 1) { ta = pt[h]; break; }
                        if (k == 0) break;
                        h = (h + 1) & (S - 1);
                    }
                }
                const bool hit = ta != 0xFFFFFFFFu;
                if constexpr (D <= 8) {
                    if (hit) {
                        const uint64_t av = tile_bits<D>(a_tiles, (size_t)a0 + ta), bv = tile_bits<D>(b_tiles, t);
                        uint64_t mm = mbits;
                        while (mm) {  // mask bit (r, c) at bit 8r + c
                            const int bit = __ffsll((long long)mm) - 1;
                            const uint32_t r = bit >> 3;
                            const uint32_t aw = (uint32_t)(av >> (8 * r)) & 0xFFu;
                            const uint32_t mw = (uint32_t)(mm >> (8 * r)) & 0xFFu;
                            mm &= ~(0xFFull << (8 * r));
                            if (!aw) continue;
                            if (work) units += __popc(mw);
                            uint32_t cc = mw;
                            while (cc) {
                                const int c = __ffs(cc) - 1;
                                cc &= cc - 1;
                                acc += __popc(aw & ((uint32_t)(bv >> (8 * c)) & 0xFFu));
                            }
                        }
                    }
                } else {
                    if (!__ballot_sync(0xffffffffu, hit)) continue;
                    uint32_t ru = rows_used;
                    while (ru) {  // warp-uniform loop over non-empty mask rows
                        const int r = __ffs(ru) - 1;
                        ru &= ru - 1;
                        uint32_t mw = __shfl_sync(0xffffffffu, mword, r);
                        if (hit) {
                            const uint32_t aw = a_tiles[((size_t)a0 + ta) * D + r];
                            if (work) units += aw ? __popc(mw) : 0u;
                            while (aw && mw) {
                                const int c = __ffs(mw) - 1;
                                mw &= mw - 1;
                                acc += __popc(aw & (uint32_t)b_tiles[(size_t)t * D + c]);
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
    if (work) {
        for (int o = 16; o; o >>= 1) units += __shfl_xor_sync(0xffffffffu, units, o);
        if (lane == 0 && units) atomicAdd(work, units);
    }
}

constexpr uint32_t TCH_BUDGET = 4096;  // probed Bt entries per row-hash work item

// parts of each eligible mask row (0: the row takes the binary-search items or is empty)
__global__ void k_tch_parts(uint32_t mntr, uint32_t m_row0, const uint32_t *__restrict__ m_trp,
                            const uint32_t *__restrict__ m_tci, const uint32_t *__restrict__ a_trp,
                            const uint32_t *__restrict__ b_trp, uint32_t *__restrict__ parts) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < mntr; i += warps) {
        const uint32_t m0 = m_trp[i], m1 = m_trp[i + 1], I = m_row0 + i;
        const uint32_t la = a_trp[I + 1] - a_trp[I];
        uint32_t p = 0;
        if (m1 > m0 && la && la <= TCH_MAX && m1 - m0 <= TCH_MAX) {
            unsigned long long w = 0;
            for (uint32_t t = m0 + lane; t < m1; t += 32) {
                const uint32_t J = m_tci[t];
                w += b_trp[J + 1] - b_trp[J];
            }
            for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            const unsigned long long q = (w + TCH_BUDGET - 1) / TCH_BUDGET;
            p = q == 0 ? 1u : (q > 0xFFFFull ? 0xFFFFu : (uint32_t)q);
        }
        if (lane == 0) parts[i] = p;
    }
}

__global__ void k_tch_fill(uint32_t mntr, const uint32_t *__restrict__ parts, const uint64_t *__restrict__ ofs,
                           uint2 *__restrict__ items) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mntr; i += gridDim.x * blockDim.x) {
        const uint32_t P = parts[i];
        const uint64_t o = ofs[i];
        for (uint32_t q = 0; q < P; q++) items[o + q] = make_uint2(i, (P << 16) | q);
    }
}

// Measured (s20, B200): row-hash 41.8 / 50.4 ms vs binary-search items 25.6 /
// 32.0 ms at d = 4 / 8 -- ncu: 25.8 G warp instructions (probe loops, partial
// 32-entry chunks of short Bt rows, 0.56 G shared-memory bank conflicts) vs
// 17.8 G.  Kept as an A/B path, off by default (B2SR_TC_HASH=1 enables it).
static bool tc_rowhash_enabled() {
    const char *e = getenv("B2SR_TC_HASH");
    return e && e[0] == '1';
}

int64_t bmm_masked_bt(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, cudaStream_t s,
                      uint64_t *work_out = nullptr) {
    if (work_out) *work_out = 0;
    if (!mask->num_tiles || !a->num_tiles || !bt->num_tiles) return 0;
    uint64_t TM = mask->num_tiles;
    Buf<uint32_t> rowid(TM, s), cnt(TM, s);
    Buf<uint64_t> ofs(TM + 1, s);
    row_ids(mask, rowid.p, s);
    const char *ce = getenv("B2SR_TC_CHUNK");  // entries of the shorter row per work item (A/B)
    const uint32_t chunk = ce ? std::max(32, atoi(ce)) : TC_CHUNK;
    const bool hashed = tc_rowhash_enabled();
    LAUNCH(k_tc_item_counts, grid_for(TM), 256, 0, s, TM, rowid.p, mask->tci, mask->row0, a->trp, bt->trp, chunk, cnt.p,
           hashed ? TCH_MAX : 0u, mask->trp);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, TM, s);
    uint64_t n_items = read_scalar(ofs.p + TM, s);
    Buf<unsigned long long> out(1, s);
    CK(cudaMemsetAsync(out.p, 0, 8, s));
    Buf<unsigned long long> work(1, s);
    if (work_out) CK(cudaMemsetAsync(work.p, 0, 8, s));
    Buf<uint2> items(std::max<uint64_t>(n_items, 1), s);
    if (n_items) LAUNCH(k_tc_item_fill, grid_for(TM), 256, 0, s, TM, cnt.p, ofs.p, items.p);
    uint64_t blocks = (n_items + 7) / 8, cap = (uint64_t)num_sms() * 16;
    unsigned g = (unsigned)std::min(blocks, cap);
    Buf<uint32_t> next_row(1, s);
    CK(cudaMemsetAsync(next_row.p, 0, 4, s));
    kernel_timer().begin(s);
    Buf<uint2> hitems;
    uint32_t n_hitems = 0;
    if (hashed) {
        // work items of the row-hash kernel: each eligible mask row cut into
        // parts of <= TCH_BUDGET probed Bt entries (bounded tail), rows handed
        // out dynamically
        const uint32_t mntr = mask->ntr;
        Buf<uint32_t> pc(std::max<uint32_t>(mntr, 1), s);
        Buf<uint64_t> pofs((size_t)mntr + 1, s);
        LAUNCH(k_tch_parts, grid_for((uint64_t)mntr * 32), 256, 0, s, mntr, mask->row0, mask->trp, mask->tci, a->trp,
               bt->trp, pc.p);
        exclusive_scan_u32_to_u64(pc.p, pofs.p, mntr, s);
        n_hitems = (uint32_t)read_scalar(pofs.p + mntr, s);
        hitems = Buf<uint2>(std::max<uint32_t>(n_hitems, 1), s);
        if (n_hitems) LAUNCH(k_tch_fill, grid_for(mntr), 256, 0, s, mntr, pc.p, pofs.p, hitems.p);
    }
    if (n_hitems) {
        const unsigned gh = (unsigned)std::min<uint64_t>((uint64_t)num_sms() * 6, ((uint64_t)n_hitems + TCH_WARPS - 1) / TCH_WARPS);
        switch (a->dim) {
#define TCH_CASE(DD, W)                                                                                          \
    case DD:                                                                                                     \
        LAUNCH(k_tc_rowhash<DD>, gh, TCH_WARPS * 32, 0, s, mask->ntr, mask->row0, mask->trp, mask->tci,         \
               (const W *)mask->tiles, a->trp, a->tci, (const W *)a->tiles, bt->trp, bt->tci,                   \
               (const W *)bt->tiles, hitems.p, n_hitems, next_row.p, out.p, work_out ? work.p : nullptr);        \
        break;
            TCH_CASE(4, uint8_t)
            TCH_CASE(8, uint8_t)
            TCH_CASE(16, uint16_t)
            TCH_CASE(32, uint32_t)
#undef TCH_CASE
        }
    }
    if (n_items) switch (a->dim) {
#define BMM_CASE(DD, W)                                                                                        \
    case DD:                                                                                                   \
        LAUNCH(k_bmm_masked_items<DD>, g, 256, 0, s, n_items, items.p, rowid.p, mask->tci,                    \
               (const W *)mask->tiles, a->trp, a->tci, (const W *)a->tiles, bt->trp, bt->tci,                 \
               (const W *)bt->tiles, mask->row0, out.p, work_out ? work.p : nullptr, chunk);                  \
        break;
        BMM_CASE(4, uint8_t)
        BMM_CASE(8, uint8_t)
        BMM_CASE(16, uint16_t)
        BMM_CASE(32, uint32_t)
#undef BMM_CASE
    }
    kernel_timer().end(s);
    if (work_out) *work_out = read_scalar(work.p, s);
    return (int64_t)read_scalar(out.p, s);
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_bmm_sum(const b2sr_matrix *a, const b2sr_matrix *b, int64_t *out, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (a->n != b->n || a->dim != b->dim) B2SR_THROW(B2SR_EINVAL, "operands must share n and tile width");
    if (b->row0 || b->ntr != tile_rows(b->n, b->dim)) B2SR_THROW(B2SR_EINVAL, "B must be a full matrix");
    const size_t rows = (size_t)tile_rows(a->n, a->dim) * a->dim;
    const size_t vb = padded_vec_bytes(b->ntr, b->dim);
    Buf<uint8_t> ones(vb, s);
    Buf<double> rowdeg(rows, s);
    Buf<unsigned long long> acc(1, s);
    CK(cudaMemsetAsync(ones.p, 0xFF, vb, s));  // bits past n meet no tile bits
    CK(cudaMemsetAsync(acc.p, 0, 8, s));
    launch_bbf(const_cast<b2sr_matrix *>(b), ones.p, nullptr, rowdeg.p, s);
    switch (a->dim) {
        case 4: bmm_sum_gather<4>(a, rowdeg.p, acc.p, s); break;
        case 8: bmm_sum_gather<8>(a, rowdeg.p, acc.p, s); break;
        case 16: bmm_sum_gather<16>(a, rowdeg.p, acc.p, s); break;
        default: bmm_sum_gather<32>(a, rowdeg.p, acc.p, s); break;
    }
    *out = (int64_t)read_scalar(acc.p, s);
    API_END
}

int b2sr_bmm_sum_masked_bt(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, int64_t *out,
                           void *stream) {
    API_BEGIN
    if (a->n != bt->n || a->dim != bt->dim || a->n != mask->n || a->dim != mask->dim)
        B2SR_THROW(B2SR_EINVAL, "operands must share n and tile width");
    if (a->row0 || bt->row0 || a->ntr != tile_rows(a->n, a->dim) || bt->ntr != a->ntr)
        B2SR_THROW(B2SR_EINVAL, "A and Bt must be full matrices (only the mask may be a row block)");
    *out = bmm_masked_bt(a, bt, mask, (cudaStream_t)stream);
    API_END
}

int b2sr_tc(const b2sr_matrix *lower, int64_t *count, void *stream) {
    API_BEGIN
    // bmm_masked(L, transpose(L), L): B = transpose(L) enters transposed, i.e. L.
    *count = bmm_masked_bt(lower, lower, lower, (cudaStream_t)stream);
    API_END
}

int b2sr_tc_work(const b2sr_matrix *lower, int64_t *count, uint64_t *work, void *stream) {
    API_BEGIN
    *count = bmm_masked_bt(lower, lower, lower, (cudaStream_t)stream, work);
    API_END
}

}  // extern "C"

// ================================================================ row-partitioned triangle count
// L replicated on every rank, the mask (L's tile rows) cut into
// contiguous blocks of equal estimated work -- per mask tile (I, J) the
// shorter of rows I and J (the intersection's search length) plus one -- each
// rank counts its block with K8, and one int64 all-reduce sums the counts.
namespace b2sr {

__global__ void k_tc_row_work(uint32_t ntr, const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                              unsigned long long *__restrict__ work) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < ntr; I += warps) {
        const uint32_t t0 = trp[I], t1 = trp[I + 1], li = t1 - t0;
        unsigned long long w = 0;
        for (uint32_t t = t0 + lane; t < t1; t += 32) {
            const uint32_t J = tci[t], lj = trp[J + 1] - trp[J];
            w += (li < lj ? li : lj) + 1;
        }
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0) work[I] = w;
    }
}

__global__ void k_work_cuts(const uint64_t *__restrict__ pre, uint32_t ntr, int world, uint32_t *__restrict__ cuts) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > world) return;
    if (k == 0 || k == world) {
        cuts[k] = k ? ntr : 0;
        return;
    }
    const unsigned long long target = (unsigned long long)pre[ntr] * k / world;
    uint32_t lo = 0, hi = ntr;
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (pre[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    cuts[k] = lo;
}

}  // namespace b2sr

#include "dist_comm.cuh"

extern "C" int b2sr_dist_tc(b2sr_comm *comm, const b2sr_matrix *lower, int64_t *count, uint32_t *rows_out,
                            void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (lower->row0 || lower->ntr != tile_rows(lower->n, lower->dim))
        B2SR_THROW(B2SR_EINVAL, "b2sr_dist_tc needs the full (replicated) lower triangle");
    Exchange *ex = comm->ex;
    const int W = ex->world, R = ex->rank;
    const uint32_t ntr = lower->ntr;
    Buf<unsigned long long> work(ntr + 1, s);
    Buf<uint64_t> pre(ntr + 1, s);
    Buf<uint32_t> cuts(W + 1, s);
    CK(cudaMemsetAsync(work.p, 0, 8 * ((size_t)ntr + 1), s));
    LAUNCH(k_tc_row_work, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, lower->trp, lower->tci, work.p);
    exclusive_scan_u64(reinterpret_cast<const uint64_t *>(work.p), pre.p, (size_t)ntr + 1, s);
    LAUNCH(k_work_cuts, 1, 64 * ((W + 64) / 64), 0, s, pre.p, ntr, W, cuts.p);
    std::vector<uint32_t> rows(W + 1);
    CK(cudaMemcpyAsync(rows.data(), cuts.p, 4 * (W + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (rows_out) std::copy(rows.begin(), rows.end(), rows_out);
    b2sr_matrix *blk = nullptr;
    int rc = b2sr_row_block(lower, rows[R], rows[R + 1], s, &blk);
    if (rc) throw Error{rc, std::string()};
    int64_t mine = 0;
    try {
        mine = bmm_masked_bt(lower, lower, blk, s);
    } catch (...) {
        free_matrix(blk);
        throw;
    }
    free_matrix(blk);
    Buf<int64_t> tot(1, s);
    CK(cudaMemcpyAsync(tot.p, &mine, 8, cudaMemcpyHostToDevice, s));
    ex->allreduce_sum_i64(tot.p, 1, s);
    *count = read_scalar(tot.p, s);
    API_END
}
