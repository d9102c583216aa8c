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
                                 uint32_t chunk, uint32_t *__restrict__ cnt,
                                 const uint8_t *__restrict__ elig, bool sym) {
    for (uint64_t mt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; mt < TM; mt += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t i = m_rowid[mt], I = i + m_row0, J = m_tci[mt];
        uint32_t la = a_trp[I + 1] - a_trp[I], lb = b_trp[J + 1] - b_trp[J];
        uint32_t sh = min(la, lb);
        // pairs the filter kernel takes get no items here: staged on mask row i
        // (non-SYM, elig per mask row), or on the longer of rows I and J (SYM,
        // elig per global row: with a mask row block the pair may belong to the
        // rank that owns row J)
        const uint32_t X = sym ? (lb > la ? J : I) : i;
        const bool filtered = elig && elig[X] != 0;
        cnt[mt] = la && lb && !filtered ? (sh + chunk - 1) / chunk : 0;
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

// ------------------------------------------------------------ row-filter items
// Staged rows of at most TCB_CAP tiles (every row of the degree-oriented DAG
// at R-MAT s20) and D <= 8: one CTA per work item (staged row X, partner
// chunk, part) stages row X in shared memory -- its tile columns, its tiles,
// a one-bit-per-column filter indexed by the low TCB_BITS_LG bits of the
// column and the first position of each of TCB_NB column buckets -- plus, per
// partner, the mask tile, the start and length of the streamed row and the
// prefix of its 32-entry chunk counts.  The item's chunks (each inside one
// streamed row) are strided over the 8 warps; per lane: one coalesced load of
// a column K (the next chunk's loads issued before this chunk's tests), one
// shared-memory filter test.  Filter hits go to a per-warp queue and are
// resolved 32 at a time with every lane busy: the bucket of K gives its
// position in row X (about one comparison), and the AND+POPC of the tile pair
// is done with byte-parallel masks.  Replaces the per-lane binary search of
// the longer row for every entry of the shorter one (~40 warp instructions
// per AND+POPC unit).  The sum over common K is order-free integer
// arithmetic, so the count is the item kernel's bit for bit.
constexpr uint32_t TCB_CAP = 1024;       // longest A row / mask row staged
constexpr uint32_t TCB_BITS_LG = 15;     // filter: 2^15 bits = 4 KB (false hits <= 1024 / 2^15, resolved cheaply)
constexpr uint32_t TCB_THREADS = 256;
constexpr uint32_t TCB_BUDGET = 32000;   // probed Bt entries per work item (B2SR_TC_BUDGET overrides; 16 K: +5 %)
constexpr uint32_t TCB_NB = 1024;        // column buckets of the staged row (hit lookup)
constexpr uint32_t TCB_MAXCH = 1024;     // 32-probe chunks per item: budget <= 32 * (TCB_MAXCH - 2)

template <int D>
using TileBits = typename std::conditional<D == 4, uint32_t, unsigned long long>::type;

template <int D>
__device__ __forceinline__ TileBits<D> tile_bits(const typename WordT<D>::T *__restrict__ tiles, size_t t) {
    // D <= 8: the whole tile in one load (row r in byte r; d = 4 keeps the high nibble clear)
    return __ldg(reinterpret_cast<const TileBits<D> *>(tiles) + t);
}

// bytes of x (< 256) replicated: byte c of the result is 0xFF iff bit c of m is set
__device__ __forceinline__ unsigned long long expand_bits8(uint32_t m) {
    unsigned long long e = ((unsigned long long)m * 0x0101010101010101ull) & 0x8040201008040201ull;
    e = ((e + 0x7F7F7F7F7F7F7F7Full) | e) & 0x8080808080808080ull;
    return (e >> 7) * 0xFFull;
}

// byte r of x non-zero -> bit r
template <int D>
__device__ __forceinline__ uint32_t nz_rows(TileBits<D> x) {
    unsigned long long y = (unsigned long long)x;
    y = (((y & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full) | y) & 0x8080808080808080ull;
    return (uint32_t)(((y >> 7) * 0x0102040810204080ull) >> 56);
}

// sum over mask bits (r, c) of m of popc(S[r] & T[c]) (S: the staged row's tile,
// T: the streamed row's tile).  units: the item kernel's AND+POPC unit count,
// sum over rows r with A[r] != 0 of popc(M[r]) in the ORIGINAL orientation --
// side 0: m = M, S = A; side 1: m = M^T, T = A.
template <int D>
__device__ __forceinline__ void tc_tile_pair(TileBits<D> m, TileBits<D> sa, TileBits<D> tb, uint32_t side,
                                             unsigned long long &acc, unsigned long long &units, bool count_units) {
    if (count_units) {
        const unsigned long long mm = (unsigned long long)m;
        units += side == 0 ? __popcll(mm & expand_bits8(nz_rows<D>(sa)))
                           : __popcll(mm & ((unsigned long long)nz_rows<D>(tb) * 0x0101010101010101ull));
    }
    while (m) {
        const uint32_t r = (uint32_t)(__ffsll((long long)m) - 1) >> 3;
        const uint32_t mw = (uint32_t)(m >> (8 * r)) & 0xFFu, aw = (uint32_t)(sa >> (8 * r)) & 0xFFu;
        m &= ~((TileBits<D>)0xFF << (8 * r));
        if (!aw) continue;
        const unsigned long long sel = expand_bits8(mw) & ((unsigned long long)aw * 0x0101010101010101ull);
        if constexpr (D == 4) acc += __popc((uint32_t)sel & (uint32_t)tb);
        else acc += __popcll(sel & (unsigned long long)tb);
    }
}

// a queued filter hit: confirm K in the staged row (binary search), then the
// tile pair (s_*: 32-bit shared addresses of the staged arrays)
template <int D>
__device__ __forceinline__ void tc_resolve(uint32_t t, const uint32_t *__restrict__ b_tci, uint32_t j, uint32_t s_acol,
                                           uint32_t s_start,
                                           uint32_t ksh, uint32_t s_atile, uint32_t s_mtile, uint32_t s_side,
                                           const typename WordT<D>::T *__restrict__ b_tiles, unsigned long long &acc,
                                           unsigned long long &units, bool count_units) {
    constexpr uint32_t TBY = sizeof(TileBits<D>);
    const uint32_t K = __ldg(b_tci + t);  // reloaded (L1): the queue keeps 6 bytes per hit
    // bucket K >> ksh of the staged row: positions [start[b], start[b+1]), ~1 entry
    const uint32_t b = K >> ksh;
    const uint32_t ab = lds_u32(s_start + 2 * (b & ~1u));  // start[b], start[b+1] (u16 pairs)
    uint32_t p = (b & 1u) ? (ab >> 16) : (ab & 0xFFFFu);
    const uint32_t pe = (b & 1u) ? lds_u16(s_start + 2 * (b + 1)) : (ab >> 16);
    while (p < pe && lds_u32(s_acol + 4 * p) < K) p++;
    if (p < pe && lds_u32(s_acol + 4 * p) == K) {
        TileBits<D> m, a;
        if constexpr (D == 4) { m = lds_u32(s_mtile + 4 * j); a = lds_u32(s_atile + 4 * p); }
        else { m = lds_u64(s_mtile + TBY * j); a = lds_u64(s_atile + TBY * p); }
        const uint32_t side = count_units ? (lds_u32(s_side + 4 * (j >> 5)) >> (j & 31u)) & 1u : 0u;
        tc_tile_pair<D>(m, a, tile_bits<D>(b_tiles, t), side, acc, units, count_units);
    }
}

// SYM: a staged row longer than TCB_CAP is cut into R column ranges of
// <= TCB_CAP of its own entries, range r covering columns [c_r, c_{r+1}) with
// c_r = the column of its entry r*CAP (c_0 = 0, c_R = infinity); a partner row
// is streamed against range r only over its entries in those columns (two
// binary searches of the sorted partner row), so every common column is met
// in exactly one range and no row needs the binary-search items.
__device__ __forceinline__ uint32_t tcf_ranges(uint32_t la) { return la ? (la + TCB_CAP - 1) / TCB_CAP : 0u; }

__device__ __forceinline__ uint32_t tcf_lower(const uint32_t *__restrict__ v, uint32_t lo, uint32_t hi, uint32_t key) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(v + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// the part of partner row [b0, b0 + lb) of Bt inside the columns of range r of
// staged row a0.. (la entries, R ranges)
__device__ __forceinline__ void tcf_restrict(const uint32_t *__restrict__ a_tci, uint32_t a0, uint32_t la,
                                             uint32_t R, uint32_t r, const uint32_t *__restrict__ b_tci,
                                             uint32_t &b0, uint32_t &lb) {
    if (R <= 1) return;
    const uint32_t b1 = b0 + lb;
    const uint32_t lo = r ? tcf_lower(b_tci, b0, b1, __ldg(a_tci + a0 + r * TCB_CAP)) : b0;
    const uint32_t hi = r + 1 < R ? tcf_lower(b_tci, lo, b1, __ldg(a_tci + a0 + (r + 1) * TCB_CAP)) : b1;
    b0 = lo;
    lb = hi - lo;
    (void)la;
}

// Work item {X, chunk, part, parts}: staged row X of A; its partners are
// positions [chunk * CAP, +CAP) of the concatenation (mask row X) ++ (row X
// of the mask's transpose MT, SYM only), and the item probes part `part` of
// `parts` of their streamed entries.
//   non-SYM (any A, Bt, M): partners = mask row X: (J, M_XJ), stream Bt row J.
//   SYM (triangle counting, A = Bt = M = L, MT = L^T): each pair (I, J) of L
//     is intersected once, staged on its LONGER row: mask row X keeps J when
//     len J <= len X (m = M_XJ), L^T row X keeps I when len I < len X (m = the
//     L^T tile = M_IX^T, and sum_{(r,c) in M} popc(A_I[r] & L_X[c]) =
//     sum_{(c,r) in M^T} popc(L_X[c] & A_I[r])): sum over pairs of the SHORTER
//     row (s20 d=4: 2.48 G probes instead of 5.0 G); excluded partners keep
//     their slot with no probes.
template <int D, bool SYM, bool RANGED>
__global__ void __launch_bounds__(TCB_THREADS, 6) k_tc_filter(
    uint32_t m_row0, const uint32_t *__restrict__ m_trp, const uint32_t *__restrict__ m_tci,
    const typename WordT<D>::T *__restrict__ m_tiles, const uint32_t *__restrict__ mt_trp,
    const uint32_t *__restrict__ mt_tci, const typename WordT<D>::T *__restrict__ mt_tiles,
    const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci, const typename WordT<D>::T *__restrict__ a_tiles,
    const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
    const typename WordT<D>::T *__restrict__ b_tiles, const uint4 *__restrict__ items, uint32_t n_items,
    uint32_t *__restrict__ next_item, unsigned long long *__restrict__ out, unsigned long long *__restrict__ work,
    uint32_t ksh) {
    using TB = TileBits<D>;
    constexpr uint32_t FLG = TCB_BITS_LG;
    constexpr uint32_t FW = 1u << (FLG - 5), FM = (1u << FLG) - 1;
    constexpr uint32_t NW = TCB_THREADS / 32, PER = TCB_CAP / TCB_THREADS;
    __shared__ uint32_t filt[FW];
    __shared__ uint32_t acol[TCB_CAP];
    __shared__ __align__(16) uint16_t bstart[TCB_NB + 2];  // staged row: first position of each column bucket
    __shared__ TB atile[TCB_CAP];
    __shared__ TB mtile[TCB_CAP];
    __shared__ uint32_t jst[TCB_CAP];
    __shared__ uint32_t jln[TCB_CAP];
    __shared__ uint32_t pre[TCB_CAP + 1];
    __shared__ uint32_t pside[TCB_CAP / 32];
    __shared__ uint16_t jfirst[TCB_MAXCH];
    __shared__ uint32_t ring_t[NW][64];
    __shared__ uint16_t ring_j[NW][64];
    __shared__ uint32_t wtot[NW];
    __shared__ uint4 s_item;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5, lt_mask = (1u << lane) - 1u;
    for (uint32_t q = tid; q < FW; q += TCB_THREADS) filt[q] = 0;
    unsigned long long acc = 0, units = 0;
    const uint32_t s_rt = smem_addr(&ring_t[wid][0]), s_rj = smem_addr(&ring_j[wid][0]);
    const uint32_t s_pre = smem_addr(pre), s_jst = smem_addr(jst), s_jf = smem_addr(jfirst), s_jln = smem_addr(jln);
    const uint32_t s_filt = smem_addr(filt), s_acol = smem_addr(acol), s_atile = smem_addr(atile);
    const uint32_t s_mtile = smem_addr(mtile), s_side = smem_addr(pside), s_start = smem_addr(bstart);
    for (;;) {
        if (tid == 0) {
            const uint32_t w = atomicAdd(next_item, 1u);
            s_item = w < n_items ? items[w] : make_uint4(0xFFFFFFFFu, 0, 0, 0);
        }
        __syncthreads();  // also orders the previous item's filter clear before this item's staging
        const uint4 it = s_item;
        if (it.x == 0xFFFFFFFFu) break;
        const uint32_t i = it.x, chunk = it.y & 0xFFFFu, rng = it.y >> 16, part = it.z, parts = it.w;
        const uint32_t I = m_row0 + i, a0f = __ldg(a_trp + I), laf = __ldg(a_trp + I + 1) - a0f;
        const uint32_t R = RANGED ? tcf_ranges(laf) : 1u;  // RANGED: the rows over TCB_CAP entries
        // this item's range of the staged row (SYM rows over TCB_CAP entries)
        const uint32_t a0 = a0f + rng * TCB_CAP, la = min(TCB_CAP, laf - rng * TCB_CAP);
        const uint32_t m0 = __ldg(m_trp + i), nL = __ldg(m_trp + i + 1) - m0;
        uint32_t t0 = 0, nT = 0;
        if constexpr (SYM) {
            t0 = __ldg(mt_trp + I);
            nT = __ldg(mt_trp + I + 1) - t0;
        }
        const uint32_t g0 = chunk * TCB_CAP, nm = min(TCB_CAP, nL + nT - g0);
        for (uint32_t q = tid; q < la; q += TCB_THREADS) {
            const uint32_t K = __ldg(a_tci + a0 + q);
            acol[q] = K;
            atile[q] = tile_bits<D>(a_tiles, (size_t)a0 + q);
            atomicOr(filt + ((K & FM) >> 5), 1u << (K & 31u));
        }
        // partners: streamed-row starts and lengths, mask tiles, block-exclusive
        // prefix of their 32-entry chunk counts
        uint32_t len[PER], run = 0;
#pragma unroll
        for (uint32_t k = 0; k < PER; k++) {
            const uint32_t q = tid * PER + k;
            len[k] = 0;
            if (q < nm) {
                const uint32_t g = g0 + q;
                uint32_t J;
                bool second = false;  // partner from MT
                if (!SYM || g < nL) {
                    J = __ldg(m_tci + m0 + g);
                    mtile[q] = tile_bits<D>(m_tiles, (size_t)m0 + g);
                } else {
                    second = true;
                    J = __ldg(mt_tci + t0 + (g - nL));
                    mtile[q] = tile_bits<D>(mt_tiles, (size_t)t0 + (g - nL));
                }
                uint32_t b0 = __ldg(b_trp + J), lb = __ldg(b_trp + J + 1) - b0;
                const bool keep_pair = !(SYM && (second ? lb >= laf : lb > laf));  // else staged on row J
                if (RANGED && keep_pair) tcf_restrict(a_tci, a0f, laf, R, rng, b_tci, b0, lb);
                const uint32_t kept = keep_pair ? lb : 0u;
                jst[q] = b0;
                jln[q] = kept;
                len[k] = (kept + 31) >> 5;  // 32-entry chunks
            }
            run += len[k];
        }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) wtot[wid] = incl;
        if (tid < TCB_CAP / 32) {  // side bit q: partner q comes from MT
            uint32_t sw = 0;
            if (SYM) {
                const uint32_t qb = tid * 32, first2 = nL > g0 ? nL - g0 : 0u;  // first MT partner slot
                if (first2 <= qb) sw = 0xFFFFFFFFu;
                else if (first2 < qb + 32) sw = 0xFFFFFFFFu << (first2 - qb);
            }
            pside[tid] = sw;
        }
        __syncthreads();
        uint32_t off = incl - run;
        for (uint32_t v = 0; v < wid; v++) off += wtot[v];
#pragma unroll
        for (uint32_t k = 0; k < PER; k++) {
            const uint32_t q = tid * PER + k;
            if (q <= nm) pre[q] = off;  // q == nm: the total
            off += len[k];
        }
        if (tid == TCB_THREADS - 1 && nm == TCB_CAP) pre[TCB_CAP] = off;
        // bucket starts of the staged row (acol is in place since the barrier above):
        // entry q fills the buckets after its predecessor's up to its own
        for (uint32_t q = tid; q <= la; q += TCB_THREADS) {
            const uint32_t bq = q < la ? acol[q] >> ksh : TCB_NB + 1;
            const uint32_t bp = q ? (acol[q - 1] >> ksh) + 1 : 0u;
            for (uint32_t bb = bp; bb <= bq && bb <= TCB_NB + 1; bb++) bstart[bb] = (uint16_t)q;
        }
        __syncthreads();
        const uint32_t total = pre[nm];  // chunks
        const uint32_t lo = (uint32_t)((unsigned long long)total * part / parts);
        const uint32_t hi = (uint32_t)((unsigned long long)total * (part + 1) / parts);
        // chunk -> its partner (each warp chunk lies inside one partner row: R-MAT
        // s20 pairs waste 10 % of the lanes on row tails, against a per-lane
        // partner search for chunks that cross rows)
        for (uint32_t j = tid; j < nm; j += TCB_THREADS) {
            const uint32_t c0 = max(pre[j], lo), c1 = min(pre[j + 1], hi);
            for (uint32_t c = c0; c < c1; c++) jfirst[c - lo] = (uint16_t)j;
        }
        __syncthreads();
        // filter hits are queued per warp (ring of 64) and resolved 32 at a
        // time with every lane busy: ~1 lane in 5 hits, so resolving them
        // in place would run the lookup on nearly every chunk
        uint32_t qh = 0, qtl = 0;
        auto locate = [&](uint32_t c, uint32_t &t, uint32_t &j) -> bool {
            j = lds_u16(s_jf + 2 * (c - lo));
            const uint32_t off = (c - lds_u32(s_pre + 4 * j)) * 32 + lane;
            t = lds_u32(s_jst + 4 * j) + off;
            return off < lds_u32(s_jln + 4 * j);
        };
        // two-deep pipeline: the column loads of the next chunk are issued
        // before the filter test of this one
        uint32_t c = lo + wid;
        uint32_t t_c = 0, j_c = 0, K_c = 0;
        bool v_c = false;
        if (c < hi) {
            v_c = locate(c, t_c, j_c);
            K_c = v_c ? __ldg(b_tci + t_c) : 0u;
        }
        for (; c < hi; c += NW) {
            uint32_t t_n = 0, j_n = 0, K_n = 0;
            bool v_n = false;
            if (c + NW < hi) {
                v_n = locate(c + NW, t_n, j_n);
                K_n = v_n ? __ldg(b_tci + t_n) : 0u;
            }
            const bool hit = v_c && ((lds_u32(s_filt + 4 * ((K_c & FM) >> 5)) >> (K_c & 31u)) & 1u);
            const uint32_t hm = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const uint32_t pos = (qtl + __popc(hm & lt_mask)) & 63u;
                sts_u32(s_rt + 4 * pos, t_c);
                sts_u16(s_rj + 2 * pos, j_c);
            }
            qtl += __popc(hm);
            if (qtl - qh >= 32) {
                __syncwarp();
                const uint32_t pos = (qh + lane) & 63u;
                tc_resolve<D>(lds_u32(s_rt + 4 * pos), b_tci, lds_u16(s_rj + 2 * pos), s_acol,
                              s_start, ksh, s_atile, s_mtile, s_side, b_tiles, acc, units, work != nullptr);
                qh += 32;
                __syncwarp();
            }
            t_c = t_n; j_c = j_n; K_c = K_n; v_c = v_n;
        }
        __syncwarp();
        if (lane < qtl - qh) {
            const uint32_t pos = (qh + lane) & 63u;
            tc_resolve<D>(lds_u32(s_rt + 4 * pos), b_tci, lds_u16(s_rj + 2 * pos), s_acol,
                          s_start, ksh, s_atile, s_mtile, s_side, b_tiles, acc, units, work != nullptr);
        }
        __syncthreads();
        for (uint32_t q = tid; q < la; q += TCB_THREADS) filt[(acol[q] & FM) >> 5] = 0;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
    if (work) {
        for (int o = 16; o; o >>= 1) units += __shfl_xor_sync(0xffffffffu, units, o);
        if (lane == 0 && units) atomicAdd(work, units);
    }
}

// Items of the filter kernel.  Per staged row X (X = mask row i, I = row0 + i):
// eligible iff 0 < len_A(X) <= CAP (D <= 8); non-SYM also needs the mask row
// <= CAP partners.  k_tcf_chunks: partner chunks of CAP per eligible row;
// k_tcf_parts: per chunk, the probes it streams cut into parts of <= budget.
__global__ void k_tcf_chunks(uint32_t mntr, uint32_t m_row0, const uint32_t *__restrict__ m_trp,
                             const uint32_t *__restrict__ mt_trp, const uint32_t *__restrict__ a_trp,
                             uint32_t *__restrict__ nch, uint8_t *__restrict__ elig) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mntr; i += gridDim.x * blockDim.x) {
        const uint32_t I = m_row0 + i, la = a_trp[I + 1] - a_trp[I];
        const uint32_t np = (m_trp[i + 1] - m_trp[i]) + (mt_trp ? mt_trp[I + 1] - mt_trp[I] : 0u);
        // SYM: any non-empty row (long rows in column ranges); else <= CAP and <= CAP partners
        const bool ok = la > 0 && (mt_trp || (la <= TCB_CAP && np <= TCB_CAP));
        elig[i] = ok;
        const uint32_t R = mt_trp ? tcf_ranges(la) : 1u;
        nch[i] = ok ? R * ((np + TCB_CAP - 1) / TCB_CAP) : 0u;
    }
}

// SYM: a row can be staged iff it is not empty (per global row)
__global__ void k_tcf_elig_global(uint32_t ntr, const uint32_t *__restrict__ a_trp, uint8_t *__restrict__ elig) {
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x) {
        elig[I] = a_trp[I + 1] > a_trp[I];  // every non-empty row can be staged (column ranges)
    }
}

__global__ void k_tcf_chunk_list(uint32_t mntr, const uint32_t *__restrict__ nch, const uint64_t *__restrict__ ofs,
                                 uint2 *__restrict__ chunks) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mntr; i += gridDim.x * blockDim.x)
        for (uint32_t c = 0; c < nch[i]; c++) chunks[ofs[i] + c] = make_uint2(i, c);  // c = range * npc + chunk
}

// warp per chunk: probes = sum of the streamed lengths of its kept partners
__global__ void k_tcf_parts(uint32_t nchunks, uint2 *__restrict__ chunks, uint32_t m_row0,
                            const uint32_t *__restrict__ m_trp, const uint32_t *__restrict__ m_tci,
                            const uint32_t *__restrict__ mt_trp, const uint32_t *__restrict__ mt_tci,
                            const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci,
                            const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci, uint32_t budget,
                            uint32_t *__restrict__ parts, uint32_t *__restrict__ parts_ranged) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += warps) {
        const uint2 ch = chunks[c];
        const uint32_t i = ch.x, I = m_row0 + i, a0 = a_trp[I], la = a_trp[I + 1] - a0;
        const uint32_t m0 = m_trp[i], nL = m_trp[i + 1] - m0;
        const uint32_t t0 = mt_trp ? mt_trp[I] : 0u, nT = mt_trp ? mt_trp[I + 1] - t0 : 0u;
        const uint32_t npc = (nL + nT + TCB_CAP - 1) / TCB_CAP, R = mt_trp ? tcf_ranges(la) : 1u;
        const uint32_t rng = ch.y / npc, pc = ch.y % npc;
        const uint32_t g0 = pc * TCB_CAP, g1 = min(g0 + TCB_CAP, nL + nT);
        unsigned long long w = 0;
        for (uint32_t g = g0 + lane; g < g1; g += 32) {
            const bool second = g >= nL;
            const uint32_t J = second ? mt_tci[t0 + (g - nL)] : m_tci[m0 + g];
            uint32_t b0 = b_trp[J], lb = b_trp[J + 1] - b0;
            if (!mt_trp || (second ? lb < la : lb <= la)) {
                if (mt_trp) tcf_restrict(a_tci, a0, la, R, rng, b_tci, b0, lb);
                w += (lb + 31) / 32;  // 32-entry chunks
            }
        }
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        const unsigned long long q = (w + budget - 1) / budget;  // budget: chunks per item
        if (lane == 0) {
            const uint32_t P = (q == 0 || w >= 0x80000000ull) ? 0u : (q > 0xFFFFull ? 0xFFFFu : (uint32_t)q);
            parts[c] = R > 1 ? 0u : P;         // items of the plain kernel
            parts_ranged[c] = R > 1 ? P : 0u;  // items of the column-range kernel
            chunks[c].y = (rng << 16) | pc;    // what the filter kernel's items carry
        }
    }
}

__global__ void k_tcf_fill(uint32_t nchunks, const uint2 *__restrict__ chunks, const uint32_t *__restrict__ parts,
                           const uint64_t *__restrict__ ofs, uint4 *__restrict__ items) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += gridDim.x * blockDim.x) {
        const uint32_t P = parts[c];
        for (uint32_t q = 0; q < P; q++) items[ofs[c] + q] = make_uint4(chunks[c].x, chunks[c].y, q, P);
    }
}

// B2SR_TC_FILTER=0: every mask tile on the binary-search items (A/B)
static bool tc_filter_enabled(int dim) {
    const char *e = getenv("B2SR_TC_FILTER");
    return dim <= 8 && !(e && e[0] == '0');
}

// mt: the mask's transpose (SYM triangle counting: a = bt = mask = L, mt = L^T), else null
int64_t bmm_masked_bt(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, cudaStream_t s,
                      uint64_t *work_out = nullptr, const b2sr_matrix *mt = nullptr) {
    if (work_out) *work_out = 0;
    if (!mask->num_tiles || !a->num_tiles || !bt->num_tiles) return 0;
    uint64_t TM = mask->num_tiles;
    Buf<uint32_t> rowid(TM, s), cnt(TM, s);
    Buf<uint64_t> ofs(TM + 1, s);
    row_ids(mask, rowid.p, s);
    const char *ce = getenv("B2SR_TC_CHUNK");  // entries of the shorter row per work item (A/B)
    const uint32_t chunk = ce ? std::max(32, atoi(ce)) : TC_CHUNK;
    const bool filtered = tc_filter_enabled(a->dim);
    const bool sym = filtered && mt != nullptr;
    Buf<uint4> fitems;  // plain items, then the column-range items (SYM rows over TCB_CAP)
    Buf<uint8_t> elig;
    uint32_t n_fitems = 0, n_ritems = 0;
    if (filtered) {
        // work items of the filter kernel, handed out dynamically
        const char *be = getenv("B2SR_TC_BUDGET");
        const uint32_t budget =  // in 32-entry chunks (the jfirst table holds TCB_MAXCH)
            (be ? (uint32_t)std::min(32 * (int)(TCB_MAXCH - 2), std::max(256, atoi(be))) : TCB_BUDGET) / 32;
        const uint32_t mntr = mask->ntr;
        elig = Buf<uint8_t>(std::max<uint32_t>(mntr, 1), s);
        Buf<uint32_t> nch(std::max<uint32_t>(mntr, 1), s);
        Buf<uint64_t> cofs((size_t)mntr + 1, s);
        LAUNCH(k_tcf_chunks, grid_for(mntr), 256, 0, s, mntr, mask->row0, mask->trp, sym ? mt->trp : nullptr, a->trp,
               nch.p, elig.p);
        exclusive_scan_u32_to_u64(nch.p, cofs.p, mntr, s);
        const uint32_t nchunks = (uint32_t)read_scalar(cofs.p + mntr, s);
        if (nchunks) {
            Buf<uint2> chunks(nchunks, s);
            Buf<uint32_t> pc(nchunks, s), pcr(nchunks, s);
            Buf<uint64_t> pofs((size_t)nchunks + 1, s), rofs((size_t)nchunks + 1, s);
            LAUNCH(k_tcf_chunk_list, grid_for(mntr), 256, 0, s, mntr, nch.p, cofs.p, chunks.p);
            LAUNCH(k_tcf_parts, grid_for((uint64_t)nchunks * 32), 256, 0, s, nchunks, chunks.p, mask->row0, mask->trp,
                   mask->tci, sym ? mt->trp : nullptr, sym ? mt->tci : nullptr, a->trp, a->tci, bt->trp, bt->tci,
                   budget, pc.p, pcr.p);
            exclusive_scan_u32_to_u64(pc.p, pofs.p, nchunks, s);
            exclusive_scan_u32_to_u64(pcr.p, rofs.p, nchunks, s);
            n_fitems = (uint32_t)read_scalar(pofs.p + nchunks, s);
            n_ritems = (uint32_t)read_scalar(rofs.p + nchunks, s);
            fitems = Buf<uint4>(std::max<uint32_t>(n_fitems + n_ritems, 1), s);
            if (n_fitems) LAUNCH(k_tcf_fill, grid_for(nchunks), 256, 0, s, nchunks, chunks.p, pc.p, pofs.p, fitems.p);
            if (n_ritems)
                LAUNCH(k_tcf_fill, grid_for(nchunks), 256, 0, s, nchunks, chunks.p, pcr.p, rofs.p, fitems.p + n_fitems);
        }
    }
    Buf<uint8_t> elig_g;
    if (sym) {
        elig_g = Buf<uint8_t>(std::max<uint32_t>(a->ntr, 1), s);
        LAUNCH(k_tcf_elig_global, grid_for(a->ntr), 256, 0, s, a->ntr, a->trp, elig_g.p);
    }
    LAUNCH(k_tc_item_counts, grid_for(TM), 256, 0, s, TM, rowid.p, mask->tci, mask->row0, a->trp, bt->trp, chunk, cnt.p,
           sym ? elig_g.p : (filtered ? elig.p : nullptr), sym);
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
    if (n_fitems || n_ritems) {
        int per_sm = 1;
        const uint32_t *mtp = sym ? mt->trp : nullptr, *mtc = sym ? mt->tci : nullptr;
        const void *mtt = sym ? mt->tiles : nullptr;
        uint32_t ksh = 0;  // column bucket shift: (ntr - 1) >> ksh < TCB_NB
        while (((uint64_t)(a->ntr ? a->ntr - 1 : 0) >> ksh) >= TCB_NB) ksh++;
        for (int ranged = 0; ranged < 2; ranged++) {
            const uint32_t ni = ranged ? n_ritems : n_fitems;
            const uint4 *its = fitems.p + (ranged ? n_fitems : 0);
            if (!ni) continue;
            CK(cudaMemsetAsync(next_row.p, 0, 4, s));
            switch (a->dim * 4 + (sym ? 2 : 0) + ranged) {
#define TCB_CASE(DD, SY, RG, W)                                                                                      \
    case DD * 4 + SY * 2 + RG:                                                                                       \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc_filter<DD, SY, RG>, TCB_THREADS, 0));         \
        LAUNCH((k_tc_filter<DD, SY, RG>),                                                                            \
               (unsigned)std::min<uint64_t>((uint64_t)num_sms() * std::max(per_sm, 1), ni), TCB_THREADS, 0, s,       \
               mask->row0, mask->trp, mask->tci, (const W *)mask->tiles, mtp, mtc, (const W *)mtt, a->trp, a->tci,   \
               (const W *)a->tiles, bt->trp, bt->tci, (const W *)bt->tiles, its, ni, next_row.p, out.p,             \
               work_out ? work.p : nullptr, ksh);                                                                     \
        break;
                TCB_CASE(4, 0, 0, uint8_t)
                TCB_CASE(4, 1, 0, uint8_t)
                TCB_CASE(4, 1, 1, uint8_t)
                TCB_CASE(8, 0, 0, uint8_t)
                TCB_CASE(8, 1, 0, uint8_t)
                TCB_CASE(8, 1, 1, uint8_t)
#undef TCB_CASE
            }
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

// triangle counting: bmm_masked(L, transpose(L), L) -- B = transpose(L) enters
// transposed, i.e. L.  With the filter kernel, pairs are staged on their longer
// row, which needs L^T (one transpose of L; B2SR_TC_SYM=0 keeps row I staged).
static int64_t tc_count(const b2sr_matrix *lower, cudaStream_t s, uint64_t *work) {
    const char *e = getenv("B2SR_TC_SYM");
    if (tc_filter_enabled(lower->dim) && !(e && e[0] == '0') && lower->num_tiles) {
        b2sr_matrix *lt = transpose_device(lower, s);
        try {
            const int64_t c = bmm_masked_bt(lower, lower, lower, s, work, lt);
            free_matrix(lt);
            return c;
        } catch (...) {
            free_matrix(lt);
            throw;
        }
    }
    return bmm_masked_bt(lower, lower, lower, s, work);
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
    *count = tc_count(lower, (cudaStream_t)stream, nullptr);
    API_END
}

int b2sr_tc_work(const b2sr_matrix *lower, int64_t *count, uint64_t *work, void *stream) {
    API_BEGIN
    *count = tc_count(lower, (cudaStream_t)stream, work);
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

// SYM triangle counting: pair (I, J) costs its shorter row and is counted by the
// owner of the longer row X
__global__ void k_tc_row_work_sym(uint32_t ntr, const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                                  unsigned long long *__restrict__ work) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < ntr; I += warps) {
        const uint32_t t0 = trp[I], t1 = trp[I + 1], li = t1 - t0;
        for (uint32_t t = t0 + lane; t < t1; t += 32) {
            const uint32_t J = tci[t], lj = trp[J + 1] - trp[J];
            const uint32_t X = lj > li ? J : I;  // every non-empty row can be staged
            atomicAdd(work + X, (unsigned long long)(li < lj ? li : lj) + 1ull);
        }
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
    const char *se = getenv("B2SR_TC_SYM");
    const bool sym = tc_filter_enabled(lower->dim) && !(se && se[0] == '0') && lower->num_tiles;
    if (sym) LAUNCH(k_tc_row_work_sym, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, lower->trp, lower->tci, work.p);
    else LAUNCH(k_tc_row_work, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, lower->trp, lower->tci, work.p);
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
    b2sr_matrix *lt = nullptr;  // SYM: L^T replicated, each pair counted by the owner of its staged row
    try {
        if (sym) lt = transpose_device(lower, s);
        mine = bmm_masked_bt(lower, lower, blk, s, nullptr, lt);
    } catch (...) {
        free_matrix(blk);
        free_matrix(lt);
        throw;
    }
    free_matrix(blk);
    free_matrix(lt);
    Buf<int64_t> tot(1, s);
    CK(cudaMemcpyAsync(tot.p, &mine, 8, cudaMemcpyHostToDevice, s));
    ex->allreduce_sum_i64(tot.p, 1, s);
    *count = read_scalar(tot.p, s);
    API_END
}
