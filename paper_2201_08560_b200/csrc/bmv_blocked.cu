// Column-strip blocked bin-SpMV (bbb and the BFS pull sweep).
//
// Why: in the row-major B2SR stream every tile gathers its x word from L2 at
// a random column -- one 32-byte sector per tile.  At d=4/8 that sector
// traffic is 4x / 2.7x the tile bytes themselves and caps the streaming
// kernel far below HBM bandwidth (profiles/r01_ncu_full_k_bmv_bbb4_v1.csv:
// 5.4 GB L1 sector traffic for 1.03 GB of matrix).
//
// Plan (built once per matrix, cached on the handle): the tile columns are cut
// into P strips whose x bits fit in shared memory (STRIP_VERTS vertices =
// 128 KB of bits); the tiles of every tile row are re-laid strip-major --
// strip p holds, row after row, the (still column-sorted) tiles of that row
// falling in strip p -- so each (row, strip) segment is contiguous.  Tile
// bytes are identical to the reference layout, only their order changes.
//
// Kernel: persistent CTAs (1024 threads, one per SM) pull (strip, row block)
// work units from an atomic counter in strip-major order; a CTA stages the x
// strip into shared memory only when its strip changes, then groups of GS
// lanes walk row segments with 128-bit streaming loads and gather x from
// shared memory.  A row's strips are OR-combined into y with one atomicOr per
// (row, strip) -- OR is order-free, so the result is bit-identical.
#include "bmv_common.cuh"

namespace b2sr {

constexpr uint32_t STRIP_VERTS = 1u << 20;               // vertices per strip
constexpr uint32_t STRIP_SMEM = STRIP_VERTS / 8;         // 128 KB of x bits
constexpr uint32_t MAX_STRIPS = 16;
constexpr int BLK_THREADS = 1024;

struct BlockedPlan {
    uint32_t P = 1, R = 1, nB = 1, strip_cols = 1;
    uint32_t *seg = nullptr;   // P x (ntr+1) tile offsets (strip-major)
    uint32_t *tci = nullptr;   // strip-major tile columns
    void *tiles = nullptr;     // strip-major tiles
    bool owns = false;         // false when P == 1 (arrays alias the matrix)
};

void free_plan(void *p) {
    BlockedPlan *bp = static_cast<BlockedPlan *>(p);
    if (!bp) return;
    if (bp->owns) {
        dfree(bp->tci, nullptr);
        dfree(bp->tiles, nullptr);
    }
    dfree(bp->seg, nullptr);
    delete bp;
}

static unsigned grid_for(uint64_t work) {
    uint64_t b = (work + 255) / 256, cap = (uint64_t)num_sms() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

__device__ __forceinline__ uint32_t lb_u32(const uint32_t *v, uint32_t lo, uint32_t hi, uint32_t key) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (v[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// cnt[p*ntr + I] = tiles of row I in strip p
__global__ void k_plan_counts(uint32_t ntr, uint32_t P, uint32_t sc, const uint32_t *trp, const uint32_t *tci,
                              uint32_t *cnt) {
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x) {
        uint32_t t0 = trp[I], t1 = trp[I + 1], prev = t0;
        for (uint32_t p = 0; p < P; p++) {
            uint32_t b = p + 1 == P ? t1 : lb_u32(tci, prev, t1, (p + 1) * sc);
            cnt[(size_t)p * ntr + I] = b - prev;
            prev = b;
        }
    }
}

// seg[p*(ntr+1) + I] = ofs[p*ntr + I]  (the scan of cnt is strip-major)
__global__ void k_plan_seg(uint32_t ntr, uint32_t P, const uint64_t *ofs, uint32_t *seg) {
    size_t total = (size_t)P * (ntr + 1);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        size_t p = i / (ntr + 1), I = i % (ntr + 1);
        seg[i] = (uint32_t)ofs[p * ntr + I];
    }
}

// warp per tile row: copy each strip segment to its strip-major place
template <int TB>
__global__ void k_plan_copy(uint32_t ntr, uint32_t P, uint32_t sc, const uint32_t *trp, const uint32_t *tci,
                            const uint8_t *tiles, const uint32_t *seg, uint32_t *tci2, uint8_t *tiles2) {
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < ntr; I += warps) {
        uint32_t t0 = trp[I], t1 = trp[I + 1], prev = t0;
        for (uint32_t p = 0; p < P; p++) {
            uint32_t b = p + 1 == P ? t1 : lb_u32(tci, prev, t1, (p + 1) * sc);
            uint32_t dst = seg[(size_t)p * (ntr + 1) + I];
            for (uint32_t k = lane; k < b - prev; k += 32) {
                tci2[dst + k] = tci[prev + k];
                const uint8_t *src = tiles + (size_t)(prev + k) * TB;
                uint8_t *out = tiles2 + (size_t)(dst + k) * TB;
                if constexpr (TB % 16 == 0) {
#pragma unroll
                    for (int q = 0; q < TB / 16; q++)
                        reinterpret_cast<uint4 *>(out)[q] = reinterpret_cast<const uint4 *>(src)[q];
                } else if constexpr (TB == 8) {
                    *reinterpret_cast<uint2 *>(out) = *reinterpret_cast<const uint2 *>(src);
                } else {
                    *reinterpret_cast<uint32_t *>(out) = *reinterpret_cast<const uint32_t *>(src);
                }
            }
            prev = b;
        }
    }
}

BlockedPlan *ensure_plan(b2sr_matrix *m, cudaStream_t s) {
    if (m->plan) return static_cast<BlockedPlan *>(m->plan);
    uint32_t d = m->dim, ntr = m->ntr;
    uint32_t ncols = tile_rows(m->n, d);        // global tile columns
    uint32_t sc = STRIP_VERTS / d;              // tile columns per strip
    uint32_t P = (ncols + sc - 1) / sc;
    if (P > MAX_STRIPS) return nullptr;         // too many strips: the row-major kernel is used
    BlockedPlan *bp = new BlockedPlan();
    try {
        bp->P = P;
        bp->strip_cols = sc;
        uint64_t units = (uint64_t)num_sms() * 16;  // ~16 work units per SM
        uint64_t rows_per = ((uint64_t)ntr * P + units - 1) / units;
        bp->R = (uint32_t)std::max<uint64_t>(64, rows_per);
        bp->nB = (ntr + bp->R - 1) / bp->R;
        bp->seg = static_cast<uint32_t *>(dalloc((size_t)P * (ntr + 1) * 4, s));
        if (P == 1) {
            CK(cudaMemcpyAsync(bp->seg, m->trp, ((size_t)ntr + 1) * 4, cudaMemcpyDeviceToDevice, s));
            bp->tci = m->tci;
            bp->tiles = m->tiles;
            bp->owns = false;
        } else {
            Buf<uint32_t> cnt((size_t)P * ntr, s);
            Buf<uint64_t> ofs((size_t)P * ntr + 1, s);
            LAUNCH(k_plan_counts, grid_for(ntr), 256, 0, s, ntr, P, sc, m->trp, m->tci, cnt.p);
            exclusive_scan_u32_to_u64(cnt.p, ofs.p, (size_t)P * ntr, s);
            LAUNCH(k_plan_seg, grid_for((uint64_t)P * (ntr + 1)), 256, 0, s, ntr, P, ofs.p, bp->seg);
            size_t tb = (size_t)d * word_bytes(d);
            bp->tci = static_cast<uint32_t *>(dalloc(m->num_tiles * 4 + 16, s));
            bp->tiles = dalloc(m->num_tiles * tb + 16, s);
            bp->owns = true;
            unsigned g = grid_for((uint64_t)ntr * 32);
            const uint8_t *src = (const uint8_t *)m->tiles;
            uint8_t *dst = (uint8_t *)bp->tiles;
            switch (d) {
                case 4: LAUNCH(k_plan_copy<4>, g, 256, 0, s, ntr, P, sc, m->trp, m->tci, src, bp->seg, bp->tci, dst); break;
                case 8: LAUNCH(k_plan_copy<8>, g, 256, 0, s, ntr, P, sc, m->trp, m->tci, src, bp->seg, bp->tci, dst); break;
                case 16: LAUNCH(k_plan_copy<32>, g, 256, 0, s, ntr, P, sc, m->trp, m->tci, src, bp->seg, bp->tci, dst); break;
                default: LAUNCH(k_plan_copy<128>, g, 256, 0, s, ntr, P, sc, m->trp, m->tci, src, bp->seg, bp->tci, dst); break;
            }
        }
    } catch (...) {
        free_plan(bp);
        throw;
    }
    m->plan = bp;
    return bp;
}

// ------------------------------------------------------------ kernel
template <int D> struct GroupSize { static constexpr int GS = D <= 8 ? 8 : (D == 16 ? 16 : 32); };

constexpr uint32_t MAX_LONG = 256;

// keep word of a row; false when the row needs no work
template <int D, int MODE>
__device__ __forceinline__ bool row_keep(const void *keep, const void *live, uint32_t grow, uint32_t I,
                                         uint32_t &keepw) {
    if constexpr (MODE == 1) {
        keepw = ~load_word<D>(keep, grow) & load_word<D>(live, I);
        return keepw != 0;
    } else {
        keepw = keep ? load_word<D>(keep, grow) : 0xffffffffu;
        return true;
    }
}

// hit bits of one group step (TILES_STEP tiles starting at base) for this lane
template <int D, int MODE>
__device__ __forceinline__ uint32_t seg_step(const uint32_t *__restrict__ tci, const uint8_t *__restrict__ tiles,
                                             const uint32_t *xs, uint32_t c0, uint32_t base, uint32_t s0, uint32_t s1,
                                             uint32_t gl, uint32_t lane, uint32_t xmask) {
    using G = Geo<D>;
    uint32_t xw[G::TPL];
    uint4 v = make_uint4(0, 0, 0, 0);
    if constexpr (G::TPL > 1) {
        uint32_t tl = base + gl * G::TPL;
        uint32_t anyx = 0;
#pragma unroll
        for (int j = 0; j < G::TPL; j++) xw[j] = 0;
        if (tl < s1 && tl + G::TPL > s0) {
            uint32_t cols[G::TPL];
            if constexpr (G::TPL == 4) {
                uint4 c = ld_stream128(tci + tl);
                cols[0] = c.x; cols[1] = c.y; cols[2] = c.z; cols[3] = c.w;
            } else {
                uint2 c = *reinterpret_cast<const uint2 *>(tci + tl);
                cols[0] = c.x; cols[1] = c.y;
            }
#pragma unroll
            for (int j = 0; j < G::TPL; j++) {
                bool ok = tl + j >= s0 && tl + j < s1;
                uint32_t bit = (cols[j] - c0) * D;
                xw[j] = ok ? (xs[bit >> 5] >> (bit & 31)) & xmask : 0u;
                anyx |= xw[j];
            }
            if (MODE == 0 || anyx) v = ld_stream128(tiles + (size_t)tl * G::TB);
        }
    } else {
        uint32_t t = base + gl / G::LPT, q = gl % G::LPT;
        xw[0] = 0;
        if (t < s1) {
            uint32_t bit = (__ldg(tci + t) - c0) * D;
            xw[0] = (xs[bit >> 5] >> (bit & 31)) & xmask;
            if (MODE == 0 || xw[0]) v = ld_stream128(tiles + (size_t)t * G::TB + q * 16);
        }
    }
    return hits16<D>(v, xw, lane);
}

// MODE 0: y = (A x) & keep (keep may be null); MODE 1: BFS pull,
// next = (A frontier) & ~visited & live with payload skipping and early exit.
template <int D, int MODE>
__global__ void __launch_bounds__(BLK_THREADS, 1)
k_blocked(uint32_t P, uint32_t R, uint32_t nB, uint32_t sc, uint32_t ntr, uint32_t ncols, uint32_t row0,
          const uint32_t *__restrict__ seg, const uint32_t *__restrict__ tci, const uint8_t *__restrict__ tiles,
          const void *__restrict__ x, const void *__restrict__ keep, const void *__restrict__ live,
          void *__restrict__ y, uint32_t *__restrict__ counter) {
    using G = Geo<D>;
    constexpr int GS = GroupSize<D>::GS;
    constexpr uint32_t TILES_STEP = GS * G::TPL / G::LPT;  // tiles per group step
    constexpr uint32_t MIN_LONG = 4 * TILES_STEP;          // pass-2 threshold floor (tiles)
    extern __shared__ uint32_t xs[];                        // strip bits
    __shared__ uint32_t s_unit, s_nlong, s_overflow;
    __shared__ uint32_t s_long[MAX_LONG];
    const uint32_t lane = lane_id();
    const uint32_t gl = threadIdx.x % GS;                   // lane within group
    const uint32_t group = threadIdx.x / GS, ngroups = blockDim.x / GS;
    const uint32_t gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1u) << (lane & ~(GS - 1u)));
    const uint32_t nunits = P * nB;
    const uint32_t xmask = D == 32 ? 0xffffffffu : ((1u << D) - 1u);
    uint32_t cur_p = 0xffffffffu;
    for (;;) {
        if (threadIdx.x == 0) {
            s_unit = atomicAdd(counter, 1u);
            s_nlong = 0;
            s_overflow = 0;
        }
        __syncthreads();
        uint32_t unit = s_unit;
        __syncthreads();
        if (unit >= nunits) break;
        uint32_t p = unit / nB, B = unit % nB;
        if (p != cur_p) {  // stage x words of tile columns [p*sc, p*sc+sc) as packed bits
            uint32_t c0 = p * sc, c1 = min(ncols, c0 + sc);
            uint32_t nwords = ((c1 - c0) * D + 31) / 32;
            for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) {
                uint32_t v = 0;
                if constexpr (D == 4) {  // 8 nibble words -> one u32
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        uint32_t c = c0 + i * 8 + j;
                        if (c < c1) v |= (load_word<4>(x, c) & 0xFu) << (4 * j);
                    }
                } else {
                    constexpr int PER = 32 / D;
#pragma unroll
                    for (int j = 0; j < PER; j++) {
                        uint32_t c = c0 + i * PER + j;
                        if (c < c1) v |= load_word<D>(x, c) << (D * j);
                    }
                }
                xs[i] = v;
            }
            cur_p = p;
            __syncthreads();
        }
        const uint32_t c0 = p * sc;
        const uint32_t *sg = seg + (size_t)p * (ntr + 1);
        const uint32_t r_end = min(ntr, (B + 1) * R);
        // a row longer than one group's fair share of the unit goes to pass 2
        const uint32_t LONG = max(MIN_LONG, (sg[r_end] - sg[B * R]) / ngroups);
        // pass 1: a group per row segment; segments longer than LONG tiles are
        // deferred to pass 2 so a hub row never serialises the CTA
        for (uint32_t I = B * R + group; I < r_end; I += ngroups) {
            uint32_t s0 = sg[I], s1 = sg[I + 1];
            if (s0 == s1) continue;
            if (s1 - s0 > LONG) {
                if (gl == 0) {
                    uint32_t k = atomicAdd(&s_nlong, 1u);
                    if (k < MAX_LONG) s_long[k] = I;
                    else s_overflow = 1;  // processed below by a slow path
                }
                continue;
            }
            uint32_t keepw;
            if (!row_keep<D, MODE>(keep, live, row0 + I, I, keepw)) continue;
            uint32_t acc = 0;
            uint32_t base = G::TPL > 1 ? (s0 & ~(uint32_t)(G::TPL - 1)) : s0;
            for (; base < s1; base += TILES_STEP) {
                acc |= seg_step<D, MODE>(tci, tiles, xs, c0, base, s0, s1, gl, lane, xmask);
                if constexpr (MODE == 1) {
                    uint32_t all = acc;
#pragma unroll
                    for (int o = GS / 2; o; o >>= 1) all |= __shfl_xor_sync(gmask, all, o);
                    if ((all & keepw) == keepw) { acc = all; break; }
                }
            }
#pragma unroll
            for (int o = GS / 2; o; o >>= 1) acc |= __shfl_xor_sync(gmask, acc, o);
            acc &= keepw;
            if (gl == 0 && acc) atomic_or_word<D>(y, I, acc);
        }
        __syncthreads();
        // pass 2: every group of the CTA takes interleaved steps of each long segment
        uint32_t nlong = min(s_nlong, MAX_LONG);
        bool overflow = s_overflow != 0;
        for (uint32_t k = 0; k < nlong + (overflow ? r_end - B * R : 0); k++) {
            uint32_t I;
            if (k < nlong) {
                I = s_long[k];
            } else {  // overflow slow path: rescan the unit for long rows not in the list
                I = B * R + (k - nlong);
                uint32_t a0 = sg[I], a1 = sg[I + 1];
                bool listed = false;
                for (uint32_t q = 0; q < nlong; q++) listed |= s_long[q] == I;
                if (a1 - a0 <= LONG || listed) continue;
            }
            uint32_t s0 = sg[I], s1 = sg[I + 1];
            uint32_t keepw;
            if (!row_keep<D, MODE>(keep, live, row0 + I, I, keepw)) continue;
            uint32_t acc = 0;
            uint32_t start = G::TPL > 1 ? (s0 & ~(uint32_t)(G::TPL - 1)) : s0;
            for (uint32_t base = start + group * TILES_STEP; base < s1; base += ngroups * TILES_STEP)
                acc |= seg_step<D, MODE>(tci, tiles, xs, c0, base, s0, s1, gl, lane, xmask);
#pragma unroll
            for (int o = GS / 2; o; o >>= 1) acc |= __shfl_xor_sync(gmask, acc, o);
            acc &= keepw;
            if (gl == 0 && acc) atomic_or_word<D>(y, I, acc);
        }
    }
}

bool blocked_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("B2SR_BLOCKED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// Returns false when the matrix has too many strips for the blocked path.
bool launch_blocked(b2sr_matrix *m, int mode, const void *x, const void *keep, void *y, cudaStream_t s) {
    BlockedPlan *bp = ensure_plan(m, s);
    if (!bp) return false;
    CK(cudaMemsetAsync(y, 0, padded_vec_bytes(m->ntr, m->dim), s));
    Buf<uint32_t> counter(1, s);
    CK(cudaMemsetAsync(counter.p, 0, 4, s));
    uint32_t ncols = tile_rows(m->n, m->dim);
    size_t smem = STRIP_SMEM;
    unsigned g = (unsigned)num_sms();
    const uint8_t *tl = (const uint8_t *)bp->tiles;
#define BLK_CASE(DD)                                                                                               \
    case DD:                                                                                                       \
        if (mode == 0) {                                                                                           \
            CK(cudaFuncSetAttribute(k_blocked<DD, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   \
            LAUNCH((k_blocked<DD, 0>), g, BLK_THREADS, smem, s, bp->P, bp->R, bp->nB, bp->strip_cols, m->ntr,      \
                   ncols, m->row0, bp->seg, bp->tci, tl, x, keep, (const void *)nullptr, y, counter.p);            \
        } else {                                                                                                   \
            CK(cudaFuncSetAttribute(k_blocked<DD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   \
            LAUNCH((k_blocked<DD, 1>), g, BLK_THREADS, smem, s, bp->P, bp->R, bp->nB, bp->strip_cols, m->ntr,      \
                   ncols, m->row0, bp->seg, bp->tci, tl, x, keep, (const void *)m->live, y, counter.p);            \
        }                                                                                                          \
        break;
    switch (m->dim) {
        BLK_CASE(4)
        BLK_CASE(8)
        BLK_CASE(16)
        BLK_CASE(32)
    }
#undef BLK_CASE
    return true;
}

}  // namespace b2sr
