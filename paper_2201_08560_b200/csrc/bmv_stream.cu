// K4 bbb as a flat tile stream (d = 4, 8) -- replaces kernels.py:97-115, 219-225.
//
// The work-item kernel (bmv.cu) gives every warp one tile row at a time, so a
// warp has a single row's loads in flight and the chain item -> tiles/tci ->
// x gather -> store is paid once per row; with ~120 tiles per tile row at R-MAT
// s22 d=4 that is one 128-bit warp load per chain.  Here the tile array is cut
// into warp loads of TPW tiles (128 at d=4, 64 at d=8) and each warp streams a
// contiguous range of them with the next loads already in flight, independent
// of row boundaries:
//   * the row of every tile is recovered from a per-load row hint (lrow[k] =
//     tile row holding tile k*TPW, built once per matrix) plus a short search
//     in tile_row_ptr (only when the load crosses a row boundary);
//   * per-tile hit words are OR-combined per row with a segmented warp scan
//     (rows are non-decreasing along the lanes) and stored with one atomicOr
//     per (row, load) -- OR is order-independent, so the bits are exactly the
//     reference's;
//   * x words come from the hot-column cache in shared memory (hot.cu) or, for
//     cold columns, from L1/L2.
#include "bfs_ctl.cuh"
#include "bmv_common.cuh"

namespace b2sr {

constexpr uint32_t SPAN = 7;  // row boundaries a load descriptor carries (more: searched)

// One descriptor per warp load k (tiles [k*TPW, (k+1)*TPW)):
//   x = ra, the tile row holding tile k*TPW;
//   y, z = byte i: offset inside the load where row ra+1+i starts (i < span),
//          0xFF when unused; the row of the tile at offset p is
//          ra + #{i : off[i] <= p} (empty rows are counted, so rows line up);
//   w = span (number of boundaries, 0 = the load lies in one row); span > SPAN
//       loads search tile_row_ptr instead (x of descriptor k+1 bounds them).
struct StreamPlan {
    uint32_t n_loads = 0;
    uint4 *desc = nullptr;  // n_loads + 1 (the last only carries the row of tile T-1)
};

void free_stream(void *p) {
    StreamPlan *sp = static_cast<StreamPlan *>(p);
    if (!sp) return;
    dfree(sp->desc, nullptr);
    delete sp;
}

__device__ __forceinline__ uint32_t row_of(const uint32_t *__restrict__ trp, uint32_t lo, uint32_t hi, uint64_t t) {
    while (lo < hi) {  // largest r in [lo, hi] with trp[r] <= t
        uint32_t mid = lo + (hi - lo + 1) / 2;
        if (trp[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void k_stream_desc(uint32_t n_loads, uint32_t tpw, uint64_t T, uint32_t ntr, const uint32_t *__restrict__ trp,
                              uint4 *__restrict__ desc) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= n_loads; k += gridDim.x * blockDim.x) {
        uint64_t t = std::min<uint64_t>((uint64_t)k * tpw, T - 1);
        uint32_t ra = row_of(trp, 0, ntr - 1, t);
        uint4 o = make_uint4(ra, 0x80808080u, 0x80808080u, 0);  // unused offset bytes: 128 (never <= p)
        if (k < n_loads) {
            uint64_t tn = std::min<uint64_t>((uint64_t)(k + 1) * tpw, T - 1);
            uint32_t rb = row_of(trp, ra, ntr - 1, tn), span = rb - ra;
            o.w = span;
            if (span <= SPAN) {
                for (uint32_t i = 0; i < span; i++) {
                    uint32_t off = (uint32_t)(trp[ra + 1 + i] - (uint64_t)k * tpw);  // 1..tpw
                    if (i < 4) o.y = (o.y & ~(0xFFu << (8 * i))) | (off << (8 * i));
                    else o.z = (o.z & ~(0xFFu << (8 * (i - 4)))) | (off << (8 * (i - 4)));
                }
            }
        }
        desc[k] = o;
    }
}

static StreamPlan *stream_plan(b2sr_matrix *m, uint32_t tpw, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (!m->stream) {
        StreamPlan *sp = new StreamPlan();
        sp->n_loads = (uint32_t)((m->num_tiles + tpw - 1) / tpw);
        try {
            Buf<uint4> desc((size_t)sp->n_loads + 65, s);  // + 64: the warps read descriptors 64 ahead
            CK(cudaMemsetAsync(desc.p, 0, ((size_t)sp->n_loads + 65) * 16, s));
            unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((sp->n_loads + 256) / 256, (uint64_t)num_sms() * 16));
            LAUNCH(k_stream_desc, g, 256, 0, s, sp->n_loads, tpw, m->num_tiles, m->ntr, m->trp, desc.p);
            sp->desc = desc.release();
        } catch (...) {
            free_stream(sp);
            throw;
        }
        m->stream = sp;
    }
    return static_cast<StreamPlan *>(m->stream);
}

// Lane geometry of one warp load of LT = 128 tiles.  A lane holds NG groups of
// GT consecutive tiles: d=4: one 16-byte group of 4 tiles at 4*lane; d=8: two
// 16-byte groups of 2 tiles, at 2*lane and 64 + 2*lane (each load instruction
// stays fully coalesced).
template <int D> struct SGeo;
template <> struct SGeo<4> {
    static constexpr int NG = 1, GT = 4;
    __device__ static uint32_t pos(uint32_t lane, int g) { return 4 * lane; }
};
template <> struct SGeo<8> {
    static constexpr int NG = 2, GT = 2;
    __device__ static uint32_t pos(uint32_t lane, int g) { return 64 * g + 2 * lane; }
};
constexpr uint32_t LT = 128;  // tiles per warp load

// masked tile words of one group: byte r (row r) non-zero iff the row hits
template <int D>
__device__ __forceinline__ void mask_group(const uint4 &v, const uint32_t *xw, uint32_t (&m)[4]) {
    if constexpr (D == 4) {
        m[0] = v.x & (xw[0] * 0x01010101u);
        m[1] = v.y & (xw[1] * 0x01010101u);
        m[2] = v.z & (xw[2] * 0x01010101u);
        m[3] = v.w & (xw[3] * 0x01010101u);
    } else {
        uint32_t a = xw[0] * 0x01010101u, b = xw[1] * 0x01010101u;
        m[0] = v.x & a; m[1] = v.y & a;  // tile 0: rows 0-3, rows 4-7
        m[2] = v.z & b; m[3] = v.w & b;  // tile 1
    }
}
// hit word of tile j of a group / of all tiles of a group
template <int D>
__device__ __forceinline__ uint32_t tile_hits(const uint32_t (&m)[4], int j) {
    if constexpr (D == 4) return nz_nibble_bytes(m[j]);
    else return nz_bytes(m[2 * j]) | (nz_bytes(m[2 * j + 1]) << 4);
}
template <int D>
__device__ __forceinline__ uint32_t group_hits(const uint32_t (&m)[4]) {
    if constexpr (D == 4) return nz_nibble_bytes(m[0] | m[1] | m[2] | m[3]);
    else return nz_bytes(m[0] | m[2]) | (nz_bytes(m[1] | m[3]) << 4);
}

template <int D>
__device__ __forceinline__ void or_row(void *__restrict__ y, uint32_t row, uint32_t acc) {
    if (acc) atomic_or_word<D>(y, row, acc);
}

// row of offset p (0..LT-1) relative to ra: #{i : off[i] <= p}.  Offsets are
// bytes in 1..128, so per byte (p + 128) - off lies in 0..254: the subtraction
// never borrows across bytes and bit 7 of a byte is set iff p >= off (three
// integer ops per word instead of the emulated __vcmpgeu4).  pp = p * 0x01010101
// + 0x80808080 is lane-constant at the call sites.
__device__ __forceinline__ uint32_t rel_row_pp(uint32_t pp, uint32_t oa, uint32_t ob) {
    return __popc((pp - oa) & 0x80808080u) + __popc((pp - ob) & 0x80808080u);
}
__device__ __forceinline__ uint32_t row_pp(uint32_t p) { return p * 0x01010101u + 0x80808080u; }

// Streams the loads at positions [p0, p1): load k = list[p] with a list (BFS
// pull over the loads that still hold an unvisited vertex), else k = p.
template <int D, bool LIST, class GX, bool LAZY = false>
__device__ __forceinline__ void bbb_stream(uint32_t p0, uint32_t p1, uint32_t n_loads, uint64_t T,
                                           const uint32_t *__restrict__ list, const uint4 *__restrict__ desc,
                                           const uint32_t *__restrict__ trp, const uint8_t *__restrict__ tiles,
                                           const uint32_t *__restrict__ tci, const GX &gx, void *__restrict__ y) {
    using SG = SGeo<D>;
    constexpr int NG = SG::NG, GT = SG::GT, TB = Geo<D>::TB;
    constexpr int SPW = 32 / D;                     // packed D-bit row slots per u32: 8 / 4
    constexpr int NW = (SPAN + 1 + SPW - 1) / SPW;  // accumulator words: 1 / 2
    const uint32_t lane = lane_id();
    struct Stage {
        uint4 v[NG];
        uint32_t cx[NG * GT];  // tile columns after issue(), x words after gather()
    };
    // per 32 positions: load index (list mode) and descriptor, one block ahead
    uint32_t bb = p0;  // first position of the current block
    uint32_t kc = 0, kn = 0;
    if constexpr (LIST) {
        kc = p0 + lane < p1 ? __ldg(list + p0 + lane) : 0u;
        kn = p0 + 32 + lane < p1 ? __ldg(list + p0 + 32 + lane) : 0u;
    } else {
        kc = p0 + lane;
        kn = p0 + 32 + lane;
    }
    uint4 dcur = __ldg(desc + std::min(kc, n_loads)), dnxt = __ldg(desc + std::min(kn, n_loads));
    auto kat = [&](uint32_t p) -> uint32_t {  // load index of position p (p - bb < 64)
        if constexpr (LIST) {
            uint32_t o = p - bb;
            uint32_t a = __shfl_sync(0xffffffffu, kc, o & 31), b = __shfl_sync(0xffffffffu, kn, o & 31);
            return o < 32 ? a : b;
        } else {
            return p;
        }
    };
    auto issue = [&](uint32_t p, Stage &st) {
        const bool live = p < p1;
        const uint32_t k = kat(p);
#pragma unroll
        for (int g = 0; g < NG; g++) {
            uint64_t t = (uint64_t)k * LT + SG::pos(lane, g);
            bool ok = live && t < T;
            // LAZY (sparse BFS frontiers): the tile bytes are fetched after the
            // x words, only by lanes whose x words are not all zero
            if constexpr (!LAZY) st.v[g] = ok ? ld_stream128(tiles + t * TB) : make_uint4(0, 0, 0, 0);
            if constexpr (GT == 4) {
                uint4 q = ok ? ld_stream128(tci + t) : make_uint4(0, 0, 0, 0);
                st.cx[0] = q.x; st.cx[1] = q.y; st.cx[2] = q.z; st.cx[3] = q.w;
            } else {
                uint2 q = ok ? *reinterpret_cast<const uint2 *>(tci + t) : make_uint2(0, 0);
                st.cx[2 * g] = q.x; st.cx[2 * g + 1] = q.y;
            }
        }
    };
    auto gather = [&](uint32_t p, Stage &st) {
        const uint32_t k = kat(p);
        const bool full = p < p1 && (k + 1 < n_loads || (uint64_t)(k + 1) * LT <= T);  // every tile of load k exists
        if (full) {
#pragma unroll
            for (int j = 0; j < NG * GT; j++) st.cx[j] = gx(st.cx[j]);
        } else {
#pragma unroll
            for (int g = 0; g < NG; g++)
#pragma unroll
                for (int j = 0; j < GT; j++) {
                    uint64_t t = (uint64_t)k * LT + SG::pos(lane, g) + j;
                    st.cx[g * GT + j] = (p < p1 && t < T) ? gx(st.cx[g * GT + j]) : 0u;
                }
        }
        if constexpr (LAZY) {
#pragma unroll
            for (int g = 0; g < NG; g++) {
                uint32_t any = 0;
#pragma unroll
                for (int j = 0; j < GT; j++) any |= st.cx[g * GT + j];
                const uint64_t t = (uint64_t)k * LT + SG::pos(lane, g);
                st.v[g] = any ? ld_stream128(tiles + t * TB) : make_uint4(0, 0, 0, 0);
            }
        }
    };
    auto compute = [&](uint32_t p, const Stage &st) {
        if (p - bb == 32) {  // next block of 32 positions
            bb = p;
            kc = kn;
            dcur = dnxt;
            uint32_t q = p + 32 + lane;
            if constexpr (LIST) kn = q < p1 ? __ldg(list + q) : 0u;
            else kn = q;
            dnxt = __ldg(desc + std::min(kn, n_loads));
        }
        const uint32_t i = p - bb;
        const uint32_t k = LIST ? __shfl_sync(0xffffffffu, kc, i) : p;
        const uint32_t ra = __shfl_sync(0xffffffffu, dcur.x, i);
        const uint32_t span = __shfl_sync(0xffffffffu, dcur.w, i);
        uint32_t m[NG][4];
#pragma unroll
        for (int g = 0; g < NG; g++) mask_group<D>(st.v[g], st.cx + g * GT, m[g]);
        if (span == 0) {  // the whole load lies in one row
            if constexpr (D == 4) {
                uint32_t raw = m[0][0] | m[0][1] | m[0][2] | m[0][3];  // OR raw words, test once
                raw = __reduce_or_sync(0xffffffffu, raw);
                if (lane == 0) or_row<D>(y, ra, nz_nibble_bytes(raw));
            } else {
                uint32_t lo = m[0][0] | m[0][2] | m[1][0] | m[1][2], hi = m[0][1] | m[0][3] | m[1][1] | m[1][3];
                lo = __reduce_or_sync(0xffffffffu, lo);
                hi = __reduce_or_sync(0xffffffffu, hi);
                if (lane == 0) or_row<D>(y, ra, nz_bytes(lo) | (nz_bytes(hi) << 4));
            }
        } else if (span <= SPAN) {
            const uint32_t oa = __shfl_sync(0xffffffffu, dcur.y, i), ob = __shfl_sync(0xffffffffu, dcur.z, i);
            uint32_t acc[NW];
#pragma unroll
            for (int u = 0; u < NW; u++) acc[u] = 0;
#pragma unroll
            for (int g = 0; g < NG; g++) {
                const uint32_t q0 = SG::pos(lane, g);
                const uint32_t qa = rel_row_pp(row_pp(q0), oa, ob), qb = rel_row_pp(row_pp(q0 + GT - 1), oa, ob);
                if (qa == qb) {  // the group's tiles share one row
                    uint32_t h = group_hits<D>(m[g]);
#pragma unroll
                    for (int u = 0; u < NW; u++) acc[u] |= (qa / SPW == (uint32_t)u) ? h << (D * (qa % SPW)) : 0u;
                } else {
#pragma unroll
                    for (int j = 0; j < GT; j++) {
                        uint32_t q = rel_row_pp(row_pp(q0 + j), oa, ob), h = tile_hits<D>(m[g], j);
#pragma unroll
                        for (int u = 0; u < NW; u++) acc[u] |= (q / SPW == (uint32_t)u) ? h << (D * (q % SPW)) : 0u;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < NW; u++) acc[u] = __reduce_or_sync(0xffffffffu, acc[u]);
            if (lane <= span) {
                uint32_t a = 0;
#pragma unroll
                for (int u = 0; u < NW; u++) a |= (lane / SPW == (uint32_t)u) ? acc[u] : 0u;
                or_row<D>(y, ra + lane, (a >> (D * (lane % SPW))) & ((1u << D) - 1u));
            }
        } else {
            // many short rows: search trp[ra..rb] per tile and write per tile
            const uint32_t rb = __ldg(&desc[k + 1].x);
#pragma unroll
            for (int g = 0; g < NG; g++)
#pragma unroll
                for (int j = 0; j < GT; j++) {
                    uint32_t h = tile_hits<D>(m[g], j);
                    if (h) or_row<D>(y, row_of(trp, ra, rb, (uint64_t)k * LT + SG::pos(lane, g) + j), h);
                }
        }
    };
    if (p0 >= p1) return;
    // three-stage pipeline, unrolled so the stages never move: while load p is
    // reduced, the x gathers of p+1 and the tile/column loads of p+2 are in flight
    Stage A, B, C;
    issue(p0, A);
    issue(p0 + 1, B);
    gather(p0, A);
    for (uint32_t p = p0; p < p1; p += 3) {
        issue(p + 2, C);
        gather(p + 1, B);
        compute(p, A);
        if (p + 1 >= p1) break;
        issue(p + 3, A);
        gather(p + 2, C);
        compute(p + 1, B);
        if (p + 2 >= p1) break;
        issue(p + 4, B);
        gather(p + 3, A);
        compute(p + 2, C);
    }
}

template <int D, int NT, bool LIST, bool LAZY = false>
__global__ void __launch_bounds__(NT, 1)
    k_bmv_bbb_stream(uint32_t n_loads, const uint32_t *__restrict__ list, const uint32_t *__restrict__ list_n,
                     uint64_t T, const uint4 *__restrict__ desc, const uint32_t *__restrict__ trp,
                     const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci2, const void *__restrict__ hx,
                     uint32_t hx_bytes16, uint32_t S, const void *__restrict__ x, void *__restrict__ y,
                     const int *__restrict__ gate, int want) {
    if (gate && *gate != want) return;  // device-side BFS direction choice (drivers.cu)
    const uint32_t n_pos = LIST ? *list_n : n_loads;
    if (n_pos == 0) return;
    stage_hot(const_cast<uint8_t *>(hot_bytes()), hx, hx_bytes16);
    __syncthreads();
    XHot<D> gx(x, S);
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t per = (n_pos + warps - 1) / warps;
    const uint32_t p0 = std::min(n_pos, w * per), p1 = std::min(n_pos, p0 + per);
    bbb_stream<D, LIST, XHot<D>, LAZY>(p0, p1, n_loads, T, list, desc, trp, tiles, tci2, gx, y);
}

// ------------------------------------------------------------ fused BFS level
// Push body: warp per (frontier tile row, 1024-tile chunk) entry of a; each
// lane holds TPL consecutive tiles of one 128-bit load; the bit-rows of the
// frontier word select the tile bytes, folded to the column word and OR'd into
// next[col] (fire-and-forget RED; visited vertices are masked by the update).
// With `visited`, bits of already visited vertices are dropped before the RED:
// on dense levels that skips most atomics, hub columns (reached early) included.
template <int D>
__device__ __forceinline__ void push_entries(uint32_t n_entries, const uint2 *__restrict__ plist,
                                             const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                                             const uint8_t *__restrict__ tiles, const void *__restrict__ frontier,
                                             void *__restrict__ next, const void *__restrict__ visited = nullptr) {
    using G = Geo<D>;
    constexpr int TPL = G::TPL;
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_entries; e += warps) {
        const uint2 ent = plist[e];
        const uint32_t I = ent.x;
        const uint32_t t0 = __ldg(trp + I) + ent.y * PUSH_CH;
        const uint32_t t1 = min(__ldg(trp + I + 1), t0 + PUSH_CH);
        const uint32_t fw = load_word<D>(frontier, I);
        // 0xFF in the bytes of the frontier bit-rows
        const uint32_t sl = ((fw & 0xFu) * 0x00204081u & 0x01010101u) * 0xFFu;
        const uint32_t sh = (((fw >> 4) & 0xFu) * 0x00204081u & 0x01010101u) * 0xFFu;
        for (uint32_t base = t0 & ~(uint32_t)(TPL - 1); base < t1; base += 2 * G::TPW) {
            uint4 v[2];
            uint32_t c[2][TPL];
#pragma unroll
            for (int u = 0; u < 2; u++) {
                uint32_t tl = base + u * G::TPW + lane * TPL;
                bool any = tl < t1 && tl + TPL > t0;
                v[u] = any ? ld_stream128(tiles + (size_t)tl * G::TB) : make_uint4(0, 0, 0, 0);
                if constexpr (TPL == 4) {
                    uint4 q = any ? ld_stream128(tci + tl) : make_uint4(0, 0, 0, 0);
                    c[u][0] = q.x; c[u][1] = q.y; c[u][2] = q.z; c[u][3] = q.w;
                } else {
                    uint2 q = any ? *reinterpret_cast<const uint2 *>(tci + tl) : make_uint2(0, 0);
                    c[u][0] = q.x; c[u][1] = q.y;
                }
            }
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const uint32_t tl = base + u * G::TPW + lane * TPL;
#pragma unroll
                for (int j = 0; j < TPL; j++) {
                    uint32_t m;
                    if constexpr (D == 4) {
                        uint32_t w = (j == 0 ? v[u].x : j == 1 ? v[u].y : j == 2 ? v[u].z : v[u].w) & sl;
                        w |= w >> 16;
                        m = (w | (w >> 8)) & 0xFFu;
                    } else {
                        uint32_t w = ((j == 0 ? v[u].x : v[u].z) & sl) | ((j == 0 ? v[u].y : v[u].w) & sh);
                        w |= w >> 16;
                        m = (w | (w >> 8)) & 0xFFu;
                    }
                    if (!(tl + j >= t0 && tl + j < t1)) m = 0;  // neighbours' / padding tiles of the load
                    if (m && visited) m &= ~load_word<D>(visited, c[u][j]);
                    if (m) atomic_or_word<D>(next, c[u][j], m);
                }
            }
        }
    }
}

// The three pull variants of the fused level kernel, each compiled out of line:
// inlined into one kernel body under the 64-register cap of a 1024-thread CTA
// they spilled (20 B per thread); as separate callees each gets the whole
// register budget.
template <int D, bool LIST, bool LAZY>
__device__ __noinline__ void bfs_pull(uint32_t p0, uint32_t p1, uint32_t n_loads, uint64_t T,
                                      const uint32_t *__restrict__ list, const uint4 *__restrict__ desc,
                                      const uint32_t *__restrict__ trp, const uint8_t *__restrict__ tiles,
                                      const uint32_t *__restrict__ tci2, const void *__restrict__ x, uint32_t S,
                                      void *__restrict__ y) {
    XHot<D> gx(x, S);
    bbb_stream<D, LIST, XHot<D>, LAZY>(p0, p1, n_loads, T, list, desc, trp, tiles, tci2, gx, y);
}

// One BFS level in one launch: the direction chosen by the device-side plan
// (BfsCtl::mode) selects the push body, the full flat-stream pull, or the
// stream over the listed active loads.
template <int D, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_bfs_level(const BfsCtl *__restrict__ ctl, const uint2 *__restrict__ plist, const uint32_t *__restrict__ a_trp,
                const uint32_t *__restrict__ a_tci, const uint8_t *__restrict__ a_tiles, uint32_t n_loads,
                const uint32_t *__restrict__ alist, uint64_t T, const uint4 *__restrict__ desc,
                const uint32_t *__restrict__ trp, const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci2,
                const void *__restrict__ hx, uint32_t hx_bytes16, uint32_t S, const void *__restrict__ frontier,
                void *__restrict__ next, const void *__restrict__ visited, const void *__restrict__ pfrontier,
                void *__restrict__ pnext) {
    pdl_prologue();
    const int mode = ctl->mode;
    if (mode == BFS_NONE) return;
    if (mode == BFS_PUSH) {
        push_entries<D>(ctl->list_n, plist, a_trp, a_tci, a_tiles, pfrontier, pnext, visited);
        return;
    }
    const bool listed = mode == BFS_PULL_ACTIVE;
    const uint32_t n_pos = listed ? ctl->active_n : n_loads;
    if (n_pos == 0) return;
    stage_hot(const_cast<uint8_t *>(hot_bytes()), hx, hx_bytes16);
    __syncthreads();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t per = (n_pos + warps - 1) / warps;
    const uint32_t p0 = std::min(n_pos, w * per), p1 = std::min(n_pos, p0 + per);
    if (listed) bfs_pull<D, true, false>(p0, p1, n_loads, T, alist, desc, trp, tiles, tci2, frontier, S, next);
    else if (ctl->sparse) bfs_pull<D, false, true>(p0, p1, n_loads, T, nullptr, desc, trp, tiles, tci2, frontier, S, next);
    else bfs_pull<D, false, false>(p0, p1, n_loads, T, nullptr, desc, trp, tiles, tci2, frontier, S, next);
}

// Push-only level (BFS without a transpose): every level top-down over a.
template <int D>
__global__ void __launch_bounds__(256) k_bfs_push_level(const BfsCtl *__restrict__ ctl, const uint2 *__restrict__ plist,
                                                        const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                                                        const uint8_t *__restrict__ tiles, const void *__restrict__ frontier,
                                                        const void *__restrict__ visited, void *__restrict__ next) {
    pdl_prologue();
    if (ctl->mode != BFS_PUSH) return;
    push_entries<D>(ctl->list_n, plist, trp, tci, tiles, frontier, next, visited);
}

void launch_bfs_push_level(const b2sr_matrix *a, const BfsCtl *ctl, const uint2 *push_list, const void *frontier,
                           const void *visited, void *next, cudaStream_t s, bool pdl) {
    const unsigned g = (unsigned)num_sms() * 8;
    if (a->dim == 4)
        LAUNCH_PDL(pdl, k_bfs_push_level<4>, g, 256, 0, s, ctl, push_list, a->trp, a->tci, (const uint8_t *)a->tiles,
                   frontier, visited, next);
    else
        LAUNCH_PDL(pdl, k_bfs_push_level<8>, g, 256, 0, s, ctl, push_list, a->trp, a->tci, (const uint8_t *)a->tiles,
                   frontier, visited, next);
}

void launch_bfs_level(b2sr_matrix *at, const b2sr_matrix *a, BfsCtl *ctl, const uint2 *push_list,
                      const uint32_t *active_list, const void *hx, size_t hb, const void *frontier, void *next,
                      const void *visited, cudaStream_t s, const void *pfrontier, void *pnext, bool pdl) {
    if (!pfrontier) pfrontier = frontier;
    if (!pnext) pnext = next;
    StreamPlan *sp = stream_plan(at, LT, s);
    HotView hv = hot_view(at, s);
    const unsigned g = (unsigned)num_sms();
    const uint32_t *atrp = a ? a->trp : nullptr, *atci = a ? a->tci : nullptr;
    const uint8_t *atl = a ? (const uint8_t *)a->tiles : nullptr;
    if (at->dim == 4) {
        hot_smem_attr(k_bfs_level<4, 1024>, hb);
        LAUNCH_PDL(pdl, (k_bfs_level<4, 1024>), g, 1024, hb, s, ctl, push_list, atrp, atci, atl, sp->n_loads, active_list,
               at->num_tiles, sp->desc, at->trp, (const uint8_t *)at->tiles, hv.tci2, hx, (uint32_t)hb, hv.S,
               frontier, next, visited, pfrontier, pnext);
    } else {
        hot_smem_attr(k_bfs_level<8, 768>, hb);
        LAUNCH_PDL(pdl, (k_bfs_level<8, 768>), g, 768, hb, s, ctl, push_list, atrp, atci, atl, sp->n_loads, active_list,
               at->num_tiles, sp->desc, at->trp, (const uint8_t *)at->tiles, hv.tci2, hx, (uint32_t)hb, hv.S,
               frontier, next, visited, pfrontier, pnext);
    }
}

// BFS pull over part of the matrix: the loads holding a tile of a row with an
// unvisited live vertex (rows [ra, next ra] of every load are checked).
template <int D>
__global__ void k_active_loads(uint32_t n_loads, const uint4 *__restrict__ desc, const void *__restrict__ visited,
                               const void *__restrict__ live, uint32_t row0, uint32_t *__restrict__ list,
                               uint32_t *__restrict__ count) {
    const uint32_t lane = lane_id();
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t iters = (n_loads + stride - 1) / stride;
    for (uint32_t it = 0; it < iters; it++) {
        uint32_t k = blockIdx.x * blockDim.x + threadIdx.x + it * stride;
        bool act = false;
        if (k < n_loads) {
            uint32_t ra = desc[k].x, rb = desc[k + 1].x;
            for (uint32_t r = ra; r <= rb && !act; r++)
                act = (~load_word<D>(visited, row0 + r) & load_word<D>(live, r)) != 0;
        }
        uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (!bal) continue;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(count, (uint32_t)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (act) list[base + __popc(bal & ((1u << lane) - 1u))] = k;
    }
}

// y &= keep (keep is indexed by global tile row: row0 offsets it for row blocks)
__global__ void k_and_words(uint32_t nw, uint32_t *__restrict__ y, const uint32_t *__restrict__ keep) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x) y[i] &= keep[i];
}
__global__ void k_and_bytes(uint32_t nb, uint8_t *__restrict__ y, const uint8_t *__restrict__ keep) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) y[i] &= keep[i];
}

bool stream_enabled(int dim) {
    const char *e = getenv("B2SR_STREAM");  // B2SR_STREAM=0: work-item kernel (A/B)
    if (e && e[0] == '0') return false;
    return (dim == 4 || dim == 8) && hot_enabled(dim);
}

// y &= ~visited & live (BFS pull: only unvisited vertices with in-edges take a level)
__global__ void k_pull_mask(uint32_t nb, uint8_t *__restrict__ y, const uint8_t *__restrict__ visited,
                            const uint8_t *__restrict__ live, bool aligned) {
    if (aligned) {
        uint32_t nw = nb / 4;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x)
            reinterpret_cast<uint32_t *>(y)[i] &= ~reinterpret_cast<const uint32_t *>(visited)[i] &
                                                  reinterpret_cast<const uint32_t *>(live)[i];
    } else {
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x)
            y[i] &= (uint8_t)(~visited[i] & live[i]);
    }
}

const uint4 *stream_desc(b2sr_matrix *m, cudaStream_t s, uint32_t *n_loads) {
    StreamPlan *sp = stream_plan(m, LT, s);
    *n_loads = sp->n_loads;
    return sp->desc;
}

// The stream kernel alone: y must be zeroed and hx filled (hot_fill) by the caller.
void launch_stream_sweep(b2sr_matrix *m, const uint32_t *list, const uint32_t *list_n, const void *hx, size_t hb,
                         const void *x, void *y, const int *gate, int want, cudaStream_t s, bool lazy) {
    if (!m->num_tiles) return;
    StreamPlan *sp = stream_plan(m, LT, s);
    HotView hv = hot_view(m, s);
    unsigned g = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)num_sms(), ((uint64_t)sp->n_loads + 31) / 32));
    const uint8_t *tl = (const uint8_t *)m->tiles;
    const char *te = getenv("B2SR_STREAM_THREADS");  // A/B: 768 / 1024 threads per CTA
    int nt = te ? atoi(te) : (m->dim == 4 ? 1024 : 768);
#define STREAM_LAUNCH3(DD, NT, LI, LZ)                                                                               \
    do {                                                                                                             \
        hot_smem_attr(k_bmv_bbb_stream<DD, NT, LI, LZ>, hb);                                                         \
        LAUNCH((k_bmv_bbb_stream<DD, NT, LI, LZ>), g, NT, hb, s, sp->n_loads, LI ? list : nullptr,                   \
               LI ? list_n : nullptr, m->num_tiles, sp->desc, m->trp, tl, hv.tci2, hx, (uint32_t)hb, hv.S, x, y,    \
               gate, want);                                                                                          \
    } while (0)
#define STREAM_LAUNCH(DD, NT)                                                                                        \
    do {                                                                                                             \
        if (list) {                                                                                                  \
            if (lazy) STREAM_LAUNCH3(DD, NT, true, true);                                                            \
            else STREAM_LAUNCH3(DD, NT, true, false);                                                                \
        } else {                                                                                                     \
            if (lazy) STREAM_LAUNCH3(DD, NT, false, true);                                                           \
            else STREAM_LAUNCH3(DD, NT, false, false);                                                               \
        }                                                                                                            \
    } while (0)
    if (m->dim == 4) {
        if (nt == 768) STREAM_LAUNCH(4, 768);
        else STREAM_LAUNCH(4, 1024);
    } else {
        STREAM_LAUNCH(8, 768);
    }
#undef STREAM_LAUNCH
#undef STREAM_LAUNCH3
}

void launch_bbb_stream(b2sr_matrix *m, const void *x, const void *keep, void *y, cudaStream_t s,
                       const void *visited, bool active_only, bool lazy) {
    const size_t yb = padded_vec_bytes(m->ntr, m->dim);
    CK(cudaMemsetAsync(y, 0, yb, s));
    if (!m->num_tiles) return;
    StreamPlan *sp = stream_plan(m, LT, s);
    HotView hv = hot_view(m, s);
    size_t hb = hot_fill_bytes(hv, m->dim);
    Buf<uint8_t> hx(hb, s);
    Buf<uint32_t> list, list_n;
    if (active_only && visited) {  // compact the loads that still matter
        list = Buf<uint32_t>(sp->n_loads, s);
        list_n = Buf<uint32_t>(1, s);
        CK(cudaMemsetAsync(list_n.p, 0, 4, s));
        unsigned ga = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((sp->n_loads + 255) / 256, (uint64_t)num_sms() * 8));
        if (m->dim == 4)
            LAUNCH(k_active_loads<4>, ga, 256, 0, s, sp->n_loads, sp->desc, visited, m->live, m->row0, list.p, list_n.p);
        else
            LAUNCH(k_active_loads<8>, ga, 256, 0, s, sp->n_loads, sp->desc, visited, m->live, m->row0, list.p, list_n.p);
    }
    hot_fill(hv, m->dim, x, hx.p, s);
    kernel_timer().begin(s);
    launch_stream_sweep(m, list.p, list_n.p, hx.p, hb, x, y, nullptr, 0, s, lazy);
    kernel_timer().end(s);
    if (visited) {  // BFS pull: keep = ~visited & live, applied once at the end
        const uint8_t *vp = static_cast<const uint8_t *>(visited) + (size_t)m->row0 * word_bytes(m->dim);
        const uint32_t nb = (uint32_t)yb;
        bool aligned = ((uintptr_t)vp & 3) == 0;
        unsigned gk = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nb / (aligned ? 4 : 1) + 255) / 256,
                                                                         (uint64_t)num_sms() * 8));
        LAUNCH(k_pull_mask, gk, 256, 0, s, nb, (uint8_t *)y, vp, (const uint8_t *)m->live, aligned);
    } else if (keep) {  // masked variant: the keep words are applied once at the end (kernels.py:219-225)
        const uint8_t *kp = static_cast<const uint8_t *>(keep) + (size_t)m->row0 * word_bytes(m->dim);
        if (((uintptr_t)kp & 3) == 0) {
            const uint32_t kw = (uint32_t)(yb / 4);
            unsigned gk = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((kw + 255) / 256, (uint64_t)num_sms() * 8));
            LAUNCH(k_and_words, gk, 256, 0, s, kw, (uint32_t *)y, (const uint32_t *)kp);
        } else {
            const uint32_t nb = (uint32_t)((size_t)m->ntr * word_bytes(m->dim));
            unsigned gk = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nb + 255) / 256, (uint64_t)num_sms() * 8));
            LAUNCH(k_and_bytes, gk, 256, 0, s, nb, (uint8_t *)y, kp);
        }
    }
}

}  // namespace b2sr
