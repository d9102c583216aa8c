// K4/K5/K6: bin-SpMV over B2SR on sm_100a (replaces kernels.py:86-249).
//
// bbb / bbf (bit and popcount outputs) are HBM-streaming kernels:
//   * the matrix is cut into work items of at most CHUNK tiles of one tile
//     row (long rows split; built once per matrix and cached);
//   * one warp per item streams its tiles with 128-bit non-allocating loads:
//     d=4 -> 4 tiles per lane (128 tiles per warp load), d=8 -> 2 (64),
//     d=16 -> half a tile per lane (16), d=32 -> a quarter tile (4), all
//     fully coalesced, tile-column indices loaded alongside, x words
//     gathered through L1/L2;
//   * per-lane partial results are reduced with redux.sync / shfl and stored
//     once per item (atomics only for split rows -- OR and integer sums, so
//     results are deterministic).
// bff (float64 semiring gather) keeps the reference's reduction order: one
// group of d lanes per tile row, lane = bit-row, tiles in ascending column
// order, bits ascending inside a tile (kernels.py:195-207) -- the sum is
// bit-identical to the reference.
#include <cmath>

#include "bmv_common.cuh"

namespace b2sr {

// ------------------------------------------------------------ work items
__global__ void k_item_counts(uint32_t ntr, const uint32_t *trp, uint32_t chunk, uint32_t *cnt) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= ntr) return;
    uint32_t len = trp[I + 1] - trp[I];
    uint32_t p = (len + chunk - 1) / chunk;
    cnt[I] = p ? p : 1u;
}

__global__ void k_item_fill(uint32_t ntr, const uint32_t *trp, uint32_t chunk, const uint64_t *ofs, WorkItem *items,
                            int *any_split) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= ntr) return;
    uint32_t t0 = trp[I], t1 = trp[I + 1];
    uint64_t b = ofs[I];
    uint32_t P = (uint32_t)(ofs[I + 1] - b);
    if (P > 1) *any_split = 1;
    for (uint32_t j = 0; j < P; j++) {
        uint32_t a = t0 + j * chunk;
        uint32_t e = min(t1, a + chunk);
        items[b + j] = WorkItem{I, a, e, P > 1 ? 1u : 0u};
    }
}

__global__ void k_ofs_u32(uint32_t n, const uint64_t *in, uint32_t *out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)in[i];
}

void ensure_items(b2sr_matrix *m, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (m->items) return;
    uint32_t chunk = m->dim == 4 ? Geo<4>::CHUNK : m->dim == 8 ? Geo<8>::CHUNK
                   : m->dim == 16 ? Geo<16>::CHUNK : Geo<32>::CHUNK;
    Buf<uint32_t> cnt(m->ntr, s);
    Buf<uint64_t> ofs((size_t)m->ntr + 1, s);
    LAUNCH(k_item_counts, (m->ntr + 255) / 256, 256, 0, s, m->ntr, m->trp, chunk, cnt.p);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, m->ntr, s);
    uint64_t n_items = read_scalar(ofs.p + m->ntr, s);
    Buf<WorkItem> items(n_items, s);
    Buf<int> split(1, s);
    CK(cudaMemsetAsync(split.p, 0, sizeof(int), s));
    LAUNCH(k_item_fill, (m->ntr + 255) / 256, 256, 0, s, m->ntr, m->trp, chunk, ofs.p, items.p, split.p);
    m->any_split = read_scalar(split.p, s) != 0;
    Buf<uint32_t> item_ofs((size_t)m->ntr + 1, s);  // per-row first item (BFS active lists)
    LAUNCH(k_ofs_u32, (m->ntr + 256) / 256, 256, 0, s, m->ntr + 1, ofs.p, item_ofs.p);
    m->n_items = (uint32_t)n_items;
    m->items = items.release();
    m->item_ofs = item_ofs.release();
}

static unsigned item_grid(const b2sr_matrix *m) {
    uint64_t blocks = ((uint64_t)m->n_items + 7) / 8;  // 8 warps per 256-thread CTA
    uint64_t cap = (uint64_t)num_sms() * 16;
    return (unsigned)(blocks < cap ? blocks : cap);
}

// ------------------------------------------------------------ one warp load
// Loads the tiles covered by this lane for the warp load starting at `base`
// and returns them with their x words; tiles outside [t0, t1) read as zero.
template <int D>
struct LaneTiles {
    uint4 v;                  // raw 16 bytes
    uint32_t xw[Geo<D>::TPL]; // x word per tile (0 when invalid)
};

template <int D, class GX>
__device__ __forceinline__ void load_lane(const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                          const GX &gx, uint32_t base, uint32_t t0, uint32_t t1,
                                          uint32_t lane, LaneTiles<D> &lt) {
    using G = Geo<D>;
    if constexpr (G::TPL > 1) {
        uint32_t tl = base + lane * G::TPL;
        bool any = tl < t1 && tl + G::TPL > t0;
        lt.v = any ? ld_stream128(tiles + (size_t)tl * G::TB) : make_uint4(0, 0, 0, 0);
        uint32_t cols[G::TPL];
        if constexpr (G::TPL == 4) {
            uint4 c = any ? ld_stream128(tci + tl) : make_uint4(0, 0, 0, 0);
            cols[0] = c.x; cols[1] = c.y; cols[2] = c.z; cols[3] = c.w;
        } else {
            uint2 c = any ? *reinterpret_cast<const uint2 *>(tci + tl) : make_uint2(0, 0);
            cols[0] = c.x; cols[1] = c.y;
        }
#pragma unroll
        for (int j = 0; j < G::TPL; j++) {
            bool ok = tl + j >= t0 && tl + j < t1;
            lt.xw[j] = ok ? gx(cols[j]) : 0u;
        }
    } else {
        uint32_t t = base + lane / G::LPT;
        uint32_t q = lane % G::LPT;
        bool ok = t < t1;
        lt.v = ok ? ld_stream128(tiles + (size_t)t * G::TB + q * 16) : make_uint4(0, 0, 0, 0);
        lt.xw[0] = ok ? gx(__ldg(tci + t)) : 0u;
    }
}

// bbb: hit bits of the rows this lane covers (positions within the row word)
template <int D>
__device__ __forceinline__ uint32_t lane_hits(const LaneTiles<D> &lt, uint32_t lane) {
    return hits16<D>(lt.v, lt.xw, lane);
}

// ------------------------------------------------------------ K4 bbb
template <int D, class GX>
__device__ __forceinline__ void bbb_items(const WorkItem *__restrict__ items, uint32_t n_items,
                                          const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                          const GX &gx, const void *__restrict__ keep, void *__restrict__ y,
                                          uint32_t row0) {
    using G = Geo<D>;
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        WorkItem it = items[w];
        uint32_t acc = 0;
        uint32_t start = G::TPL > 1 ? (it.t0 & ~(uint32_t)(G::TPL - 1)) : it.t0;
        uint32_t base = start;
        // two warp loads in flight per iteration
        for (; base + G::TPW < it.t1; base += 2 * G::TPW) {
            LaneTiles<D> a, b;
            load_lane<D>(tiles, tci, gx, base, it.t0, it.t1, lane, a);
            load_lane<D>(tiles, tci, gx, base + G::TPW, it.t0, it.t1, lane, b);
            acc |= lane_hits<D>(a, lane) | lane_hits<D>(b, lane);
        }
        if (base < it.t1) {
            LaneTiles<D> a;
            load_lane<D>(tiles, tci, gx, base, it.t0, it.t1, lane, a);
            acc |= lane_hits<D>(a, lane);
        }
        acc = __reduce_or_sync(0xffffffffu, acc);
        if (lane == 0) {
            uint32_t grow = row0 + it.row;
            if (keep) acc &= load_word<D>(keep, grow);
            if (it.split) {
                if (acc) atomic_or_word<D>(y, it.row, acc);
            } else {
                reinterpret_cast<typename WordT<D>::T *>(y)[it.row] = (typename WordT<D>::T)acc;
            }
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_bmv_bbb(const WorkItem *__restrict__ items, uint32_t n_items,
                                                 const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                                 const void *__restrict__ x, const void *__restrict__ keep,
                                                 void *__restrict__ y, uint32_t row0) {
    bbb_items<D>(items, n_items, tiles, tci, XGlobal<D>{x}, keep, y, row0);
}

// ------------------------------------------------------------ K5 bbf
template <int D> struct NCnt { static constexpr int N = D == 4 ? 4 : (D == 32 ? 4 : 8); };

template <int D>
__device__ __forceinline__ void lane_counts(const LaneTiles<D> &lt, uint32_t (&c)[NCnt<D>::N]) {
    if constexpr (D == 4) {
        uint32_t s = popc_bytes(lt.v.x & (lt.xw[0] * 0x01010101u)) + popc_bytes(lt.v.y & (lt.xw[1] * 0x01010101u)) +
                     popc_bytes(lt.v.z & (lt.xw[2] * 0x01010101u)) + popc_bytes(lt.v.w & (lt.xw[3] * 0x01010101u));
#pragma unroll
        for (int i = 0; i < 4; i++) c[i] += (s >> (8 * i)) & 0xFFu;
    } else if constexpr (D == 8) {
        uint32_t x0 = lt.xw[0] * 0x01010101u, x1 = lt.xw[1] * 0x01010101u;
        uint32_t lo = popc_bytes(lt.v.x & x0) + popc_bytes(lt.v.z & x1);
        uint32_t hi = popc_bytes(lt.v.y & x0) + popc_bytes(lt.v.w & x1);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            c[i] += (lo >> (8 * i)) & 0xFFu;
            c[4 + i] += (hi >> (8 * i)) & 0xFFu;
        }
    } else if constexpr (D == 16) {
        uint32_t xr = lt.xw[0] | (lt.xw[0] << 16), w[4] = {lt.v.x, lt.v.y, lt.v.z, lt.v.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            uint32_t v = w[i] & xr;
            c[2 * i] += __popc(v & 0xFFFFu);
            c[2 * i + 1] += __popc(v >> 16);
        }
    } else {
        uint32_t x = lt.xw[0];
        c[0] += __popc(lt.v.x & x);
        c[1] += __popc(lt.v.y & x);
        c[2] += __popc(lt.v.z & x);
        c[3] += __popc(lt.v.w & x);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_bmv_bbf(const WorkItem *__restrict__ items, uint32_t n_items, uint32_t n,
                                                 const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                                 const void *__restrict__ x, const void *__restrict__ keep,
                                                 double *__restrict__ y, uint32_t row0) {
    using G = Geo<D>;
    constexpr int NC = NCnt<D>::N;
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        WorkItem it = items[w];
        uint32_t c[NC];
#pragma unroll
        for (int i = 0; i < NC; i++) c[i] = 0;
        uint32_t start = G::TPL > 1 ? (it.t0 & ~(uint32_t)(G::TPL - 1)) : it.t0;
        uint32_t base = start;
        for (; base + G::TPW < it.t1; base += 2 * G::TPW) {
            LaneTiles<D> a, b;
            load_lane<D>(tiles, tci, XGlobal<D>{x}, base, it.t0, it.t1, lane, a);
            load_lane<D>(tiles, tci, XGlobal<D>{x}, base + G::TPW, it.t0, it.t1, lane, b);
            lane_counts<D>(a, c);
            lane_counts<D>(b, c);
        }
        if (base < it.t1) {
            LaneTiles<D> a;
            load_lane<D>(tiles, tci, XGlobal<D>{x}, base, it.t0, it.t1, lane, a);
            lane_counts<D>(a, c);
        }
        // reduce lanes that cover the same rows, then lane i takes row i
        uint32_t mine = 0;
        if constexpr (D == 4 || D == 8) {
#pragma unroll
            for (int i = 0; i < NC; i++) {
                uint32_t t = __reduce_add_sync(0xffffffffu, c[i]);
                if (lane == (uint32_t)i) mine = t;
            }
        } else if constexpr (D == 16) {
#pragma unroll
            for (int i = 0; i < NC; i++)
                for (int o = 2; o < 32; o <<= 1) c[i] += __shfl_xor_sync(0xffffffffu, c[i], o);
#pragma unroll
            for (int i = 0; i < NC; i++) {  // row r = 8*q + i lives in lanes with lane%2 == q
                uint32_t t = __shfl_sync(0xffffffffu, c[i], lane / 8);
                if ((lane & 7) == (uint32_t)i) mine = t;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NC; i++) {
                c[i] += __shfl_xor_sync(0xffffffffu, c[i], 8);
                c[i] += __shfl_xor_sync(0xffffffffu, c[i], 16);
            }
#pragma unroll
            for (int i = 0; i < NC; i++) {  // row r = 4*q + i lives in lanes with lane%8 == q
                uint32_t t = __shfl_sync(0xffffffffu, c[i], lane / 4);
                if ((lane & 3) == (uint32_t)i) mine = t;
            }
        }
        if (lane < (uint32_t)D) {
            uint32_t grow = row0 + it.row;
            uint64_t vrow = (uint64_t)grow * D + lane;
            if (vrow < n) {
                if (keep && !((load_word<D>(keep, grow) >> lane) & 1u)) mine = 0;
                size_t o = (size_t)it.row * D + lane;
                if (it.split) {
                    if (mine) atomicAdd(y + o, (double)mine);
                } else {
                    y[o] = (double)mine;
                }
            }
        }
    }
}

// ------------------------------------------------------------ K6 plans
// Rows longer than this many tiles take bmv_vlong.cu (segmented scatter +
// fold).  At d = 32 a tile row of 1024 tiles still holds only ~40 terms per
// bit-row on R-MAT, so the group walk keeps more rows (s16: 0.59 -> 0.45 ms).
static uint32_t vlong_row_tiles(int dim) { return dim == 32 ? 1024u : (dim == 4 ? 512u : 256u); }  // s24 d=4 PR: 512 -> 96.8 vs 98.8 ms at 256

// Row-length thresholds are fixed per matrix when its plan is built; the env
// override exists so parity tests can push small matrices through both paths.
static uint32_t vlong_thresh(int dim) {
    const char *ev = getenv("B2SR_VLONG_TILES");
    return ev ? (uint32_t)atoi(ev) : vlong_row_tiles(dim);
}

static void ensure_vlong(b2sr_matrix *m, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (!m->vlong) m->vlong = build_vlong(m, vlong_thresh(m->dim), s);
}

// ------------------------------------------------------------ used columns / scale
template <int D>
__global__ void k_used_words(uint64_t T, const uint32_t *__restrict__ tci, const typename WordT<D>::T *__restrict__ tiles,
                             uint32_t *__restrict__ colw) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t o = 0;
#pragma unroll
        for (int r = 0; r < D; r++) o |= tiles[t * D + r];
        if (o) atomicOr(colw + tci[t], o);
    }
}

__global__ void k_expand_used(uint32_t n, uint32_t d, const uint32_t *colw, uint8_t *out) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        out[j] = (colw[j / d] >> (j % d)) & 1u;
}

// zero scale at a used column -> *bad = min such j; otherwise xs = x / scale
__global__ void k_prescale(uint32_t n, uint32_t d, const uint32_t *colw, const double *x, const double *scale,
                           double *xs, unsigned long long *bad) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double sc = scale[j];
        if (sc == 0.0) {
            if ((colw[j / d] >> (j % d)) & 1u) atomicMin(bad, (unsigned long long)j);
            xs[j] = 0.0;
        } else {
            xs[j] = __ddiv_rn(x[j], sc);
        }
    }
}

void used_column_words(const b2sr_matrix *m, uint32_t *colw, cudaStream_t s) {
    uint32_t ntr_global = tile_rows(m->n, m->dim);
    CK(cudaMemsetAsync(colw, 0, (size_t)ntr_global * 4, s));
    if (!m->num_tiles) return;
    unsigned g = (unsigned)std::min<uint64_t>((m->num_tiles + 255) / 256, (uint64_t)num_sms() * 16);
    switch (m->dim) {
        case 4: LAUNCH(k_used_words<4>, g, 256, 0, s, m->num_tiles, m->tci, (const uint8_t *)m->tiles, colw); break;
        case 8: LAUNCH(k_used_words<8>, g, 256, 0, s, m->num_tiles, m->tci, (const uint8_t *)m->tiles, colw); break;
        case 16: LAUNCH(k_used_words<16>, g, 256, 0, s, m->num_tiles, m->tci, (const uint16_t *)m->tiles, colw); break;
        default: LAUNCH(k_used_words<32>, g, 256, 0, s, m->num_tiles, m->tci, (const uint32_t *)m->tiles, colw); break;
    }
}

// xs = x / scale with the reference's zero-scale rules (kernels.py:159-173).
// Returns -1 on success or the first offending column.
int64_t prescale(const b2sr_matrix *m, const double *x, const double *scale, double *xs, cudaStream_t s) {
    uint32_t ntr_global = tile_rows(m->n, m->dim);
    Buf<uint32_t> colw(ntr_global, s);
    used_column_words(m, colw.p, s);
    Buf<unsigned long long> bad(1, s);
    CK(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
    unsigned g = std::max(1u, std::min((m->n + 255) / 256, (uint32_t)num_sms() * 8));
    LAUNCH(k_prescale, g, 256, 0, s, m->n, m->dim, colw.p, x, scale, xs, bad.p);
    unsigned long long b = read_scalar(bad.p, s);
    return b == ~0ull ? -1 : (int64_t)b;
}

// ------------------------------------------------------------ launchers
void launch_bbb(b2sr_matrix *m, const void *x, const void *keep, void *y, cudaStream_t s) {
    if (stream_enabled(m->dim)) {
        launch_bbb_stream(m, x, keep, y, s);
        return;
    }
    ensure_items(m, s);
    if (m->any_split) CK(cudaMemsetAsync(y, 0, padded_vec_bytes(m->ntr, m->dim), s));
    const uint8_t *tl = (const uint8_t *)m->tiles;
    unsigned g = item_grid(m);
    kernel_timer().begin(s);
#define BBB_CASE(DD)                                                                                              \
    case DD:                                                                                                      \
        LAUNCH((k_bmv_bbb<DD>), g, 256, 0, s, m->items, m->n_items, tl, m->tci, x, keep, y, m->row0);          \
        break;
    switch (m->dim) {
        BBB_CASE(4)
        BBB_CASE(8)
        BBB_CASE(16)
        BBB_CASE(32)
    }
    kernel_timer().end(s);
#undef BBB_CASE
}

static size_t local_rows(const b2sr_matrix *m) {
    uint64_t lo = (uint64_t)m->row0 * m->dim;
    uint64_t hi = std::min<uint64_t>((uint64_t)(m->row0 + m->ntr) * m->dim, m->n);
    return hi > lo ? hi - lo : 0;
}

void launch_bbf(b2sr_matrix *m, const void *x, const void *keep, double *y, cudaStream_t s) {
    ensure_items(m, s);
    if (m->any_split) CK(cudaMemsetAsync(y, 0, local_rows(m) * sizeof(double), s));
    unsigned g = item_grid(m);
    const uint8_t *tl = (const uint8_t *)m->tiles;
    switch (m->dim) {
        case 4: LAUNCH(k_bmv_bbf<4>, g, 256, 0, s, m->items, m->n_items, m->n, tl, m->tci, x, keep, y, m->row0); break;
        case 8: LAUNCH(k_bmv_bbf<8>, g, 256, 0, s, m->items, m->n_items, m->n, tl, m->tci, x, keep, y, m->row0); break;
        case 16: LAUNCH(k_bmv_bbf<16>, g, 256, 0, s, m->items, m->n_items, m->n, tl, m->tci, x, keep, y, m->row0); break;
        default: LAUNCH(k_bmv_bbf<32>, g, 256, 0, s, m->items, m->n_items, m->n, tl, m->tci, x, keep, y, m->row0); break;
    }
}

// ARITHMETIC with add identity -0.0 (a public Semiring may carry it): the
// reference adds +0.0 for every unset bit it walks (kernels.py:201-207,
// cur + where(bit, term, 0.0)), which turns a -0.0 accumulator into +0.0; the
// set-bit fold keeps -0.0.  They differ only where the fold ends at -0.0, so
// those positions -- rare: every term was -0.0 -- are rescanned: if the
// bit-row meets an unset bit in any tile of its tile row, the reference holds
// +0.0.  Masked-off positions keep the identity.
template <int D>
__global__ void k_fix_negzero(uint32_t n, const uint32_t *__restrict__ trp, const typename WordT<D>::T *__restrict__ tiles,
                              const void *__restrict__ keep, double *__restrict__ y, uint32_t row0, uint32_t nrows) {
    constexpr uint32_t FULL = D == 32 ? 0xFFFFFFFFu : ((1u << D) - 1u);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows * D; i += gridDim.x * blockDim.x) {
        const double v = y[i];
        if (v != 0.0 || !signbit(v)) continue;
        const uint32_t I = i / D, r = i % D, grow = row0 + I;
        if ((uint64_t)grow * D + r >= n) continue;
        if (keep && !((load_word<D>(keep, grow) >> r) & 1u)) continue;
        const uint32_t t0 = trp[I], t1 = trp[I + 1];
        uint32_t walked_unset = 0;
        for (uint32_t t = t0; t < t1 && !walked_unset; t++) walked_unset = (uint32_t)tiles[(size_t)t * D + r] != FULL;
        if (walked_unset) y[i] = 0.0;
    }
}

// Rows up to the segmented-plan threshold: pipelined group-per-row walk
// (bmv_bff.cu), overlapped with the hub rows' segmented scatter + warp folds
// (bmv_vlong.cu).
void launch_bff(const b2sr_matrix *m_, const double *x, int ring, double inc, const void *keep, double *y,
                cudaStream_t s, double ident) {
    b2sr_matrix *m = const_cast<b2sr_matrix *>(m_);
    if (bff_csr_enabled(m)) {  // wide tiles: the cached CSR column lists (bmv_csr.cu)
        launch_bff_csr(m, x, ring, inc, ident, keep, y, s);
    } else {
        ensure_vlong(m, s);
        const uint32_t hi = vlong_thresh(m->dim);
        launch_bff_rows(m, x, ring, inc, ident, keep, y, hi, s, /*plan_only=*/true);
        // large x: gather from a hot-first relabelled copy (bmv_xperm.cu)
        Buf<double> xp;
        const uint32_t *gtci = nullptr;
        if (xperm_enabled(m)) {
            const size_t xbytes = (size_t)tile_rows(m->n, m->dim) * m->dim * sizeof(double);
            xp = Buf<double>(xbytes / sizeof(double), s);
            gtci = xperm_apply(m, x, xp.p, s);
            x = xp.p;
        }
        launch_vlong(m, x, ring, inc, ident, keep, y, s,
                     [&](cudaStream_t so) { launch_bff_rows(m, x, ring, inc, ident, keep, y, hi, so, false, gtci); },
                     gtci);
    }
    if (ring == B2SR_RING_ARITHMETIC && ident == 0.0 && std::signbit(ident) && m->ntr) {
        unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)m->ntr * m->dim + 255) / 256,
                                                                          (uint64_t)num_sms() * 8));
        switch (m->dim) {
            case 4: LAUNCH(k_fix_negzero<4>, g, 256, 0, s, m->n, m->trp, (const uint8_t *)m->tiles, keep, y, m->row0, m->ntr); break;
            case 8: LAUNCH(k_fix_negzero<8>, g, 256, 0, s, m->n, m->trp, (const uint8_t *)m->tiles, keep, y, m->row0, m->ntr); break;
            case 16: LAUNCH(k_fix_negzero<16>, g, 256, 0, s, m->n, m->trp, (const uint16_t *)m->tiles, keep, y, m->row0, m->ntr); break;
            default: LAUNCH(k_fix_negzero<32>, g, 256, 0, s, m->n, m->trp, (const uint32_t *)m->tiles, keep, y, m->row0, m->ntr); break;
        }
    }
}
}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_bmv_bbb(const b2sr_matrix *m, const void *d_x, const void *d_keep, void *d_y, void *stream) {
    API_BEGIN
    launch_bbb(const_cast<b2sr_matrix *>(m), d_x, d_keep, d_y, (cudaStream_t)stream);
    API_END
}

int b2sr_bmv_bbf(const b2sr_matrix *m, const void *d_x, const void *d_keep, double *d_y, void *stream) {
    API_BEGIN
    launch_bbf(const_cast<b2sr_matrix *>(m), d_x, d_keep, d_y, (cudaStream_t)stream);
    API_END
}

int b2sr_bmv_bff(const b2sr_matrix *m, const double *d_x, int ring, double inc, const double *d_scale,
                 const void *d_keep, double *d_y, int64_t *bad_col, void *stream) {
    return b2sr_bmv_bff_ex(m, d_x, ring, inc, ring_identity(ring), d_scale, d_keep, d_y, bad_col, stream);
}

int b2sr_bmv_bff_ex(const b2sr_matrix *m, const double *d_x, int ring, double inc, double add_identity,
                    const double *d_scale, const void *d_keep, double *d_y, int64_t *bad_col, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (ring == B2SR_RING_BOOLEAN)
        B2SR_THROW(B2SR_EINVAL, "boolean semiring has no full-precision gather; use bmv_bin_bin_bin");
    if (ring < 0 || ring > 3) B2SR_THROW(B2SR_EINVAL, "unknown semiring id %d", ring);
    if (d_scale && ring != B2SR_RING_ARITHMETIC)
        B2SR_THROW(B2SR_EINVAL, "scale is only supported with the arithmetic semiring");
    const double *x = d_x;
    Buf<double> xs;
    if (d_scale) {
        xs = Buf<double>(m->n, s);
        int64_t bad = prescale(m, d_x, d_scale, xs.p, s);
        if (bad >= 0) {
            if (bad_col) *bad_col = bad;
            B2SR_THROW(B2SR_EINVAL, "scale is zero at column %lld, which has incident bits", (long long)bad);
        }
        x = xs.p;
    }
    launch_bff(m, x, ring, inc, d_keep, d_y, s, add_identity);
    API_END
}

int b2sr_used_columns(const b2sr_matrix *m, uint8_t *d_out, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    Buf<uint32_t> colw(tile_rows(m->n, m->dim), s);
    used_column_words(m, colw.p, s);
    unsigned g = std::max(1u, std::min((m->n + 255) / 256, (uint32_t)num_sms() * 8));
    LAUNCH(k_expand_used, g, 256, 0, s, m->n, m->dim, colw.p, d_out);
    API_END
}

}  // extern "C"
