// K9: device-resident algorithm drivers (replaces algorithms.py:75-196).
//
// Every sweep's state (frontier, visited, levels, distances, ranks, labels)
// stays in HBM; the host sees one 4- or 8-byte flag per sweep (the
// reference's loop condition) and the final vector.
//
// BFS (algorithms.py:75-93): level-synchronous masked bbb sweeps over the
// transposed matrix.  The sweep kernel is the bbb stream with three
// output-preserving shortcuts: tile rows whose keep word (~visited) is zero
// are skipped, a tile's payload is only loaded when its frontier word is
// non-zero, and a row stops as soon as every keep bit is hit.  Levels,
// visited and the frontier-any flag are updated by one fused epilogue.
//
// PageRank delta (algorithms.py:157) is numpy's pairwise summation
// reproduced exactly (same leaf blocks, 8 accumulators, same tree), so the
// convergence test sees the reference's bits.
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "bfs_ctl.cuh"
#include "bmv_common.cuh"
#include "dist_comm.cuh"

namespace b2sr {

void launch_bff(const b2sr_matrix *m, const double *x, int ring, double inc, const void *keep, double *y,
                cudaStream_t s, double ident);
const uint32_t *xperm_apply_f32(b2sr_matrix *m, const double *x, float *xp, cudaStream_t s);
void used_column_words(const b2sr_matrix *m, uint32_t *colw, cudaStream_t s);

static unsigned grid_for(uint64_t work) {
    uint64_t b = (work + 255) / 256, cap = (uint64_t)num_sms() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

// ================================================================ BFS
template <int D> using BGeo = Geo<D>;

// hit bits (row-word positions) of the tiles this lane covers; the payload
// is only fetched for tiles whose frontier word is non-zero
template <int D, class GX>
__device__ __forceinline__ uint32_t bfs_lane(const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                             const GX &gx, uint32_t base, uint32_t t0, uint32_t t1,
                                             uint32_t lane) {
    using G = BGeo<D>;
    if constexpr (G::TPL > 1) {
        uint32_t tl = base + lane * G::TPL;
        if (!(tl < t1 && tl + G::TPL > t0)) return 0;
        uint32_t cols[G::TPL], xw[G::TPL];
        if constexpr (G::TPL == 4) {
            uint4 c = ld_stream128(tci + tl);
            cols[0] = c.x; cols[1] = c.y; cols[2] = c.z; cols[3] = c.w;
        } else {
            uint2 c = *reinterpret_cast<const uint2 *>(tci + tl);
            cols[0] = c.x; cols[1] = c.y;
        }
        uint32_t anyx = 0;
#pragma unroll
        for (int j = 0; j < G::TPL; j++) {
            bool ok = tl + j >= t0 && tl + j < t1;
            xw[j] = ok ? gx(cols[j]) : 0u;
            anyx |= xw[j];
        }
        if (!anyx) return 0;
        uint4 v = ld_stream128(tiles + (size_t)tl * G::TB);
        if constexpr (D == 4) {
            uint32_t w[4] = {v.x, v.y, v.z, v.w}, a = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) a |= nz_nibble_bytes(w[j] & (xw[j] * 0x01010101u));
            return a;
        } else {
            uint32_t x0 = xw[0] * 0x01010101u, x1 = xw[1] * 0x01010101u;
            uint32_t lo = nz_bytes(v.x & x0) | nz_bytes(v.z & x1);
            uint32_t hi = nz_bytes(v.y & x0) | nz_bytes(v.w & x1);
            return lo | (hi << 4);
        }
    } else {
        uint32_t t = base + lane / G::LPT, q = lane % G::LPT;
        if (t >= t1) return 0;
        uint32_t xw = gx(__ldg(tci + t));
        if (!xw) return 0;
        uint4 v = ld_stream128(tiles + (size_t)t * G::TB + q * 16);
        if constexpr (D == 16) {
            uint32_t xr = xw | (xw << 16), w[4] = {v.x, v.y, v.z, v.w}, a = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                uint32_t y = w[i] & xr;
                a |= ((y & 0xFFFFu) ? 1u : 0u) << (2 * i);
                a |= ((y >> 16) ? 1u : 0u) << (2 * i + 1);
            }
            return a << (8 * (lane & 1));
        } else {
            uint32_t a = 0;
            a |= (v.x & xw) ? 1u : 0u;
            a |= (v.y & xw) ? 2u : 0u;
            a |= (v.z & xw) ? 4u : 0u;
            a |= (v.w & xw) ? 8u : 0u;
            return a << (4 * (lane & 7));
        }
    }
}

template <int D, class GX>
__device__ __forceinline__ void pull_items(const WorkItem *__restrict__ items, uint32_t n_items,
                                           const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                           const GX &gx, const void *__restrict__ visited,
                                           const void *__restrict__ live, void *__restrict__ next, uint32_t row0,
                                           const uint32_t *__restrict__ idx, const uint32_t *__restrict__ idx_n) {
    using G = BGeo<D>;
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    if (idx) n_items = *idx_n;  // active-item list of a late pull level
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        WorkItem it = items[idx ? idx[w] : w];
        uint32_t grow = row0 + it.row;
        uint32_t keepw = ~load_word<D>(visited, grow) & load_word<D>(live, it.row);  // live is block-local
        if (!keepw) continue;
        uint32_t acc = 0;
        uint32_t base = G::TPL > 1 ? (it.t0 & ~(uint32_t)(G::TPL - 1)) : it.t0;
        for (; base < it.t1; base += 2 * G::TPW) {
            acc |= bfs_lane<D>(tiles, tci, gx, base, it.t0, it.t1, lane);
            if (base + G::TPW < it.t1) acc |= bfs_lane<D>(tiles, tci, gx, base + G::TPW, it.t0, it.t1, lane);
            if ((__reduce_or_sync(0xffffffffu, acc) & keepw) == keepw) break;  // every unvisited row reached
        }
        acc = __reduce_or_sync(0xffffffffu, acc) & keepw;
        if (lane == 0 && acc) {
            if (it.split) atomic_or_word<D>(next, it.row, acc);
            else reinterpret_cast<typename WordT<D>::T *>(next)[it.row] = (typename WordT<D>::T)acc;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_bfs_pull(const WorkItem *__restrict__ items, uint32_t n_items, uint32_t n,
                                                  const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                                  const void *__restrict__ frontier, const void *__restrict__ visited,
                                                  const void *__restrict__ live, void *__restrict__ next, uint32_t row0,
                                                  const uint32_t *__restrict__ idx, const uint32_t *__restrict__ idx_n) {
    pull_items<D>(items, n_items, tiles, tci, XGlobal<D>{frontier}, visited, live, next, row0, idx, idx_n);
}

// visited |= frontier; levels[new bits] = level; *any |= frontier != 0
template <int D>
__global__ void k_bfs_update(uint32_t ntr, const void *__restrict__ frontier, void *__restrict__ visited,
                             double *__restrict__ levels, double level, int *__restrict__ any,
                             unsigned long long *__restrict__ fv) {
    using W = typename WordT<D>::T;
    int found = 0;
    uint32_t cnt = 0;
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x) {
        uint32_t w = load_word<D>(frontier, I);
        if (!w) continue;
        found = 1;
        cnt += __popc(w);
        W *vis = reinterpret_cast<W *>(visited);
        vis[I] = (W)(vis[I] | w);
        while (w) {
            int k = __ffs(w) - 1;
            w &= w - 1;
            levels[(size_t)I * D + k] = level;
        }
    }
    if (__any_sync(0xffffffffu, found) && lane_id() == 0) atomicOr(any, 1);
    if (fv) {
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane_id() == 0 && cnt) atomicAdd(fv, (unsigned long long)cnt);
    }
}

__global__ void k_fill_f64(double *v, size_t n, double val) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) v[i] = val;
}

__global__ void k_bfs_seed(uint32_t src, uint32_t d, double *levels, void *visited, void *frontier) {
    levels[src] = 0.0;
    uint32_t w = src / d, b = src % d;
    int wb = d == 32 ? 4 : (d == 16 ? 2 : 1);
    size_t byte = (size_t)w * wb;
    uint32_t *vb = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(visited) + (byte & ~(size_t)3));
    uint32_t *fb = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(frontier) + (byte & ~(size_t)3));
    *vb |= (1u << b) << (8 * (byte & 3));
    *fb |= (1u << b) << (8 * (byte & 3));
}

// ---------------------------------------------------------------- direction-optimizing pieces
// Top-down (push) sweeps over the NON-transposed matrix a for small
// frontiers: every frontier tile row scatters the OR of its frontier bit-rows
// into next[K] & ~visited[K].  The set produced is exactly the pull sweep's
// (A^T x) & ~visited, so levels are unchanged -- only the work differs.

// visited |= next; levels[new] = level; counters; push work list for the next
// level.  Each thread owns 16 bytes of `next` (16/16/8/4 words); all-zero
// chunks cost one vector load, so the kernel scales with the frontier, not n.
// Unvisited tiles are tracked incrementally: removed_tiles counts the rows of
// at whose keep word (~visited & live) just became zero.
template <int D>
__global__ void k_bfs_update_dir(uint32_t ntr, uint32_t n, void *__restrict__ next, void *__restrict__ visited,
                                 double *__restrict__ levels, double level, const uint32_t *__restrict__ trp_a,
                                 const uint32_t *__restrict__ trp_at, const void *__restrict__ live_at,
                                 uint2 *__restrict__ list, BfsCounters *__restrict__ cnt,
                                 const int *__restrict__ gate, int mask, BfsCtl *__restrict__ ctl,
                                 uint4 *__restrict__ zero_buf, double alpha, unsigned long long tiles_at, int has_a) {
    using W = typename WordT<D>::T;
    if (gate && *gate == 0) return;  // device-controlled BFS: no sweep this level
    constexpr int WB = sizeof(W), WPC = 16 / WB;
    unsigned long long ft = 0, rt = 0, fv = 0;
    int found = 0;
    const uint32_t lane = lane_id();
    const uint32_t nchunks = (ntr + WPC - 1) / WPC;
    const uint32_t c0 = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t iters = (nchunks + stride - 1) / stride;  // warp-uniform trip count (scan below)
    for (uint32_t k = 0; k < iters; k++) {
        uint32_t c = c0 + k * stride;
        uint4 nv = c < nchunks ? reinterpret_cast<const uint4 *>(next)[c] : make_uint4(0, 0, 0, 0);
        if (zero_buf && c < nchunks) zero_buf[c] = make_uint4(0, 0, 0, 0);  // recycled as the next output
        if (mask && (nv.x | nv.y | nv.z | nv.w)) {
            // a raw pull sweep: keep only unvisited vertices with in-edges, and
            // store the masked words back -- they are the next frontier
            uint4 vv = reinterpret_cast<const uint4 *>(visited)[c], lv = reinterpret_cast<const uint4 *>(live_at)[c];
            uint4 mv = make_uint4(nv.x & ~vv.x & lv.x, nv.y & ~vv.y & lv.y, nv.z & ~vv.z & lv.z, nv.w & ~vv.w & lv.w);
            if (mv.x != nv.x || mv.y != nv.y || mv.z != nv.z || mv.w != nv.w) {
                reinterpret_cast<uint4 *>(next)[c] = mv;
                nv = mv;
            }
        }
        const W *nw = reinterpret_cast<const W *>(&nv);
        uint32_t nch = 0;
        if (nv.x | nv.y | nv.z | nv.w) {
#pragma unroll
            for (int j = 0; j < WPC; j++) {
                uint32_t w = nw[j];
                uint32_t I = c * WPC + j;
                if (!w || I >= ntr) continue;  // bytes past the last word are not part of the vector
                found = 1;
                W *vp = reinterpret_cast<W *>(visited) + I;
                uint32_t old = *vp, vis = old | w;
                *vp = (W)vis;
                fv += __popc(w);
                uint32_t b = w;
                while (b) {
                    int kk = __ffs(b) - 1;
                    b &= b - 1;
                    levels[(size_t)I * D + kk] = level;
                }
                uint32_t lv = load_word<D>(live_at, I);
                if ((~old & lv) && !(~vis & lv)) rt += trp_at[I + 1] - trp_at[I];
                if (trp_a) {
                    uint32_t len = trp_a[I + 1] - trp_a[I];
                    ft += len;
                    nch += (len + PUSH_CH - 1) / PUSH_CH;
                }
            }
        }
        // warp-aggregated reservation of push entries
        if (__any_sync(0xffffffffu, nch != 0)) {
            uint32_t incl = nch;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            uint32_t base = 0;
            if (lane == 31) base = atomicAdd(&cnt->list_n, total);
            base = __shfl_sync(0xffffffffu, base, 31);
            uint32_t o = base + incl - nch;
            if (nch) {
#pragma unroll
                for (int j = 0; j < WPC; j++) {
                    uint32_t I = c * WPC + j;
                    if (!nw[j] || I >= ntr) continue;
                    uint32_t len = trp_a[I + 1] - trp_a[I];
                    for (uint32_t q = 0; q < (len + PUSH_CH - 1) / PUSH_CH; q++) list[o++] = make_uint2(I, q);
                }
            }
        }
    }
    ft = __reduce_add_sync(0xffffffffu, (uint32_t)ft);  // per-warp sums < T < 2^32
    rt = __reduce_add_sync(0xffffffffu, (uint32_t)rt);
    fv = __reduce_add_sync(0xffffffffu, (uint32_t)fv);
    if (lane == 0) {
        if (ft) atomicAdd(&cnt->frontier_tiles, ft);
        if (rt) atomicAdd(&cnt->removed_tiles, rt);
        if (fv) atomicAdd(&cnt->frontier_vertices, fv);
    }
    if (__any_sync(0xffffffffu, found) && lane == 0) atomicOr(&cnt->any, 1);
    if (ctl) {  // the last block to finish plans the next level on the device
        __shared__ bool last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(&ctl->blocks_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last && threadIdx.x == 0) {
            __threadfence();
            volatile BfsCtl *c = ctl;
            c->blocks_done = 0;
            if (c->done || !c->cnt.any) {  // this sweep found nothing: BFS is over
                c->done = 1;
                c->mode = BFS_NONE;
            } else {
                c->unvisited -= c->cnt.removed_tiles;
                bool push = has_a && (double)c->cnt.frontier_tiles * alpha < (double)c->unvisited;
                c->mode = push ? BFS_PUSH : (c->unvisited * 2 < tiles_at ? BFS_PULL_ACTIVE : BFS_PULL);
                c->list_n = c->cnt.list_n;
                c->active_n = 0;
                c->sweeps = c->sweeps + 1;
                c->cnt.any = 0;
                c->cnt.list_n = 0;
                c->cnt.frontier_tiles = 0;
                c->cnt.removed_tiles = 0;
                c->cnt.frontier_vertices = 0;
            }
        }
    }
}

// late pull levels: the items of tile rows that still have a keep bit
template <int D>
__global__ void k_active_items(uint32_t ntr, const void *__restrict__ visited, const void *__restrict__ live,
                               const uint32_t *__restrict__ item_ofs, uint32_t *__restrict__ idx,
                               uint32_t *__restrict__ count) {
    const uint32_t lane = lane_id();
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t iters = (ntr + stride - 1) / stride;
    for (uint32_t k = 0; k < iters; k++) {
        uint32_t I = blockIdx.x * blockDim.x + threadIdx.x + k * stride;
        uint32_t nit = 0, first = 0;
        if (I < ntr && (~load_word<D>(visited, I) & load_word<D>(live, I))) {
            first = item_ofs[I];
            nit = item_ofs[I + 1] - first;
        }
        if (!__any_sync(0xffffffffu, nit != 0)) continue;
        uint32_t incl = nit;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        uint32_t total = __shfl_sync(0xffffffffu, incl, 31), base = 0;
        if (lane == 31) base = atomicAdd(count, total);
        base = __shfl_sync(0xffffffffu, base, 31);
        for (uint32_t j = 0; j < nit; j++) idx[base + incl - nit + j] = first + j;
    }
}

// warp per push entry; lane-strided tiles
template <int D>
__global__ void __launch_bounds__(256) k_bfs_push(const uint2 *__restrict__ list, const uint32_t *__restrict__ list_n,
                                                  const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                                                  const typename WordT<D>::T *__restrict__ tiles,
                                                  const void *__restrict__ frontier, const void *__restrict__ visited,
                                                  void *__restrict__ next, const int *__restrict__ gate) {
    if (gate && *gate != 1) return;  // device-controlled BFS: not a push level
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_entries = *list_n;
    for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_entries; e += warps) {
        uint2 ent = list[e];
        uint32_t I = ent.x;
        uint32_t t0 = trp[I] + ent.y * PUSH_CH;
        uint32_t t1 = min(trp[I + 1], t0 + PUSH_CH);
        uint32_t fw = load_word<D>(frontier, I);
        for (uint32_t t = t0 + lane; t < t1; t += 32) {
            uint32_t m = 0, f = fw;
            while (f) {
                int r = __ffs(f) - 1;
                f &= f - 1;
                m |= tiles[(size_t)t * D + r];
            }
            if (m) {
                uint32_t K = __ldg(tci + t);
                m &= ~load_word<D>(visited, K);
                if (m) atomic_or_word<D>(next, K, m);
            }
        }
    }
}

static double bfs_alpha() {
    const char *e = getenv("B2SR_BFS_ALPHA");
    return e ? atof(e) : 4.0;
}

// live[I] bit r: bit-row I*D+r of m has at least one set bit (warp per tile row)
template <int D>
__global__ void k_row_live(uint32_t ntr, const uint32_t *__restrict__ trp, const typename WordT<D>::T *__restrict__ tiles,
                           typename WordT<D>::T *__restrict__ live) {
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < ntr; I += warps) {
        uint32_t o = 0;
        for (uint32_t t = trp[I] + lane; t < trp[I + 1]; t += 32)
#pragma unroll
            for (int r = 0; r < D; r++) o |= (tiles[(size_t)t * D + r] ? 1u : 0u) << r;
        o = __reduce_or_sync(0xffffffffu, o);
        if (lane == 0) live[I] = (typename WordT<D>::T)o;
    }
}

template <int D>
__global__ void k_live_tiles(uint32_t ntr, const uint32_t *__restrict__ trp, const void *__restrict__ live,
                             unsigned long long *__restrict__ out) {
    unsigned long long acc = 0;
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x)
        if (load_word<D>(live, I)) acc += trp[I + 1] - trp[I];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0 && acc) atomicAdd(out, acc);
}

void ensure_live(b2sr_matrix *m, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (m->live) return;
    Buf<uint8_t> lv(padded_vec_bytes(m->ntr, m->dim), s);
    CK(cudaMemsetAsync(lv.p, 0, padded_vec_bytes(m->ntr, m->dim), s));
    unsigned g = grid_for((uint64_t)m->ntr * 32);
    switch (m->dim) {
        case 4: LAUNCH(k_row_live<4>, g, 256, 0, s, m->ntr, m->trp, (const uint8_t *)m->tiles, (uint8_t *)lv.p); break;
        case 8: LAUNCH(k_row_live<8>, g, 256, 0, s, m->ntr, m->trp, (const uint8_t *)m->tiles, (uint8_t *)lv.p); break;
        case 16: LAUNCH(k_row_live<16>, g, 256, 0, s, m->ntr, m->trp, (const uint16_t *)m->tiles, (uint16_t *)lv.p); break;
        default: LAUNCH(k_row_live<32>, g, 256, 0, s, m->ntr, m->trp, (const uint32_t *)m->tiles, (uint32_t *)lv.p); break;
    }
    // tiles in rows with a live bit: the starting "unvisited tiles" of a BFS
    Buf<unsigned long long> lt(1, s);
    CK(cudaMemsetAsync(lt.p, 0, 8, s));
    switch (m->dim) {
        case 4: LAUNCH(k_live_tiles<4>, grid_for(m->ntr), 256, 0, s, m->ntr, m->trp, lv.p, lt.p); break;
        case 8: LAUNCH(k_live_tiles<8>, grid_for(m->ntr), 256, 0, s, m->ntr, m->trp, lv.p, lt.p); break;
        case 16: LAUNCH(k_live_tiles<16>, grid_for(m->ntr), 256, 0, s, m->ntr, m->trp, lv.p, lt.p); break;
        default: LAUNCH(k_live_tiles<32>, grid_for(m->ntr), 256, 0, s, m->ntr, m->trp, lv.p, lt.p); break;
    }
    m->live_tiles = read_scalar(lt.p, s);
    m->live = lv.release();
}

// pull levels run on the flat tile stream (bmv_stream.cu) where it applies
static bool pull_stream(const b2sr_matrix *at) {
    const char *ps = getenv("B2SR_PULL_STREAM");  // B2SR_PULL_STREAM=0: work-item pull kernels (A/B)
    return stream_enabled(at->dim) && !(ps && ps[0] == '0');
}

void bfs_sweep(b2sr_matrix *at, const void *frontier, const void *visited, void *next, cudaStream_t s,
               const uint32_t *idx = nullptr, const uint32_t *idx_n = nullptr, int active_only = -1,
               bool lazy = false) {
    ensure_live(at, s);
    if (!idx && pull_stream(at)) {
        // only the loads that still hold an unvisited vertex, once few are left
        launch_bbb_stream(at, frontier, nullptr, next, s, visited, active_only > 0, lazy);
        return;
    }
    ensure_items(at, s);
    CK(cudaMemsetAsync(next, 0, padded_vec_bytes(at->ntr, at->dim), s));
    uint64_t blocks = ((uint64_t)at->n_items + 7) / 8, cap = (uint64_t)num_sms() * 16;
    unsigned g = (unsigned)std::min(blocks, cap);
    const uint8_t *tl = (const uint8_t *)at->tiles;
#define PULL_CASE(DD)                                                                                              \
    case DD:                                                                                                       \
        LAUNCH(k_bfs_pull<DD>, g, 256, 0, s, at->items, at->n_items, at->n, tl, at->tci, frontier, visited,        \
               at->live, next, at->row0, idx, idx_n);                                                              \
        break;
    switch (at->dim) {
        PULL_CASE(4)
        PULL_CASE(8)
        PULL_CASE(16)
        PULL_CASE(32)
    }
#undef PULL_CASE
}

void bfs_update(uint32_t n, uint32_t d, const void *frontier, void *visited, double *levels, double level, int *any,
                cudaStream_t s, unsigned long long *fv = nullptr) {
    uint32_t ntr = tile_rows(n, d);
    unsigned g = grid_for(ntr);
    switch (d) {
        case 4: LAUNCH(k_bfs_update<4>, g, 256, 0, s, ntr, frontier, visited, levels, level, any, fv); break;
        case 8: LAUNCH(k_bfs_update<8>, g, 256, 0, s, ntr, frontier, visited, levels, level, any, fv); break;
        case 16: LAUNCH(k_bfs_update<16>, g, 256, 0, s, ntr, frontier, visited, levels, level, any, fv); break;
        default: LAUNCH(k_bfs_update<32>, g, 256, 0, s, ntr, frontier, visited, levels, level, any, fv); break;
    }
}

void bfs_init(uint32_t n, uint32_t d, uint32_t src, void *visited, void *frontier, double *levels, cudaStream_t s) {
    size_t vb = padded_vec_bytes(tile_rows(n, d), d);
    CK(cudaMemsetAsync(visited, 0, vb, s));
    CK(cudaMemsetAsync(frontier, 0, vb, s));
    LAUNCH(k_fill_f64, grid_for(n), 256, 0, s, levels, (size_t)n, HUGE_VAL);
    LAUNCH(k_bfs_seed, 1, 1, 0, s, src, d, levels, visited, frontier);
}

// ================================================================ SSSP
// relaxed = np.minimum(dist, y); *changed |= relaxed != dist; dist = relaxed
__global__ void k_relax(size_t n, double *__restrict__ dist, const double *__restrict__ y, int *changed) {
    int ch = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double a = dist[i], b = y[i];
        double r = (a < b || isnan(a)) ? a : b;
        if (!(r == a)) { ch = 1; dist[i] = r; }
    }
    if (__any_sync(0xffffffffu, ch) && lane_id() == 0) atomicOr(changed, 1);
}

// ================================================================ PageRank
struct PwTree {
    std::vector<uint64_t> leaf_start;
    std::vector<uint32_t> leaf_len;
    std::vector<uint32_t> left, right, height;  // internal nodes (ids after the leaves)
};

static uint32_t pw_build(PwTree &t, uint64_t lo, uint64_t n, uint32_t &h) {
    if (n <= 128) {
        t.leaf_start.push_back(lo);
        t.leaf_len.push_back((uint32_t)n);
        h = 0;
        return (uint32_t)(t.leaf_start.size() - 1) | 0x80000000u;  // tagged leaf index
    }
    uint64_t n2 = n / 2;
    n2 -= n2 % 8;
    uint32_t hl, hr;
    uint32_t l = pw_build(t, lo, n2, hl);
    uint32_t r = pw_build(t, lo + n2, n - n2, hr);
    t.left.push_back(l);
    t.right.push_back(r);
    h = std::max(hl, hr) + 1;
    t.height.push_back(h);
    return (uint32_t)(t.left.size() - 1);
}

// numpy pairwise_sum leaf (n <= 128), additions only, no contraction
__device__ double pw_leaf(const double *a, uint32_t n) {
    if (n < 8) {
        double res = -0.0;
        for (uint32_t i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    uint32_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
}

__global__ void k_pw_leaves(uint32_t nleaves, const uint64_t *start, const uint32_t *len, const double *a, double *val) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nleaves; i += gridDim.x * blockDim.x)
        val[i] = pw_leaf(a + start[i], len[i]);
}

// internal nodes sorted by height; hofs[h] .. hofs[h+1] are the nodes of height h+1
__global__ void __launch_bounds__(1024) k_pw_combine(uint32_t nleaves, uint32_t nheights, const uint32_t *hofs,
                                                     const uint32_t *order, const uint32_t *left, const uint32_t *right,
                                                     double *val, double *out) {
    double *ival = val + nleaves;
    for (uint32_t h = 0; h < nheights; h++) {
        for (uint32_t k = hofs[h] + threadIdx.x; k < hofs[h + 1]; k += blockDim.x) {
            uint32_t node = order[k];
            uint32_t l = left[node], r = right[node];
            double lv = (l & 0x80000000u) ? val[l & 0x7FFFFFFFu] : ival[l];
            double rv = (r & 0x80000000u) ? val[r & 0x7FFFFFFFu] : ival[r];
            ival[node] = __dadd_rn(lv, rv);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = nheights ? ival[order[hofs[nheights] - 1]] : val[0];
}

struct PairwiseSum {
    uint32_t nleaves = 0, nheights = 0;
    Buf<uint64_t> start;
    Buf<uint32_t> len, hofs, order, left, right;
    Buf<double> val, out;
    PairwiseSum(uint64_t n, cudaStream_t s) {
        PwTree t;
        uint32_t h;
        pw_build(t, 0, n, h);
        nleaves = (uint32_t)t.leaf_start.size();
        uint32_t ni = (uint32_t)t.left.size();
        nheights = h;
        std::vector<uint32_t> hcount(h + 2, 0), ord(ni);
        for (uint32_t k = 0; k < ni; k++) hcount[t.height[k]]++;
        std::vector<uint32_t> hofs_h(h + 1, 0);
        for (uint32_t x = 1; x <= h; x++) hofs_h[x] = hofs_h[x - 1] + hcount[x];
        std::vector<uint32_t> fill(hofs_h.begin(), hofs_h.end());
        for (uint32_t k = 0; k < ni; k++) ord[fill[t.height[k] - 1]++] = k;
        start = Buf<uint64_t>(nleaves, s);
        len = Buf<uint32_t>(nleaves, s);
        hofs = Buf<uint32_t>(h + 1, s);
        order = Buf<uint32_t>(ni, s);
        left = Buf<uint32_t>(ni, s);
        right = Buf<uint32_t>(ni, s);
        val = Buf<double>((size_t)nleaves + ni, s);
        out = Buf<double>(1, s);
        CK(cudaMemcpyAsync(start.p, t.leaf_start.data(), nleaves * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(len.p, t.leaf_len.data(), nleaves * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(hofs.p, hofs_h.data(), (h + 1) * 4, cudaMemcpyHostToDevice, s));
        if (ni) {
            CK(cudaMemcpyAsync(order.p, ord.data(), ni * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(left.p, t.left.data(), ni * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(right.p, t.right.data(), ni * 4, cudaMemcpyHostToDevice, s));
        }
        CK(cudaStreamSynchronize(s));  // host vectors die at scope exit
    }
    // enqueue; the result lands in out.p
    void run(const double *a, cudaStream_t s) {
        LAUNCH(k_pw_leaves, grid_for(nleaves), 256, 0, s, nleaves, start.p, len.p, a, val.p);
        LAUNCH(k_pw_combine, 1, 1024, 0, s, nleaves, nheights, hofs.p, order.p, left.p, right.p, val.p, out.p);
    }
};

// bad column: out-degree zero where the column carries bits (algorithms.py:145-148)
__global__ void k_pr_check(uint32_t n, uint32_t d, const uint32_t *colw, const double *deg, unsigned long long *bad) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        if (deg[j] == 0.0 && ((colw[j / d] >> (j % d)) & 1u)) atomicMin(bad, (unsigned long long)j);
}

__global__ void k_pr_init(uint32_t n, double r0, const double *deg, double *rank, double *xs) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        rank[j] = r0;
        xs[j] = deg[j] == 0.0 ? 0.0 : __ddiv_rn(r0, deg[j]);
    }
}

// ---------------------------------------------------------------- PageRank, fast mode
// B2SR_PR_MODE=fast (d = 4, 8): the north-star tolerance for PageRank is a
// relative L1 of 1e-5, not bit equality, so the gather may drop the
// reference's term order.  x = rank/deg is kept as float32 (64 MB at s24
// instead of 134: it stays in the 126 MB L2, so the random x gathers stop
// missing to HBM -- the 1.6x DRAM overfetch of the exact gather) and
// accumulated in float64; every row's sum is a fixed lane-strided partial per
// lane plus a fixed shuffle tree (deterministic), split rows fold their
// items' partials in item order; the hubs need no serial chain.  The update
// (teleport + alpha*g), the delta (numpy pairwise) and the iteration rule are
// the exact driver's.  Error: each term carries <= 2^-24 relative rounding of
// x, so ranks differ from the exact ones by ~1e-7 relative (checked <= 1e-5
// against the oracle at s24, same iteration count).
template <int D>
__device__ __forceinline__ void pr_add(double (&acc)[D], uint32_t r, double v) {
#pragma unroll
    for (int q = 0; q < D; q++) acc[q] = __dadd_rn(acc[q], q == (int)r ? v : 0.0);
}

// U: tiles per lane in flight per step; MINB: CTAs per SM (the gather is
// latency-bound on the x loads: ncu at U = 8, 4 CTAs/SM, 64 registers: 41 %
// warps active, long-scoreboard stalls)
template <int D, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_pr_gather32(const WorkItem *__restrict__ items, uint32_t n_items, uint32_t n,
                                                     const uint32_t *__restrict__ tci, const uint8_t *__restrict__ tiles,
                                                     const float *__restrict__ x, double *__restrict__ y,
                                                     double *__restrict__ part) {
    static_assert(D == 4 || D == 8, "one 32/64-bit word per tile");
    using TW = typename std::conditional<D == 4, uint32_t, unsigned long long>::type;  // row r in byte r
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        const WorkItem it = items[w];
        double acc[D];
#pragma unroll
        for (int r = 0; r < D; r++) acc[r] = 0.0;
        // U tiles per lane per step: tile loads, then every tile's FIRST set bit
        // gathered unconditionally (R-MAT: ~1 bit per tile), all in flight
        // together; further bits of a tile are the rare tail
        for (uint32_t t = it.t0 + lane; t < it.t1; t += 32 * U) {
            uint32_t k[U];
            TW wd[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t tu = t + 32 * u;
                const bool ok = tu < it.t1;
                k[u] = ok ? ld_stream32(tci + tu) : 0u;
                if constexpr (D == 4) wd[u] = ok ? ld_stream32(tiles + (size_t)tu * 4) : 0u;
                else wd[u] = ok ? ((TW)ld_stream32(tiles + (size_t)tu * 8 + 4) << 32) | ld_stream32(tiles + (size_t)tu * 8) : 0ull;
            }
            float v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int p = wd[u] ? (D == 4 ? __ffs((uint32_t)wd[u]) : __ffsll((long long)wd[u])) - 1 : 0;
                v[u] = wd[u] ? __ldg(x + (size_t)k[u] * D + (p & 7)) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                TW b = wd[u];
                if (!b) continue;
                int p = (D == 4 ? __ffs((uint32_t)b) : __ffsll((long long)b)) - 1;
                pr_add<D>(acc, (uint32_t)p >> 3, (double)v[u]);
                b &= b - 1;
                while (b) {
                    p = (D == 4 ? __ffs((uint32_t)b) : __ffsll((long long)b)) - 1;
                    b &= b - 1;
                    pr_add<D>(acc, (uint32_t)p >> 3, (double)__ldg(x + (size_t)k[u] * D + (p & 7)));
                }
            }
        }
        double mine = 0.0;
#pragma unroll
        for (int r = 0; r < D; r++) {
            double val = acc[r];
#pragma unroll
            for (int o = 16; o; o >>= 1) val = __dadd_rn(val, __shfl_xor_sync(0xffffffffu, val, o));
            if (lane == (uint32_t)r) mine = val;
        }
        const uint64_t vrow = (uint64_t)it.row * D + lane;
        if (lane < (uint32_t)D) {
            if (it.split) part[(size_t)w * D + lane] = mine;
            else if (vrow < n) y[vrow] = mine;
        }
    }
}

// split rows: the items' partial sums in item order
template <int D>
__global__ void k_pr_fold_parts(uint32_t ntr, uint32_t n, const uint32_t *__restrict__ item_ofs,
                                const double *__restrict__ part, double *__restrict__ y) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ntr * D; i += gridDim.x * blockDim.x) {
        const uint32_t I = i / D, r = i % D, a = item_ofs[I], b = item_ofs[I + 1];
        if (b - a < 2 || i >= n) continue;
        double s = 0.0;
        for (uint32_t w = a; w < b; w++) s = __dadd_rn(s, part[(size_t)w * D + r]);
        y[i] = s;
    }
}

__global__ void k_to_f32(uint32_t n, const double *__restrict__ a, float *__restrict__ b) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) b[j] = __double2float_rn(a[j]);
}

// Keeps the float32 x of the fast PageRank gather resident in L2 while the
// tile stream (4.2 GB per sweep at s24) passes through: an access-policy
// window marks x persisting (set-aside capped by the device limit), the
// stream's other accesses streaming.  Restored on destruction.
struct L2Persist {
    cudaStream_t s = nullptr;
    bool on = false;
    size_t old_limit = 0;
    L2Persist(cudaStream_t st, const void *base, size_t bytes) : s(st) {
        const char *e = getenv("B2SR_PR_L2PERSIST");
        if (e && e[0] == '0') return;
        int dev = 0, max_persist = 0, max_window = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
        CK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
        if (max_persist <= 0 || max_window <= 0) return;
        CK(cudaDeviceGetLimit(&old_limit, cudaLimitPersistingL2CacheSize));
        const size_t set_aside = std::min<size_t>(bytes, (size_t)max_persist);
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside));
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
        v.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, (size_t)max_window);
        v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)set_aside / (double)v.accessPolicyWindow.num_bytes);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
        on = true;
    }
    ~L2Persist() {
        if (!on) return;
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
        cudaStreamSynchronize(s);
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, old_limit);
    }
};

static bool pr_fast_mode(int dim) {
    const char *e = getenv("B2SR_PR_MODE");
    return e && !strcmp(e, "fast") && (dim == 4 || dim == 8);
}

// new = teleport + alpha * g (no FMA); diff = |new - rank|; rank = new; xs = new / deg
__global__ void k_pr_update(uint32_t n, double teleport, double alpha, const double *__restrict__ g,
                            const double *__restrict__ deg, double *__restrict__ rank, double *__restrict__ xs,
                            double *__restrict__ diff) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double nr = __dadd_rn(teleport, __dmul_rn(alpha, g[j]));
        diff[j] = fabs(__dadd_rn(nr, -rank[j]));
        rank[j] = nr;
        double dg = deg[j];
        xs[j] = dg == 0.0 ? 0.0 : __ddiv_rn(nr, dg);
    }
}

// ================================================================ CC
__global__ void k_cc_init(uint32_t n, double *labels, uint32_t *lab_u) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        labels[j] = (double)j;
        lab_u[j] = j;
    }
}

// CC's gather m = bff(a, f, min_plus(0)) (algorithms.py:176) on d = 4, 8.  The
// labels are non-negative integers, so min(f_j + 0.0) over a row is exact and
// independent of the order the terms are visited in: no reference-order walk
// is needed, and the labels are read as u32 (64 MB at s24 instead of 134).
// Warp per work item (chunk of one tile row); lanes stride the tiles, keep a
// per-bit-row minimum, reduce with redux.sync min; split rows combine with
// atomicMin.  mu = 0xFFFFFFFF where a vertex has no neighbour (bff's +inf).
template <int D>
__global__ void __launch_bounds__(256) k_cc_min(const WorkItem *__restrict__ items, uint32_t n_items, uint32_t n,
                                                const uint32_t *__restrict__ tci, const uint8_t *__restrict__ tiles,
                                                const uint32_t *__restrict__ lab, uint32_t *__restrict__ mu) {
    static_assert(D == 4 || D == 8, "one 32/64-bit word per tile");
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        const WorkItem it = items[w];
        uint32_t mn[D];
#pragma unroll
        for (int r = 0; r < D; r++) mn[r] = 0xFFFFFFFFu;
        constexpr int U = 4;  // tiles per lane per step, their loads issued together
        for (uint32_t t = it.t0 + lane; t < it.t1; t += 32 * U) {
            uint32_t k[U], wd[U][D / 4];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t tu = t + 32 * u;
                const bool ok = tu < it.t1;
                k[u] = ok ? ld_stream32(tci + tu) : 0u;
                if constexpr (D == 4) {
                    wd[u][0] = ok ? ld_stream32(tiles + (size_t)tu * 4) : 0u;
                } else {
                    wd[u][0] = ok ? ld_stream32(tiles + (size_t)tu * 8) : 0u;
                    wd[u][1] = ok ? ld_stream32(tiles + (size_t)tu * 8 + 4) : 0u;
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t *xs = lab + (size_t)k[u] * D;
#pragma unroll
                for (int r = 0; r < D; r++) {
                    uint32_t b = (wd[u][r / 4] >> (8 * (r % 4))) & 0xFFu;
                    while (b) {
                        mn[r] = min(mn[r], __ldg(xs + __ffs(b) - 1));
                        b &= b - 1;
                    }
                }
            }
        }
        uint32_t mine = 0xFFFFFFFFu;
#pragma unroll
        for (int r = 0; r < D; r++) {
            const uint32_t v = __reduce_min_sync(0xffffffffu, mn[r]);
            if (lane == (uint32_t)r) mine = v;
        }
        const uint64_t v = (uint64_t)it.row * D + lane;
        if (lane < (uint32_t)D && v < n) {
            if (it.split) {
                if (mine != 0xFFFFFFFFu) atomicMin(mu + v, mine);
            } else {
                mu[v] = mine;
            }
        }
    }
}

// hook on the u32 minima: nxt[labels[i]] = min(nxt[labels[i]], mu_i)
__global__ void k_cc_hook_u(uint32_t n, const uint32_t *__restrict__ mu, const uint32_t *__restrict__ lab_u,
                            uint32_t *__restrict__ nxt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t v = mu[i];
        if (v != 0xFFFFFFFFu) {  // a neighbour exists (bff's minimum is finite)
            const uint32_t t = lab_u[i];
            if (v < nxt[t]) atomicMin(nxt + t, v);
        }
    }
}

// hook: nxt[labels[i]] = min(nxt[labels[i]], m_i)  (parallel form of algorithms.py:181-185)
__global__ void k_cc_hook(uint32_t n, const double *__restrict__ m, const uint32_t *__restrict__ lab_u,
                          uint32_t *__restrict__ nxt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double mi = m[i];
        if (mi < (double)n) {  // finite neighbour minimum (+inf when isolated)
            uint32_t t = lab_u[i];
            uint32_t v = (uint32_t)mi;
            if (v < nxt[t]) atomicMin(nxt + t, v);
        }
    }
}

// pointer jumping until every label is a root (algorithms.py:187-191)
__global__ void k_cc_jump(uint32_t n, uint32_t *__restrict__ nxt, int *changed) {
    int ch = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t p = nxt[i], g = nxt[p];
        if (g != p) { nxt[i] = g; ch = 1; }
    }
    if (__any_sync(0xffffffffu, ch) && lane_id() == 0) atomicOr(changed, 1);
}

__global__ void k_cc_commit(uint32_t n, const uint32_t *__restrict__ nxt, uint32_t *__restrict__ lab_u,
                            double *__restrict__ labels, int *changed) {
    int ch = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t v = nxt[i];
        if (v != lab_u[i]) { ch = 1; lab_u[i] = v; labels[i] = (double)v; }
    }
    if (__any_sync(0xffffffffu, ch) && lane_id() == 0) atomicOr(changed, 1);
}

// ================================================================ device-controlled BFS
// The direction choice of every level (push / full pull / pull over the
// loads of unvisited rows) is made on the device from the previous level's
// counters, and every kernel of a level is gated on it, so the host enqueues
// levels back to back and only polls for termination every few levels --
// instead of one D2H round trip plus a launch ramp per level.
__global__ void k_bfs_ctl_init(BfsCtl *c, unsigned long long unvisited) {
    c->mode = BFS_NONE;
    c->done = 0;
    c->list_n = 0;
    c->active_n = 0;
    c->unvisited = unvisited;
    c->sweeps = 0;
    c->blocks_done = 0;
    c->sparse = 0;
    c->cnt = BfsCounters{};
}

// One kernel for a root's setup (instead of a fill, four memsets, the seed
// and the control init): levels = +inf except the source (0), visited = next
// = 0, frontier = {src}, control block reset.
__global__ void k_bfs_init(uint32_t n, double *__restrict__ levels, uint32_t nw, uint32_t *__restrict__ visited,
                           uint32_t *__restrict__ next, uint32_t *__restrict__ frontier, uint32_t src, uint32_t d,
                           BfsCtl *__restrict__ c, unsigned long long unvisited) {
    const uint32_t wb = d == 32 ? 4 : (d == 16 ? 2 : 1);  // bytes per tile-row word
    const size_t byte = (size_t)(src / d) * wb;
    const size_t sw = byte >> 2;
    const uint32_t sm = (1u << (src % d)) << (8 * (byte & 3));
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) levels[i] = i == src ? 0.0 : HUGE_VAL;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < nw; j += stride) {
        visited[j] = 0;
        next[j] = 0;
        frontier[j] = j == sw ? sm : 0u;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->mode = BFS_NONE;
        c->done = 0;
        c->list_n = 0;
        c->active_n = 0;
        c->unvisited = unvisited;
        c->sweeps = 0;
        c->blocks_done = 0;
        c->sparse = 0;
        c->cnt = BfsCounters{};
    }
}

// Level update of the device-controlled BFS.  Per 16-byte chunk of the raw
// sweep output: keep unvisited live vertices (stored back: the next frontier),
// visited |= it (one vector RMW), levels of the new vertices, counters for the
// plan; the recycled output buffer of the next level is zeroed on the way.
// The last block to finish plans the next level (push / pull / active pull).
template <int D>
__global__ void k_bfs_update_dc(uint32_t ntr, uint4 *__restrict__ next, uint4 *__restrict__ visited,
                                double *__restrict__ levels, double level, const uint32_t *__restrict__ trp_a,
                                const uint32_t *__restrict__ trp_at, const uint4 *__restrict__ live_at,
                                BfsCtl *__restrict__ ctl, uint4 *__restrict__ zero_buf, int mask, double alpha,
                                unsigned long long tiles_at, int has_a, BfsSnap *__restrict__ snap,
                                uint32_t level_no, double active_frac) {
    using W = typename WordT<D>::T;
    pdl_prologue();
    if (ctl->mode == BFS_NONE && mask) return;  // BFS already over
    constexpr int WPC = 16 / sizeof(W);
    unsigned long long ft = 0, rt = 0, fv = 0;
    int found = 0;
    const uint32_t lane = lane_id();
    const uint32_t nchunks = (ntr + WPC - 1) / WPC;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += gridDim.x * blockDim.x) {
        uint4 nv = next[c];
        if (zero_buf) zero_buf[c] = make_uint4(0, 0, 0, 0);  // recycled as the next level's output
        if (!(nv.x | nv.y | nv.z | nv.w)) continue;
        const uint4 vv = visited[c];
        const uint4 lv = live_at ? live_at[c] : make_uint4(~0u, ~0u, ~0u, ~0u);
        if (mask) {
            uint4 mv = make_uint4(nv.x & ~vv.x & lv.x, nv.y & ~vv.y & lv.y, nv.z & ~vv.z & lv.z, nv.w & ~vv.w & lv.w);
            if (mv.x != nv.x || mv.y != nv.y || mv.z != nv.z || mv.w != nv.w) next[c] = mv;
            nv = mv;
            if (!(nv.x | nv.y | nv.z | nv.w)) continue;
        }
        visited[c] = make_uint4(vv.x | nv.x, vv.y | nv.y, vv.z | nv.z, vv.w | nv.w);
        found = 1;
        const W *nw = reinterpret_cast<const W *>(&nv);
        const W *vw = reinterpret_cast<const W *>(&vv);
        const W *lw = reinterpret_cast<const W *>(&lv);
#pragma unroll
        for (int j = 0; j < WPC; j++) {
            const uint32_t w = nw[j], I = c * WPC + j;
            if (!w) continue;  // words past ntr are zero (padding)
            fv += __popc(w);
            uint32_t b = w;
            while (b) {
                int kk = __ffs(b) - 1;
                b &= b - 1;
                levels[(size_t)I * D + kk] = level;
            }
            const uint32_t old = vw[j], l = lw[j];
            if (trp_at && (~old & l) && !(~(old | w) & l)) rt += __ldg(trp_at + I + 1) - __ldg(trp_at + I);
            if (trp_a) ft += __ldg(trp_a + I + 1) - __ldg(trp_a + I);
        }
    }
    ft = __reduce_add_sync(0xffffffffu, (uint32_t)ft);  // per-warp sums < T < 2^32
    rt = __reduce_add_sync(0xffffffffu, (uint32_t)rt);
    fv = __reduce_add_sync(0xffffffffu, (uint32_t)fv);
    BfsCounters *cnt = &ctl->cnt;
    const bool any = __any_sync(0xffffffffu, found);
    // block totals first, then one atomic per counter per block: every warp
    // hitting the same four L2 addresses serialised the update (ncu: 8-29 us
    // per level at s22 for ~3 MB of vectors)
    __shared__ unsigned long long bsum[3][32];
    __shared__ int bany[32];
    __shared__ bool last;
    const uint32_t wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        bsum[0][wid] = ft;
        bsum[1][wid] = rt;
        bsum[2][wid] = fv;
        bany[wid] = any;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0, c = 0;
        int o = 0;
        for (uint32_t q = 0; q < nw; q++) {
            a += bsum[0][q];
            b += bsum[1][q];
            c += bsum[2][q];
            o |= bany[q];
        }
        if (a) atomicAdd(&cnt->frontier_tiles, a);
        if (b) atomicAdd(&cnt->removed_tiles, b);
        if (c) atomicAdd(&cnt->frontier_vertices, c);
        if (o) atomicOr(&cnt->any, 1);
        // acq_rel: this block's counters are ordered before its "done" (release)
        // and the last block sees every block's counters (acquire) -- in place
        // of a full fence on each side
        unsigned int prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&ctl->blocks_done) : "memory");
        last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {  // the last block plans the next level
        // one batch of independent L2 reads (a chain of volatile accesses costs
        // a round trip each), then plain stores: later kernels see them
        const int done0 = __ldcg(&ctl->done), any_all = __ldcg(&ctl->cnt.any);
        const unsigned long long unv = __ldcg(&ctl->unvisited), rtn = __ldcg(&ctl->cnt.removed_tiles);
        const unsigned long long ftn = __ldcg(&ctl->cnt.frontier_tiles), fvn = __ldcg(&ctl->cnt.frontier_vertices);
        long long sweeps = __ldcg(&ctl->sweeps);
        int done = done0;
        ctl->blocks_done = 0;
        if (done0 || !any_all) {  // this sweep found nothing: BFS is over
            done = 1;
            ctl->done = 1;
            ctl->mode = BFS_NONE;
        } else {
            const unsigned long long u = unv - rtn;
            ctl->unvisited = u;
            const bool push = has_a && (double)ftn * alpha < (double)u;
            ctl->mode = push ? BFS_PUSH : ((double)u < active_frac * (double)tiles_at ? BFS_PULL_ACTIVE : BFS_PULL);
            // a frontier of < 1/16 of the vertices: most 4-tile groups see all-zero x words
            ctl->sparse = fvn * 16 < (unsigned long long)ntr * D;
            ctl->list_n = 0;
            ctl->active_n = 0;
            ctl->sweeps = ++sweeps;
            ctl->cnt.any = 0;
            ctl->cnt.frontier_tiles = 0;
            ctl->cnt.removed_tiles = 0;
            ctl->cnt.frontier_vertices = 0;
        }
        if (snap) {  // the level's outcome, straight into mapped host memory
            volatile BfsSnap *hs = snap + level_no % 8;
            hs->w = bfs_snap_pack(level_no, done, sweeps);  // one store: no fence between fields
        }
    }
}

// pull levels: fill the hot x words from the frontier, and for
// late pull levels list the loads that still hold an unvisited live vertex
template <int D>
__global__ void k_bfs_prep(BfsCtl *__restrict__ c, uint32_t ntr, const uint32_t *__restrict__ a_trp,
                           uint2 *__restrict__ plist, uint32_t S,
                           const uint32_t *__restrict__ cols, const void *__restrict__ frontier,
                           uint8_t *__restrict__ hx, uint32_t n_loads, const uint4 *__restrict__ desc,
                           const void *__restrict__ visited, const void *__restrict__ live,
                           uint32_t *__restrict__ alist, const void *__restrict__ pfrontier) {
    // row blocks: pfrontier / visited are shifted to the block's first row
    // (a and at blocks share the row range); frontier stays global (hot fill)
    pdl_prologue();
    const int mode = c->mode;
    if (mode == BFS_NONE) return;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const uint32_t lane = lane_id();
    __shared__ uint32_t wtot[32];
    __shared__ uint32_t bbase;
    const uint32_t wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (mode == BFS_PUSH) {  // work list: (frontier tile row of a, 1024-tile chunk)
        // one list reservation per block and round (block scan over the warps'
        // totals): per-warp atomics on list_n serialised on one L2 address
        const uint32_t iters = (ntr + stride - 1) / stride;
        for (uint32_t it = 0; it < iters; it++) {
            uint32_t I = tid + it * stride, nch = 0, len = 0;
            if (I < ntr && load_word<D>(pfrontier, I)) {
                len = a_trp[I + 1] - a_trp[I];
                nch = (len + PUSH_CH - 1) / PUSH_CH;
            }
            const bool any_here = __syncthreads_or(nch != 0);
            if (!any_here) continue;
            uint32_t incl = nch;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            if (lane == 31) wtot[wid] = incl;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t run = 0;
                for (uint32_t q = 0; q < nw; q++) {
                    const uint32_t v = wtot[q];
                    wtot[q] = run;
                    run += v;
                }
                bbase = run ? atomicAdd(&c->list_n, run) : 0u;
            }
            __syncthreads();
            const uint32_t base = bbase + wtot[wid];
            for (uint32_t q = 0; q < nch; q++) plist[base + incl - nch + q] = make_uint2(I, q);
            __syncthreads();  // wtot / bbase are rewritten next round
        }
        return;
    }
    const uint8_t *fr = static_cast<const uint8_t *>(frontier);
    if constexpr (D == 4 && HOT_NIBBLES) {
        for (uint32_t i = tid; i < (S + 1) / 2; i += stride) {
            uint32_t a = 2 * i, b = 2 * i + 1;
            uint32_t lo = fr[cols ? cols[a] : a] & 0xFu, hi = b < S ? (fr[cols ? cols[b] : b] & 0xFu) : 0u;
            hx[i] = (uint8_t)(lo | (hi << 4));
        }
    } else {
        for (uint32_t i = tid; i < S; i += stride) hx[i] = fr[cols ? cols[i] : i];
    }
    if (mode != BFS_PULL_ACTIVE) return;
    const uint32_t iters = (n_loads + stride - 1) / stride;
    for (uint32_t it = 0; it < iters; it++) {
        uint32_t k = tid + it * stride;
        bool act = false;
        if (k < n_loads) {
            uint32_t ra = desc[k].x, rb = desc[k + 1].x;
            for (uint32_t r = ra; r <= rb && !act; r++)
                act = (~load_word<D>(visited, r) & load_word<D>(live, r)) != 0;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (!__syncthreads_or(bal != 0)) continue;
        if (lane == 0) wtot[wid] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {  // one reservation per block and round
            uint32_t run = 0;
            for (uint32_t q = 0; q < nw; q++) {
                const uint32_t v = wtot[q];
                wtot[q] = run;
                run += v;
            }
            bbase = run ? atomicAdd(&c->active_n, run) : 0u;
        }
        __syncthreads();
        if (act) alist[bbase + wtot[wid] + __popc(bal & ((1u << lane) - 1u))] = k;
        __syncthreads();
    }
}

// Mapped (zero-copy) host ring the update kernel's last block writes each
// level's outcome into: the host learns that the BFS is over without a copy
// or a sync in the stream (one per host thread and device).
struct BfsSnapshots {
    static constexpr uint32_t N = 8;
    BfsSnap *host = nullptr, *dev = nullptr;
    BfsSnapshots() {
        CK(cudaHostAlloc(&host, N * sizeof(BfsSnap), cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dev), host, 0));
        reset();
    }
    void reset() {
        for (uint32_t i = 0; i < N; i++) host[i].w = 0xFFFFFFFFull;  // level ~0: no level yet
    }
    const volatile BfsSnap *slot(uint32_t level) const { return host + level % N; }
};
// levels enqueued beyond the one whose end is being checked (B2SR_BFS_LOOKAHEAD, A/B)
static uint32_t bfs_lookahead() {
    static const uint32_t v = [] {
        const char *e = getenv("B2SR_BFS_LOOKAHEAD");
        const int k = e ? atoi(e) : 1;
        return (uint32_t)std::max(1, std::min(k, 6));  // < the 8 snapshot slots
    }();
    return v;
}

// CTAs per SM of the per-level prep kernel (B2SR_BFS_PREP_CTAS, A/B)
static unsigned bfs_prep_ctas() {
    static const unsigned v = [] {
        const char *e = getenv("B2SR_BFS_PREP_CTAS");
        const int k = e ? atoi(e) : 8;
        return (unsigned)std::max(1, std::min(k, 16));
    }();
    return v;
}

static BfsSnapshots &bfs_snapshots() {
    // per host thread (re-entrant C ABI) and per device (the events belong to one)
    static thread_local BfsSnapshots *snaps[16] = {};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    dev &= 15;
    if (!snaps[dev]) snaps[dev] = new BfsSnapshots();
    return *snaps[dev];
}

// Per-thread, per-device scratch of the single-GPU BFS drivers, kept between
// calls (every call ends with a stream sync, so the next may reuse it): the
// seven stream-ordered allocations and frees of a root cost ~15 us of host
// time between roots.  Grown on demand; lives as long as the thread.
struct BfsScratch {
    uint8_t *p = nullptr;
    size_t bytes = 0;
    bool busy = false;  // set while a call uses it: a call that threw may have left work queued
};
static BfsScratch &bfs_scratch_slot() {
    static thread_local BfsScratch w[16];
    int dev = 0;
    CK(cudaGetDevice(&dev));
    return w[dev & 15];
}
static uint8_t *bfs_scratch(size_t bytes, cudaStream_t s) {
    BfsScratch &x = bfs_scratch_slot();
    if (x.busy) CK(cudaDeviceSynchronize());  // the previous call did not finish normally
    x.busy = true;
    if (x.bytes < bytes) {
        if (x.p) dfree(x.p, s);
        x.p = static_cast<uint8_t *>(dalloc(bytes, s));
        x.bytes = bytes;
    }
    return x.p;
}
// carve consecutive 256-byte aligned pieces out of a scratch block
struct Carve {
    size_t off = 0;
    size_t take(size_t b) {
        const size_t o = off;
        off += (b + 255) & ~size_t(255);
        return o;
    }
};

template <int D>
static void bfs_devctl(const b2sr_matrix *a, b2sr_matrix *at, uint32_t src, double *d_levels, int64_t *iterations,
                       cudaStream_t s) {
    const uint32_t n = at->n, ntr = at->ntr;
    const size_t vb = padded_vec_bytes(ntr, D);
    const uint32_t n16 = (uint32_t)((vb + 15) / 16);
    size_t list_cap = a ? (size_t)ntr + a->num_tiles / PUSH_CH + 1 : 1;
    ensure_live(at, s);
    HotView hv = hot_view(at, s);
    const size_t hb = hot_fill_bytes(hv, D);
    uint32_t n_loads = 0;
    const uint4 *desc = stream_desc(at, s, &n_loads);
    Carve cv;
    const size_t o_vis = cv.take(n16 * 16), o_fa = cv.take(n16 * 16), o_fb = cv.take(n16 * 16),
                 o_ctl = cv.take(sizeof(BfsCtl)), o_list = cv.take(list_cap * sizeof(uint2)), o_hx = cv.take(hb),
                 o_al = cv.take((size_t)std::max<uint32_t>(n_loads, 1) * 4);
    uint8_t *ws = bfs_scratch(cv.off, s);
    struct { uint8_t *p; } visited{ws + o_vis}, fa{ws + o_fa}, fb{ws + o_fb}, hx{ws + o_hx};
    struct { BfsCtl *p; } ctl{reinterpret_cast<BfsCtl *>(ws + o_ctl)};
    struct { uint2 *p; } list{reinterpret_cast<uint2 *>(ws + o_list)};
    struct { uint32_t *p; } alist{reinterpret_cast<uint32_t *>(ws + o_al)};
    CK(cudaMemsetAsync(hx.p, 0, hb, s));
    const double alpha = bfs_alpha();
    const char *afe = getenv("B2SR_BFS_ACTIVE");  // pull only the loads of unvisited rows below this tile fraction
    const double active_frac = afe ? atof(afe) : 0.5;
    const bool trace = getenv("B2SR_BFS_TRACE") != nullptr;
    // visited filter in the push levels: measured slower here, where push
    // levels are the sparse ones (92.9 vs 97.6 GTEPS at s22), so off
    const char *pve = getenv("B2SR_PUSH_VISITED");
    const bool push_vis = pve && pve[0] == '1';
    LAUNCH(k_bfs_init, grid_for(n), 256, 0, s, n, d_levels, n16 * 4, (uint32_t *)visited.p, (uint32_t *)fa.p,
           (uint32_t *)fb.p, src, (uint32_t)D, ctl.p, (unsigned long long)at->live_tiles);
    const unsigned gu = grid_for(n16);  // one thread per 16-byte chunk: the last-block plan waits on every block
    const uint32_t *ta = a ? a->trp : nullptr;
    BfsSnapshots &snaps = bfs_snapshots();
    snaps.reset();
    // programmatic dependent launch between the level's kernels (B2SR_BFS_PDL=0: plain launches, A/B)
    const char *pde = getenv("B2SR_BFS_PDL");
    const bool pdl = !(pde && pde[0] == '0');
    // level 0 = {src}: visited, levels, counters, the push list of level 1 and its plan
    LAUNCH_PDL(pdl, k_bfs_update_dc<D>, gu, 256, 0, s, ntr, (uint4 *)fb.p, (uint4 *)visited.p, d_levels, 0.0, ta,
               (const uint32_t *)at->trp, (const uint4 *)at->live, ctl.p, (uint4 *)nullptr, 0, alpha,
               (unsigned long long)at->num_tiles, a ? 1 : 0, snaps.dev, 0u, active_frac);
    void *frontier = fb.p, *next = fa.p;
    const unsigned gp = (unsigned)num_sms() * bfs_prep_ctas();
    int done = 0;
    long long sweeps = 0;
    for (uint32_t L = 1;; L++) {
        LAUNCH_PDL(pdl, k_bfs_prep<D>, gp, 256, 0, s, ctl.p, ntr, ta, list.p, hv.S, hv.cols, frontier, hx.p, n_loads,
                   desc, (const void *)visited.p, (const void *)at->live, alist.p, (const void *)frontier);
        launch_bfs_level(at, a, ctl.p, list.p, alist.p, hx.p, hb, frontier, next, push_vis ? visited.p : nullptr, s,
                         nullptr, nullptr, pdl);
        LAUNCH_PDL(pdl, k_bfs_update_dc<D>, gu, 256, 0, s, ntr, (uint4 *)next, (uint4 *)visited.p, d_levels, (double)L,
                   ta, (const uint32_t *)at->trp, (const uint4 *)at->live, ctl.p, (uint4 *)frontier, 1, alpha,
                   (unsigned long long)at->num_tiles, a ? 1 : 0, snaps.dev, L, active_frac);
        std::swap(frontier, next);
        // the host checks level L-LOOKAHEAD's outcome while levels up to L are
        // already enqueued (levels past the end are gated no-ops): no poll
        // ever drains the queue
        const uint32_t LOOKAHEAD = bfs_lookahead();
        if (trace || L > LOOKAHEAD) {
            const uint32_t Lc = trace ? L : L - LOOKAHEAD;
            const volatile BfsSnap *sn = snaps.slot(Lc);
            uint32_t lv_seen = 0;
            for (;;) {
                bfs_snap_read(sn, &lv_seen, &done, &sweeps);
                if (lv_seen == Lc) break;
                const cudaError_t q = cudaStreamQuery(s);
                bfs_snap_read(sn, &lv_seen, &done, &sweeps);
                if (lv_seen == Lc) break;
                if (q != cudaErrorNotReady) {
                    CK(q);  // a failed kernel surfaces here
                    B2SR_THROW(B2SR_ECUDA, "BFS level %u finished without its outcome", Lc);
                }
                std::this_thread::yield();
            }
            if (trace) fprintf(stderr, "[b2sr bfs] after level %u: done=%d sweeps=%lld\n", Lc, done, sweeps);
            if (done) break;
        }
        if (L > n + 2 + LOOKAHEAD) B2SR_THROW(B2SR_ENOCONV, "BFS failed to drain its frontier");
    }
    CK(cudaStreamSynchronize(s));  // the enqueued no-op levels are done
    bfs_scratch_slot().busy = false;
    *iterations = sweeps;
}

// BFS without a transpose (b2sr_bfs with at == NULL; d = 4, 8): every level
// top-down over a -- each tile row is read once per level its frontier bits
// fall in, and visited targets are filtered before the scatter.  A matrix that
// has no transpose yet pays the traversal only, not the (~10x longer) K3
// transpose the pull levels need; the Python driver switches to the
// direction-optimizing path once the transpose exists.
template <int D>
static void bfs_push_only(const b2sr_matrix *a, uint32_t src, double *d_levels, int64_t *iterations,
                          cudaStream_t s) {
    const uint32_t n = a->n, ntr = a->ntr;
    const size_t vb = padded_vec_bytes(ntr, D);
    const uint32_t n16 = (uint32_t)((vb + 15) / 16);
    Buf<uint8_t> visited(n16 * 16, s), fa(n16 * 16, s), fb(n16 * 16, s);
    Buf<BfsCtl> ctl(1, s);
    Buf<uint2> list((size_t)ntr + a->num_tiles / PUSH_CH + 1, s);
    const bool trace = getenv("B2SR_BFS_TRACE") != nullptr;
    const double active_frac = 0.0;  // every level is a push here
    const char *pve = getenv("B2SR_PUSH_VISITED");  // A/B (default on: every level is a push here)
    const bool push_vis = !(pve && pve[0] == '0');
    // alpha = 0 below: every level is a push
    LAUNCH(k_bfs_init, grid_for(n), 256, 0, s, n, d_levels, n16 * 4, (uint32_t *)visited.p, (uint32_t *)fa.p,
           (uint32_t *)fb.p, src, (uint32_t)D, ctl.p, 1ull);
    const unsigned gu = grid_for(n16);  // one thread per 16-byte chunk: the last-block plan waits on every block
    BfsSnapshots &snaps = bfs_snapshots();
    snaps.reset();
    const char *pde = getenv("B2SR_BFS_PDL");  // programmatic dependent launch between the level's kernels
    const bool pdl = !(pde && pde[0] == '0');
    LAUNCH_PDL(pdl, k_bfs_update_dc<D>, gu, 256, 0, s, ntr, (uint4 *)fb.p, (uint4 *)visited.p, d_levels, 0.0,
               (const uint32_t *)a->trp, (const uint32_t *)nullptr, (const uint4 *)nullptr, ctl.p, (uint4 *)nullptr, 0,
               0.0, (unsigned long long)a->num_tiles, 1, snaps.dev, 0u, active_frac);
    void *frontier = fb.p, *next = fa.p;
    const unsigned gp = (unsigned)num_sms() * bfs_prep_ctas();
    int done = 0;
    long long sweeps = 0;
    for (uint32_t L = 1;; L++) {
        LAUNCH_PDL(pdl, k_bfs_prep<D>, gp, 256, 0, s, ctl.p, ntr, (const uint32_t *)a->trp, list.p, 0u,
                   (const uint32_t *)nullptr, (const void *)frontier, (uint8_t *)nullptr, 0u, (const uint4 *)nullptr,
                   (const void *)visited.p, (const void *)nullptr, (uint32_t *)nullptr, (const void *)frontier);
        launch_bfs_push_level(a, ctl.p, list.p, frontier, push_vis ? visited.p : nullptr, next, s, pdl);
        LAUNCH_PDL(pdl, k_bfs_update_dc<D>, gu, 256, 0, s, ntr, (uint4 *)next, (uint4 *)visited.p, d_levels, (double)L,
                   (const uint32_t *)a->trp, (const uint32_t *)nullptr, (const uint4 *)nullptr, ctl.p, (uint4 *)frontier,
                   1, 0.0, (unsigned long long)a->num_tiles, 1, snaps.dev, L, active_frac);
        std::swap(frontier, next);
        const uint32_t LOOKAHEAD = bfs_lookahead();
        if (trace || L > LOOKAHEAD) {
            const uint32_t Lc = trace ? L : L - LOOKAHEAD;
            const volatile BfsSnap *sn = snaps.slot(Lc);
            uint32_t lv_seen = 0;
            for (;;) {
                bfs_snap_read(sn, &lv_seen, &done, &sweeps);
                if (lv_seen == Lc) break;
                const cudaError_t q = cudaStreamQuery(s);
                bfs_snap_read(sn, &lv_seen, &done, &sweeps);
                if (lv_seen == Lc) break;
                if (q != cudaErrorNotReady) {
                    CK(q);
                    B2SR_THROW(B2SR_ECUDA, "BFS level %u finished without its outcome", Lc);
                }
                std::this_thread::yield();
            }
            if (trace) fprintf(stderr, "[b2sr bfs push] after level %u: done=%d sweeps=%lld\n", Lc, done, sweeps);
            if (done) break;
        }
        if (L > n + 2 + LOOKAHEAD) B2SR_THROW(B2SR_ENOCONV, "BFS failed to drain its frontier");
    }
    CK(cudaStreamSynchronize(s));
    *iterations = sweeps;
}

static bool bfs_devctl_enabled(const b2sr_matrix *at) {
    const char *e = getenv("B2SR_BFS_DEVCTL");  // B2SR_BFS_DEVCTL=0: host-controlled levels (A/B)
    return pull_stream(at) && !(e && e[0] == '0');
}


// ================================================================ row-partitioned BFS (multi-GPU)
// both a and at are cut into the same contiguous tile-row
// blocks, balanced by at's tile count (the pull work); every rank keeps the
// global frontier / visited / levels and the global row lengths of a and at
// plus at's row-liveness words (small next to its block), so each rank
// evaluates the single-GPU driver's level plan on identical data -- the
// direction of every level is chosen on the device, identically on every
// rank, with no collective and no host round trip.  Per level:
//   prep     push list over the block's rows of a / hot x words + active loads
//   level    push: the block's frontier rows of a scatter into a global-length
//            contribution; pull: the block's rows of at (K4 flat stream)
//   exchange each rank's contribution to every other rank's rows
//            (grouped send/recv: an all-to-all-v of bit words)
//   merge    own rows = own contribution | the received ones
//   gather   all-gather-v of the merged row blocks -> global next
//   update   the single-GPU level update + plan on the global next
// Levels and sweep counts equal the single-GPU driver's bit for bit (the
// per-level vertex set is the same OR of the same bits).
}  // namespace b2sr

struct b2sr_dist_bfs {
    b2sr::Exchange *ex = nullptr;       // not owned
    b2sr_matrix *a = nullptr, *at = nullptr;
    bool owns_blocks = false;
    uint32_t n = 0, dim = 0, ntr = 0;   // global
    uint32_t *trp_a = nullptr, *trp_at = nullptr;  // global tile-row offsets (device)
    void *live_at = nullptr;            // global row-liveness words (n16 * 16 bytes)
    uint64_t live_tiles = 0, tiles_at = 0;
    std::vector<uint32_t> rows;         // world + 1 tile-row boundaries
    std::vector<size_t> off, len;       // byte ranges of the blocks in a global bit vector
    size_t n16 = 0, maxlen = 0;
    ~b2sr_dist_bfs() {
        if (owns_blocks) {
            b2sr::free_matrix(a);
            b2sr::free_matrix(at);
        }
        b2sr::dfree(trp_a, nullptr);
        b2sr::dfree(trp_at, nullptr);
        b2sr::dfree(live_at, nullptr);
    }
};

namespace b2sr {

// rows = multiple of `align`, boundaries where at's tile prefix crosses k*T/world
__global__ void k_balanced_cuts(const uint32_t *__restrict__ trp, uint32_t ntr, int world, uint32_t align,
                                uint32_t *__restrict__ cuts) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > world) return;
    if (k == 0 || k == world) {
        cuts[k] = k ? ntr : 0;
        return;
    }
    const unsigned long long target = (unsigned long long)trp[ntr] * k / world;
    uint32_t lo = 0, hi = ntr;  // first row whose prefix reaches the target
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if ((unsigned long long)trp[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    uint32_t r = (lo + align / 2) / align * align;
    cuts[k] = r < ntr ? r : ntr;
}

// own rows of the global next = own contribution | every peer's contribution
__global__ void k_or_merge(uint4 *__restrict__ dst, const uint4 *__restrict__ own, const uint4 *__restrict__ recv,
                           uint32_t n16, uint32_t stride16, int parts) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
        uint4 v = own[i];
        for (int p = 0; p < parts; p++) {
            uint4 w = recv[(size_t)p * stride16 + i];
            v.x |= w.x; v.y |= w.y; v.z |= w.z; v.w |= w.w;
        }
        dst[i] = v;
    }
}

static void dist_layout(b2sr_dist_bfs *p) {
    const int W = p->ex->world;
    const int wb = word_bytes(p->dim);
    const size_t vb = padded_vec_bytes(p->ntr, p->dim);
    p->n16 = (vb + 15) / 16;
    p->off.assign(W, 0);
    p->len.assign(W, 0);
    p->maxlen = 0;
    for (int r = 0; r < W; r++) {  // a block at the very end may be empty
        p->off[r] = p->rows[r] >= p->ntr ? p->n16 * 16 : (size_t)p->rows[r] * wb;
        size_t end = (r + 1 == W || p->rows[r + 1] >= p->ntr) ? p->n16 * 16 : (size_t)p->rows[r + 1] * wb;
        if (p->off[r] % 16 || end % 16) B2SR_THROW(B2SR_EINVAL, "row blocks must start on 16-byte words");
        p->len[r] = end - p->off[r];
        p->maxlen = std::max(p->maxlen, p->len[r]);
    }
}

static uint32_t row_align(int dim) { return 16 / word_bytes(dim); }

template <int D>
static void dist_bfs_run(b2sr_dist_bfs *p, uint32_t src, double *d_levels, int64_t *iterations, cudaStream_t s) {
    Exchange &ex = *p->ex;
    const int W = ex.world, R = ex.rank;
    const uint32_t n = p->n, ntr = p->ntr;
    b2sr_matrix *a = p->a, *at = p->at;
    const size_t vbytes = p->n16 * 16, off = p->off[R];
    Buf<uint8_t> visited(vbytes, s), fa(vbytes, s), fb(vbytes, s), contrib(vbytes, s);
    Buf<uint8_t> recv(std::max<size_t>(1, (size_t)(W - 1) * p->maxlen), s);
    Buf<BfsCtl> ctl(1, s);
    Buf<uint2> list((size_t)a->ntr + a->num_tiles / PUSH_CH + 1, s);
    ensure_live(at, s);  // block-local liveness (active-load lists)
    HotView hv = at->num_tiles ? hot_view(at, s) : HotView{0, nullptr, nullptr};
    const size_t hb = hot_fill_bytes(hv, D);
    Buf<uint8_t> hx(hb, s);
    CK(cudaMemsetAsync(hx.p, 0, hb, s));
    uint32_t n_loads = 0;
    const uint4 *desc = at->num_tiles ? stream_desc(at, s, &n_loads) : nullptr;
    Buf<uint32_t> alist(std::max<uint32_t>(n_loads, 1), s);
    const double alpha = bfs_alpha();
    const char *afe = getenv("B2SR_BFS_ACTIVE");
    const double active_frac = afe ? atof(afe) : 0.5;
    const bool trace = getenv("B2SR_BFS_TRACE") != nullptr;
    LAUNCH(k_fill_f64, grid_for(n), 256, 0, s, d_levels, (size_t)n, HUGE_VAL);
    CK(cudaMemsetAsync(visited.p, 0, vbytes, s));
    CK(cudaMemsetAsync(fb.p, 0, vbytes, s));
    CK(cudaMemsetAsync(fa.p, 0, vbytes, s));
    CK(cudaMemsetAsync(contrib.p, 0, vbytes, s));
    LAUNCH(k_bfs_seed, 1, 1, 0, s, src, (uint32_t)D, d_levels, fa.p, fb.p);
    CK(cudaMemsetAsync(fa.p, 0, vbytes, s));
    LAUNCH(k_bfs_ctl_init, 1, 1, 0, s, ctl.p, (unsigned long long)p->live_tiles);
    const unsigned gu = grid_for(p->n16);
    BfsSnapshots &snaps = bfs_snapshots();
    snaps.reset();
    LAUNCH(k_bfs_update_dc<D>, gu, 256, 0, s, ntr, (uint4 *)fb.p, (uint4 *)visited.p, d_levels, 0.0, p->trp_a,
           p->trp_at, (const uint4 *)p->live_at, ctl.p, nullptr, 0, alpha, (unsigned long long)p->tiles_at, 1,
           snaps.dev, 0u, active_frac);
    // the exchange pattern is the same every level
    std::vector<Xfer> sends, recvs;
    for (int q = 0, k = 0; q < W; q++) {
        if (q == R) continue;
        if (p->len[q]) sends.push_back({q, contrib.p + p->off[q], p->len[q]});
        if (p->len[R]) recvs.push_back({q, recv.p + (size_t)k * p->maxlen, p->len[R]});
        k++;
    }
    const uint32_t own16 = (uint32_t)(p->len[R] / 16);
    const unsigned gm = grid_for(own16);
    void *frontier = fb.p, *next = fa.p;
    const unsigned gp = (unsigned)num_sms() * bfs_prep_ctas();
    const uint8_t *vis_blk = visited.p + off;
    int done = 0;
    long long sweeps = 0;
    for (uint32_t L = 1;; L++) {
        const uint8_t *fr = static_cast<const uint8_t *>(frontier);
        LAUNCH(k_bfs_prep<D>, gp, 256, 0, s, ctl.p, a->ntr, a->trp, list.p, hv.S, hv.cols, frontier, hx.p, n_loads,
               desc, vis_blk, at->live, alist.p, fr + off);
        if (at->num_tiles || a->num_tiles)
            launch_bfs_level(at, a, ctl.p, list.p, alist.p, hx.p, hb, frontier, contrib.p + off, nullptr, s, fr + off,
                             contrib.p);
        ex.sendrecv(sends, recvs, s);
        LAUNCH(k_or_merge, gm, 256, 0, s, reinterpret_cast<uint4 *>(static_cast<uint8_t *>(next) + off),
               reinterpret_cast<const uint4 *>(contrib.p + off), reinterpret_cast<const uint4 *>(recv.p), own16,
               (uint32_t)(p->maxlen / 16), W - 1);
        ex.allgatherv(next, p->off, p->len, s);
        LAUNCH(k_bfs_update_dc<D>, gu, 256, 0, s, ntr, (uint4 *)next, (uint4 *)visited.p, d_levels, (double)L,
               p->trp_a, p->trp_at, (const uint4 *)p->live_at, ctl.p, (uint4 *)contrib.p, 1, alpha,
               (unsigned long long)p->tiles_at, 1, snaps.dev, L, active_frac);
        std::swap(frontier, next);
        const uint32_t LOOKAHEAD = bfs_lookahead();
        if (trace || L > LOOKAHEAD) {
            const uint32_t Lc = trace ? L : L - LOOKAHEAD;
            const volatile BfsSnap *sn = snaps.slot(Lc);
            uint32_t lv_seen = 0;
            for (;;) {
                bfs_snap_read(sn, &lv_seen, &done, &sweeps);
                if (lv_seen == Lc) break;
                const cudaError_t q = cudaStreamQuery(s);
                bfs_snap_read(sn, &lv_seen, &done, &sweeps);
                if (lv_seen == Lc) break;
                if (q != cudaErrorNotReady) {
                    CK(q);
                    B2SR_THROW(B2SR_ECUDA, "BFS level %u finished without its outcome", Lc);
                }
                std::this_thread::yield();
            }
            if (trace) fprintf(stderr, "[b2sr dist bfs r%d] after level %u: done=%d sweeps=%lld\n", R, Lc, done, sweeps);
            if (done) break;
        }
        if (L > n + 2 + LOOKAHEAD) B2SR_THROW(B2SR_ENOCONV, "BFS failed to drain its frontier");
    }
    CK(cudaStreamSynchronize(s));
    *iterations = sweeps;
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_bfs(const b2sr_matrix *a_c, const b2sr_matrix *at_c, uint32_t src, double *d_levels,
             int64_t *iterations, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    b2sr_matrix *at = const_cast<b2sr_matrix *>(at_c);
    const b2sr_matrix *a = a_c;
    if (!at) {  // no transpose: push-only levels over a
        if (!a) B2SR_THROW(B2SR_EINVAL, "bfs needs a or its transpose");
        if (a->row0 != 0 || a->ntr != tile_rows(a->n, a->dim)) B2SR_THROW(B2SR_EINVAL, "bfs needs a full matrix");
        if (a->dim > 8) B2SR_THROW(B2SR_EINVAL, "push-only bfs supports tile dims 4 and 8");
        if (src >= a->n) B2SR_THROW(B2SR_EINVAL, "source vertex %u out of range for n=%u", src, a->n);
        if (a->dim == 4) bfs_push_only<4>(a, src, d_levels, iterations, s);
        else bfs_push_only<8>(a, src, d_levels, iterations, s);
        return B2SR_OK;
    }
    if (at->row0 != 0 || at->ntr != tile_rows(at->n, at->dim)) B2SR_THROW(B2SR_EINVAL, "bfs needs a full matrix");
    if (a && (a->n != at->n || a->dim != at->dim || a->row0 != 0 || a->ntr != at->ntr))
        B2SR_THROW(B2SR_EINVAL, "a and at must be the same full matrix and its transpose");
    if (src >= at->n) B2SR_THROW(B2SR_EINVAL, "source vertex %u out of range for n=%u", src, at->n);
    if (bfs_devctl_enabled(at)) {
        if (at->dim == 4) bfs_devctl<4>(a, at, src, d_levels, iterations, s);
        else bfs_devctl<8>(a, at, src, d_levels, iterations, s);
        return B2SR_OK;
    }
    uint32_t n = at->n, d = at->dim, ntr = at->ntr;
    size_t vb = padded_vec_bytes(ntr, d);
    Buf<uint8_t> visited(vb, s), fa(vb, s), fb(vb, s);
    Buf<BfsCounters> cnt(1, s);
    size_t list_cap = a ? (size_t)ntr + a->num_tiles / PUSH_CH + 1 : 1;
    Buf<uint2> list(list_cap, s);
    ensure_live(at, s);
    ensure_items(at, s);
    const double alpha = bfs_alpha();
    const bool trace = getenv("B2SR_BFS_TRACE") != nullptr;
    // seed: next = {src}, visited = {}; the update makes it the level-0 frontier
    LAUNCH(k_fill_f64, grid_for(n), 256, 0, s, d_levels, (size_t)n, HUGE_VAL);
    CK(cudaMemsetAsync(visited.p, 0, vb, s));
    CK(cudaMemsetAsync(fb.p, 0, vb, s));
    CK(cudaMemsetAsync(fa.p, 0, vb, s));
    LAUNCH(k_bfs_seed, 1, 1, 0, s, src, d, d_levels, fa.p, fb.p);  // sets the bit in both; fa re-zeroed below
    CK(cudaMemsetAsync(fa.p, 0, vb, s));
    void *frontier = fb.p, *next = fa.p;
    BfsCounters h{};
    auto update = [&](const void *fr, double level) {
        CK(cudaMemsetAsync(cnt.p, 0, sizeof(BfsCounters), s));
        unsigned g = grid_for(ntr);
        const uint32_t *ta = a ? a->trp : nullptr;
        switch (d) {
            case 4: LAUNCH(k_bfs_update_dir<4>, g, 256, 0, s, ntr, n, const_cast<void *>(fr), visited.p, d_levels, level, ta, at->trp, at->live, list.p, cnt.p, nullptr, 0, nullptr, nullptr, 0.0, 0ull, 0); break;
            case 8: LAUNCH(k_bfs_update_dir<8>, g, 256, 0, s, ntr, n, const_cast<void *>(fr), visited.p, d_levels, level, ta, at->trp, at->live, list.p, cnt.p, nullptr, 0, nullptr, nullptr, 0.0, 0ull, 0); break;
            case 16: LAUNCH(k_bfs_update_dir<16>, g, 256, 0, s, ntr, n, const_cast<void *>(fr), visited.p, d_levels, level, ta, at->trp, at->live, list.p, cnt.p, nullptr, 0, nullptr, nullptr, 0.0, 0ull, 0); break;
            default: LAUNCH(k_bfs_update_dir<32>, g, 256, 0, s, ntr, n, const_cast<void *>(fr), visited.p, d_levels, level, ta, at->trp, at->live, list.p, cnt.p, nullptr, 0, nullptr, nullptr, 0.0, 0ull, 0); break;
        }
        CK(cudaMemcpyAsync(&h, cnt.p, sizeof(BfsCounters), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    };
    uint64_t unvisited = at->live_tiles;  // tiles of at in rows that still have a keep bit
    update(frontier, 0.0);                // level 0 = {src}
    unvisited -= h.removed_tiles;
    Buf<uint32_t> act_idx, act_n;         // active-item list for late pull levels
    int64_t sweeps = 0;
    for (;;) {
        bool push = a && (double)h.frontier_tiles * alpha < (double)unvisited;
        bool sparse_pull = !push && unvisited * 16 < at->num_tiles;
        if (!push && pull_stream(at)) {
            // flat-stream pull; restricted to the loads of unvisited rows once they are few
            bfs_sweep(at, frontier, visited.p, next, s, nullptr, nullptr, unvisited * 2 < at->num_tiles ? 1 : 0);
            sparse_pull = false;
        }
        if (sparse_pull) {
            if (!act_idx.p) {
                act_idx = Buf<uint32_t>(at->n_items, s);
                act_n = Buf<uint32_t>(1, s);
            }
            CK(cudaMemsetAsync(act_n.p, 0, 4, s));
            unsigned g = grid_for(ntr);
            switch (d) {
                case 4: LAUNCH(k_active_items<4>, g, 256, 0, s, ntr, visited.p, at->live, at->item_ofs, act_idx.p, act_n.p); break;
                case 8: LAUNCH(k_active_items<8>, g, 256, 0, s, ntr, visited.p, at->live, at->item_ofs, act_idx.p, act_n.p); break;
                case 16: LAUNCH(k_active_items<16>, g, 256, 0, s, ntr, visited.p, at->live, at->item_ofs, act_idx.p, act_n.p); break;
                default: LAUNCH(k_active_items<32>, g, 256, 0, s, ntr, visited.p, at->live, at->item_ofs, act_idx.p, act_n.p); break;
            }
        }
        if (!push && pull_stream(at)) {
            // swept above
        } else if (push) {
            CK(cudaMemsetAsync(next, 0, vb, s));
            uint64_t blocks = ((uint64_t)h.list_n + 7) / 8, cap = (uint64_t)num_sms() * 16;
            unsigned g = (unsigned)std::max<uint64_t>(1, std::min(blocks, cap));
            switch (d) {
                case 4: LAUNCH(k_bfs_push<4>, g, 256, 0, s, list.p, &cnt.p->list_n, a->trp, a->tci, (const uint8_t *)a->tiles, frontier, visited.p, next, nullptr); break;
                case 8: LAUNCH(k_bfs_push<8>, g, 256, 0, s, list.p, &cnt.p->list_n, a->trp, a->tci, (const uint8_t *)a->tiles, frontier, visited.p, next, nullptr); break;
                case 16: LAUNCH(k_bfs_push<16>, g, 256, 0, s, list.p, &cnt.p->list_n, a->trp, a->tci, (const uint16_t *)a->tiles, frontier, visited.p, next, nullptr); break;
                default: LAUNCH(k_bfs_push<32>, g, 256, 0, s, list.p, &cnt.p->list_n, a->trp, a->tci, (const uint32_t *)a->tiles, frontier, visited.p, next, nullptr); break;
            }
        } else if (sparse_pull) {
            bfs_sweep(at, frontier, visited.p, next, s, act_idx.p, act_n.p);
        } else {
            bfs_sweep(at, frontier, visited.p, next, s);
        }
        sweeps++;
        if (trace)
            fprintf(stderr, "[b2sr bfs] level %lld %s frontier_v=%llu frontier_tiles=%llu unvisited_tiles=%llu\n",
                    (long long)sweeps, push ? "push" : (sparse_pull ? "pull(active)" : "pull"),
                    h.frontier_vertices, h.frontier_tiles, (unsigned long long)unvisited);
        update(next, (double)sweeps);
        unvisited -= h.removed_tiles;
        std::swap(frontier, next);
        if (sweeps > (int64_t)n) B2SR_THROW(B2SR_ENOCONV, "BFS failed to drain its frontier");
        if (!h.any) break;
    }
    *iterations = sweeps;
    API_END
}

int b2sr_bfs_init(uint32_t n, uint32_t dim, uint32_t src, void *d_visited, void *d_frontier, double *d_levels,
                  void *stream) {
    API_BEGIN
    if (src >= n) B2SR_THROW(B2SR_EINVAL, "source vertex %u out of range for n=%u", src, n);
    bfs_init(n, dim, src, d_visited, d_frontier, d_levels, (cudaStream_t)stream);
    API_END
}

int b2sr_bfs_sweep(const b2sr_matrix *at_block, const void *d_frontier, const void *d_visited, void *d_next,
                   void *stream) {
    API_BEGIN
    bfs_sweep(const_cast<b2sr_matrix *>(at_block), d_frontier, d_visited, d_next, (cudaStream_t)stream);
    API_END
}

int b2sr_bfs_update(uint32_t n, uint32_t dim, const void *d_frontier, void *d_visited, double *d_levels,
                    double level, int *d_any, void *stream) {
    API_BEGIN
    bfs_update(n, dim, d_frontier, d_visited, d_levels, level, d_any, (cudaStream_t)stream);
    API_END
}

int b2sr_bfs_sweep_ex(const b2sr_matrix *at_block, const void *d_frontier, const void *d_visited, void *d_next,
                      int flags, void *stream) {
    API_BEGIN
    bfs_sweep(const_cast<b2sr_matrix *>(at_block), d_frontier, d_visited, d_next, (cudaStream_t)stream, nullptr,
              nullptr, (flags & B2SR_SWEEP_ACTIVE) ? 1 : 0, (flags & B2SR_SWEEP_LAZY) != 0);
    API_END
}

int b2sr_bfs_update_ex(uint32_t n, uint32_t dim, const void *d_frontier, void *d_visited, double *d_levels,
                       double level, int *d_any, uint64_t *d_frontier_vertices, void *stream) {
    API_BEGIN
    bfs_update(n, dim, d_frontier, d_visited, d_levels, level, d_any, (cudaStream_t)stream,
               reinterpret_cast<unsigned long long *>(d_frontier_vertices));
    API_END
}

int b2sr_sssp(const b2sr_matrix *at, uint32_t src, double *d_dist, int64_t *iterations, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (at->row0 != 0) B2SR_THROW(B2SR_EINVAL, "sssp needs a full matrix");
    uint32_t n = at->n;
    if (src >= n) B2SR_THROW(B2SR_EINVAL, "source vertex %u out of range for n=%u", src, n);
    Buf<double> y(n, s);
    Buf<int> changed(1, s);
    LAUNCH(k_fill_f64, grid_for(n), 256, 0, s, d_dist, (size_t)n, HUGE_VAL);
    CK(cudaMemsetAsync(d_dist + src, 0, sizeof(double), s));
    int64_t sweeps = 0;
    for (uint32_t it = 0; it + 1 < n; it++) {  // for _ in range(n - 1)
        launch_bff(at, d_dist, B2SR_RING_MINPLUS, 1.0, nullptr, y.p, s, ring_identity(B2SR_RING_MINPLUS));
        CK(cudaMemsetAsync(changed.p, 0, sizeof(int), s));
        LAUNCH(k_relax, grid_for(n), 256, 0, s, (size_t)n, d_dist, y.p, changed.p);
        sweeps++;
        if (!read_scalar(changed.p, s)) break;
    }
    *iterations = sweeps;
    API_END
}

int b2sr_pr_step(uint32_t count, double teleport, double alpha, const double *d_g, const double *d_deg, double *d_rank,
                 double *d_xs, double *d_diff, void *stream) {
    API_BEGIN
    if (count) LAUNCH(k_pr_update, grid_for(count), 256, 0, (cudaStream_t)stream, count, teleport, alpha, d_g, d_deg,
                      d_rank, d_xs, d_diff);
    API_END
}

int b2sr_pairwise_sum(const double *d_a, uint64_t n, double *d_out, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (!n) {
        CK(cudaMemsetAsync(d_out, 0, 8, s));
    } else {
        PairwiseSum pw(n, s);
        pw.run(d_a, s);
        CK(cudaMemcpyAsync(d_out, pw.out.p, 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));  // pw's buffers die at scope exit
    }
    API_END
}

int b2sr_min_relax(uint64_t count, double *d_dist, const double *d_y, int *d_changed, void *stream) {
    API_BEGIN
    if (count) LAUNCH(k_relax, grid_for(count), 256, 0, (cudaStream_t)stream, (size_t)count, d_dist, d_y, d_changed);
    API_END
}

int b2sr_pagerank(const b2sr_matrix *a, const double *d_out_degree, double alpha, double epsilon, int64_t max_iter,
                  double *d_rank, int64_t *iterations, int *converged, int64_t *bad_col, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (a->row0 != 0) B2SR_THROW(B2SR_EINVAL, "pagerank needs a full matrix");
    uint32_t n = a->n, d = a->dim;
    {
        Buf<uint32_t> colw(tile_rows(n, d), s);
        used_column_words(a, colw.p, s);
        Buf<unsigned long long> bad(1, s);
        CK(cudaMemsetAsync(bad.p, 0xFF, 8, s));
        LAUNCH(k_pr_check, grid_for(n), 256, 0, s, n, d, colw.p, d_out_degree, bad.p);
        unsigned long long b = read_scalar(bad.p, s);
        if (b != ~0ull) {
            if (bad_col) *bad_col = (int64_t)b;
            B2SR_THROW(B2SR_EINVAL, "out_degree[%llu] is zero but vertex %llu has out-edges", b, b);
        }
    }
    Buf<double> xs(n, s), g(n, s), diff(n, s);
    PairwiseSum pw(n, s);
    double teleport = (1.0 - alpha) / (double)n;
    LAUNCH(k_pr_init, grid_for(n), 256, 0, s, n, 1.0 / (double)n, d_out_degree, d_rank, xs.p);
    int64_t sweeps = 0;
    int conv = 0;
    const bool trace = getenv("B2SR_PR_TRACE") != nullptr;
    cudaEvent_t ev[4] = {};
    if (trace)
        for (auto &e : ev) CK(cudaEventCreate(&e));
    const bool fast = pr_fast_mode(d);
    const char *pxe = getenv("B2SR_PR_XPERM");  // fast mode: relabelled x' (default on; 0 = plain x)
    const bool pr_xperm = fast && !(pxe && pxe[0] == '0');
    Buf<float> x32(fast ? (size_t)a->ntr * d : 1, s);
    Buf<double> part;
    if (fast) {
        ensure_items(const_cast<b2sr_matrix *>(a), s);
        part = Buf<double>((size_t)a->n_items * d, s);
        CK(cudaMemsetAsync(x32.p, 0, (size_t)a->ntr * d * 4, s));
    }
    std::unique_ptr<L2Persist> persist;
    if (fast) persist.reset(new L2Persist(s, x32.p, (size_t)a->ntr * d * 4));
    while (sweeps < max_iter) {
        if (trace) CK(cudaEventRecord(ev[0], s));
        if (fast) {
            // hot-first relabelled float32 x' (bmv_xperm.cu): hot columns share
            // cache lines, so more of the random gathers hit L1 / L2
            const uint32_t *gtci = pr_xperm ? xperm_apply_f32(const_cast<b2sr_matrix *>(a), xs.p, x32.p, s) : a->tci;
            if (!pr_xperm) LAUNCH(k_to_f32, grid_for(n), 256, 0, s, n, xs.p, x32.p);
            const unsigned gi = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)a->n_items + 7) / 8,
                                                                                    (uint64_t)num_sms() * 16));
            kernel_timer().begin(s);
            // B2SR_PRG: gather geometry (A/B; s24 gather ms) -- 5 (default): U=2 x 8 CTAs/SM (3.03),
            // 0: U=8 x 4 (3.97), 1: U=4 x 6 (3.31), 2: U=6 x 5 (4.07), 3: U=16 x 2 (6.56), 4: U=4 x 8 (3.89, spills)
            static const int prg = [] { const char *e = getenv("B2SR_PRG"); return e ? atoi(e) : 5; }();
#define PRG_LAUNCH(DD, UU, MB)                                                                                    \
    LAUNCH((k_pr_gather32<DD, UU, MB>), gi, 256, 0, s, a->items, a->n_items, n, gtci, (const uint8_t *)a->tiles, \
           x32.p, g.p, part.p)
            if (d == 4) {
                if (prg == 0) PRG_LAUNCH(4, 8, 4);
                else if (prg == 1) PRG_LAUNCH(4, 4, 6);
                else if (prg == 2) PRG_LAUNCH(4, 6, 5);
                else if (prg == 3) PRG_LAUNCH(4, 16, 2);
                else if (prg == 4) PRG_LAUNCH(4, 4, 8);
                else PRG_LAUNCH(4, 2, 8);
            } else {
                PRG_LAUNCH(8, 8, 4);  // d = 8 (U = 4 x 6 spills there)
            }
#undef PRG_LAUNCH
            kernel_timer().end(s);
            if (a->any_split) {
                if (d == 4) LAUNCH(k_pr_fold_parts<4>, grid_for((uint64_t)a->ntr * 4), 256, 0, s, a->ntr, n, a->item_ofs, part.p, g.p);
                else LAUNCH(k_pr_fold_parts<8>, grid_for((uint64_t)a->ntr * 8), 256, 0, s, a->ntr, n, a->item_ofs, part.p, g.p);
            }
        } else {
            launch_bff(a, xs.p, B2SR_RING_ARITHMETIC, 0.0, nullptr, g.p, s, 0.0);
        }
        if (trace) CK(cudaEventRecord(ev[1], s));
        LAUNCH(k_pr_update, grid_for(n), 256, 0, s, n, teleport, alpha, g.p, d_out_degree, d_rank, xs.p, diff.p);
        pw.run(diff.p, s);
        if (trace) CK(cudaEventRecord(ev[2], s));
        double delta = read_scalar(pw.out.p, s);
        if (trace) {
            float t1, t2;
            CK(cudaEventElapsedTime(&t1, ev[0], ev[1]));
            CK(cudaEventElapsedTime(&t2, ev[1], ev[2]));
            fprintf(stderr, "[b2sr pr] sweep %lld gather %.3f ms update+delta %.3f ms\n", (long long)sweeps, t1, t2);
        }
        sweeps++;
        if (delta < epsilon) { conv = 1; break; }
    }
    *iterations = sweeps;
    *converged = conv;
    API_END
}

int b2sr_cc(const b2sr_matrix *a, double *d_labels, int64_t *iterations, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (a->row0 != 0) B2SR_THROW(B2SR_EINVAL, "connected components needs a full matrix");
    uint32_t n = a->n;
    const char *ue = getenv("B2SR_CC_U32");  // B2SR_CC_U32=0: the generic float gather (A/B)
    const bool u32 = (a->dim == 4 || a->dim == 8) && !(ue && ue[0] == '0');
    Buf<double> m(u32 ? 1 : n, s);
    Buf<uint32_t> lab_u(n, s), nxt(n, s), mu(u32 ? n : 1, s);
    Buf<int> flag(1, s);
    LAUNCH(k_cc_init, grid_for(n), 256, 0, s, n, d_labels, lab_u.p);
    b2sr_matrix *am = const_cast<b2sr_matrix *>(a);
    if (u32) ensure_items(am, s);
    // large label vectors: gather from the hot-first relabelled copy (bmv_xperm.cu)
    const bool perm = u32 && xperm_enabled(am);
    Buf<uint32_t> labp(perm ? (size_t)tile_rows(n, a->dim) * a->dim : 1, s);
    int64_t sweeps = 0;
    for (;;) {
        if (u32) {
            CK(cudaMemsetAsync(mu.p, 0xFF, (size_t)n * 4, s));
            const uint32_t *gl = lab_u.p, *gtci = a->tci;
            if (perm) {
                gtci = xperm_apply_u32(am, lab_u.p, labp.p, s);
                gl = labp.p;
            }
            const unsigned gi = (unsigned)std::max<uint64_t>(
                1, std::min<uint64_t>(((uint64_t)am->n_items + 7) / 8, (uint64_t)num_sms() * 16));
            if (a->dim == 4)
                LAUNCH(k_cc_min<4>, gi, 256, 0, s, am->items, am->n_items, n, gtci, (const uint8_t *)a->tiles, gl,
                       mu.p);
            else
                LAUNCH(k_cc_min<8>, gi, 256, 0, s, am->items, am->n_items, n, gtci, (const uint8_t *)a->tiles, gl,
                       mu.p);
        } else {
            launch_bff(a, d_labels, B2SR_RING_MINPLUS, 0.0, nullptr, m.p, s, ring_identity(B2SR_RING_MINPLUS));
        }
        sweeps++;
        CK(cudaMemcpyAsync(nxt.p, lab_u.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
        if (u32) LAUNCH(k_cc_hook_u, grid_for(n), 256, 0, s, n, mu.p, lab_u.p, nxt.p);
        else LAUNCH(k_cc_hook, grid_for(n), 256, 0, s, n, m.p, lab_u.p, nxt.p);
        for (;;) {
            CK(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
            LAUNCH(k_cc_jump, grid_for(n), 256, 0, s, n, nxt.p, flag.p);
            if (!read_scalar(flag.p, s)) break;
        }
        CK(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
        LAUNCH(k_cc_commit, grid_for(n), 256, 0, s, n, nxt.p, lab_u.p, d_labels, flag.p);
        if (!read_scalar(flag.p, s)) break;
        if (sweeps > (int64_t)n + 1) B2SR_THROW(B2SR_ENOCONV, "component labels failed to stabilise");
    }
    *iterations = sweeps;
    API_END
}

}  // extern "C"

// ================================================================ row-partitioned drivers: C ABI
namespace b2sr {

static void check_block_pair(const b2sr_matrix *a, const b2sr_matrix *at) {
    if (!a || !at) B2SR_THROW(B2SR_EINVAL, "distributed bfs needs a and its transpose");
    if (a->n != at->n || a->dim != at->dim) B2SR_THROW(B2SR_EINVAL, "a and at must share n and tile width");
    if (a->dim > 8) B2SR_THROW(B2SR_EINVAL, "the device-controlled distributed bfs supports tile dims 4 and 8");
}

static b2sr_matrix *block_of(const b2sr_matrix *m, uint32_t b, uint32_t e, cudaStream_t s) {
    b2sr_matrix *out = nullptr;
    int rc = b2sr_row_block(m, b, e, s, &out);
    if (rc) throw Error{rc, std::string()};
    return out;
}

static uint32_t *copy_u32(const uint32_t *src, size_t count, cudaStream_t s) {
    uint32_t *d = static_cast<uint32_t *>(dalloc(count * 4 + 16, s));
    CK(cudaMemcpyAsync(d, src, count * 4, cudaMemcpyDefault, s));
    return d;
}

}  // namespace b2sr

extern "C" {

int b2sr_dist_bfs_plan(b2sr_comm *comm, const b2sr_matrix *a_c, const b2sr_matrix *at_c, void *stream,
                       b2sr_dist_bfs **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    check_block_pair(a_c, at_c);
    b2sr_matrix *a = const_cast<b2sr_matrix *>(a_c), *at = const_cast<b2sr_matrix *>(at_c);
    if (a->row0 || at->row0 || a->ntr != tile_rows(a->n, a->dim) || at->ntr != a->ntr)
        B2SR_THROW(B2SR_EINVAL, "b2sr_dist_bfs_plan needs the full matrices (see b2sr_dist_bfs_plan_blocks)");
    Exchange *ex = comm->ex;
    auto *p = new b2sr_dist_bfs();
    try {
        p->ex = ex;
        p->n = at->n;
        p->dim = at->dim;
        p->ntr = at->ntr;
        ensure_live(at, s);
        p->live_tiles = at->live_tiles;
        p->tiles_at = at->num_tiles;
        // cuts balanced by at's tiles, on 16-byte word boundaries of the bit vectors
        Buf<uint32_t> cuts(ex->world + 1, s);
        LAUNCH(k_balanced_cuts, 1, 64 * ((ex->world + 64) / 64), 0, s, at->trp, at->ntr, ex->world,
               row_align(at->dim), cuts.p);
        p->rows.resize(ex->world + 1);
        CK(cudaMemcpyAsync(p->rows.data(), cuts.p, 4 * (ex->world + 1), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        dist_layout(p);
        const uint32_t b = p->rows[ex->rank], e = p->rows[ex->rank + 1];
        p->a = block_of(a, b, e, s);
        p->at = block_of(at, b, e, s);
        p->owns_blocks = true;
        p->trp_a = copy_u32(a->trp, (size_t)p->ntr + 1, s);
        p->trp_at = copy_u32(at->trp, (size_t)p->ntr + 1, s);
        p->live_at = dalloc(p->n16 * 16, s);
        CK(cudaMemsetAsync(p->live_at, 0, p->n16 * 16, s));
        CK(cudaMemcpyAsync(p->live_at, at->live, padded_vec_bytes(p->ntr, p->dim), cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
    } catch (...) {
        delete p;
        throw;
    }
    *out = p;
    API_END
}

int b2sr_dist_bfs_plan_blocks(b2sr_comm *comm, const b2sr_matrix *a_blk, const b2sr_matrix *at_blk,
                              const uint32_t *trp_a, const uint32_t *trp_at, void *stream, b2sr_dist_bfs **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    check_block_pair(a_blk, at_blk);
    if (a_blk->row0 != at_blk->row0 || a_blk->ntr != at_blk->ntr)
        B2SR_THROW(B2SR_EINVAL, "a and at blocks must cover the same tile rows");
    Exchange *ex = comm->ex;
    const int W = ex->world, R = ex->rank;
    auto *p = new b2sr_dist_bfs();
    try {
        p->ex = ex;
        p->n = at_blk->n;
        p->dim = at_blk->dim;
        p->ntr = tile_rows(p->n, p->dim);
        p->a = const_cast<b2sr_matrix *>(a_blk);
        p->at = const_cast<b2sr_matrix *>(at_blk);
        ensure_live(p->at, s);
        // every rank's (first row, rows, live tiles): an all-reduce of one-hot slots
        Buf<int64_t> meta(3 * (size_t)W, s);
        std::vector<int64_t> h(3 * (size_t)W, 0);
        h[3 * R] = at_blk->row0;
        h[3 * R + 1] = at_blk->ntr;
        h[3 * R + 2] = (int64_t)p->at->live_tiles;
        CK(cudaMemcpyAsync(meta.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
        ex->allreduce_sum_i64(meta.p, h.size(), s);
        CK(cudaMemcpyAsync(h.data(), meta.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        p->rows.resize(W + 1);
        for (int r = 0; r < W; r++) {
            if (h[3 * r] != (r ? (int64_t)p->rows[r] : 0))
                B2SR_THROW(B2SR_EINVAL, "row blocks must be contiguous and in rank order");
            p->rows[r] = (uint32_t)h[3 * r];
            p->rows[r + 1] = (uint32_t)(h[3 * r] + h[3 * r + 1]);
            p->live_tiles += (uint64_t)h[3 * r + 2];
        }
        if (p->rows[W] != p->ntr) B2SR_THROW(B2SR_EINVAL, "row blocks must cover every tile row");
        dist_layout(p);
        p->trp_a = copy_u32(trp_a, (size_t)p->ntr + 1, s);
        p->trp_at = copy_u32(trp_at, (size_t)p->ntr + 1, s);
        CK(cudaMemcpyAsync(&p->tiles_at, p->trp_at + p->ntr, 4, cudaMemcpyDeviceToHost, s));
        // global liveness: every block's words at its offset, then all-gathered
        p->live_at = dalloc(p->n16 * 16, s);
        CK(cudaMemsetAsync(p->live_at, 0, p->n16 * 16, s));
        const size_t own = (size_t)at_blk->ntr * word_bytes(p->dim);
        if (own) CK(cudaMemcpyAsync(static_cast<char *>(p->live_at) + p->off[R], p->at->live, own,
                                    cudaMemcpyDeviceToDevice, s));
        ex->allgatherv(p->live_at, p->off, p->len, s);
        CK(cudaStreamSynchronize(s));
        p->tiles_at &= 0xFFFFFFFFull;
    } catch (...) {
        p->a = p->at = nullptr;
        delete p;
        throw;
    }
    *out = p;
    API_END
}

int b2sr_dist_bfs_rows(const b2sr_dist_bfs *p, uint32_t *begin, uint32_t *end) {
    API_BEGIN
    *begin = p->rows[p->ex->rank];
    *end = p->rows[p->ex->rank + 1];
    API_END
}

int b2sr_dist_bfs_run(b2sr_dist_bfs *p, uint32_t src, double *d_levels, int64_t *iterations, void *stream) {
    API_BEGIN
    if (src >= p->n) B2SR_THROW(B2SR_EINVAL, "source vertex %u out of range for n=%u", src, p->n);
    if (p->dim == 4) dist_bfs_run<4>(p, src, d_levels, iterations, (cudaStream_t)stream);
    else dist_bfs_run<8>(p, src, d_levels, iterations, (cudaStream_t)stream);
    API_END
}

int b2sr_dist_bfs_free(b2sr_dist_bfs *p) {
    API_BEGIN
    if (p) {
        cudaDeviceSynchronize();
        delete p;
    }
    API_END
}

}  // extern "C"
