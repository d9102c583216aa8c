// Column-strip blocked bin-SpMV (bbb and the BFS pull sweep).
//
// Why: in the row-major B2SR stream every tile gathers its x word at a random
// column.  ncu on k_bmv_bbb<4> at R-MAT s22 (profiles/r01_ncu_*): L1tex
// throughput 71 % of peak, 167 M L1 sectors for a 1.03 GB matrix -- each
// 32-lane gather costs 32 L1 wavefronts, which caps d=4/8 at ~2 TB/s no
// matter how the tiles are streamed.  Shared memory serves the same random
// gather in a few wavefronts.
//
// Plan (built once per matrix, cached on the handle):
//   * tile columns are cut into P strips of STRIP_VERTS vertices whose x
//     bits (128 KB) fit in shared memory;
//   * tiles are re-laid strip-major (strip p = every row's column-sorted
//     tiles that fall in strip p, row after row) -- same bytes, new order;
//   * per strip, a work-item list of (row, tile range) chunks of at most
//     ITEM_STEPS group steps (hub rows split);
//   * CTAs are assigned to strips in proportion to the strip's tiles.
// Kernel: one 1024-thread CTA per SM stages its strip's x bits with a TMA
// bulk copy (cp.async.bulk + mbarrier), then groups of GS lanes walk the
// strip's items with 128-bit streaming loads and gather x from shared memory.
// No CTA barrier after the staging.  Each item ORs its hits into y with one
// atomicOr (OR is order-free: bit-identical to the reference).
#include <vector>

#include "bmv_common.cuh"

namespace b2sr {

constexpr uint32_t STRIP_VERTS = 1u << 20;        // vertices per strip
constexpr uint32_t STRIP_SMEM = STRIP_VERTS / 8;  // 128 KB of x bits
constexpr uint32_t MAX_STRIPS = 16;
constexpr int BLK_THREADS = 1024;
constexpr uint32_t ITEM_STEPS = 8;                // group steps per work item

template <int D> struct GroupSize { static constexpr int GS = D <= 8 ? 8 : (D == 16 ? 16 : 32); };
template <int D> constexpr uint32_t tiles_step() {
    return GroupSize<D>::GS * Geo<D>::TPL / Geo<D>::LPT;
}

struct BlockedPlan {
    uint32_t P = 1, strip_cols = 1, n_items = 0, n_ctas = 0;
    uint32_t *seg = nullptr;          // P x (ntr+1) tile offsets (strip-major)
    uint32_t *tci = nullptr;          // strip-major tile columns
    void *tiles = nullptr;            // strip-major tiles
    uint4 *items = nullptr;           // (row, t0, t1, 0) per strip, strip-major
    uint32_t *strip_items = nullptr;  // P+1 item offsets per strip (device)
    uint32_t *strip_ctas = nullptr;   // P+1 CTA offsets per strip (device)
    bool owns = false;                // false when P == 1 (tile arrays alias the matrix)
};

void free_plan(void *p) {
    BlockedPlan *bp = static_cast<BlockedPlan *>(p);
    if (!bp) return;
    if (bp->owns) {
        dfree(bp->tci, nullptr);
        dfree(bp->tiles, nullptr);
    }
    dfree(bp->seg, nullptr);
    dfree(bp->items, nullptr);
    dfree(bp->strip_items, nullptr);
    dfree(bp->strip_ctas, nullptr);
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

// items per (strip, row): ceil(len / chunk), strip-major
__global__ void k_plan_item_counts(uint32_t ntr, uint32_t P, uint32_t chunk, const uint32_t *seg, uint32_t *cnt) {
    size_t total = (size_t)P * ntr;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        size_t p = i / ntr, I = i % ntr;
        uint32_t len = seg[p * (ntr + 1) + I + 1] - seg[p * (ntr + 1) + I];
        cnt[i] = (len + chunk - 1) / chunk;
    }
}

__global__ void k_plan_item_fill(uint32_t ntr, uint32_t P, uint32_t chunk, const uint32_t *seg, const uint64_t *ofs,
                                 uint4 *items) {
    size_t total = (size_t)P * ntr;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        size_t p = i / ntr, I = i % ntr;
        uint32_t s0 = seg[p * (ntr + 1) + I], s1 = seg[p * (ntr + 1) + I + 1];
        uint64_t o = ofs[i];
        for (uint32_t t = s0; t < s1; t += chunk) items[o++] = make_uint4((uint32_t)I, t, min(s1, t + chunk), 0);
    }
}

BlockedPlan *ensure_plan(b2sr_matrix *m, cudaStream_t s) {
    if (m->plan) return static_cast<BlockedPlan *>(m->plan);
    uint32_t d = m->dim, ntr = m->ntr;
    uint32_t ncols = tile_rows(m->n, d);  // global tile columns
    uint32_t sc = STRIP_VERTS / d;        // tile columns per strip
    uint32_t P = (ncols + sc - 1) / sc;
    if (P > MAX_STRIPS) return nullptr;   // too many strips: the row-major kernel is used
    uint32_t chunk = ITEM_STEPS * (d == 4 ? tiles_step<4>() : d == 8 ? tiles_step<8>()
                                   : d == 16 ? tiles_step<16>() : tiles_step<32>());
    BlockedPlan *bp = new BlockedPlan();
    try {
        bp->P = P;
        bp->strip_cols = sc;
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
        // work items per strip
        Buf<uint32_t> icnt((size_t)P * ntr, s);
        Buf<uint64_t> iofs((size_t)P * ntr + 1, s);
        LAUNCH(k_plan_item_counts, grid_for((uint64_t)P * ntr), 256, 0, s, ntr, P, chunk, bp->seg, icnt.p);
        exclusive_scan_u32_to_u64(icnt.p, iofs.p, (size_t)P * ntr, s);
        std::vector<uint64_t> h_iofs(P + 1);
        std::vector<uint32_t> h_seg_end(P);
        for (uint32_t p = 0; p <= P; p++)
            CK(cudaMemcpyAsync(&h_iofs[p], iofs.p + (size_t)p * ntr, 8, cudaMemcpyDeviceToHost, s));
        for (uint32_t p = 0; p < P; p++)
            CK(cudaMemcpyAsync(&h_seg_end[p], bp->seg + (size_t)p * (ntr + 1) + ntr, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        bp->n_items = (uint32_t)h_iofs[P];
        bp->items = static_cast<uint4 *>(dalloc((size_t)bp->n_items * 16 + 16, s));
        LAUNCH(k_plan_item_fill, grid_for((uint64_t)P * ntr), 256, 0, s, ntr, P, chunk, bp->seg, iofs.p, bp->items);
        // CTAs per strip in proportion to the strip's tiles (at least one each)
        uint32_t G = (uint32_t)num_sms();
        std::vector<uint32_t> h_items(P + 1), h_ctas(P + 1, 0);
        uint64_t prev_end = 0, T = m->num_tiles ? m->num_tiles : 1, assigned = 0;
        for (uint32_t p = 0; p < P; p++) {
            uint64_t tiles_p = h_seg_end[p] - prev_end;
            prev_end = h_seg_end[p];
            h_items[p] = (uint32_t)h_iofs[p];
            h_ctas[p] = (uint32_t)assigned;
            assigned += std::max<uint64_t>(1, (tiles_p * G + T / 2) / T);
        }
        h_items[P] = (uint32_t)h_iofs[P];
        h_ctas[P] = (uint32_t)assigned;
        bp->n_ctas = (uint32_t)assigned;
        bp->strip_items = static_cast<uint32_t *>(dalloc((P + 1) * 4, s));
        bp->strip_ctas = static_cast<uint32_t *>(dalloc((P + 1) * 4, s));
        CK(cudaMemcpyAsync(bp->strip_items, h_items.data(), (P + 1) * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(bp->strip_ctas, h_ctas.data(), (P + 1) * 4, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // host vectors die here
    } catch (...) {
        free_plan(bp);
        throw;
    }
    m->plan = bp;
    return bp;
}

// ------------------------------------------------------------ x bit packing
// d=4 BitVector words are bytes with a low nibble; pack 8 of them per u32 so
// every width hands the kernel a plain little-endian bitset
__global__ void k_pack_nibbles(uint32_t nwords, const uint8_t *__restrict__ x, uint32_t *__restrict__ bits) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += gridDim.x * blockDim.x) {
        uint2 v = reinterpret_cast<const uint2 *>(x)[i];
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            o |= ((v.x >> (8 * j)) & 0xFu) << (4 * j);
            o |= ((v.y >> (8 * j)) & 0xFu) << (16 + 4 * j);
        }
        bits[i] = o;
    }
}

// ------------------------------------------------------------ TMA staging
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Bulk-copy `bytes` (multiple of 16) from global to shared memory with the
// TMA bulk path; completion is tracked by an mbarrier (transaction bytes).
__device__ __forceinline__ void tma_stage(void *dst, const void *src, uint32_t bytes, uint64_t *mbar) {
    uint32_t mb = smem_addr(mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        const uint32_t CH = 32768;
        for (uint32_t off = 0; off < bytes; off += CH) {
            uint32_t len = min(CH, bytes - off);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr((char *)dst + off)),
                "l"((const char *)src + off), "r"(len), "r"(mb)
                : "memory");
        }
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra WAIT_%=;\n}" ::"r"(
            mb)
        : "memory");
}

// ------------------------------------------------------------ kernel
template <int D, int MODE>
__device__ __forceinline__ uint32_t seg_step(const uint32_t *__restrict__ tci, const uint8_t *__restrict__ tiles,
                                             const uint32_t *xs, uint32_t c0, uint32_t base, uint32_t s0, uint32_t s1,
                                             uint32_t gl, uint32_t lane) {
    using G = Geo<D>;
    constexpr uint32_t xmask = D == 32 ? 0xffffffffu : ((1u << D) - 1u);
    uint32_t xw[G::TPL];
    uint4 v = make_uint4(0, 0, 0, 0);
    if constexpr (G::TPL > 1) {
        uint32_t tl = base + gl * G::TPL;
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
            uint32_t anyx = 0;
            if (MODE == 0) v = ld_stream128(tiles + (size_t)tl * G::TB);
#pragma unroll
            for (int j = 0; j < G::TPL; j++) {
                bool ok = tl + j >= s0 && tl + j < s1;
                uint32_t bit = (cols[j] - c0) * D;
                xw[j] = ok ? (xs[bit >> 5] >> (bit & 31)) & xmask : 0u;
                anyx |= xw[j];
            }
            if (MODE == 1 && anyx) v = ld_stream128(tiles + (size_t)tl * G::TB);
        }
    } else {
        uint32_t t = base + gl / G::LPT, q = gl % G::LPT;
        xw[0] = 0;
        if (t < s1) {
            if (MODE == 0) v = ld_stream128(tiles + (size_t)t * G::TB + q * 16);
            uint32_t bit = (__ldg(tci + t) - c0) * D;
            xw[0] = (xs[bit >> 5] >> (bit & 31)) & xmask;
            if (MODE == 1 && xw[0]) v = ld_stream128(tiles + (size_t)t * G::TB + q * 16);
        }
    }
    return hits16<D>(v, xw, lane);
}

// MODE 0: y = (A x) & keep (keep may be null);  MODE 1: BFS pull,
// next = (A frontier) & ~visited & live, payload skipping + early exit.
// xbits is the little-endian bitset of x (vertex v = bit v).
template <int D, int MODE>
__global__ void __launch_bounds__(BLK_THREADS, 1)
k_blocked(uint32_t P, uint32_t sc, uint32_t nbits_bytes, uint32_t row0, const uint4 *__restrict__ items,
          const uint32_t *__restrict__ strip_items, const uint32_t *__restrict__ strip_ctas,
          const uint32_t *__restrict__ tci, const uint8_t *__restrict__ tiles, const uint8_t *__restrict__ xbits,
          const void *__restrict__ keep, const void *__restrict__ live, void *__restrict__ y) {
    constexpr int GS = GroupSize<D>::GS;
    constexpr uint32_t TILES_STEP = tiles_step<D>();
    extern __shared__ __align__(128) uint32_t xs[];
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t lane = lane_id();
    const uint32_t gl = threadIdx.x % GS;
    const uint32_t gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1u) << (lane & ~(GS - 1u)));
    // this CTA's strip
    uint32_t p = 0;
    while (p + 1 < P && strip_ctas[p + 1] <= blockIdx.x) p++;
    const uint32_t lcta = blockIdx.x - strip_ctas[p], ncta = strip_ctas[p + 1] - strip_ctas[p];
    // stage x bits of vertices [p*STRIP_VERTS, (p+1)*STRIP_VERTS)
    uint32_t b0 = p * STRIP_SMEM;
    uint32_t bytes = min(STRIP_SMEM, nbits_bytes - b0);
    bytes = (bytes + 15) & ~15u;
    tma_stage(xs, xbits + b0, bytes, &mbar);
    const uint32_t c0 = p * sc;
    const uint32_t groups = ncta * (blockDim.x / GS);
    const uint32_t gid = lcta * (blockDim.x / GS) + threadIdx.x / GS;
    const uint32_t i1 = strip_items[p + 1];
    for (uint32_t k = strip_items[p] + gid; k < i1; k += groups) {
        uint4 it = items[k];
        uint32_t I = it.x, s0 = it.y, s1 = it.z;
        uint32_t grow = row0 + I;
        uint32_t keepw;
        if constexpr (MODE == 1) {
            keepw = ~load_word<D>(keep, grow) & load_word<D>(live, I);
            if (!keepw) continue;
        } else {
            keepw = keep ? load_word<D>(keep, grow) : 0xffffffffu;
        }
        uint32_t acc = 0;
        uint32_t base = Geo<D>::TPL > 1 ? (s0 & ~(uint32_t)(Geo<D>::TPL - 1)) : s0;
        for (; base < s1; base += TILES_STEP) {
            acc |= seg_step<D, MODE>(tci, tiles, xs, c0, base, s0, s1, gl, lane);
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
}

bool blocked_enabled() {
    // opt-in: measured 1.42 TB/s vs 1.55 TB/s for the row-major stream at
    // s22 d=4 (profiles/r01_ab_blocked.txt) -- kept as an experiment
    const char *e = getenv("B2SR_BLOCKED");
    return e && e[0] == '1';
}

// Returns false when the matrix has too many strips for the blocked path.
bool launch_blocked(b2sr_matrix *m, int mode, const void *x, const void *keep, void *y, cudaStream_t s) {
    BlockedPlan *bp = ensure_plan(m, s);
    if (!bp) return false;
    CK(cudaMemsetAsync(y, 0, padded_vec_bytes(m->ntr, m->dim), s));
    uint32_t ncols = tile_rows(m->n, m->dim);
    uint32_t nbits_bytes = (uint32_t)(((uint64_t)ncols * m->dim + 7) / 8);
    const uint8_t *xbits = (const uint8_t *)x;
    Buf<uint32_t> packed;
    if (m->dim == 4) {  // nibble words -> bitset
        uint32_t nwords = (ncols + 7) / 8;
        packed = Buf<uint32_t>(nwords + 4, s);
        LAUNCH(k_pack_nibbles, grid_for(nwords), 256, 0, s, nwords, (const uint8_t *)x, packed.p);
        xbits = (const uint8_t *)packed.p;
    }
    unsigned g = bp->n_ctas;
    size_t smem = STRIP_SMEM;
    const uint8_t *tl = (const uint8_t *)bp->tiles;
#define BLK_CASE(DD)                                                                                             \
    case DD:                                                                                                     \
        if (mode == 0) {                                                                                         \
            CK(cudaFuncSetAttribute(k_blocked<DD, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
            LAUNCH((k_blocked<DD, 0>), g, BLK_THREADS, smem, s, bp->P, bp->strip_cols, nbits_bytes, m->row0,     \
                   bp->items, bp->strip_items, bp->strip_ctas, bp->tci, tl, xbits, keep, (const void *)nullptr,  \
                   y);                                                                                           \
        } else {                                                                                                 \
            CK(cudaFuncSetAttribute(k_blocked<DD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
            LAUNCH((k_blocked<DD, 1>), g, BLK_THREADS, smem, s, bp->P, bp->strip_cols, nbits_bytes, m->row0,     \
                   bp->items, bp->strip_items, bp->strip_ctas, bp->tci, tl, xbits, keep,                         \
                   (const void *)m->live, y);                                                                    \
        }                                                                                                        \
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
