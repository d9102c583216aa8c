// K6 float gather for the tile rows below the segmented-plan threshold
// (replaces kernels.py:140-216 for those rows; bmv_vlong.cu takes the hubs).
//
// A group of d lanes per tile row, lane = bit-row, walks the row's tiles in
// ascending order and, inside a tile, the set bits in ascending column order:
// the reference's reduction order, so ARITHMETIC is bit-identical and the
// min/max rings keep numpy's NaN / tie behaviour (bff_op below).
//
// What makes it fast is keeping the loads independent of the fold:
//   * four tiles per step, fetched as 16-byte vectors (d=4: the four tile
//     words; d=8: two vectors) plus one 16-byte load of their columns;
//   * the first set bit of each tile row word is gathered unconditionally
//     (predicated on the word), so a step issues its four x gathers at once --
//     R-MAT tiles carry ~1 bit, further bits take a short loop;
//   * a three-stage register pipeline: the tiles/columns of step s+2 and the
//     gathers of step s+1 are in flight while step s is folded;
//   * rows are visited in descending length order (a per-matrix plan), so the
//     groups of a warp walk rows of similar length.
#include "bmv_common.cuh"

namespace b2sr {

constexpr int BFF_THREADS = 256;

struct BffPlan {
    uint32_t n_rows = 0;
    uint32_t *rows = nullptr;  // rows with <= thresh tiles, longest first
};

void free_bff(void *p) {
    BffPlan *b = static_cast<BffPlan *>(p);
    if (!b) return;
    dfree(b->rows, nullptr);
    delete b;
}

__global__ void k_bff_keys(uint32_t ntr, const uint32_t *__restrict__ trp, uint32_t thresh, uint32_t *__restrict__ key,
                           uint32_t *__restrict__ row, uint32_t *__restrict__ count) {
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x) {
        uint32_t len = trp[I + 1] - trp[I];
        key[I] = len <= thresh ? thresh - len : 0xFFFFFFFFu;  // longest first; excluded rows sort last
        row[I] = I;
        if (len <= thresh) atomicAdd(count, 1u);
    }
}

static BffPlan *bff_plan(b2sr_matrix *m, uint32_t thresh, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (!m->bff) {
        BffPlan *b = new BffPlan();
        try {
            const uint32_t ntr = m->ntr;
            Buf<uint32_t> key(ntr, s), row(ntr, s), cnt(1, s);
            CK(cudaMemsetAsync(cnt.p, 0, 4, s));
            unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ntr + 255) / 256, (uint64_t)num_sms() * 16));
            LAUNCH(k_bff_keys, g, 256, 0, s, ntr, m->trp, thresh, key.p, row.p, cnt.p);
            uint32_t *ko, *vo;
            Buf<uint32_t> kalt, valt;
            radix_sort_pairs_u32(key.p, row.p, ntr, 32, s, &ko, &vo, &kalt, &valt);
            b->n_rows = read_scalar(cnt.p, s);
            Buf<uint32_t> rows(std::max<uint32_t>(b->n_rows, 1), s);
            if (b->n_rows) CK(cudaMemcpyAsync(rows.p, vo, (size_t)b->n_rows * 4, cudaMemcpyDeviceToDevice, s));
            b->rows = rows.release();
            CK(cudaStreamSynchronize(s));
        } catch (...) {
            free_bff(b);
            throw;
        }
        m->bff = b;
    }
    return static_cast<BffPlan *>(m->bff);
}

template <int RING>
__device__ __forceinline__ double bff_op(double cur, double term, double inc) {
    if constexpr (RING == B2SR_RING_ARITHMETIC) {
        return __dadd_rn(cur, term);
    } else if constexpr (RING == B2SR_RING_MINPLUS) {
        double t = __dadd_rn(term, inc);
        return (cur < t || isnan(cur)) ? cur : t;  // np.minimum
    } else {
        return (cur > term || isnan(cur)) ? cur : term;  // np.maximum
    }
}

// One step: the row words of this lane's bit-row in 4 tiles, their columns,
// and the x value of each word's lowest set bit.
struct BffStep {
    uint32_t w[4], c[4];
    double v[4];
};

template <int D>
__device__ __forceinline__ void bff_load(const uint8_t *__restrict__ tiles, const uint32_t *__restrict__ tci,
                                         uint32_t b, uint32_t t0, uint32_t t1, uint32_t r, BffStep &st) {
    using W = typename WordT<D>::T;
    if (b >= t1) {
#pragma unroll
        for (int j = 0; j < 4; j++) st.w[j] = 0, st.c[j] = 0;
        return;
    }
    uint4 q = ld_stream128(tci + b);  // b % 4 == 0: 16-byte aligned
    st.c[0] = q.x; st.c[1] = q.y; st.c[2] = q.z; st.c[3] = q.w;
    uint32_t w[4];
    if constexpr (D == 4) {
        uint4 t = ld_stream128(tiles + (size_t)b * 4);
        w[0] = (t.x >> (8 * r)) & 0xFFu; w[1] = (t.y >> (8 * r)) & 0xFFu;
        w[2] = (t.z >> (8 * r)) & 0xFFu; w[3] = (t.w >> (8 * r)) & 0xFFu;
    } else if constexpr (D == 8) {
        uint4 a = ld_stream128(tiles + (size_t)b * 8);
        uint4 e = b + 2 < t1 ? ld_stream128(tiles + (size_t)b * 8 + 16) : make_uint4(0, 0, 0, 0);
        uint32_t sh = 8 * (r & 3);
        w[0] = ((r < 4 ? a.x : a.y) >> sh) & 0xFFu; w[1] = ((r < 4 ? a.z : a.w) >> sh) & 0xFFu;
        w[2] = ((r < 4 ? e.x : e.y) >> sh) & 0xFFu; w[3] = ((r < 4 ? e.z : e.w) >> sh) & 0xFFu;
    } else {
        const W *tw = reinterpret_cast<const W *>(tiles);
#pragma unroll
        for (int j = 0; j < 4; j++) w[j] = b + j < t1 ? (uint32_t)tw[(size_t)(b + j) * D + r] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 4; j++) st.w[j] = (b + j >= t0 && b + j < t1) ? w[j] : 0u;
}

template <int D>
__device__ __forceinline__ void bff_gather(const double *__restrict__ x, BffStep &st) {
#pragma unroll
    for (int j = 0; j < 4; j++)
        st.v[j] = st.w[j] ? __ldg(x + (size_t)st.c[j] * D + (__ffs(st.w[j]) - 1)) : 0.0;
}

template <int D, int RING>
__device__ __forceinline__ double bff_fold(const double *__restrict__ x, const BffStep &st, double acc, double inc) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
        uint32_t w = st.w[j];
        if (!w) continue;
        acc = bff_op<RING>(acc, st.v[j], inc);
        w &= w - 1;
        const double *xs = x + (size_t)st.c[j] * D;
        while (w) {  // further bits of the same tile row word (rare on R-MAT)
            int k = __ffs(w) - 1;
            w &= w - 1;
            acc = bff_op<RING>(acc, __ldg(xs + k), inc);
        }
    }
    return acc;
}

template <int D, int RING>
__global__ void __launch_bounds__(BFF_THREADS, 4) k_bff_rows(uint32_t n_rows, const uint32_t *__restrict__ rows, uint32_t n,
                                                         const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                                                         const uint8_t *__restrict__ tiles, const double *__restrict__ x,
                                                         double inc, double ident, const void *__restrict__ keep,
                                                         double *__restrict__ y, uint32_t row0) {
    constexpr uint32_t GPW = 32 / D;
    const uint32_t lane = lane_id(), r = lane % D;
    const uint32_t groups = ((gridDim.x * blockDim.x) >> 5) * GPW;
    for (uint32_t i = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * GPW + lane / D; i < n_rows; i += groups) {
        const uint32_t I = rows[i];
        const uint32_t t0 = trp[I], t1 = trp[I + 1];
        double acc = ident;
        uint32_t b = t0 & ~3u;
        BffStep s0, s1;
        bff_load<D>(tiles, tci, b, t0, t1, r, s0);
        bff_gather<D>(x, s0);
        for (; b < t1; b += 8) {
            bff_load<D>(tiles, tci, b + 4, t0, t1, r, s1);
            acc = bff_fold<D, RING>(x, s0, acc, inc);
            if (b + 4 >= t1) break;
            bff_gather<D>(x, s1);
            bff_load<D>(tiles, tci, b + 8, t0, t1, r, s0);
            acc = bff_fold<D, RING>(x, s1, acc, inc);
            if (b + 8 >= t1) break;
            bff_gather<D>(x, s0);
        }
        const uint32_t grow = row0 + I;
        const uint64_t vrow = (uint64_t)grow * D + r;
        if (vrow < n) {
            if (keep && !((load_word<D>(keep, grow) >> r) & 1u)) acc = ident;
            y[(size_t)I * D + r] = acc;
        }
    }
}

template <int D>
static void bff_rows_ring(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                          uint32_t thresh, cudaStream_t s, const uint32_t *gtci) {
    BffPlan *p = static_cast<BffPlan *>(m->bff);  // built by a plan_only call on the caller's stream
    if (!p || !p->n_rows) return;
    constexpr uint32_t GPW = 32 / D;
    uint64_t warps = ((uint64_t)p->n_rows + GPW - 1) / GPW;
    unsigned g = (unsigned)std::min<uint64_t>((warps + BFF_THREADS / 32 - 1) / (BFF_THREADS / 32),
                                              (uint64_t)num_sms() * 8);
    const uint8_t *tl = (const uint8_t *)m->tiles;
    if (ring == B2SR_RING_ARITHMETIC)
        LAUNCH((k_bff_rows<D, B2SR_RING_ARITHMETIC>), g, BFF_THREADS, 0, s, p->n_rows, p->rows, m->n, m->trp, gtci, tl,
               x, inc, ident, keep, y, m->row0);
    else if (ring == B2SR_RING_MINPLUS)
        LAUNCH((k_bff_rows<D, B2SR_RING_MINPLUS>), g, BFF_THREADS, 0, s, p->n_rows, p->rows, m->n, m->trp, gtci, tl,
               x, inc, ident, keep, y, m->row0);
    else
        LAUNCH((k_bff_rows<D, B2SR_RING_MAXTIMES>), g, BFF_THREADS, 0, s, p->n_rows, p->rows, m->n, m->trp, gtci, tl,
               x, inc, ident, keep, y, m->row0);
}

void launch_bff_rows(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                     uint32_t thresh, cudaStream_t s, bool plan_only, const uint32_t *gtci) {
    bff_plan(m, thresh, s);
    if (plan_only) return;
    if (!gtci) gtci = m->tci;
    switch (m->dim) {
        case 4: bff_rows_ring<4>(m, x, ring, inc, ident, keep, y, thresh, s, gtci); break;
        case 8: bff_rows_ring<8>(m, x, ring, inc, ident, keep, y, thresh, s, gtci); break;
        case 16: bff_rows_ring<16>(m, x, ring, inc, ident, keep, y, thresh, s, gtci); break;
        default: bff_rows_ring<32>(m, x, ring, inc, ident, keep, y, thresh, s, gtci); break;
    }
}

}  // namespace b2sr
