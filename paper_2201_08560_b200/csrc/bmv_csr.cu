// K6 float gather for wide tiles (d = 16, 32): a per-matrix row plan.
//
// The reference folds each bit-row in ascending column order (kernels.py:
// 176-207: tiles ascending, bits ascending inside a tile row word) -- exactly
// the column order of the matrix's CSR form.  At d = 16/32 the tile walk of
// bmv_bff.cu gives each tile row to one warp, whose lanes (bit-rows) step
// through ~600 tiles of which ~95 % hold no bit of theirs (R-MAT s16 d=32:
// 2048 tile rows, 14 warps per SM, latency-bound at 0.44 ms).  Here the
// matrix's CSR column lists (b2sr_to_csr on the device, cached on the
// immutable matrix: 4 B per entry + 4 B per row) are the plan: one warp per
// row gathers 32 terms at a time in parallel and folds them in order with
// shuffles, so the sum is the reference's bit for bit while every row is in
// flight at once.  Full matrices only (row blocks keep the tile walk).
#include <vector>

#include "bmv_common.cuh"

extern "C" int b2sr_to_csr_rowptr(const b2sr_matrix *m, uint32_t *d_row_ptr, uint64_t *nnz, void *stream);
extern "C" int b2sr_to_csr_fill(const b2sr_matrix *m, const uint32_t *d_row_ptr, uint32_t *d_col_ind, void *stream);
extern "C" const char *b2sr_last_error(void);

namespace b2sr {

struct CsrPlan {
    uint32_t *rp = nullptr;     // n + 1
    uint32_t *ci = nullptr;     // nnz
    uint32_t *order = nullptr;  // rows, longest first: the hub rows' serial folds start at once
    uint64_t nnz = 0;
};

void free_csrplan(void *p) {
    CsrPlan *c = static_cast<CsrPlan *>(p);
    if (!c) return;
    dfree(c->rp, nullptr);
    dfree(c->ci, nullptr);
    dfree(c->order, nullptr);
    delete c;
}

// B2SR_BFF_CSR=0: wide tiles keep the tile walk (A/B)
bool bff_csr_enabled(const b2sr_matrix *m) {
    const char *e = getenv("B2SR_BFF_CSR");  // read per call: tests switch it; "all": d = 4, 8 too (A/B)
    const bool wide = m->dim >= 16 || (e && e[0] == 'a');
    return !(e && e[0] == '0') && wide && m->row0 == 0 && m->ntr == tile_rows(m->n, m->dim) && m->num_tiles;
}

__global__ void k_csr_len_keys(uint32_t n, const uint32_t *__restrict__ rp, uint32_t *__restrict__ key,
                               uint32_t *__restrict__ row) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        key[i] = 0xFFFFFFFFu - (rp[i + 1] - rp[i]);  // ascending key = descending length
        row[i] = i;
    }
}

static CsrPlan *csr_plan(b2sr_matrix *m, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (!m->csrplan) {
        CsrPlan *c = new CsrPlan();
        try {
            Buf<uint32_t> rp((size_t)m->n + 1, s);
            uint64_t nnz = 0;
            if (b2sr_to_csr_rowptr(m, rp.p, &nnz, s) != B2SR_OK) B2SR_THROW(B2SR_ECUDA, "%s", b2sr_last_error());
            Buf<uint32_t> ci(std::max<uint64_t>(nnz, 1), s);
            if (b2sr_to_csr_fill(m, rp.p, ci.p, s) != B2SR_OK) B2SR_THROW(B2SR_ECUDA, "%s", b2sr_last_error());
            const uint32_t n = m->n;
            Buf<uint32_t> key(n, s), row(n, s), kalt, valt;
            const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 16));
            LAUNCH(k_csr_len_keys, g, 256, 0, s, n, rp.p, key.p, row.p);
            uint32_t *ko = nullptr, *vo = nullptr;
            radix_sort_pairs_u32(key.p, row.p, n, 32, s, &ko, &vo, &kalt, &valt);
            Buf<uint32_t> order(n, s);
            CK(cudaMemcpyAsync(order.p, vo, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
            c->nnz = nnz;
            c->rp = rp.release();
            c->ci = ci.release();
            c->order = order.release();
        } catch (...) {
            free_csrplan(c);
            throw;
        }
        m->csrplan = c;
    }
    return static_cast<CsrPlan *>(m->csrplan);
}

template <int RING>
__device__ __forceinline__ double csr_op(double cur, double term, double inc) {
    if constexpr (RING == B2SR_RING_ARITHMETIC) {
        return __dadd_rn(cur, term);
    } else if constexpr (RING == B2SR_RING_MINPLUS) {
        const double t = __dadd_rn(term, inc);
        return (cur < t || isnan(cur)) ? cur : t;  // np.minimum
    } else {
        return (cur > term || isnan(cur)) ? cur : term;  // np.maximum
    }
}

// np.minimum / np.maximum step of the reference (NaN sticks, ties take the
// later term): associative, so an order-preserving tree gives its bits
template <int RING>
__device__ __forceinline__ double csr_pick(double a, double b) {
    if constexpr (RING == B2SR_RING_MINPLUS) return (a < b || isnan(a)) ? a : b;
    else return (a > b || isnan(a)) ? a : b;
}

#ifndef CSR_G
#define CSR_G 4  // s16 d=32: 4 -> 0.159 ms, 8 -> 0.187 ms (63 registers)
#endif
template <int D, int RING>
__global__ void __launch_bounds__(256) k_bff_csr(uint32_t n, const uint32_t *__restrict__ order,
                                                 const uint32_t *__restrict__ rp,
                                                 const uint32_t *__restrict__ ci, const double *__restrict__ x,
                                                 double inc, double ident, const void *__restrict__ keep,
                                                 double *__restrict__ y) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    constexpr int G = CSR_G;  // 32-term chunks in flight: a hub row's gathers overlap its fold
    __shared__ double2 csr_sbuf[8][16];  // per warp: one chunk of terms (ARITHMETIC)
    double *sb = reinterpret_cast<double *>(csr_sbuf[threadIdx.x >> 5]);
    const double2 *sbuf2 = csr_sbuf[threadIdx.x >> 5];
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
        const uint32_t i = __ldg(order + w);  // longest rows first
        const uint32_t a = __ldg(rp + i), b = __ldg(rp + i + 1);
        double acc = ident;
        double cur[G], nxt[G];
        auto fetch = [&](uint32_t base, double (&v)[G]) {
#pragma unroll
            for (int g = 0; g < G; g++) {
                const uint32_t k = base + 32 * g + lane;
                v[g] = k < b ? __ldg(x + __ldg(ci + k)) : 0.0;
            }
        };
        if (a < b) fetch(a, cur);
        for (uint32_t base = a; base < b; base += 32 * G) {
            if (base + 32 * G < b) fetch(base + 32 * G, nxt);
#pragma unroll
            for (int g = 0; g < G; g++) {
                const uint32_t cb = base + 32 * g;
                if (cb >= b) break;  // warp-uniform
                const uint32_t cnt = min(32u, b - cb);
                double v = cur[g];
                if constexpr (RING == B2SR_RING_ARITHMETIC) {
                    // the serial chain of the reference: the 32 terms go through
                    // shared memory and are read back as 16 broadcast 16-byte
                    // loads before the chain, so only the dependent adds are
                    // serial (a shuffle per term put its latency on the chain:
                    // ~30 instead of 8 cycles per term on a hub row)
                    __syncwarp();
                    sb[lane] = v;
                    __syncwarp();
                    if (cnt == 32) {
                        double2 t[16];
#pragma unroll
                        for (int q = 0; q < 16; q++) t[q] = sbuf2[q];
#pragma unroll
                        for (int q = 0; q < 16; q++) {
                            acc = __dadd_rn(acc, t[q].x);
                            acc = __dadd_rn(acc, t[q].y);
                        }
                    } else {
                        for (uint32_t q = 0; q < cnt; q++) acc = __dadd_rn(acc, sb[q]);
                    }
                } else {
                    if constexpr (RING == B2SR_RING_MINPLUS) v = __dadd_rn(v, inc);
                    bool has = lane < cnt;
#pragma unroll
                    for (uint32_t o = 1; o < 32; o <<= 1) {  // ordered tree: lane i takes lane i + o
                        const double w = __shfl_down_sync(0xffffffffu, v, o);
                        const bool hw = __shfl_down_sync(0xffffffffu, has, o) && lane + o < 32;
                        if ((lane & (2 * o - 1)) == 0 && hw) {
                            v = has ? csr_pick<RING>(v, w) : w;
                            has = true;
                        }
                    }
                    if (lane == 0) acc = csr_pick<RING>(acc, v);  // cnt >= 1: lane 0's term is valid
                }
            }
#pragma unroll
            for (int g = 0; g < G; g++) cur[g] = nxt[g];
        }
        if (lane == 0) {
            if (keep && !((load_word<D>(keep, i / D) >> (i % D)) & 1u)) acc = ident;
            y[i] = acc;
        }
    }
}

template <int D>
static void bff_csr_ring(const CsrPlan *c, uint32_t n, const double *x, int ring, double inc, double ident,
                         const void *keep, double *y, cudaStream_t s) {
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)n + 7) / 8, (uint64_t)num_sms() * 8));
    if (ring == B2SR_RING_ARITHMETIC)
        LAUNCH((k_bff_csr<D, B2SR_RING_ARITHMETIC>), g, 256, 0, s, n, c->order, c->rp, c->ci, x, inc, ident, keep, y);
    else if (ring == B2SR_RING_MINPLUS)
        LAUNCH((k_bff_csr<D, B2SR_RING_MINPLUS>), g, 256, 0, s, n, c->order, c->rp, c->ci, x, inc, ident, keep, y);
    else
        LAUNCH((k_bff_csr<D, B2SR_RING_MAXTIMES>), g, 256, 0, s, n, c->order, c->rp, c->ci, x, inc, ident, keep, y);
}

void launch_bff_csr(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                    cudaStream_t s) {
    const CsrPlan *c = csr_plan(m, s);
    switch (m->dim) {
        case 4: bff_csr_ring<4>(c, m->n, x, ring, inc, ident, keep, y, s); break;
        case 8: bff_csr_ring<8>(c, m->n, x, ring, inc, ident, keep, y, s); break;
        case 16: bff_csr_ring<16>(c, m->n, x, ring, inc, ident, keep, y, s); break;
        default: bff_csr_ring<32>(c, m->n, x, ring, inc, ident, keep, y, s); break;
    }
}

}  // namespace b2sr
