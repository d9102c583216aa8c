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
    uint32_t *rp = nullptr;  // n + 1
    uint32_t *ci = nullptr;  // nnz
    uint64_t nnz = 0;
};

void free_csrplan(void *p) {
    CsrPlan *c = static_cast<CsrPlan *>(p);
    if (!c) return;
    dfree(c->rp, nullptr);
    dfree(c->ci, nullptr);
    delete c;
}

// B2SR_BFF_CSR=0: wide tiles keep the tile walk (A/B)
bool bff_csr_enabled(const b2sr_matrix *m) {
    const char *e = getenv("B2SR_BFF_CSR");  // read per call: tests switch it
    return !(e && e[0] == '0') && m->dim >= 16 && m->row0 == 0 && m->ntr == tile_rows(m->n, m->dim) && m->num_tiles;
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
            c->nnz = nnz;
            c->rp = rp.release();
            c->ci = ci.release();
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
__global__ void __launch_bounds__(256) k_bff_csr(uint32_t n, const uint32_t *__restrict__ rp,
                                                 const uint32_t *__restrict__ ci, const double *__restrict__ x,
                                                 double inc, double ident, const void *__restrict__ keep,
                                                 double *__restrict__ y) {
    const uint32_t lane = lane_id(), warps = (gridDim.x * blockDim.x) >> 5;
    constexpr int G = CSR_G;  // 32-term chunks in flight: a hub row's gathers overlap its fold
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
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
                    // the serial chain of the reference: the shuffles are independent
                    // of acc, so unrolled they issue ahead of the dependent adds
#pragma unroll
                    for (uint32_t j = 0; j < 32; j++) {
                        const double t = __shfl_sync(0xffffffffu, v, j);
                        if (j < cnt) acc = __dadd_rn(acc, t);
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
        LAUNCH((k_bff_csr<D, B2SR_RING_ARITHMETIC>), g, 256, 0, s, n, c->rp, c->ci, x, inc, ident, keep, y);
    else if (ring == B2SR_RING_MINPLUS)
        LAUNCH((k_bff_csr<D, B2SR_RING_MINPLUS>), g, 256, 0, s, n, c->rp, c->ci, x, inc, ident, keep, y);
    else
        LAUNCH((k_bff_csr<D, B2SR_RING_MAXTIMES>), g, 256, 0, s, n, c->rp, c->ci, x, inc, ident, keep, y);
}

void launch_bff_csr(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                    cudaStream_t s) {
    const CsrPlan *c = csr_plan(m, s);
    if (m->dim == 16) bff_csr_ring<16>(c, m->n, x, ring, inc, ident, keep, y, s);
    else bff_csr_ring<32>(c, m->n, x, ring, inc, ident, keep, y, s);
}

}  // namespace b2sr
