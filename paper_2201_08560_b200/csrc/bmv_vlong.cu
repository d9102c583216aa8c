// K6 for the very longest tile rows (R-MAT hubs, ~1e5 tiles per row at s24).
//
// The reference reduces every output element sequentially in ascending column
// order (kernels.py:195-207), so a hub row is an inherently serial chain of
// float64 adds.  What is NOT serial is finding its terms: here the row is cut
// into segments of VSEG tiles spread over many CTAs, each of which gathers its
// segment's x terms for every bit-row and writes them, compacted and in order,
// into a per-(row, bit-row) region of a global buffer.  One thread per
// (row, bit-row) then folds its region -- a pure dependent-add chain over
// contiguous memory, bit-identical to the reference.  The region layout only
// depends on the matrix's bits, so it is planned once and cached.
#include <vector>

#include "bmv_common.cuh"

namespace b2sr {

constexpr uint32_t VSEG = 2048;          // tiles per scatter unit
constexpr int VTHREADS = 256;

struct VLongPlan {
    uint32_t n_rows = 0, n_units = 0;
    uint64_t n_terms = 0;
    uint32_t *rows = nullptr;      // tile rows handled here
    uint4 *units = nullptr;        // (row index into rows, t0, t1, 0)
    uint32_t *unit_off = nullptr;  // n_units * D: first term of the unit inside its (row, r) region
    uint64_t *base = nullptr;      // n_rows * D: region starts
    uint32_t *total = nullptr;     // n_rows * D: region lengths
    double *terms = nullptr;       // n_terms
};

void free_vlong(void *p) {
    VLongPlan *v = static_cast<VLongPlan *>(p);
    if (!v) return;
    dfree(v->rows, nullptr);
    dfree(v->units, nullptr);
    dfree(v->unit_off, nullptr);
    dfree(v->base, nullptr);
    dfree(v->total, nullptr);
    dfree(v->terms, nullptr);
    delete v;
}

__global__ void k_vlong_flags(uint32_t ntr, const uint32_t *__restrict__ trp, uint32_t thresh, uint32_t *__restrict__ f) {
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x)
        f[I] = trp[I + 1] - trp[I] > thresh ? 1u : 0u;
}

// rows (ascending) and their unit counts
__global__ void k_vlong_rows(uint32_t ntr, const uint32_t *__restrict__ trp, const uint32_t *__restrict__ f,
                             const uint64_t *__restrict__ pos, uint32_t *__restrict__ rows, uint32_t *__restrict__ nu) {
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x)
        if (f[I]) {
            uint32_t i = (uint32_t)pos[I];
            rows[i] = I;
            nu[i] = (trp[I + 1] - trp[I] + VSEG - 1) / VSEG;
        }
}

__global__ void k_vlong_units(uint32_t nr, const uint32_t *__restrict__ rows, const uint32_t *__restrict__ trp,
                              const uint64_t *__restrict__ uofs, uint4 *__restrict__ units) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x) {
        uint32_t t0 = trp[rows[i]], t1 = trp[rows[i] + 1];
        uint64_t u = uofs[i];
        for (uint32_t t = t0; t < t1; t += VSEG, u++) units[u] = make_uint4(i, t, min(t1, t + VSEG), 0);
    }
}

// per (row, bit-row): offsets of its units inside the region, and the region length
template <int D>
__global__ void k_vlong_offsets(uint32_t nr, const uint64_t *__restrict__ uofs, const uint32_t *__restrict__ cnt,
                                uint32_t *__restrict__ unit_off, uint32_t *__restrict__ total) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nr * D; k += gridDim.x * blockDim.x) {
        uint32_t i = k / D, r = k % D, off = 0;
        for (uint64_t u = uofs[i]; u < uofs[i + 1]; u++) {
            unit_off[u * D + r] = off;
            off += cnt[u * D + r];
        }
        total[k] = off;
    }
}

// per (unit, bit-row) term counts
template <int D>
__global__ void __launch_bounds__(VTHREADS) k_vlong_counts(uint32_t n_units, const uint4 *__restrict__ units,
                                                           const typename WordT<D>::T *__restrict__ tiles,
                                                           uint32_t *__restrict__ cnt) {
    __shared__ uint32_t red[VTHREADS / 32][D];
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    for (uint32_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        uint4 un = units[u];
        uint32_t c[D];
#pragma unroll
        for (int r = 0; r < D; r++) c[r] = 0;
        for (uint32_t t = un.y + tid; t < un.z; t += blockDim.x)
#pragma unroll
            for (int r = 0; r < D; r++) c[r] += __popc((uint32_t)tiles[(size_t)t * D + r]);
#pragma unroll
        for (int r = 0; r < D; r++) {
            uint32_t v = __reduce_add_sync(0xffffffffu, c[r]);
            if (lane == 0) red[wid][r] = v;
        }
        __syncthreads();
        if (tid < (uint32_t)D) {
            uint32_t s = 0;
            for (int w = 0; w < VTHREADS / 32; w++) s += red[w][tid];
            cnt[(size_t)u * D + tid] = s;
        }
        __syncthreads();
    }
}

void *build_vlong(b2sr_matrix *m, uint32_t thresh, cudaStream_t s) {
    const uint32_t D = m->dim, ntr = m->ntr;
    VLongPlan *v = new VLongPlan();
    auto grid = [](uint64_t work) {
        return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)num_sms() * 16));
    };
    try {
        Buf<uint32_t> f(ntr, s);
        Buf<uint64_t> pos((size_t)ntr + 1, s);
        LAUNCH(k_vlong_flags, grid(ntr), 256, 0, s, ntr, m->trp, thresh, f.p);
        exclusive_scan_u32_to_u64(f.p, pos.p, ntr, s);
        const uint32_t nr = (uint32_t)read_scalar(pos.p + ntr, s);
        v->n_rows = nr;
        if (nr) {
            Buf<uint32_t> rows(nr, s), nu(nr, s);
            Buf<uint64_t> uofs((size_t)nr + 1, s);
            LAUNCH(k_vlong_rows, grid(ntr), 256, 0, s, ntr, m->trp, f.p, pos.p, rows.p, nu.p);
            exclusive_scan_u32_to_u64(nu.p, uofs.p, nr, s);
            v->n_units = (uint32_t)read_scalar(uofs.p + nr, s);
            Buf<uint4> units(v->n_units, s);
            LAUNCH(k_vlong_units, grid(nr), 256, 0, s, nr, rows.p, m->trp, uofs.p, units.p);
            Buf<uint32_t> cnt((size_t)v->n_units * D, s), unit_off((size_t)v->n_units * D, s), total((size_t)nr * D, s);
            unsigned gu = std::min<unsigned>(v->n_units, (unsigned)num_sms() * 8);
            switch (D) {
                case 4:
                    LAUNCH(k_vlong_counts<4>, gu, VTHREADS, 0, s, v->n_units, units.p, (const uint8_t *)m->tiles, cnt.p);
                    LAUNCH(k_vlong_offsets<4>, grid(nr * 4), 256, 0, s, nr, uofs.p, cnt.p, unit_off.p, total.p);
                    break;
                case 8:
                    LAUNCH(k_vlong_counts<8>, gu, VTHREADS, 0, s, v->n_units, units.p, (const uint8_t *)m->tiles, cnt.p);
                    LAUNCH(k_vlong_offsets<8>, grid(nr * 8), 256, 0, s, nr, uofs.p, cnt.p, unit_off.p, total.p);
                    break;
                case 16:
                    LAUNCH(k_vlong_counts<16>, gu, VTHREADS, 0, s, v->n_units, units.p, (const uint16_t *)m->tiles, cnt.p);
                    LAUNCH(k_vlong_offsets<16>, grid(nr * 16), 256, 0, s, nr, uofs.p, cnt.p, unit_off.p, total.p);
                    break;
                default:
                    LAUNCH(k_vlong_counts<32>, gu, VTHREADS, 0, s, v->n_units, units.p, (const uint32_t *)m->tiles, cnt.p);
                    LAUNCH(k_vlong_offsets<32>, grid(nr * 32), 256, 0, s, nr, uofs.p, cnt.p, unit_off.p, total.p);
                    break;
            }
            Buf<uint64_t> base((size_t)nr * D + 1, s);
            exclusive_scan_u32_to_u64(total.p, base.p, (size_t)nr * D, s);
            v->n_terms = read_scalar(base.p + (size_t)nr * D, s);
            v->terms = static_cast<double *>(dalloc(std::max<uint64_t>(v->n_terms, 1) * 8, s));
            v->rows = rows.release();
            v->units = units.release();
            v->unit_off = unit_off.release();
            v->base = base.release();
            v->total = total.release();
            CK(cudaStreamSynchronize(s));  // scratch buffers die here
        }
    } catch (...) {
        free_vlong(v);
        throw;
    }
    return v;
}

// scatter every unit's terms (x values in reference order) into the regions
template <int D>
__global__ void __launch_bounds__(VTHREADS) k_vlong_scatter(uint32_t n_units, const uint4 *__restrict__ units,
                                                            const uint32_t *__restrict__ unit_off,
                                                            const uint64_t *__restrict__ base,
                                                            const uint32_t *__restrict__ tci,
                                                            const typename WordT<D>::T *__restrict__ tiles,
                                                            const double *__restrict__ x, double *__restrict__ terms) {
    __shared__ uint32_t wsum[VTHREADS / 32][D];
    __shared__ uint32_t run_s[D];
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    for (uint32_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        uint4 un = units[u];
        if (tid < (uint32_t)D) run_s[tid] = unit_off[(size_t)u * D + tid];
        __syncthreads();
        for (uint32_t cb = un.y; cb < un.z; cb += VTHREADS) {
            uint32_t t = cb + tid;
            bool ok = t < un.z;
            uint32_t w[D];
            const double *xs = x;
#pragma unroll
            for (int r = 0; r < D; r++) w[r] = ok ? (uint32_t)tiles[(size_t)t * D + r] : 0u;
            if (ok) xs = x + (size_t)__ldg(tci + t) * D;
            uint32_t off[D];
#pragma unroll
            for (int r = 0; r < D; r++) {
                uint32_t c = __popc(w[r]), inc = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= (uint32_t)o) inc += y;
                }
                off[r] = inc - c;
                if (lane == 31) wsum[wid][r] = inc;
            }
            __syncthreads();
            if (tid < (uint32_t)D) {  // warp offsets, then advance the unit's running offset
                uint32_t r = tid, acc = run_s[r];
                for (int q = 0; q < VTHREADS / 32; q++) {
                    uint32_t v = wsum[q][r];
                    wsum[q][r] = acc;
                    acc += v;
                }
                run_s[r] = acc;
            }
            __syncthreads();
            if (ok) {
                uint32_t row = un.x;
#pragma unroll
                for (int r = 0; r < D; r++) {
                    uint32_t b = w[r];
                    if (!b) continue;
                    double *dst = terms + base[(size_t)row * D + r] + wsum[wid][r] + off[r];
                    while (b) {
                        int k = __ffs(b) - 1;
                        b &= b - 1;
                        *dst++ = __ldg(xs + k);
                    }
                }
            }
            __syncthreads();
        }
    }
}

// RING_MIN_COMBINE: the min-plus step without the increment (combining
// partial minima that already include it)
constexpr int RING_MIN_COMBINE = B2SR_RING_MAXTIMES + 1;

template <int RING>
__device__ __forceinline__ double vring_op(double cur, double term, double inc) {
    if constexpr (RING == B2SR_RING_ARITHMETIC) {
        return __dadd_rn(cur, term);
    } else if constexpr (RING == B2SR_RING_MINPLUS) {
        double t = __dadd_rn(term, inc);
        return (cur < t || isnan(cur)) ? cur : t;
    } else if constexpr (RING == RING_MIN_COMBINE) {
        return (cur < term || isnan(cur)) ? cur : term;
    } else {
        return (cur > term || isnan(cur)) ? cur : term;
    }
}

// One warp per (row, bit-row) over its contiguous term region.
//  * ARITHMETIC: the reference-order fold (kernels.py:195-207) is a dependent
//    chain of float64 adds (8 cycles each on B200); lanes keep four chunks of
//    32 terms in flight (coalesced) and every lane applies them in order from
//    shuffles, so the chain itself is the only serial part.
//  * MINPLUS / MAXTIMES: the reference's np.minimum / np.maximum step
//    f(cur, t) = (cur < t || isnan(cur)) ? cur : t (ties to the later term, the
//    first NaN sticks) is associative, so each lane folds one contiguous
//    segment and the segments are combined in order by a shuffle tree --
//    bit-identical to the sequential fold.
template <int D, int RING>
__global__ void __launch_bounds__(256) k_vlong_fold(uint32_t n_rows, const uint32_t *__restrict__ rows,
                                                    const uint64_t *__restrict__ base,
                                                    const uint32_t *__restrict__ total,
                                                    const double *__restrict__ terms, double inc, uint32_t n,
                                                    const void *__restrict__ keep, double *__restrict__ y,
                                                    uint32_t row0) {
    const double ident = RING == B2SR_RING_MINPLUS ? __longlong_as_double(0x7FF0000000000000ll) : 0.0;
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_rows * D; k += warps) {
        const uint32_t i = k / D, r = k % D, I = rows[i];
        const double *p = terms + base[k];
        const uint32_t nt = total[k];
        double acc = ident;
        if constexpr (RING == B2SR_RING_ARITHMETIC) {
            double c0 = lane < nt ? p[lane] : 0.0, c1 = 32 + lane < nt ? p[32 + lane] : 0.0;
            double c2 = 64 + lane < nt ? p[64 + lane] : 0.0, c3 = 96 + lane < nt ? p[96 + lane] : 0.0;
            for (uint32_t q = 0; q < nt; q += 32) {
                double c4 = q + 128 + lane < nt ? p[q + 128 + lane] : 0.0;  // four chunks ahead
                const uint32_t m = min(32u, nt - q);
                if (m == 32) {
#pragma unroll
                    for (int j0 = 0; j0 < 32; j0 += 8) {
                        double t[8];
#pragma unroll
                        for (int j = 0; j < 8; j++) t[j] = __shfl_sync(0xffffffffu, c0, j0 + j);
#pragma unroll
                        for (int j = 0; j < 8; j++) acc = __dadd_rn(acc, t[j]);
                    }
                } else {
                    for (uint32_t j = 0; j < m; j++) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, c0, j));
                }
                c0 = c1;
                c1 = c2;
                c2 = c3;
                c3 = c4;
            }
        } else {
            const uint32_t seg = (nt + 31) / 32, a = min(nt, lane * seg), b = min(nt, a + seg);
            for (uint32_t q = a; q < b; q++) acc = vring_op<RING>(acc, p[q], inc);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {  // ordered combine: lane l's segments precede lane l+o's
                double other = __shfl_down_sync(0xffffffffu, acc, o);
                if (lane + o < 32) acc = vring_op<RING == B2SR_RING_MINPLUS ? RING_MIN_COMBINE : RING>(acc, other, 0.0);
            }
        }
        if (lane == 0) {
            uint32_t grow = row0 + I;
            uint64_t vrow = (uint64_t)grow * D + r;
            if (vrow < n) {
                if (keep && !((load_word<D>(keep, grow) >> r) & 1u)) acc = ident;
                y[(size_t)I * D + r] = acc;
            }
        }
    }
}

void launch_vlong(b2sr_matrix *m, const double *x, int ring, double inc, const void *keep, double *y,
                  cudaStream_t s) {
    VLongPlan *v = static_cast<VLongPlan *>(m->vlong);
    if (!v || !v->n_rows) return;
    unsigned gu = std::min<unsigned>(v->n_units, (unsigned)num_sms() * 8);
    unsigned gf = (unsigned)std::min<uint64_t>(((uint64_t)v->n_rows * m->dim + 7) / 8, (uint64_t)num_sms() * 8);
#define VL_CASE(DD, W)                                                                                            \
    case DD:                                                                                                      \
        LAUNCH(k_vlong_scatter<DD>, gu, VTHREADS, 0, s, v->n_units, v->units, v->unit_off, v->base, m->tci,      \
               (const W *)m->tiles, x, v->terms);                                                                 \
        if (ring == B2SR_RING_ARITHMETIC)                                                                         \
            LAUNCH((k_vlong_fold<DD, B2SR_RING_ARITHMETIC>), gf, 256, 0, s, v->n_rows, v->rows, v->base, v->total, \
                   v->terms, inc, m->n, keep, y, m->row0);                                                        \
        else if (ring == B2SR_RING_MINPLUS)                                                                       \
            LAUNCH((k_vlong_fold<DD, B2SR_RING_MINPLUS>), gf, 256, 0, s, v->n_rows, v->rows, v->base, v->total,   \
                   v->terms, inc, m->n, keep, y, m->row0);                                                        \
        else                                                                                                      \
            LAUNCH((k_vlong_fold<DD, B2SR_RING_MAXTIMES>), gf, 256, 0, s, v->n_rows, v->rows, v->base, v->total,  \
                   v->terms, inc, m->n, keep, y, m->row0);                                                        \
        break;
    switch (m->dim) {
        VL_CASE(4, uint8_t)
        VL_CASE(8, uint8_t)
        VL_CASE(16, uint16_t)
        VL_CASE(32, uint32_t)
    }
#undef VL_CASE
}

}  // namespace b2sr
