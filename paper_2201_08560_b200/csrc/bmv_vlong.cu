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

__global__ void k_find_vlong(uint32_t ntr, const uint32_t *trp, uint32_t thresh, uint32_t *rows, uint32_t *count) {
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < ntr; I += gridDim.x * blockDim.x)
        if (trp[I + 1] - trp[I] > thresh) rows[atomicAdd(count, 1u)] = I;
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
    try {
        Buf<uint32_t> rows(ntr, s), cnt1(1, s);
        CK(cudaMemsetAsync(cnt1.p, 0, 4, s));
        unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ntr + 255) / 256, (uint64_t)num_sms() * 16));
        LAUNCH(k_find_vlong, g, 256, 0, s, ntr, m->trp, thresh, rows.p, cnt1.p);
        uint32_t nr = read_scalar(cnt1.p, s);
        v->n_rows = nr;
        if (nr) {
            std::vector<uint32_t> h_rows(nr), h_t0(nr), h_t1(nr);
            CK(cudaMemcpyAsync(h_rows.data(), rows.p, nr * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (uint32_t i = 0; i < nr; i++) {
                CK(cudaMemcpyAsync(&h_t0[i], m->trp + h_rows[i], 4, cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(&h_t1[i], m->trp + h_rows[i] + 1, 4, cudaMemcpyDeviceToHost, s));
            }
            CK(cudaStreamSynchronize(s));
            std::vector<uint4> h_units;
            for (uint32_t i = 0; i < nr; i++)
                for (uint32_t t = h_t0[i]; t < h_t1[i]; t += VSEG)
                    h_units.push_back(make_uint4(i, t, std::min(h_t1[i], t + VSEG), 0));
            v->n_units = (uint32_t)h_units.size();
            v->rows = static_cast<uint32_t *>(dalloc(nr * 4, s));
            v->units = static_cast<uint4 *>(dalloc(h_units.size() * 16, s));
            CK(cudaMemcpyAsync(v->rows, h_rows.data(), nr * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(v->units, h_units.data(), h_units.size() * 16, cudaMemcpyHostToDevice, s));
            Buf<uint32_t> cnt((size_t)v->n_units * D, s);
            unsigned gu = std::min<unsigned>(v->n_units, (unsigned)num_sms() * 8);
            switch (D) {
                case 4: LAUNCH(k_vlong_counts<4>, gu, VTHREADS, 0, s, v->n_units, v->units, (const uint8_t *)m->tiles, cnt.p); break;
                case 8: LAUNCH(k_vlong_counts<8>, gu, VTHREADS, 0, s, v->n_units, v->units, (const uint8_t *)m->tiles, cnt.p); break;
                case 16: LAUNCH(k_vlong_counts<16>, gu, VTHREADS, 0, s, v->n_units, v->units, (const uint16_t *)m->tiles, cnt.p); break;
                default: LAUNCH(k_vlong_counts<32>, gu, VTHREADS, 0, s, v->n_units, v->units, (const uint32_t *)m->tiles, cnt.p); break;
            }
            std::vector<uint32_t> h_cnt((size_t)v->n_units * D), h_off((size_t)v->n_units * D), h_tot((size_t)nr * D, 0);
            CK(cudaMemcpyAsync(h_cnt.data(), cnt.p, h_cnt.size() * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (uint32_t u = 0; u < v->n_units; u++)  // units of a row are consecutive, in tile order
                for (uint32_t r = 0; r < D; r++) {
                    uint32_t row = h_units[u].x;
                    h_off[(size_t)u * D + r] = h_tot[(size_t)row * D + r];
                    h_tot[(size_t)row * D + r] += h_cnt[(size_t)u * D + r];
                }
            std::vector<uint64_t> h_base((size_t)nr * D);
            uint64_t run = 0;
            for (size_t k = 0; k < h_base.size(); k++) {
                h_base[k] = run;
                run += h_tot[k];
            }
            v->n_terms = run;
            v->unit_off = static_cast<uint32_t *>(dalloc(h_off.size() * 4, s));
            v->base = static_cast<uint64_t *>(dalloc(h_base.size() * 8, s));
            v->total = static_cast<uint32_t *>(dalloc(h_tot.size() * 4, s));
            v->terms = static_cast<double *>(dalloc(std::max<uint64_t>(run, 1) * 8, s));
            CK(cudaMemcpyAsync(v->unit_off, h_off.data(), h_off.size() * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(v->base, h_base.data(), h_base.size() * 8, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(v->total, h_tot.data(), h_tot.size() * 4, cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));  // host vectors die here
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

template <int RING>
__device__ __forceinline__ double vring_op(double cur, double term, double inc) {
    if constexpr (RING == B2SR_RING_ARITHMETIC) {
        return __dadd_rn(cur, term);
    } else if constexpr (RING == B2SR_RING_MINPLUS) {
        double t = __dadd_rn(term, inc);
        return (cur < t || isnan(cur)) ? cur : t;
    } else {
        return (cur > term || isnan(cur)) ? cur : term;
    }
}

// one thread per (row, bit-row): the reference-order fold
template <int D, int RING>
__global__ void k_vlong_fold(uint32_t n_rows, const uint32_t *__restrict__ rows, const uint64_t *__restrict__ base,
                             const uint32_t *__restrict__ total, const double *__restrict__ terms, double inc, uint32_t n,
                             const void *__restrict__ keep, double *__restrict__ y, uint32_t row0) {
    const double ident = RING == B2SR_RING_MINPLUS ? __longlong_as_double(0x7FF0000000000000ll) : 0.0;
    uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_rows * D) return;
    uint32_t i = k / D, r = k % D, I = rows[i];
    const double *p = terms + base[k];
    uint32_t nt = total[k];
    double acc = ident;
    uint32_t q = 0;
    for (; q + 4 <= nt; q += 4) {  // loads batched ahead of the dependent adds
        double a = p[q], b = p[q + 1], c = p[q + 2], d = p[q + 3];
        acc = vring_op<RING>(acc, a, inc);
        acc = vring_op<RING>(acc, b, inc);
        acc = vring_op<RING>(acc, c, inc);
        acc = vring_op<RING>(acc, d, inc);
    }
    for (; q < nt; q++) acc = vring_op<RING>(acc, p[q], inc);
    uint32_t grow = row0 + I;
    uint64_t vrow = (uint64_t)grow * D + r;
    if (vrow < n) {
        if (keep && !((load_word<D>(keep, grow) >> r) & 1u)) acc = ident;
        y[(size_t)I * D + r] = acc;
    }
}

void launch_vlong(b2sr_matrix *m, const double *x, int ring, double inc, const void *keep, double *y,
                  cudaStream_t s) {
    VLongPlan *v = static_cast<VLongPlan *>(m->vlong);
    if (!v || !v->n_rows) return;
    unsigned gu = std::min<unsigned>(v->n_units, (unsigned)num_sms() * 8);
    unsigned gf = (v->n_rows * m->dim + 127) / 128;
#define VL_CASE(DD, W)                                                                                            \
    case DD:                                                                                                      \
        LAUNCH(k_vlong_scatter<DD>, gu, VTHREADS, 0, s, v->n_units, v->units, v->unit_off, v->base, m->tci,      \
               (const W *)m->tiles, x, v->terms);                                                                 \
        if (ring == B2SR_RING_ARITHMETIC)                                                                         \
            LAUNCH((k_vlong_fold<DD, B2SR_RING_ARITHMETIC>), gf, 128, 0, s, v->n_rows, v->rows, v->base, v->total, \
                   v->terms, inc, m->n, keep, y, m->row0);                                                        \
        else if (ring == B2SR_RING_MINPLUS)                                                                       \
            LAUNCH((k_vlong_fold<DD, B2SR_RING_MINPLUS>), gf, 128, 0, s, v->n_rows, v->rows, v->base, v->total,   \
                   v->terms, inc, m->n, keep, y, m->row0);                                                        \
        else                                                                                                      \
            LAUNCH((k_vlong_fold<DD, B2SR_RING_MAXTIMES>), gf, 128, 0, s, v->n_rows, v->rows, v->base, v->total,  \
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
