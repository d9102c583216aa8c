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
#include <functional>
#include <vector>

#include "bmv_common.cuh"

namespace b2sr {

constexpr uint32_t VSEG = 128;           // tiles per scatter unit (one warp, four rounds of 32)
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
    uint32_t *order = nullptr;     // n_rows * D vertices (row*D + r), fewest terms first
    uint32_t n_small = 0;          // the first n_small fold lane-per-vertex, the rest warp-per-vertex
    // rows are ordered longest first; the first top_rows rows' units
    // [0, top_units) are scattered first so their big vertices (big_top) can
    // start their long fold chains while everything else is still running
    uint32_t top_rows = 0, top_units = 0, n_big_top = 0, n_big_rest = 0;
    uint32_t *big_top = nullptr;   // big vertices of the top rows, fewest terms first
    uint32_t *big_rest = nullptr;  // the other big vertices, fewest terms first
};

constexpr uint32_t TOP_ROWS = 64;  // rows whose big vertices fold on the side stream first

constexpr uint32_t LANE_FOLD_MAX = 2048;  // terms: above, one warp folds the vertex

void free_vlong(void *p) {
    VLongPlan *v = static_cast<VLongPlan *>(p);
    if (!v) return;
    dfree(v->rows, nullptr);
    dfree(v->units, nullptr);
    dfree(v->unit_off, nullptr);
    dfree(v->base, nullptr);
    dfree(v->total, nullptr);
    dfree(v->terms, nullptr);
    dfree(v->order, nullptr);
    dfree(v->big_top, nullptr);
    dfree(v->big_rest, nullptr);
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

__global__ void k_vlong_order_keys(uint32_t nv, const uint32_t *__restrict__ total, uint32_t *__restrict__ key,
                                   uint32_t *__restrict__ val, uint32_t *__restrict__ n_small) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += gridDim.x * blockDim.x) {
        key[k] = total[k];
        val[k] = k;
        if (total[k] <= LANE_FOLD_MAX) atomicAdd(n_small, 1u);
    }
}

__global__ void k_vlong_len_keys(uint32_t nr, const uint32_t *__restrict__ rows, const uint32_t *__restrict__ trp,
                                 uint32_t *__restrict__ key) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x)
        key[i] = 0xFFFFFFFFu - (trp[rows[i] + 1] - trp[rows[i]]);
}

__global__ void k_vlong_nu(uint32_t nr, const uint32_t *__restrict__ rows, const uint32_t *__restrict__ trp,
                           uint32_t *__restrict__ nu) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x)
        nu[i] = (trp[rows[i] + 1] - trp[rows[i]] + VSEG - 1) / VSEG;
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
            {  // longest rows first (their hub vertices start folding first)
                Buf<uint32_t> key(nr, s);
                LAUNCH(k_vlong_len_keys, grid(nr), 256, 0, s, nr, rows.p, m->trp, key.p);
                uint32_t *ko, *vo;
                Buf<uint32_t> kalt, valt;
                radix_sort_pairs_u32(key.p, rows.p, nr, 32, s, &ko, &vo, &kalt, &valt);
                if (vo != rows.p) CK(cudaMemcpyAsync(rows.p, vo, (size_t)nr * 4, cudaMemcpyDeviceToDevice, s));
                LAUNCH(k_vlong_nu, grid(nr), 256, 0, s, nr, rows.p, m->trp, nu.p);
                CK(cudaStreamSynchronize(s));
            }
            exclusive_scan_u32_to_u64(nu.p, uofs.p, nr, s);
            v->top_rows = std::min<uint32_t>(nr, TOP_ROWS);
            v->top_units = (uint32_t)read_scalar(uofs.p + v->top_rows, s);
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
            {  // fold order: vertices sorted by term count
                const uint32_t nv = nr * D;
                Buf<uint32_t> key(nv, s), val(nv, s), nsm(1, s);
                CK(cudaMemsetAsync(nsm.p, 0, 4, s));
                LAUNCH(k_vlong_order_keys, grid(nv), 256, 0, s, nv, total.p, key.p, val.p, nsm.p);
                uint32_t *ko, *vo;
                Buf<uint32_t> kalt, valt;
                radix_sort_pairs_u32(key.p, val.p, nv, 32, s, &ko, &vo, &kalt, &valt);
                Buf<uint32_t> order(nv, s);
                CK(cudaMemcpyAsync(order.p, vo, (size_t)nv * 4, cudaMemcpyDeviceToDevice, s));
                v->n_small = read_scalar(nsm.p, s);
                // split the big vertices by row (host side: a few thousand entries)
                const uint32_t nb = nv - v->n_small;
                std::vector<uint32_t> big(nb), top, rest;
                if (nb) CK(cudaMemcpyAsync(big.data(), order.p + v->n_small, (size_t)nb * 4, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                for (uint32_t k : big) (k / D < v->top_rows ? top : rest).push_back(k);
                v->n_big_top = (uint32_t)top.size();
                v->n_big_rest = (uint32_t)rest.size();
                v->big_top = static_cast<uint32_t *>(dalloc(std::max<size_t>(top.size(), 1) * 4, s));
                v->big_rest = static_cast<uint32_t *>(dalloc(std::max<size_t>(rest.size(), 1) * 4, s));
                if (!top.empty()) CK(cudaMemcpyAsync(v->big_top, top.data(), top.size() * 4, cudaMemcpyHostToDevice, s));
                if (!rest.empty()) CK(cudaMemcpyAsync(v->big_rest, rest.data(), rest.size() * 4, cudaMemcpyHostToDevice, s));
                CK(cudaStreamSynchronize(s));
                v->order = order.release();
            }
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

// d = 4, 8: one warp per 128-tile unit, four rounds of one tile per lane.
// The per-bit-row term counts of a tile are packed into byte (d=4) or 16-bit
// (d=8) fields of one or two words, so a single shuffle scan gives every lane
// its output positions for all bit-rows at once; the running offsets of the
// unit's bit-rows live in registers.  Terms are the x values in reference
// order (tile, then column), written into each (row, bit-row) region.
template <int D>
__global__ void __launch_bounds__(256) k_vlong_scatter_w(uint32_t n_units, const uint4 *__restrict__ units,
                                                         const uint32_t *__restrict__ unit_off,
                                                         const uint64_t *__restrict__ base,
                                                         const uint32_t *__restrict__ tci,
                                                         const uint8_t *__restrict__ tiles,
                                                         const double *__restrict__ x, double *__restrict__ terms) {
    constexpr int NPW = D == 4 ? 1 : 4;       // packed count words
    constexpr int FPW = D == 4 ? 4 : 2;       // fields per word
    constexpr int FB = 32 / FPW;              // field bits
    const uint32_t lane = lane_id();
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n_units; u += warps) {
        const uint4 un = units[u];
        uint64_t off[D];
#pragma unroll
        for (int r = 0; r < D; r++) off[r] = base[(size_t)un.x * D + r] + unit_off[(size_t)u * D + r];
        for (uint32_t t = un.y + lane; t - lane < un.z; t += 32) {
            const bool ok = t < un.z;
            uint32_t rw[D];  // row words of this lane's tile
            uint32_t c = 0;
            if (ok) {
                c = __ldg(tci + t);
                if constexpr (D == 4) {
                    uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(tiles) + t);
#pragma unroll
                    for (int r = 0; r < 4; r++) rw[r] = (w >> (8 * r)) & 0xFFu;
                } else {
                    uint2 w = __ldg(reinterpret_cast<const uint2 *>(tiles) + t);
#pragma unroll
                    for (int r = 0; r < 8; r++) rw[r] = ((r < 4 ? w.x : w.y) >> (8 * (r & 3))) & 0xFFu;
                }
            } else {
#pragma unroll
                for (int r = 0; r < D; r++) rw[r] = 0;
            }
            uint32_t pk[NPW], inc[NPW];
#pragma unroll
            for (int q = 0; q < NPW; q++) pk[q] = 0;
#pragma unroll
            for (int r = 0; r < D; r++) pk[r / FPW] |= (uint32_t)__popc(rw[r]) << (FB * (r % FPW));
#pragma unroll
            for (int q = 0; q < NPW; q++) {
                inc[q] = pk[q];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t v = __shfl_up_sync(0xffffffffu, inc[q], o);
                    if (lane >= (uint32_t)o) inc[q] += v;
                }
            }
            const double *xs = x + (size_t)c * D;
#pragma unroll
            for (int r = 0; r < D; r++) {
                const uint32_t mask = FB == 32 ? 0xFFFFFFFFu : ((1u << FB) - 1u);
                const uint32_t incl = (inc[r / FPW] >> (FB * (r % FPW))) & mask;
                const uint32_t mine = (pk[r / FPW] >> (FB * (r % FPW))) & mask;
                uint32_t b = rw[r];
                double *dst = terms + off[r] + (incl - mine);
                while (b) {
                    int k = __ffs(b) - 1;
                    b &= b - 1;
                    *dst++ = __ldg(xs + k);
                }
                off[r] += __shfl_sync(0xffffffffu, incl, 31);  // the round's total for this bit-row
            }
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
    } else if constexpr (RING == RING_MIN_COMBINE) {
        return (cur < term || isnan(cur)) ? cur : term;
    } else {
        return (cur > term || isnan(cur)) ? cur : term;
    }
}

template <int D, int RING>
__device__ __forceinline__ void vlong_store(uint32_t k, double acc, double ident, const uint32_t *__restrict__ rows,
                                            uint32_t n, const void *__restrict__ keep, double *__restrict__ y,
                                            uint32_t row0) {
    const uint32_t I = rows[k / D], r = k % D, grow = row0 + I;
    if ((uint64_t)grow * D + r < n) {
        if (keep && !((load_word<D>(keep, grow) >> r) & 1u)) acc = ident;
        y[(size_t)I * D + r] = acc;
    }
}

// Vertices with few terms: one lane per vertex folds its region in order
// (kernels.py:195-207); 32 independent chains per warp, 16-byte loads two
// terms at a time, the next four already in flight.
template <int D, int RING>
__global__ void __launch_bounds__(256) k_vlong_fold_lanes(uint32_t n_small, const uint32_t *__restrict__ order,
                                                          const uint32_t *__restrict__ rows,
                                                          const uint64_t *__restrict__ base,
                                                          const uint32_t *__restrict__ total,
                                                          const double *__restrict__ terms, double inc, double ident, uint32_t n,
                                                          const void *__restrict__ keep, double *__restrict__ y,
                                                          uint32_t row0) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_small; i += gridDim.x * blockDim.x) {
        const uint32_t k = order[i];
        const uint64_t b0 = base[k];
        const uint32_t nt = total[k];
        const double *p = terms + b0;
        double acc = ident;
        uint32_t q = 0;
        if ((b0 & 1) && nt) acc = vring_op<RING>(acc, p[q++], inc);  // to a 16-byte boundary
        for (; q + 8 <= nt; q += 8) {
            const double2 *v = reinterpret_cast<const double2 *>(p + q);
            double2 a = __ldg(v), b = __ldg(v + 1), c = __ldg(v + 2), e = __ldg(v + 3);
            acc = vring_op<RING>(acc, a.x, inc); acc = vring_op<RING>(acc, a.y, inc);
            acc = vring_op<RING>(acc, b.x, inc); acc = vring_op<RING>(acc, b.y, inc);
            acc = vring_op<RING>(acc, c.x, inc); acc = vring_op<RING>(acc, c.y, inc);
            acc = vring_op<RING>(acc, e.x, inc); acc = vring_op<RING>(acc, e.y, inc);
        }
        for (; q < nt; q++) acc = vring_op<RING>(acc, p[q], inc);
        vlong_store<D, RING>(k, acc, ident, rows, n, keep, y, row0);
    }
}

// Vertices with many terms (the hubs): one warp per vertex.
//  * ARITHMETIC: the reference-order fold is a dependent chain of float64
//    adds (8 cycles each on B200, tools/micro_dadd.cu); lanes load 32
//    consecutive terms per step (coalesced, four steps ahead) into a per-warp
//    shared buffer and every lane applies them in order from broadcast 16-byte
//    reads, so the chain itself is the only serial part.
//  * MINPLUS / MAXTIMES: the reference's np.minimum / np.maximum step
//    f(cur, t) = (cur < t || isnan(cur)) ? cur : t (ties to the later term, the
//    first NaN sticks) is associative, so each lane folds one contiguous
//    segment and the segments are combined in order by a shuffle tree --
//    bit-identical to the sequential fold.
template <int D, int RING>
__global__ void __launch_bounds__(256) k_vlong_fold(uint32_t n_big, const uint32_t *__restrict__ order,
                                                    const uint32_t *__restrict__ rows,
                                                    const uint64_t *__restrict__ base,
                                                    const uint32_t *__restrict__ total,
                                                    const double *__restrict__ terms, double inc, double ident, uint32_t n,
                                                    const void *__restrict__ keep, double *__restrict__ y,
                                                    uint32_t row0) {
    __shared__ double2 sbuf[256 / 32][16];
const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_big; i += warps) {
        const uint32_t k = order[n_big - 1 - i];  // largest first: the longest chain starts at once
        const double *p = terms + base[k];
        const uint32_t nt = total[k];
        double acc = ident;
        if constexpr (RING == B2SR_RING_ARITHMETIC) {
            double c0 = lane < nt ? p[lane] : 0.0, c1 = 32 + lane < nt ? p[32 + lane] : 0.0;
            double c2 = 64 + lane < nt ? p[64 + lane] : 0.0, c3 = 96 + lane < nt ? p[96 + lane] : 0.0;
            double *sb = reinterpret_cast<double *>(sbuf[wid]);
            for (uint32_t q = 0; q < nt; q += 32) {
                if (q + 2048 + lane < nt)  // 16 KB ahead into L2: the region streams from HBM
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + q + 2048 + lane));
                double c4 = q + 128 + lane < nt ? p[q + 128 + lane] : 0.0;  // four steps ahead
                __syncwarp();
                sb[lane] = c0;
                __syncwarp();
                const uint32_t m = min(32u, nt - q);
                if (m == 32) {
                    // all 16 broadcast reads first, then the 32-add chain: the
                    // shared-memory latency is paid once per 32 terms, not per pair
                    double2 t[16];
#pragma unroll
                    for (int j = 0; j < 16; j++) t[j] = sbuf[wid][j];
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        acc = __dadd_rn(acc, t[j].x);
                        acc = __dadd_rn(acc, t[j].y);
                    }
                } else {
                    for (uint32_t j = 0; j < m; j++) acc = __dadd_rn(acc, sb[j]);
                }
                c0 = c1;
                c1 = c2;
                c2 = c3;
                c3 = c4;
            }
        } else {
            const uint32_t seg = (nt + 31) / 32, a = min(nt, lane * seg), b = min(nt, a + seg);
            uint32_t q = a;
            for (; q + 8 <= b; q += 8) {  // eight independent loads, then the ordered steps
                double t[8];
#pragma unroll
                for (int j = 0; j < 8; j++) t[j] = __ldg(p + q + j);
#pragma unroll
                for (int j = 0; j < 8; j++) acc = vring_op<RING>(acc, t[j], inc);
            }
            for (; q < b; q++) acc = vring_op<RING>(acc, p[q], inc);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {  // ordered combine: lane l's segments precede lane l+o's
                double other = __shfl_down_sync(0xffffffffu, acc, o);
                if (lane + o < 32) acc = vring_op<RING == B2SR_RING_MINPLUS ? RING_MIN_COMBINE : RING>(acc, other, 0.0);
            }
        }
        if (lane == 0) vlong_store<D, RING>(k, acc, ident, rows, n, keep, y, row0);
    }
}

// Side stream for the hub folds (one per device and host thread), so their
// long dependent chains overlap the rest of the sweep.
static cudaStream_t side_stream(int which = 0) {
    static thread_local cudaStream_t ss[1][16] = {};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev >= 16) return nullptr;
    if (!ss[which][dev]) CK(cudaStreamCreateWithFlags(&ss[which][dev], cudaStreamNonBlocking));
    return ss[which][dev];
}

// Scatter, then the folds; `overlap` runs while the hub folds proceed on the
// side stream (the main stream waits for them before returning).
void launch_vlong(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                  cudaStream_t s, const std::function<void(cudaStream_t)> &overlap, const uint32_t *gtci) {
    const uint32_t *tci = gtci ? gtci : m->tci;  // gather columns (relabelled with x, or the matrix's)
    VLongPlan *v = static_cast<VLongPlan *>(m->vlong);
    if (!v || !v->n_rows) {
        if (overlap) overlap(s);
        return;
    }
    auto scatter = [&](uint32_t u0, uint32_t u1) {  // units [u0, u1)
        if (u1 <= u0) return;
        const uint32_t nu = u1 - u0;
        unsigned gu = std::min<unsigned>(nu, (unsigned)num_sms() * 8);
        unsigned gw = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)nu + 7) / 8, (uint64_t)num_sms() * 16));
        const uint4 *un = v->units + u0;
        const uint32_t *uo = v->unit_off + (size_t)u0 * m->dim;
        switch (m->dim) {
            case 4: LAUNCH(k_vlong_scatter_w<4>, gw, 256, 0, s, nu, un, uo, v->base, tci, (const uint8_t *)m->tiles, x, v->terms); break;
            case 8: LAUNCH(k_vlong_scatter_w<8>, gw, 256, 0, s, nu, un, uo, v->base, tci, (const uint8_t *)m->tiles, x, v->terms); break;
            case 16: LAUNCH(k_vlong_scatter<16>, gu, VTHREADS, 0, s, nu, un, uo, v->base, tci, (const uint16_t *)m->tiles, x, v->terms); break;
            default: LAUNCH(k_vlong_scatter<32>, gu, VTHREADS, 0, s, nu, un, uo, v->base, tci, (const uint32_t *)m->tiles, x, v->terms); break;
        }
    };
    // 1. the top rows' terms, then their big vertices' chains on the side stream
    scatter(0, v->top_units);
    cudaStream_t s2 = v->n_big_top ? side_stream() : nullptr;
    cudaEvent_t e1 = nullptr, e2 = nullptr;
    const size_t top_smem = 160 * 1024;  // one fold warp per SM: its chain is the critical path
    if (s2) {
        CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamWaitEvent(s2, e1, 0));
    }
    // 2. the rest of the terms, the other big vertices, the small ones, then `overlap`
    const unsigned gr = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(((uint64_t)v->n_big_rest + 7) / 8, (uint64_t)num_sms() * 8));
    const unsigned gl = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((v->n_small + 255) / 256, (uint64_t)num_sms() * 8));
#define VL_RING(DD, RR)                                                                                             \
    do {                                                                                                            \
        if (s2) {                                                                                                   \
            hot_smem_attr(k_vlong_fold<DD, RR>, top_smem);                                                          \
            LAUNCH((k_vlong_fold<DD, RR>), std::min<uint32_t>(v->n_big_top, (uint32_t)num_sms()), 32, top_smem, s2, \
                   v->n_big_top, v->big_top, v->rows, v->base, v->total, v->terms, inc, ident, m->n, keep, y, m->row0);    \
        }                                                                                                           \
        scatter(v->top_units, v->n_units);                                                                          \
        if (v->n_big_rest)                                                                                          \
            LAUNCH((k_vlong_fold<DD, RR>), gr, 256, 0, s, v->n_big_rest, v->big_rest, v->rows, v->base, v->total,   \
                   v->terms, inc, ident, m->n, keep, y, m->row0);                                                          \
        if (v->n_small)                                                                                             \
            LAUNCH((k_vlong_fold_lanes<DD, RR>), gl, 256, 0, s, v->n_small, v->order, v->rows, v->base, v->total,   \
                   v->terms, inc, ident, m->n, keep, y, m->row0);                                                          \
    } while (0)
#define VL_DIM(DD)                                                                                                  \
    do {                                                                                                            \
        if (ring == B2SR_RING_ARITHMETIC) VL_RING(DD, B2SR_RING_ARITHMETIC);                                        \
        else if (ring == B2SR_RING_MINPLUS) VL_RING(DD, B2SR_RING_MINPLUS);                                         \
        else VL_RING(DD, B2SR_RING_MAXTIMES);                                                                       \
    } while (0)
    switch (m->dim) {
        case 4: VL_DIM(4); break;
        case 8: VL_DIM(8); break;
        case 16: VL_DIM(16); break;
        default: VL_DIM(32); break;
    }
#undef VL_DIM
#undef VL_RING
    // `overlap` (the short-row kernel) follows on the main stream: running it on
    // a third stream as well was measured slower (memory contention)
    if (overlap) overlap(s);
    if (s2) {
        CK(cudaEventRecord(e2, s2));
        CK(cudaStreamWaitEvent(s, e2, 0));
        cudaEventDestroy(e1);  // released once the recorded work completes
        cudaEventDestroy(e2);
    }
}

}  // namespace b2sr
