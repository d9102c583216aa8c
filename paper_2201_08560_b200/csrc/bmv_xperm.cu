// Hot-first relabelling of the x vector for the float gather (K6).
//
// At R-MAT s24 the x vector of a float gather (134 MB) is larger than L2, and
// K6 is DRAM-bound on x misses (9.9 GB per sweep in k_bff_rows alone).  At
// d = 4 one tile column's D values are exactly one 32-byte sector, but the
// hot columns are spread over the whole vector, so every cached 128-byte line
// holds one hot sector next to three cold ones and L2 keeps a quarter of the
// hot set it could.  The plan below ranks the tile columns by tile count,
// stores x' = x with column c moved to slot rank[c] (one coalesced pass per
// sweep), and gives the gather kernels tci_p[t] = rank[tci[t]] in place of
// tci.  Only the gather addresses change: tiles are still walked in the
// matrix's order, so every row folds its terms in the reference's order and
// the results are bit-identical.  (s24 PageRank sweep: 7.78 -> 7.02 ms,
// k_bff_rows DRAM reads 9.9 -> 7.5 GB; an L2 access-policy window marking the
// head of x' persisting on top of this measured no better.)
#include "b2sr_internal.cuh"

namespace b2sr {

struct XPerm {
    uint32_t ncols = 0;
    uint32_t *rank = nullptr;   // tile column -> slot in x'
    uint32_t *tci_p = nullptr;  // rank[tci[t]] per tile
};

void free_xperm(void *p) {
    XPerm *x = static_cast<XPerm *>(p);
    if (!x) return;
    dfree(x->rank, nullptr);
    dfree(x->tci_p, nullptr);
    delete x;
}

static unsigned xgrid(uint64_t work) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)num_sms() * 16));
}

__global__ void k_xp_hist(uint64_t T, const uint32_t *__restrict__ tci, uint32_t *__restrict__ cnt) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + tci[t], 1u);
}

__global__ void k_xp_keys(uint32_t ncols, const uint32_t *__restrict__ cnt, uint32_t *__restrict__ key,
                          uint32_t *__restrict__ col) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        key[c] = ~cnt[c];  // ascending sort = most tiles first (stable: ties by column)
        col[c] = c;
    }
}

__global__ void k_xp_rank(uint32_t ncols, const uint32_t *__restrict__ order, uint32_t *__restrict__ rank) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncols; i += gridDim.x * blockDim.x) rank[order[i]] = i;
}

__global__ void k_xp_tci(uint64_t T, const uint32_t *__restrict__ tci, const uint32_t *__restrict__ rank,
                         uint32_t *__restrict__ tci_p) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x)
        tci_p[t] = rank[tci[t]];
}

// x'[rank[c]*D + b] = x[c*D + b] (x has n entries; the tail of the last
// column reads as 0.0 and is never gathered: no tile bit lies past n)
template <int D>
__global__ void k_xp_permute(uint32_t ncols, uint32_t n, const uint32_t *__restrict__ rank,
                             const double *__restrict__ x, double *__restrict__ xp) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const size_t src = (size_t)c * D, dst = (size_t)rank[c] * D;
        if (src + D <= n) {
#pragma unroll
            for (int b = 0; b < D; b += 2)
                *reinterpret_cast<double2 *>(xp + dst + b) = __ldg(reinterpret_cast<const double2 *>(x + src + b));
        } else {
            for (int b = 0; b < D; b++) xp[dst + b] = src + b < n ? x[src + b] : 0.0;
        }
    }
}

// float32 copy for the fast PageRank gather: x'[rank[c]*D + b] = (float)x[c*D + b]
template <int D>
__global__ void k_xp_permute_f32(uint32_t ncols, uint32_t n, const uint32_t *__restrict__ rank,
                                 const double *__restrict__ x, float *__restrict__ xp) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const size_t src = (size_t)c * D, dst = (size_t)rank[c] * D;
#pragma unroll
        for (int b = 0; b < D; b++) xp[dst + b] = src + b < n ? __double2float_rn(__ldg(x + src + b)) : 0.0f;
    }
}

// u32 vectors (CC labels): lab'[rank[c]*D + b] = lab[c*D + b]
template <int D>
__global__ void k_xp_permute_u32(uint32_t ncols, uint32_t n, const uint32_t *__restrict__ rank,
                                 const uint32_t *__restrict__ x, uint32_t *__restrict__ xp) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const size_t src = (size_t)c * D, dst = (size_t)rank[c] * D;
        for (int b = 0; b < D; b++) xp[dst + b] = src + b < n ? __ldg(x + src + b) : 0xFFFFFFFFu;
    }
}

// Relabel when x' would not stay L2-resident anyway (B2SR_XPERM=1 / 0 forces).
bool xperm_enabled(const b2sr_matrix *m) {
    const char *e = getenv("B2SR_XPERM");
    if (e) return e[0] == '1';
    const uint64_t xbytes = (uint64_t)tile_rows(m->n, m->dim) * m->dim * sizeof(double);
    return m->num_tiles && xbytes > ((uint64_t)64 << 20);
}

static XPerm *xperm_plan(b2sr_matrix *m, cudaStream_t s) {
    B2SR_PLAN_LOCK(m);
    if (!m->xperm) {
        XPerm *p = new XPerm();
        try {
            const uint32_t ncols = tile_rows(m->n, m->dim);
            const uint64_t T = m->num_tiles;
            p->ncols = ncols;
            Buf<uint32_t> cnt(ncols, s), key(ncols, s), col(ncols, s), rank(ncols, s), tci_p(T, s);
            CK(cudaMemsetAsync(cnt.p, 0, (size_t)ncols * 4, s));
            LAUNCH(k_xp_hist, xgrid(T), 256, 0, s, T, m->tci, cnt.p);
            LAUNCH(k_xp_keys, xgrid(ncols), 256, 0, s, ncols, cnt.p, key.p, col.p);
            uint32_t *ko, *vo;
            Buf<uint32_t> kalt, valt;
            radix_sort_pairs_u32(key.p, col.p, ncols, 32, s, &ko, &vo, &kalt, &valt);
            LAUNCH(k_xp_rank, xgrid(ncols), 256, 0, s, ncols, vo, rank.p);
            LAUNCH(k_xp_tci, xgrid(T), 256, 0, s, T, m->tci, rank.p, tci_p.p);
            CK(cudaStreamSynchronize(s));  // the sort's scratch buffers die here
            p->rank = rank.release();
            p->tci_p = tci_p.release();
        } catch (...) {
            free_xperm(p);
            throw;
        }
        m->xperm = p;
    }
    return static_cast<XPerm *>(m->xperm);
}

// x' into xp (ncols * dim doubles); returns the gather column array to use
const uint32_t *xperm_apply(b2sr_matrix *m, const double *x, double *xp, cudaStream_t s) {
    XPerm *p = xperm_plan(m, s);
    switch (m->dim) {
        case 4: LAUNCH(k_xp_permute<4>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp); break;
        case 8: LAUNCH(k_xp_permute<8>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp); break;
        case 16: LAUNCH(k_xp_permute<16>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp); break;
        default: LAUNCH(k_xp_permute<32>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp); break;
    }
    return p->tci_p;
}

const uint32_t *xperm_apply_u32(b2sr_matrix *m, const uint32_t *x, uint32_t *xp, cudaStream_t s) {
    XPerm *p = xperm_plan(m, s);
    if (m->dim == 4) LAUNCH(k_xp_permute_u32<4>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp);
    else LAUNCH(k_xp_permute_u32<8>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp);
    return p->tci_p;
}

// float32 x' for the fast PageRank gather (d = 4, 8); returns the gather column array
const uint32_t *xperm_apply_f32(b2sr_matrix *m, const double *x, float *xp, cudaStream_t s) {
    XPerm *p = xperm_plan(m, s);
    if (m->dim == 4) LAUNCH(k_xp_permute_f32<4>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp);
    else LAUNCH(k_xp_permute_f32<8>, xgrid(p->ncols), 256, 0, s, p->ncols, m->n, p->rank, x, xp);
    return p->tci_p;
}

}  // namespace b2sr
