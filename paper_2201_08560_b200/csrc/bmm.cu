// K7/K8: bin-SpGEMM reductions (replaces kernels.py:271-367).
//
// bmm_bin_bin_sum: sum_ij (A B)_ij = sum_k colsum_A(k) * rowdeg_B(k), an
// O(T) pass (the reference's per-pair colpop*rowpop sum regrouped by k;
// integer arithmetic, so the regrouping is exact).
//
// bmm_bin_bin_sum_masked with B supplied transposed (Bt): for every stored
// mask tile (I,J) the tile columns of A's row I and Bt's row J are
// intersected, and each common K contributes, for every mask bit (r,c),
// popc(A_IK[r] & Bt_JK[c]) == sum_k A[i,k] B[k,j] inside the tile pair.
// One warp per mask tile: lanes take 32 entries of the shorter tile row and
// binary-search them in the longer one; AND+POPC on the integer pipe (b1
// MMA has no native sm_100a path -- SURVEY.md §0).  Triangle counting is
// the instance A = Bt = M = L (transpose(transpose(L)) == L).
#include "b2sr_internal.cuh"

namespace b2sr {

template <int D>
__global__ void k_colsum_rowdeg(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                                const typename WordT<D>::T *__restrict__ tiles, uint32_t *__restrict__ colsum,
                                uint32_t *__restrict__ rowdeg) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t I = rowid[t], K = tci[t];
#pragma unroll
        for (int r = 0; r < D; r++) {
            uint32_t w = tiles[t * D + r];
            if (rowdeg && w) atomicAdd(rowdeg + (size_t)I * D + r, (uint32_t)__popc(w));
            if (colsum) {
                while (w) {
                    int c = __ffs(w) - 1;
                    w &= w - 1;
                    atomicAdd(colsum + (size_t)K * D + c, 1u);
                }
            }
        }
    }
}

__global__ void k_dot_u32(size_t n, const uint32_t *a, const uint32_t *b, unsigned long long *out) {
    unsigned long long acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += (unsigned long long)a[i] * b[i];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

static unsigned grid_for(uint64_t work) {
    uint64_t b = (work + 255) / 256, cap = (uint64_t)num_sms() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

static void row_ids(const b2sr_matrix *m, uint32_t *rowid, cudaStream_t s) { launch_row_ids(m, rowid, s); }

static void colsum_rowdeg(const b2sr_matrix *m, uint32_t *colsum, uint32_t *rowdeg, cudaStream_t s) {
    if (!m->num_tiles) return;
    Buf<uint32_t> rowid(m->num_tiles, s);
    row_ids(m, rowid.p, s);
    unsigned g = grid_for(m->num_tiles);
    switch (m->dim) {
        case 4: LAUNCH(k_colsum_rowdeg<4>, g, 256, 0, s, m->num_tiles, rowid.p, m->tci, (const uint8_t *)m->tiles, colsum, rowdeg); break;
        case 8: LAUNCH(k_colsum_rowdeg<8>, g, 256, 0, s, m->num_tiles, rowid.p, m->tci, (const uint8_t *)m->tiles, colsum, rowdeg); break;
        case 16: LAUNCH(k_colsum_rowdeg<16>, g, 256, 0, s, m->num_tiles, rowid.p, m->tci, (const uint16_t *)m->tiles, colsum, rowdeg); break;
        default: LAUNCH(k_colsum_rowdeg<32>, g, 256, 0, s, m->num_tiles, rowid.p, m->tci, (const uint32_t *)m->tiles, colsum, rowdeg); break;
    }
}

// ------------------------------------------------------------ masked
// lower_bound of `key` in v[lo, hi)
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *__restrict__ v, uint32_t lo, uint32_t hi, uint32_t key) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(v + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <int D>
__global__ void __launch_bounds__(256) k_bmm_masked(uint64_t TM, const uint32_t *__restrict__ m_rowid,
                                                    const uint32_t *__restrict__ m_tci,
                                                    const typename WordT<D>::T *__restrict__ m_tiles,
                                                    const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci,
                                                    const typename WordT<D>::T *__restrict__ a_tiles,
                                                    const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
                                                    const typename WordT<D>::T *__restrict__ b_tiles,
                                                    uint32_t m_row0, unsigned long long *__restrict__ out) {
    const uint32_t lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0;
    for (uint64_t mt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; mt < TM; mt += warps) {
        uint32_t I = m_rowid[mt] + m_row0, J = m_tci[mt];
        uint32_t mword = lane < (uint32_t)D ? (uint32_t)m_tiles[mt * D + lane] : 0u;
        uint32_t rows_used = __ballot_sync(0xffffffffu, mword != 0);  // bit r: mask row r non-empty
        uint32_t a0 = a_trp[I], a1 = a_trp[I + 1], b0 = b_trp[J], b1 = b_trp[J + 1];
        if (a0 == a1 || b0 == b1 || rows_used == 0) continue;
        // iterate the shorter tile row, search the longer one
        bool a_short = (a1 - a0) <= (b1 - b0);
        uint32_t s0 = a_short ? a0 : b0, s1 = a_short ? a1 : b1;
        uint32_t l0 = a_short ? b0 : a0, l1 = a_short ? b1 : a1;
        const uint32_t *stci = a_short ? a_tci : b_tci;
        const uint32_t *ltci = a_short ? b_tci : a_tci;
        for (uint32_t base = s0; base < s1; base += 32) {
            uint32_t si = base + lane;
            uint32_t ta = 0, tb = 0;
            bool hit = false;
            if (si < s1) {
                uint32_t K = __ldg(stci + si);
                uint32_t li = lower_bound_u32(ltci, l0, l1, K);
                if (li < l1 && __ldg(ltci + li) == K) {
                    hit = true;
                    ta = a_short ? si : li;
                    tb = a_short ? li : si;
                }
            }
            uint32_t hits = __ballot_sync(0xffffffffu, hit);
            if (!hits) continue;
            uint32_t ru = rows_used;
            while (ru) {  // warp-uniform loop over non-empty mask rows
                int r = __ffs(ru) - 1;
                ru &= ru - 1;
                uint32_t mw = __shfl_sync(0xffffffffu, mword, r);
                if (hit) {
                    uint32_t aw = a_tiles[(size_t)ta * D + r];
                    if (aw) {
                        while (mw) {
                            int c = __ffs(mw) - 1;
                            mw &= mw - 1;
                            acc += __popc(aw & (uint32_t)b_tiles[(size_t)tb * D + c]);
                        }
                    }
                }
            }
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
}

// ------------------------------------------------------------ chunked items
// A mask tile whose two tile rows are both long (hub x hub) would pin one
// warp for milliseconds; split every mask tile into chunks of TC_CHUNK
// entries of its shorter tile row so such pairs spread over many warps.
constexpr uint32_t TC_CHUNK = 256;

__global__ void k_tc_item_counts(uint64_t TM, const uint32_t *__restrict__ m_rowid, const uint32_t *__restrict__ m_tci,
                                 uint32_t m_row0, const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ b_trp,
                                 uint32_t *__restrict__ cnt) {
    for (uint64_t mt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; mt < TM; mt += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t I = m_rowid[mt] + m_row0, J = m_tci[mt];
        uint32_t la = a_trp[I + 1] - a_trp[I], lb = b_trp[J + 1] - b_trp[J];
        uint32_t sh = min(la, lb);
        cnt[mt] = la && lb ? (sh + TC_CHUNK - 1) / TC_CHUNK : 0;
    }
}

__global__ void k_tc_item_fill(uint64_t TM, const uint32_t *__restrict__ cnt, const uint64_t *__restrict__ ofs,
                               uint2 *__restrict__ items) {
    for (uint64_t mt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; mt < TM; mt += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t o = ofs[mt];
        for (uint32_t j = 0; j < cnt[mt]; j++) items[o + j] = make_uint2((uint32_t)mt, j);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_bmm_masked_items(uint64_t n_items, const uint2 *__restrict__ items,
                                                          const uint32_t *__restrict__ m_rowid,
                                                          const uint32_t *__restrict__ m_tci,
                                                          const typename WordT<D>::T *__restrict__ m_tiles,
                                                          const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci,
                                                          const typename WordT<D>::T *__restrict__ a_tiles,
                                                          const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
                                                          const typename WordT<D>::T *__restrict__ b_tiles,
                                                          uint32_t m_row0, unsigned long long *__restrict__ out,
                                                          unsigned long long *__restrict__ work) {
    const uint32_t lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0, units = 0;
    for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_items; w += warps) {
        uint2 it = items[w];
        uint64_t mt = it.x;
        uint32_t I = m_rowid[mt] + m_row0, J = m_tci[mt];
        uint32_t mword = lane < (uint32_t)D ? (uint32_t)m_tiles[mt * D + lane] : 0u;
        uint32_t rows_used = __ballot_sync(0xffffffffu, mword != 0);
        uint32_t a0 = a_trp[I], a1 = a_trp[I + 1], b0 = b_trp[J], b1 = b_trp[J + 1];
        bool a_short = (a1 - a0) <= (b1 - b0);
        uint32_t s0 = a_short ? a0 : b0, s1 = a_short ? a1 : b1;
        uint32_t l0 = a_short ? b0 : a0, l1 = a_short ? b1 : a1;
        const uint32_t *stci = a_short ? a_tci : b_tci;
        const uint32_t *ltci = a_short ? b_tci : a_tci;
        uint32_t c0 = s0 + it.y * TC_CHUNK, c1 = min(s1, c0 + TC_CHUNK);
        // narrow the long row to the chunk's value range once per warp
        uint32_t first = __ldg(stci + c0), last = __ldg(stci + c1 - 1);
        uint32_t lo = lower_bound_u32(ltci, l0, l1, first);
        uint32_t hi = lower_bound_u32(ltci, lo, l1, last + 1);
        if (lo == hi || rows_used == 0) continue;
        for (uint32_t base = c0; base < c1; base += 32) {
            uint32_t si = base + lane;
            uint32_t ta = 0, tb = 0;
            bool hit = false;
            if (si < c1) {
                uint32_t K = __ldg(stci + si);
                uint32_t li = lower_bound_u32(ltci, lo, hi, K);
                if (li < hi && __ldg(ltci + li) == K) {
                    hit = true;
                    ta = a_short ? si : li;
                    tb = a_short ? li : si;
                }
            }
            if (!__ballot_sync(0xffffffffu, hit)) continue;
            uint32_t ru = rows_used;
            while (ru) {  // warp-uniform loop over non-empty mask rows
                int r = __ffs(ru) - 1;
                ru &= ru - 1;
                uint32_t mw = __shfl_sync(0xffffffffu, mword, r);
                if (hit) {
                    uint32_t aw = a_tiles[(size_t)ta * D + r];
                    if (work) units += aw ? __popc(mw) : 0u;  // AND+POPC units
                    while (aw && mw) {
                        int c = __ffs(mw) - 1;
                        mw &= mw - 1;
                        acc += __popc(aw & (uint32_t)b_tiles[(size_t)tb * D + c]);
                    }
                }
            }
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
    if (work) {
        for (int o = 16; o; o >>= 1) units += __shfl_xor_sync(0xffffffffu, units, o);
        if (lane == 0 && units) atomicAdd(work, units);
    }
}

// ------------------------------------------------------------ register-table rows
// Work unit = (mask tile row I, up to RT_UNIT of its mask tiles).  The warp
// keeps A's tile row I (<= 32*RT_K columns) in registers, lane l holding
// columns [l*k, l*k+k) (k = ceil(len/32)), and finds every column of Bt's row
// J by a 5-step shuffle search over the lanes' first columns plus k shuffles --
// no dependent memory round trips.  Longer A rows search global memory.
constexpr uint32_t RT_UNIT = 64;
constexpr int RT_K = 8;

__global__ void k_rt_counts(uint32_t mntr, const uint32_t *__restrict__ mtrp, uint32_t *__restrict__ cnt) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < mntr; r += gridDim.x * blockDim.x)
        cnt[r] = (mtrp[r + 1] - mtrp[r] + RT_UNIT - 1) / RT_UNIT;
}

__global__ void k_rt_fill(uint32_t mntr, const uint32_t *__restrict__ mtrp, const uint32_t *__restrict__ cnt,
                          const uint64_t *__restrict__ ofs, uint4 *__restrict__ units) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < mntr; r += gridDim.x * blockDim.x) {
        uint64_t o = ofs[r];
        uint32_t m0 = mtrp[r], m1 = mtrp[r + 1];
        for (uint32_t j = 0; j < cnt[r]; j++) units[o + j] = make_uint4(r, m0 + j * RT_UNIT, min(m1, m0 + (j + 1) * RT_UNIT), 0);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_bmm_rowtable(uint64_t n_units, const uint4 *__restrict__ units, uint32_t m_row0,
                                                      const uint32_t *__restrict__ m_tci,
                                                      const typename WordT<D>::T *__restrict__ m_tiles,
                                                      const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci,
                                                      const typename WordT<D>::T *__restrict__ a_tiles,
                                                      const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
                                                      const typename WordT<D>::T *__restrict__ b_tiles,
                                                      unsigned long long *__restrict__ out,
                                                      unsigned long long *__restrict__ work) {
    const uint32_t lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0, units_done = 0;
    for (uint64_t u = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n_units; u += warps) {
        const uint4 un = units[u];
        const uint32_t I = un.x + m_row0;
        const uint32_t a0 = a_trp[I], a1 = a_trp[I + 1], la = a1 - a0;
        if (!la) continue;
        const bool table = la <= 32u * RT_K;
        const uint32_t k = (la + 31) / 32;
        uint32_t key[RT_K];
#pragma unroll
        for (int j = 0; j < RT_K; j++) {
            uint32_t i = lane * k + j;
            key[j] = (table && j < (int)k && i < la) ? __ldg(a_tci + a0 + i) : 0xFFFFFFFFu;
        }
        const uint32_t first = key[0];
        // the unit's mask tiles, 32 at a time: column, Bt row range and mask
        // words loaded by all lanes at once (no dependent round trips per tile)
        for (uint32_t mb = un.y; mb < un.z; mb += 32) {
        const uint32_t mi = mb + lane;
        const bool mok = mi < un.z;
        const uint32_t Jl = mok ? m_tci[mi] : 0u;
        const uint32_t b0l = mok ? b_trp[Jl] : 0u, b1l = mok ? b_trp[Jl + 1] : 0u;
        uint32_t mwl = 0, mwh = 0;  // d <= 8: the whole mask tile in one or two words
        if constexpr (D == 4) mwl = mok ? reinterpret_cast<const uint32_t *>(m_tiles)[mi] : 0u;
        if constexpr (D == 8) {
            uint2 q = mok ? reinterpret_cast<const uint2 *>(m_tiles)[mi] : make_uint2(0, 0);
            mwl = q.x;
            mwh = q.y;
        }
        const uint32_t mcount = min(32u, un.z - mb);
        for (uint32_t q = 0; q < mcount; q++) {
            const uint32_t mt = mb + q;
            uint32_t mword;
            if constexpr (D == 4) {
                const uint32_t w = __shfl_sync(0xffffffffu, mwl, q);  // every lane takes part
                mword = lane < 4 ? (w >> (8 * lane)) & 0xFFu : 0u;
            } else if constexpr (D == 8) {
                uint32_t lo = __shfl_sync(0xffffffffu, mwl, q), hi = __shfl_sync(0xffffffffu, mwh, q);
                mword = lane < 8 ? ((lane < 4 ? lo : hi) >> (8 * (lane & 3))) & 0xFFu : 0u;
            } else {
                mword = lane < (uint32_t)D ? (uint32_t)m_tiles[(size_t)mt * D + lane] : 0u;
            }
            const uint32_t rows_used = __ballot_sync(0xffffffffu, mword != 0);
            const uint32_t b0 = __shfl_sync(0xffffffffu, b0l, q), b1 = __shfl_sync(0xffffffffu, b1l, q);
            if (!rows_used || b0 == b1) continue;
            for (uint32_t base = b0; base < b1; base += 32) {
                const uint32_t bi = base + lane;
                const uint32_t K = bi < b1 ? __ldg(b_tci + bi) : 0xFFFFFFFEu;
                uint32_t ta = 0;
                bool hit = false;
                if (table) {
                    // the last lane whose first column is <= K
                    uint32_t c = 0;
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        uint32_t f = __shfl_sync(0xffffffffu, first, c + o);
                        if (f <= K) c += o;
                    }
#pragma unroll
                    for (int j = 0; j < RT_K; j++) {
                        if (j >= (int)k) break;  // warp-uniform
                        uint32_t v = __shfl_sync(0xffffffffu, key[j], c);
                        if (v == K && bi < b1) {
                            hit = true;
                            ta = a0 + c * k + j;
                        }
                    }
                } else if (bi < b1) {
                    uint32_t li = lower_bound_u32(a_tci, a0, a1, K);
                    if (li < a1 && __ldg(a_tci + li) == K) {
                        hit = true;
                        ta = li;
                    }
                }
                if (!__ballot_sync(0xffffffffu, hit)) continue;
                uint32_t ru = rows_used;
                while (ru) {  // warp-uniform loop over non-empty mask rows
                    int r = __ffs(ru) - 1;
                    ru &= ru - 1;
                    uint32_t mw = __shfl_sync(0xffffffffu, mword, r);
                    if (hit) {
                        uint32_t aw = a_tiles[(size_t)ta * D + r];
                        if (work) units_done += aw ? __popc(mw) : 0u;
                        while (aw && mw) {
                            int cc = __ffs(mw) - 1;
                            mw &= mw - 1;
                            acc += __popc(aw & (uint32_t)b_tiles[(size_t)bi * D + cc]);
                        }
                    }
                }
            }
        }
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
    if (work) {
        for (int o = 16; o; o >>= 1) units_done += __shfl_xor_sync(0xffffffffu, units_done, o);
        if (lane == 0 && units_done) atomicAdd(work, units_done);
    }
}

int64_t bmm_masked_rowtable(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, cudaStream_t s,
                            uint64_t *work_out) {
    uint32_t mntr = mask->ntr;
    Buf<uint32_t> cnt(mntr, s);
    Buf<uint64_t> ofs((size_t)mntr + 1, s);
    LAUNCH(k_rt_counts, grid_for(mntr), 256, 0, s, mntr, mask->trp, cnt.p);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, mntr, s);
    uint64_t n_units = read_scalar(ofs.p + mntr, s);
    Buf<unsigned long long> out(1, s), work(1, s);
    CK(cudaMemsetAsync(out.p, 0, 8, s));
    CK(cudaMemsetAsync(work.p, 0, 8, s));
    if (!n_units) return 0;
    Buf<uint4> units(n_units, s);
    LAUNCH(k_rt_fill, grid_for(mntr), 256, 0, s, mntr, mask->trp, cnt.p, ofs.p, units.p);
    uint64_t blocks = (n_units + 7) / 8, cap = (uint64_t)num_sms() * 16;
    unsigned g = (unsigned)std::min(blocks, cap);
    kernel_timer().begin(s);
    switch (a->dim) {
#define RT_CASE(DD, W)                                                                                         \
    case DD:                                                                                                   \
        LAUNCH(k_bmm_rowtable<DD>, g, 256, 0, s, n_units, units.p, mask->row0, mask->tci,                     \
               (const W *)mask->tiles, a->trp, a->tci, (const W *)a->tiles, bt->trp, bt->tci,                 \
               (const W *)bt->tiles, out.p, work_out ? work.p : nullptr);                                     \
        break;
        RT_CASE(4, uint8_t)
        RT_CASE(8, uint8_t)
        RT_CASE(16, uint16_t)
        RT_CASE(32, uint32_t)
#undef RT_CASE
    }
    kernel_timer().end(s);
    if (work_out) *work_out = read_scalar(work.p, s);
    return (int64_t)read_scalar(out.p, s);
}

// ------------------------------------------------------------ row-hash path
// Work unit = (mask tile row I, up to ROW_UNIT of its mask tiles).  The CTA
// hashes A's tile row I (column -> position) into shared memory once; each
// warp then takes a mask tile (I, J), streams Bt's row J 32 columns at a
// time (coalesced) and probes the table -- one memory round trip per 32
// candidates instead of a dependent binary search per candidate.  Rows of A
// longer than HASH_MAX fall back to the binary-search warp loop.
constexpr uint32_t ROW_UNIT = 128;
constexpr uint32_t HASH_MAX = 4096;              // A-row entries that fit the table
constexpr uint32_t HASH_SLOTS = 2 * HASH_MAX;    // 64 KB of keys + positions
constexpr uint32_t EMPTY_KEY = 0xFFFFFFFFu;

__global__ void k_rowunit_counts(uint32_t mntr, uint32_t m_row0, const uint32_t *__restrict__ mtrp,
                                 const uint32_t *__restrict__ a_trp, uint32_t *__restrict__ cnt) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < mntr; r += gridDim.x * blockDim.x) {
        uint32_t I = r + m_row0, len = mtrp[r + 1] - mtrp[r];
        cnt[r] = (a_trp[I + 1] > a_trp[I]) ? (len + ROW_UNIT - 1) / ROW_UNIT : 0;
    }
}

__global__ void k_rowunit_fill(uint32_t mntr, const uint32_t *__restrict__ mtrp, const uint32_t *__restrict__ cnt,
                               const uint64_t *__restrict__ ofs, uint4 *__restrict__ units) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < mntr; r += gridDim.x * blockDim.x) {
        uint64_t o = ofs[r];
        uint32_t m0 = mtrp[r], m1 = mtrp[r + 1];
        for (uint32_t j = 0; j < cnt[r]; j++) units[o + j] = make_uint4(r, m0 + j * ROW_UNIT, min(m1, m0 + (j + 1) * ROW_UNIT), 0);
    }
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t k, uint32_t mask) { return (k * 0x9E3779B1u >> 7) & mask; }

template <int D>
__device__ __forceinline__ unsigned long long mask_tile_pops(uint32_t mword, uint32_t rows_used, bool hit, uint32_t ta,
                                                             uint32_t tb, const typename WordT<D>::T *__restrict__ a_tiles,
                                                             const typename WordT<D>::T *__restrict__ b_tiles) {
    unsigned long long acc = 0;
    uint32_t ru = rows_used;
    while (ru) {  // warp-uniform loop over non-empty mask rows
        int r = __ffs(ru) - 1;
        ru &= ru - 1;
        uint32_t mw = __shfl_sync(0xffffffffu, mword, r);
        if (hit) {
            uint32_t aw = a_tiles[(size_t)ta * D + r];
            while (aw && mw) {
                int c = __ffs(mw) - 1;
                mw &= mw - 1;
                acc += __popc(aw & (uint32_t)b_tiles[(size_t)tb * D + c]);
            }
        }
    }
    return acc;
}

template <int D>
__global__ void __launch_bounds__(256) k_bmm_rowhash(uint32_t n_units, const uint4 *__restrict__ units, uint32_t m_row0,
                                                     const uint32_t *__restrict__ m_tci,
                                                     const typename WordT<D>::T *__restrict__ m_tiles,
                                                     const uint32_t *__restrict__ a_trp, const uint32_t *__restrict__ a_tci,
                                                     const typename WordT<D>::T *__restrict__ a_tiles,
                                                     const uint32_t *__restrict__ b_trp, const uint32_t *__restrict__ b_tci,
                                                     const typename WordT<D>::T *__restrict__ b_tiles,
                                                     unsigned long long *__restrict__ out) {
    extern __shared__ uint32_t hsm[];  // HASH_SLOTS keys then HASH_SLOTS positions
    uint32_t *hkey = hsm, *hval = hsm + HASH_SLOTS;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    unsigned long long acc = 0;
    for (uint32_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        uint4 un = units[u];
        uint32_t I = un.x + m_row0;
        uint32_t a0 = a_trp[I], a1 = a_trp[I + 1], la = a1 - a0;
        bool hashed = la <= HASH_MAX;
        uint32_t hs = 64;
        while (hs < 2 * la) hs <<= 1;
        uint32_t hmask = hs - 1;
        if (hashed) {
            for (uint32_t i = threadIdx.x; i < hs; i += blockDim.x) hkey[i] = EMPTY_KEY;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < la; i += blockDim.x) {
                uint32_t K = __ldg(a_tci + a0 + i), h = hash_slot(K, hmask);
                while (atomicCAS(&hkey[h], EMPTY_KEY, K) != EMPTY_KEY) h = (h + 1) & hmask;
                hval[h] = i;
            }
            __syncthreads();
        }
        for (uint32_t mt = un.y + warp; mt < un.z; mt += nwarps) {
            uint32_t J = m_tci[mt];
            uint32_t mword = lane < (uint32_t)D ? (uint32_t)m_tiles[(size_t)mt * D + lane] : 0u;
            uint32_t rows_used = __ballot_sync(0xffffffffu, mword != 0);
            uint32_t b0 = b_trp[J], b1 = b_trp[J + 1];
            if (!rows_used || b0 == b1) continue;
            if (hashed) {
                for (uint32_t base = b0; base < b1; base += 32) {
                    uint32_t bi = base + lane, ta = 0;
                    bool hit = false;
                    if (bi < b1) {
                        uint32_t K = __ldg(b_tci + bi), h = hash_slot(K, hmask), key;
                        while ((key = hkey[h]) != EMPTY_KEY && key != K) h = (h + 1) & hmask;
                        if (key == K) { hit = true; ta = a0 + hval[h]; }
                    }
                    if (__ballot_sync(0xffffffffu, hit)) acc += mask_tile_pops<D>(mword, rows_used, hit, ta, bi, a_tiles, b_tiles);
                }
            } else {  // long A row: binary-search Bt's entries in it
                for (uint32_t base = b0; base < b1; base += 32) {
                    uint32_t bi = base + lane, ta = 0;
                    bool hit = false;
                    if (bi < b1) {
                        uint32_t K = __ldg(b_tci + bi);
                        uint32_t li = lower_bound_u32(a_tci, a0, a1, K);
                        if (li < a1 && __ldg(a_tci + li) == K) { hit = true; ta = li; }
                    }
                    if (__ballot_sync(0xffffffffu, hit)) acc += mask_tile_pops<D>(mword, rows_used, hit, ta, bi, a_tiles, b_tiles);
                }
            }
        }
        __syncthreads();  // the table is rebuilt for the next unit
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(out, acc);
}

int64_t bmm_masked_rowhash(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, cudaStream_t s) {
    uint32_t mntr = mask->ntr;
    Buf<uint32_t> cnt(mntr, s);
    Buf<uint64_t> ofs((size_t)mntr + 1, s);
    LAUNCH(k_rowunit_counts, grid_for(mntr), 256, 0, s, mntr, mask->row0, mask->trp, a->trp, cnt.p);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, mntr, s);
    uint64_t n_units = read_scalar(ofs.p + mntr, s);
    Buf<unsigned long long> out(1, s);
    CK(cudaMemsetAsync(out.p, 0, 8, s));
    if (!n_units) return 0;
    Buf<uint4> units(n_units, s);
    LAUNCH(k_rowunit_fill, grid_for(mntr), 256, 0, s, mntr, mask->trp, cnt.p, ofs.p, units.p);
    unsigned g = (unsigned)std::min<uint64_t>(n_units, (uint64_t)num_sms() * 3);
    const int smem = 2 * HASH_SLOTS * 4;
    switch (a->dim) {
#define RH_CASE(DD, W)                                                                                          \
    case DD:                                                                                                    \
        CK(cudaFuncSetAttribute(k_bmm_rowhash<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));        \
        LAUNCH(k_bmm_rowhash<DD>, g, 256, smem, s, (uint32_t)n_units, units.p, mask->row0, mask->tci,          \
               (const W *)mask->tiles, a->trp, a->tci, (const W *)a->tiles, bt->trp, bt->tci,                  \
               (const W *)bt->tiles, out.p);                                                                   \
        break;
        RH_CASE(4, uint8_t)
        RH_CASE(8, uint8_t)
        RH_CASE(16, uint16_t)
        RH_CASE(32, uint32_t)
#undef RH_CASE
    }
    return (int64_t)read_scalar(out.p, s);
}

int64_t bmm_masked_bt(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, cudaStream_t s,
                      uint64_t *work_out = nullptr) {
    if (work_out) *work_out = 0;
    if (!mask->num_tiles || !a->num_tiles || !bt->num_tiles) return 0;
    // B2SR_TC_ALG=rowhash selects the smem row-hash kernel (measured 176 ms vs
    // 34 ms for the chunked items at s20 d=4, profiles/r01_pull_ab.txt)
    const char *alg = getenv("B2SR_TC_ALG");
    if (alg && alg[0] == 'r') return bmm_masked_rowhash(a, bt, mask, s);
    // B2SR_TC_ALG=table: the register-table rows kernel -- measured slower at
    // R-MAT s20 d=4 on the degree-oriented DAG (32.6 vs 27.2 ms): it always
    // scans Bt's row (5.0 G probes) where the items kernel scans the shorter
    if (alg && alg[0] == 't') return bmm_masked_rowtable(a, bt, mask, s, work_out);
    uint64_t TM = mask->num_tiles;
    Buf<uint32_t> rowid(TM, s), cnt(TM, s);
    Buf<uint64_t> ofs(TM + 1, s);
    row_ids(mask, rowid.p, s);
    LAUNCH(k_tc_item_counts, grid_for(TM), 256, 0, s, TM, rowid.p, mask->tci, mask->row0, a->trp, bt->trp, cnt.p);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, TM, s);
    uint64_t n_items = read_scalar(ofs.p + TM, s);
    Buf<unsigned long long> out(1, s);
    CK(cudaMemsetAsync(out.p, 0, 8, s));
    if (!n_items) return 0;
    Buf<uint2> items(n_items, s);
    LAUNCH(k_tc_item_fill, grid_for(TM), 256, 0, s, TM, cnt.p, ofs.p, items.p);
    uint64_t blocks = (n_items + 7) / 8, cap = (uint64_t)num_sms() * 16;
    unsigned g = (unsigned)std::min(blocks, cap);
    Buf<unsigned long long> work(1, s);
    if (work_out) CK(cudaMemsetAsync(work.p, 0, 8, s));
    kernel_timer().begin(s);
    switch (a->dim) {
#define BMM_CASE(DD, W)                                                                                        \
    case DD:                                                                                                   \
        LAUNCH(k_bmm_masked_items<DD>, g, 256, 0, s, n_items, items.p, rowid.p, mask->tci,                    \
               (const W *)mask->tiles, a->trp, a->tci, (const W *)a->tiles, bt->trp, bt->tci,                 \
               (const W *)bt->tiles, mask->row0, out.p, work_out ? work.p : nullptr);                         \
        break;
        BMM_CASE(4, uint8_t)
        BMM_CASE(8, uint8_t)
        BMM_CASE(16, uint16_t)
        BMM_CASE(32, uint32_t)
#undef BMM_CASE
    }
    kernel_timer().end(s);
    if (work_out) *work_out = read_scalar(work.p, s);
    return (int64_t)read_scalar(out.p, s);
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_bmm_sum(const b2sr_matrix *a, const b2sr_matrix *b, int64_t *out, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (a->n != b->n || a->dim != b->dim) B2SR_THROW(B2SR_EINVAL, "operands must share n and tile width");
    size_t rows = (size_t)tile_rows(a->n, a->dim) * a->dim;
    Buf<uint32_t> colsum(rows, s), rowdeg(rows, s);
    Buf<unsigned long long> acc(1, s);
    CK(cudaMemsetAsync(colsum.p, 0, rows * 4, s));
    CK(cudaMemsetAsync(rowdeg.p, 0, rows * 4, s));
    CK(cudaMemsetAsync(acc.p, 0, 8, s));
    colsum_rowdeg(a, colsum.p, nullptr, s);
    colsum_rowdeg(b, nullptr, rowdeg.p, s);
    LAUNCH(k_dot_u32, grid_for(rows), 256, 0, s, rows, colsum.p, rowdeg.p, acc.p);
    *out = (int64_t)read_scalar(acc.p, s);
    API_END
}

int b2sr_bmm_sum_masked_bt(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask, int64_t *out,
                           void *stream) {
    API_BEGIN
    if (a->n != bt->n || a->dim != bt->dim || a->n != mask->n || a->dim != mask->dim)
        B2SR_THROW(B2SR_EINVAL, "operands must share n and tile width");
    if (a->row0 || bt->row0 || a->ntr != tile_rows(a->n, a->dim) || bt->ntr != a->ntr)
        B2SR_THROW(B2SR_EINVAL, "A and Bt must be full matrices (only the mask may be a row block)");
    *out = bmm_masked_bt(a, bt, mask, (cudaStream_t)stream);
    API_END
}

int b2sr_tc(const b2sr_matrix *lower, int64_t *count, void *stream) {
    API_BEGIN
    // bmm_masked(L, transpose(L), L): B = transpose(L) enters transposed, i.e. L.
    *count = bmm_masked_bt(lower, lower, lower, (cudaStream_t)stream);
    API_END
}

int b2sr_tc_work(const b2sr_matrix *lower, int64_t *count, uint64_t *work, void *stream) {
    API_BEGIN
    *count = bmm_masked_bt(lower, lower, lower, (cudaStream_t)stream, work);
    API_END
}

}  // extern "C"
