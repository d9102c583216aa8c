// K3 tile transpose (formats.py:477-489), b2sr_to_csr (formats.py:467-474),
// diagonal drop in tile form (algorithms.py:96-101, 111).
//
// Transpose = stable radix sort of (tile column, tile id) + a gather that
// bit-transposes each tile in registers (Hacker's-Delight block swaps, one
// thread per tile, 16-byte loads/stores of whole tiles).  The reference
// unpacks every tile into a (T, d, d) uint64 temporary (~16*d^2 bytes per
// tile); here the working set is 16 bytes of indices per tile.
#include "b2sr_internal.cuh"

namespace b2sr {

// In-register transpose of a D x D bit tile, row r = a[r], LSB = column 0.
template <int D>
__device__ __forceinline__ void bit_transpose(uint32_t (&a)[D]) {
    uint32_t m = (D == 32) ? 0x0000FFFFu : (D == 16) ? 0x00FFu : (D == 8) ? 0x0Fu : 0x3u;
#pragma unroll
    for (int j = D / 2; j; j >>= 1) {
#pragma unroll
        for (int k = 0; k < D; k = (k + j + 1) & ~j) {
            uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k] ^= t << j;
            a[k + j] ^= t;
        }
        m ^= m << (j / 2);
    }
}

template <int D>
__device__ __forceinline__ void load_tile(const void *tiles, size_t t, uint32_t (&a)[D]) {
    if constexpr (D == 32) {
        const uint4 *p = reinterpret_cast<const uint4 *>(tiles) + t * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            uint4 v = __ldg(p + i);
            a[4 * i] = v.x; a[4 * i + 1] = v.y; a[4 * i + 2] = v.z; a[4 * i + 3] = v.w;
        }
    } else if constexpr (D == 16) {
        const uint4 *p = reinterpret_cast<const uint4 *>(tiles) + t * 2;
#pragma unroll
        for (int i = 0; i < 2; i++) {
            uint4 v = __ldg(p + i);
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; k++) { a[8 * i + 2 * k] = w[k] & 0xFFFFu; a[8 * i + 2 * k + 1] = w[k] >> 16; }
        }
    } else if constexpr (D == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2 *>(tiles) + t);
#pragma unroll
        for (int k = 0; k < 4; k++) { a[k] = (v.x >> (8 * k)) & 0xFFu; a[4 + k] = (v.y >> (8 * k)) & 0xFFu; }
    } else {
        uint32_t v = __ldg(reinterpret_cast<const uint32_t *>(tiles) + t);
#pragma unroll
        for (int k = 0; k < 4; k++) a[k] = (v >> (8 * k)) & 0xFFu;
    }
}

template <int D>
__device__ __forceinline__ void store_tile(void *tiles, size_t t, const uint32_t (&a)[D]) {
    if constexpr (D == 32) {
        uint4 *p = reinterpret_cast<uint4 *>(tiles) + t * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) p[i] = make_uint4(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]);
    } else if constexpr (D == 16) {
        uint4 *p = reinterpret_cast<uint4 *>(tiles) + t * 2;
#pragma unroll
        for (int i = 0; i < 2; i++)
            p[i] = make_uint4(a[8 * i] | (a[8 * i + 1] << 16), a[8 * i + 2] | (a[8 * i + 3] << 16),
                              a[8 * i + 4] | (a[8 * i + 5] << 16), a[8 * i + 6] | (a[8 * i + 7] << 16));
    } else if constexpr (D == 8) {
        uint2 v;
        v.x = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
        v.y = a[4] | (a[5] << 8) | (a[6] << 16) | (a[7] << 24);
        reinterpret_cast<uint2 *>(tiles)[t] = v;
    } else {
        reinterpret_cast<uint32_t *>(tiles)[t] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
    }
}

__global__ void k_col_hist(uint64_t T, const uint32_t *tci, uint32_t *cnt) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + tci[t], 1u);
}

__global__ void k_u64_to_u32(const uint64_t *in, uint32_t *out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// one warp per tile row: rowid[t] = I for t in [trp[I], trp[I+1])
__global__ void k_row_ids(uint32_t ntr, const uint32_t *trp, uint32_t *rowid) {
    uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < ntr; I += warps)
        for (uint32_t t = trp[I] + lane_id(); t < trp[I + 1]; t += 32) rowid[t] = I;
}

__global__ void k_iota(uint32_t *v, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

template <int D>
__global__ void __launch_bounds__(256) k_transpose_gather(uint64_t T, const uint32_t *__restrict__ order,
                                                          const uint32_t *__restrict__ rowid,
                                                          const void *__restrict__ tiles, uint32_t *__restrict__ tci_out,
                                                          void *__restrict__ tiles_out) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < T; p += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t t = order[p];
        tci_out[p] = rowid[t];
        uint32_t a[D];
        load_tile<D>(tiles, t, a);
        bit_transpose<D>(a);
        store_tile<D>(tiles_out, p, a);
    }
}

// d=4 fast path: a 4x4 tile is 16 bits of payload, so (column | row | tile)
// fits one 64-bit key and a stable radix sort over the column bits carries
// every tile to its transposed position -- no random gathers afterwards.
__global__ void k_pack4(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                        const uint32_t *__restrict__ tiles, int cb, uint64_t *__restrict__ keys) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t w = tiles[t];  // four row bytes, low nibbles
        uint32_t nib = (w & 0xFu) | ((w >> 4) & 0xF0u) | ((w >> 8) & 0xF00u) | ((w >> 12) & 0xF000u);
        keys[t] = (uint64_t)tci[t] | ((uint64_t)rowid[t] << cb) | ((uint64_t)nib << (2 * cb));
    }
}

__global__ void k_unpack4(uint64_t T, const uint64_t *__restrict__ keys, int cb, uint32_t *__restrict__ tci_out,
                          uint32_t *__restrict__ tiles_out) {
    const uint64_t mask = (1ull << cb) - 1;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < T; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[p];
        tci_out[p] = (uint32_t)((k >> cb) & mask);  // the source row is the transposed column
        uint32_t nib = (uint32_t)(k >> (2 * cb));
        uint32_t a[4] = {nib & 0xFu, (nib >> 4) & 0xFu, (nib >> 8) & 0xFu, (nib >> 12) & 0xFu};
        bit_transpose<4>(a);
        tiles_out[p] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
    }
}

void launch_row_ids(const b2sr_matrix *m, uint32_t *rowid, cudaStream_t s) {
    uint64_t b = ((uint64_t)m->ntr * 32 + 255) / 256, cap = (uint64_t)num_sms() * 16;
    LAUNCH(k_row_ids, (unsigned)std::max<uint64_t>(1, std::min(b, cap)), 256, 0, s, m->ntr, m->trp, rowid);
}

static int bits_for(uint32_t maxval) {
    int b = 0;
    while (b < 32 && (maxval >> b)) b++;
    return b;
}

static unsigned grid_for(uint64_t work, unsigned per = 256) {
    uint64_t b = (work + per - 1) / per, cap = (uint64_t)num_sms() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

b2sr_matrix *transpose_device(const b2sr_matrix *m, cudaStream_t s) {
    if (m->row0 != 0 || m->ntr != tile_rows(m->n, m->dim))
        B2SR_THROW(B2SR_EINVAL, "transpose needs a full matrix, not a row block");
    uint32_t ntr = m->ntr;
    uint64_t T = m->num_tiles;
    b2sr_matrix *o = new_matrix(m->n, m->dim, ntr, T, s);
    try {
        Buf<uint32_t> cnt(ntr, s);
        Buf<uint64_t> ofs((size_t)ntr + 1, s);
        CK(cudaMemsetAsync(cnt.p, 0, (size_t)ntr * 4, s));
        if (T) LAUNCH(k_col_hist, grid_for(T), 256, 0, s, T, m->tci, cnt.p);
        exclusive_scan_u32_to_u64(cnt.p, ofs.p, ntr, s);
        LAUNCH(k_u64_to_u32, grid_for(ntr + 1), 256, 0, s, ofs.p, o->trp, (size_t)ntr + 1);
        const int cb = bits_for(ntr - 1);
        if (T && m->dim == 4 && 2 * cb + 16 <= 64) {
            Buf<uint64_t> keys(T, s), kalt;
            {
                Buf<uint32_t> rowid(T, s);
                LAUNCH(k_row_ids, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, m->trp, rowid.p);
                LAUNCH(k_pack4, grid_for(T), 256, 0, s, T, rowid.p, m->tci, (const uint32_t *)m->tiles, cb, keys.p);
            }
            uint64_t *ks = nullptr;
            radix_sort_keys_u64(keys.p, T, cb, s, &ks, &kalt);
            LAUNCH(k_unpack4, grid_for(T), 256, 0, s, T, ks, cb, o->tci, (uint32_t *)o->tiles);
        } else if (T) {
            Buf<uint32_t> keys(T, s), vals(T, s), rowid(T, s), kalt, valt;
            CK(cudaMemcpyAsync(keys.p, m->tci, T * 4, cudaMemcpyDeviceToDevice, s));
            LAUNCH(k_iota, grid_for(T), 256, 0, s, vals.p, T);
            LAUNCH(k_row_ids, grid_for((uint64_t)ntr * 32), 256, 0, s, ntr, m->trp, rowid.p);
            uint32_t *ks = nullptr, *vs = nullptr;
            radix_sort_pairs_u32(keys.p, vals.p, T, bits_for(ntr - 1), s, &ks, &vs, &kalt, &valt);
            unsigned g = grid_for(T);
            switch (m->dim) {
                case 4: LAUNCH(k_transpose_gather<4>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
                case 8: LAUNCH(k_transpose_gather<8>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
                case 16: LAUNCH(k_transpose_gather<16>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
                default: LAUNCH(k_transpose_gather<32>, g, 256, 0, s, T, vs, rowid.p, m->tiles, o->tci, o->tiles); break;
            }
        }
    } catch (...) {
        free_matrix(o);
        throw;
    }
    return o;
}

// ------------------------------------------------------------ b2sr -> csr
template <int D>
__global__ void k_row_degrees(uint64_t T, const uint32_t *__restrict__ rowid, const typename WordT<D>::T *__restrict__ tiles,
                              uint32_t *__restrict__ deg) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t I = rowid[t];
#pragma unroll
        for (int r = 0; r < D; r++) {
            uint32_t c = __popc((uint32_t)tiles[t * D + r]);
            if (c) atomicAdd(deg + (size_t)I * D + r, c);
        }
    }
}

// group of D lanes per tile row, lane = bit-row, columns emitted in order
template <int D>
__global__ void k_csr_fill(uint32_t ntr, uint32_t n, const uint32_t *__restrict__ trp, const uint32_t *__restrict__ tci,
                           const typename WordT<D>::T *__restrict__ tiles, const uint32_t *__restrict__ row_ptr,
                           uint32_t *__restrict__ col_ind) {
    constexpr uint32_t GPW = 32 / D;
    const uint32_t lane = lane_id(), r = lane % D;
    const uint32_t groups = ((gridDim.x * blockDim.x) >> 5) * GPW;
    for (uint32_t I = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * GPW + lane / D; I < ntr; I += groups) {
        uint64_t row = (uint64_t)I * D + r;
        if (row >= n) continue;
        uint32_t pos = row_ptr[row];
        for (uint32_t t = trp[I]; t < trp[I + 1]; t++) {
            uint32_t w = tiles[(size_t)t * D + r];
            uint32_t base = tci[t] * D;
            while (w) {
                col_ind[pos++] = base + (__ffs(w) - 1);
                w &= w - 1;
            }
        }
    }
}

// ------------------------------------------------------------ diagonal drop
template <int D>
__global__ void k_diag_flags(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                             const typename WordT<D>::T *__restrict__ tiles, uint32_t *__restrict__ keep) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t k = 1;
        if (rowid[t] == tci[t]) {
            uint32_t o = 0;
#pragma unroll
            for (int r = 0; r < D; r++) o |= (uint32_t)tiles[t * D + r] & ~(1u << r);
            k = o != 0;
        }
        keep[t] = k;
    }
}

template <int D>
__global__ void k_diag_compact(uint64_t T, const uint32_t *__restrict__ rowid, const uint32_t *__restrict__ tci,
                               const typename WordT<D>::T *__restrict__ tiles, const uint32_t *__restrict__ keep,
                               const uint64_t *__restrict__ ofs, uint32_t *__restrict__ tci_out,
                               typename WordT<D>::T *__restrict__ tiles_out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        if (!keep[t]) continue;
        uint64_t o = ofs[t];
        bool diag = rowid[t] == tci[t];
        tci_out[o] = tci[t];
#pragma unroll
        for (int r = 0; r < D; r++) {
            uint32_t w = tiles[t * D + r];
            if (diag) w &= ~(1u << r);
            tiles_out[o * D + r] = (typename WordT<D>::T)w;
        }
    }
}

__global__ void k_diag_trp(uint32_t ntr, const uint32_t *trp, const uint64_t *ofs, uint32_t *trp_out) {
    uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I <= ntr) trp_out[I] = (uint32_t)ofs[trp[I]];
}

template <int D>
static b2sr_matrix *drop_diag_impl(const b2sr_matrix *m, cudaStream_t s) {
    using W = typename WordT<D>::T;
    uint64_t T = m->num_tiles;
    Buf<uint32_t> rowid(T, s), keep(T, s);
    Buf<uint64_t> ofs(T + 1, s);
    LAUNCH(k_row_ids, grid_for((uint64_t)m->ntr * 32), 256, 0, s, m->ntr, m->trp, rowid.p);
    LAUNCH(k_diag_flags<D>, grid_for(T), 256, 0, s, T, rowid.p, m->tci, (const W *)m->tiles, keep.p);
    exclusive_scan_u32_to_u64(keep.p, ofs.p, T, s);
    uint64_t T2 = read_scalar(ofs.p + T, s);
    b2sr_matrix *o = new_matrix(m->n, m->dim, m->ntr, T2, s);
    try {
        LAUNCH(k_diag_trp, (m->ntr + 256) / 256, 256, 0, s, m->ntr, m->trp, ofs.p, o->trp);
        LAUNCH(k_diag_compact<D>, grid_for(T), 256, 0, s, T, rowid.p, m->tci, (const W *)m->tiles, keep.p, ofs.p,
               o->tci, (W *)o->tiles);
    } catch (...) {
        free_matrix(o);
        throw;
    }
    return o;
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_transpose(const b2sr_matrix *m, void *stream, b2sr_matrix **out) {
    API_BEGIN
    *out = transpose_device(m, (cudaStream_t)stream);
    API_END
}

int b2sr_to_csr_rowptr(const b2sr_matrix *m, uint32_t *d_row_ptr, uint64_t *nnz, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (m->row0 != 0) B2SR_THROW(B2SR_EINVAL, "b2sr_to_csr needs a full matrix");
    uint64_t T = m->num_tiles;
    size_t rows = (size_t)m->ntr * m->dim;
    Buf<uint32_t> deg(rows, s), rowid(T, s);
    Buf<uint64_t> ofs((size_t)m->n + 1, s);
    CK(cudaMemsetAsync(deg.p, 0, rows * 4, s));
    if (T) {
        LAUNCH(k_row_ids, grid_for((uint64_t)m->ntr * 32), 256, 0, s, m->ntr, m->trp, rowid.p);
        unsigned g = grid_for(T);
        switch (m->dim) {
            case 4: LAUNCH(k_row_degrees<4>, g, 256, 0, s, T, rowid.p, (const uint8_t *)m->tiles, deg.p); break;
            case 8: LAUNCH(k_row_degrees<8>, g, 256, 0, s, T, rowid.p, (const uint8_t *)m->tiles, deg.p); break;
            case 16: LAUNCH(k_row_degrees<16>, g, 256, 0, s, T, rowid.p, (const uint16_t *)m->tiles, deg.p); break;
            default: LAUNCH(k_row_degrees<32>, g, 256, 0, s, T, rowid.p, (const uint32_t *)m->tiles, deg.p); break;
        }
    }
    exclusive_scan_u32_to_u64(deg.p, ofs.p, m->n, s);
    uint64_t total = read_scalar(ofs.p + m->n, s);
    if (total > 0xFFFFFFFFull) B2SR_THROW(B2SR_EFORMAT, "nnz exceeds the 32-bit CSR index range");
    LAUNCH(k_u64_to_u32, grid_for((uint64_t)m->n + 1), 256, 0, s, ofs.p, d_row_ptr, (size_t)m->n + 1);
    *nnz = total;
    API_END
}

int b2sr_to_csr_fill(const b2sr_matrix *m, const uint32_t *d_row_ptr, uint32_t *d_col_ind, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (!m->num_tiles) return B2SR_OK;
    uint32_t gpw = 32 / m->dim;
    unsigned g = grid_for(((uint64_t)m->ntr + gpw - 1) / gpw * 32);
    switch (m->dim) {
        case 4: LAUNCH(k_csr_fill<4>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint8_t *)m->tiles, d_row_ptr, d_col_ind); break;
        case 8: LAUNCH(k_csr_fill<8>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint8_t *)m->tiles, d_row_ptr, d_col_ind); break;
        case 16: LAUNCH(k_csr_fill<16>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint16_t *)m->tiles, d_row_ptr, d_col_ind); break;
        default: LAUNCH(k_csr_fill<32>, g, 256, 0, s, m->ntr, m->n, m->trp, m->tci, (const uint32_t *)m->tiles, d_row_ptr, d_col_ind); break;
    }
    API_END
}

int b2sr_drop_diagonal(const b2sr_matrix *m, void *stream, b2sr_matrix **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (m->row0 != 0) B2SR_THROW(B2SR_EINVAL, "drop_diagonal needs a full matrix");
    switch (m->dim) {
        case 4: *out = drop_diag_impl<4>(m, s); break;
        case 8: *out = drop_diag_impl<8>(m, s); break;
        case 16: *out = drop_diag_impl<16>(m, s); break;
        default: *out = drop_diag_impl<32>(m, s); break;
    }
    API_END
}

}  // extern "C"
