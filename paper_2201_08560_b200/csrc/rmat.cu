// Synthetic input on the device: Graph500-style R-MAT edges and COO -> CSR
// with CsrMatrix.from_coo semantics (formats.py:156-190: row-major sort,
// duplicates merged), plus the strict lower triangle (algorithms.py:218-222).
//
// The generator is counter-based (splitmix64 of (seed, edge, level)), so the
// CPU twin in oracle/b2sr_oracle.c (orc_rmat_edges) produces the same graph.
#include "b2sr_internal.cuh"

namespace b2sr {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr uint32_t RMAT_T_AB = 3264175144u;  // floor(0.76 * 2^32): P(row bit) = c + d
constexpr uint32_t RMAT_T_A = 3221225472u;   // a / (a + b) = 0.75
constexpr uint32_t RMAT_T_C = 3400182442u;   // floor(19/24 * 2^32) = c / (c + d)

__device__ __forceinline__ uint32_t rmat_perm(uint32_t v, int scale, uint64_t key) {
    uint32_t mask = scale >= 32 ? 0xFFFFFFFFu : ((1u << scale) - 1u);
    int sh = (scale + 1) / 2;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint32_t M = (uint32_t)mix64(key ^ (uint64_t)(2 * i + 1)) | 1u;
        uint32_t A = (uint32_t)mix64(key ^ (uint64_t)(2 * i + 2));
        v = (v * M + A) & mask;
        v ^= v >> sh;
    }
    return v;
}

__global__ void k_rmat(int scale, uint64_t m, uint64_t key, uint32_t *src, uint32_t *dst) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u = 0, v = 0;
        for (int l = 0; l < scale; l++) {
            uint64_t r = mix64(key + (e * (uint64_t)scale + (uint64_t)l + 1) * 0x9E3779B97F4A7C15ull);
            uint32_t lo = (uint32_t)r, hi = (uint32_t)(r >> 32);
            uint32_t rb = lo >= RMAT_T_AB;
            uint32_t cb = hi >= (rb ? RMAT_T_C : RMAT_T_A);
            u |= rb << l;
            v |= cb << l;
        }
        src[e] = rmat_perm(u, scale, key);
        dst[e] = rmat_perm(v, scale, key);
    }
}

// keys (u << B) | v; symmetric pairs side by side; dropped self-loops -> the
// all-ones 2B-bit sentinel, which sorts last and equals only a self-loop key
__global__ void k_coo_keys(uint64_t m, const uint32_t *src, const uint32_t *dst, int B, int sym, int drop,
                           uint64_t *keys) {
    const uint64_t dead_key = (1ull << (2 * B)) - 1;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t u = src[e], v = dst[e];
        bool dead = drop && u == v;
        if (sym) {
            keys[2 * e] = dead ? dead_key : (u << B) | v;
            keys[2 * e + 1] = dead ? dead_key : (v << B) | u;
        } else {
            keys[e] = dead ? dead_key : (u << B) | v;
        }
    }
}

__global__ void k_uniq_flags(uint64_t k, const uint64_t *keys, uint64_t dead_key, uint32_t *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = keys[i] != dead_key && (i == 0 || keys[i] != keys[i - 1]);
}

__global__ void k_uniq_scatter(uint64_t k, const uint64_t *keys, const uint32_t *flag, const uint64_t *ofs, int B,
                               uint32_t *col_ind, uint32_t *deg) {
    uint64_t mask = (1ull << B) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        col_ind[ofs[i]] = (uint32_t)(keys[i] & mask);
        atomicAdd(deg + (keys[i] >> B), 1u);
    }
}

__global__ void k_to_u32(const uint64_t *in, uint32_t *out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// strict lower triangle: entries c < r are a prefix of each sorted row
__global__ void k_lower_count(uint32_t n, const uint32_t *row_ptr, const uint32_t *col_ind, uint32_t *cnt) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        uint32_t a = row_ptr[r], b = row_ptr[r + 1];
        while (a < b) {
            uint32_t mid = (a + b) >> 1;
            if (col_ind[mid] < r) a = mid + 1; else b = mid;
        }
        cnt[r] = a - row_ptr[r];
    }
}

__global__ void k_lower_fill(uint32_t n, const uint32_t *row_ptr, const uint32_t *col_ind, const uint32_t *lrow_ptr,
                             uint32_t *lcol_ind) {
    uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        uint32_t src = row_ptr[r], dst = lrow_ptr[r], len = lrow_ptr[r + 1] - dst;
        for (uint32_t i = lane_id(); i < len; i += 32) lcol_ind[dst + i] = col_ind[src + i];
    }
}

// Degree orientation for triangle counting: keep (u, v) iff (deg u, u) <
// (deg v, v) -- every vertex points at higher-degree neighbours.  Any total
// order counts every triangle exactly once in sum_{(i,j) in L} (L L^T)_ij;
// this one bounds the out-degrees (R-MAT s20: max 671 instead of 30 078 for
// the ID-ordered lower triangle), so no hub row enters the intersections.
__device__ __forceinline__ bool orient_keep(const uint32_t *row_ptr, uint32_t u, uint32_t du, uint32_t v) {
    uint32_t dv = __ldg(row_ptr + v + 1) - __ldg(row_ptr + v);
    return dv > du || (dv == du && v < u);
}

__global__ void k_orient_count(uint32_t n, const uint32_t *__restrict__ row_ptr, const uint32_t *__restrict__ col_ind,
                               uint32_t *__restrict__ cnt) {
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5, lane = lane_id();
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint32_t a = row_ptr[u], b = row_ptr[u + 1], du = b - a;
        uint32_t c = 0;
        for (uint32_t i = a + lane; i - lane < b; i += 32) {
            bool k = i < b && orient_keep(row_ptr, u, du, __ldg(col_ind + i));
            c += __popc(__ballot_sync(0xffffffffu, k));
        }
        if (lane == 0) cnt[u] = c;
    }
}

__global__ void k_orient_fill(uint32_t n, const uint32_t *__restrict__ row_ptr, const uint32_t *__restrict__ col_ind,
                              const uint32_t *__restrict__ orow_ptr, uint32_t *__restrict__ ocol_ind) {
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5, lane = lane_id();
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint32_t a = row_ptr[u], b = row_ptr[u + 1], du = b - a;
        uint32_t o = orow_ptr[u];
        for (uint32_t i = a + lane; i - lane < b; i += 32) {
            uint32_t v = i < b ? __ldg(col_ind + i) : 0u;
            bool k = i < b && orient_keep(row_ptr, u, du, v);
            uint32_t bal = __ballot_sync(0xffffffffu, k);
            if (k) ocol_ind[o + __popc(bal & ((1u << lane) - 1u))] = v;  // column order is preserved
            o += __popc(bal);
        }
    }
}

static unsigned grid_for(uint64_t work) {
    uint64_t b = (work + 255) / 256, cap = (uint64_t)num_sms() * 32;
    return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

static int bits_for(uint32_t maxval) {
    int b = 0;
    while (b < 32 && (maxval >> b)) b++;
    return b;
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_rmat_edges(int scale, uint64_t m, uint64_t seed, uint32_t *d_src, uint32_t *d_dst, void *stream) {
    API_BEGIN
    if (scale < 1 || scale > 31) B2SR_THROW(B2SR_EINVAL, "scale must be in [1, 31]");
    uint64_t key = 0;
    {  // mix64(seed + golden) on the host, same as the oracle
        uint64_t z = seed + 0x9E3779B97F4A7C15ull;
        z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
        z ^= z >> 27; z *= 0x94D049BB133111EBull;
        key = z ^ (z >> 31);
    }
    LAUNCH(k_rmat, grid_for(m), 256, 0, (cudaStream_t)stream, scale, m, key, d_src, d_dst);
    API_END
}

int b2sr_coo_to_csr(uint32_t n, uint64_t m, const uint32_t *d_src, const uint32_t *d_dst, int symmetrize,
                    int drop_loops, uint32_t *d_row_ptr, uint32_t *d_col_ind, uint64_t *nnz, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    int B = bits_for(n ? n - 1 : 0);
    if (B == 0) B = 1;
    uint64_t k = symmetrize ? 2 * m : m;
    Buf<uint64_t> keys(k, s), alt;
    Buf<uint32_t> deg(n, s);
    Buf<uint64_t> rofs((size_t)n + 1, s);
    CK(cudaMemsetAsync(deg.p, 0, (size_t)n * 4, s));
    uint64_t total = 0;
    if (k) {
        LAUNCH(k_coo_keys, grid_for(m), 256, 0, s, m, d_src, d_dst, B, symmetrize, drop_loops, keys.p);
        uint64_t *sorted = nullptr;
        radix_sort_keys_u64(keys.p, k, 2 * B, s, &sorted, &alt);
        uint64_t dead_key = drop_loops ? (1ull << (2 * B)) - 1 : ~0ull;
        Buf<uint32_t> flag(k, s);
        Buf<uint64_t> ofs(k + 1, s);
        LAUNCH(k_uniq_flags, grid_for(k), 256, 0, s, k, sorted, dead_key, flag.p);
        exclusive_scan_u32_to_u64(flag.p, ofs.p, k, s);
        total = read_scalar(ofs.p + k, s);
        if (total > 0xFFFFFFFFull) B2SR_THROW(B2SR_EFORMAT, "nnz exceeds the 32-bit CSR index range");
        LAUNCH(k_uniq_scatter, grid_for(k), 256, 0, s, k, sorted, flag.p, ofs.p, B, d_col_ind, deg.p);
    }
    exclusive_scan_u32_to_u64(deg.p, rofs.p, n, s);
    LAUNCH(k_to_u32, grid_for((uint64_t)n + 1), 256, 0, s, rofs.p, d_row_ptr, (size_t)n + 1);
    *nnz = total;
    API_END
}

int b2sr_csr_lower_rowptr(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind, uint32_t *d_lrow_ptr,
                          uint64_t *lnnz, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    Buf<uint32_t> cnt(n, s);
    Buf<uint64_t> ofs((size_t)n + 1, s);
    LAUNCH(k_lower_count, grid_for(n), 256, 0, s, n, d_row_ptr, d_col_ind, cnt.p);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, n, s);
    LAUNCH(k_to_u32, grid_for((uint64_t)n + 1), 256, 0, s, ofs.p, d_lrow_ptr, (size_t)n + 1);
    *lnnz = read_scalar(ofs.p + n, s);
    API_END
}

int b2sr_csr_lower_fill(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind, const uint32_t *d_lrow_ptr,
                        uint32_t *d_lcol_ind, void *stream) {
    API_BEGIN
    LAUNCH(k_lower_fill, grid_for((uint64_t)n * 32), 256, 0, (cudaStream_t)stream, n, d_row_ptr, d_col_ind,
           d_lrow_ptr, d_lcol_ind);
    API_END
}

int b2sr_csr_orient_rowptr(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind, uint32_t *d_orow_ptr,
                           uint64_t *onnz, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    Buf<uint32_t> cnt(n, s);
    Buf<uint64_t> ofs((size_t)n + 1, s);
    LAUNCH(k_orient_count, grid_for((uint64_t)n * 32), 256, 0, s, n, d_row_ptr, d_col_ind, cnt.p);
    exclusive_scan_u32_to_u64(cnt.p, ofs.p, n, s);
    LAUNCH(k_to_u32, grid_for((uint64_t)n + 1), 256, 0, s, ofs.p, d_orow_ptr, (size_t)n + 1);
    *onnz = read_scalar(ofs.p + n, s);
    API_END
}

int b2sr_csr_orient_fill(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind, const uint32_t *d_orow_ptr,
                         uint32_t *d_ocol_ind, void *stream) {
    API_BEGIN
    LAUNCH(k_orient_fill, grid_for((uint64_t)n * 32), 256, 0, (cudaStream_t)stream, n, d_row_ptr, d_col_ind,
           d_orow_ptr, d_ocol_ind);
    API_END
}

}  // extern "C"
