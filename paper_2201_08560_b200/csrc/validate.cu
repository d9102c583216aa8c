// B2SR invariants checked on the device (formats.py:242-295), for matrices
// that arrive as raw arrays -- the .b2sr container (formats.py:517-554) or a
// caller's host arrays -- so a multi-GB matrix is validated at HBM speed
// instead of the reference's O(T*d) numpy passes.  The first violated
// invariant in the reference's order is reported with its message.
#include "b2sr_internal.cuh"

namespace b2sr {

enum : uint32_t {
    V_START = 1u << 0,      // tile_row_ptr[0] != 0
    V_MONO = 1u << 1,       // tile_row_ptr decreases
    V_LAST = 1u << 2,       // tile_row_ptr[ntr] != T
    V_COLRANGE = 1u << 3,   // tile column >= ntr
    V_ORDER = 1u << 4,      // tile columns not strictly increasing within a row
    V_EMPTY = 1u << 5,      // a stored tile without set bits
    V_NIBBLE = 1u << 6,     // d = 4 word with the high nibble set
    V_PADROW = 1u << 7,     // bits in the padding bit-rows of the last tile row
    V_PADCOL = 1u << 8,     // bits in the padding bit-columns of the last tile column
};

static const char *violation_message(uint32_t bit) {
    switch (bit) {
        case V_START: return "tile_row_ptr must start at 0";
        case V_MONO: return "tile_row_ptr must be non-decreasing";
        case V_LAST: return "tile_row_ptr[-1] must equal the tile count";
        case V_COLRANGE: return "tile column index out of range";
        case V_ORDER: return "tile columns must be strictly increasing within a tile row";
        case V_EMPTY: return "stored tiles must contain at least one set bit";
        case V_NIBBLE: return "4-wide tiles must keep the high nibble clear";
        case V_PADROW: return "padding bit-rows must be zero";
        default: return "padding bit-columns must be zero";
    }
}

// row pointer: start, monotone, last; segment starts into a bitmap over tiles
__global__ void k_check_rows(uint32_t ntr, uint64_t T, const uint32_t *__restrict__ trp, uint32_t *__restrict__ starts,
                             uint32_t *__restrict__ flags) {
    uint32_t f = 0;
    for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I <= ntr; I += gridDim.x * blockDim.x) {
        const uint32_t p = trp[I];
        if (I == 0 && p != 0) f |= V_START;
        if (I > 0 && p < trp[I - 1]) f |= V_MONO;
        if (I == ntr && (uint64_t)p != T) f |= V_LAST;
        if (I > 0 && I < ntr && p > 0 && (uint64_t)p < T) atomicOr(starts + (p >> 5), 1u << (p & 31));
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane_id() == 0 && f) atomicOr(flags, f);
}

template <typename W>
__global__ void k_check_tiles(uint64_t T, uint32_t ntr, uint32_t d, uint32_t n, const uint32_t *__restrict__ tci,
                              const W *__restrict__ tiles, const uint32_t *__restrict__ starts,
                              uint32_t *__restrict__ flags) {
    const uint32_t pad = ntr * d - n;
    const uint32_t colmask = pad ? (~((1u << (d - pad)) - 1u)) & (d == 32 ? 0xFFFFFFFFu : ((1u << d) - 1u)) : 0u;
    uint32_t f = 0;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = tci[t];
        if (c >= ntr) f |= V_COLRANGE;
        if (t > 0 && !((starts[t >> 5] >> (t & 31)) & 1u) && c <= tci[t - 1]) f |= V_ORDER;
        uint32_t any = 0;
        for (uint32_t r = 0; r < d; r++) {
            const uint32_t w = tiles[t * d + r];
            any |= w;
            if (d == 4 && (w & 0xF0u)) f |= V_NIBBLE;
            if (c == ntr - 1 && (w & colmask)) f |= V_PADCOL;
        }
        if (!any) f |= V_EMPTY;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane_id() == 0 && f) atomicOr(flags, f);
}

// padding bit-rows: the tiles of the last tile row, rows d-pad .. d-1
template <typename W>
__global__ void k_check_pad_rows(uint32_t t0, uint32_t t1, uint32_t d, uint32_t pad, const W *__restrict__ tiles,
                                 uint32_t *__restrict__ flags) {
    uint32_t f = 0;
    for (uint32_t t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x)
        for (uint32_t r = d - pad; r < d; r++)
            if (tiles[(size_t)t * d + r]) f |= V_PADROW;
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane_id() == 0 && f) atomicOr(flags, f);
}

// all invariants; returns the violation bits (0 = valid)
static uint32_t validate(const b2sr_matrix *m, cudaStream_t s) {
    const uint32_t ntr = m->ntr, d = m->dim, n = m->n;
    const uint64_t T = m->num_tiles;
    Buf<uint32_t> flags(1, s), starts(T / 32 + 1, s);
    CK(cudaMemsetAsync(flags.p, 0, 4, s));
    CK(cudaMemsetAsync(starts.p, 0, (T / 32 + 1) * 4, s));
    const unsigned cap = (unsigned)num_sms() * 8;
    LAUNCH(k_check_rows, std::min<unsigned>(cap, (ntr + 256) / 256), 256, 0, s, ntr, T, m->trp, starts.p, flags.p);
    uint32_t f = read_scalar(flags.p, s);
    if (f) return f;  // the row pointer is unusable: report it before anything indexed by it
    if (T) {
        const unsigned g = (unsigned)std::min<uint64_t>(cap, (T + 255) / 256);
        switch (word_bytes(d)) {
            case 1: LAUNCH(k_check_tiles<uint8_t>, g, 256, 0, s, T, ntr, d, n, m->tci, (const uint8_t *)m->tiles, starts.p, flags.p); break;
            case 2: LAUNCH(k_check_tiles<uint16_t>, g, 256, 0, s, T, ntr, d, n, m->tci, (const uint16_t *)m->tiles, starts.p, flags.p); break;
            default: LAUNCH(k_check_tiles<uint32_t>, g, 256, 0, s, T, ntr, d, n, m->tci, (const uint32_t *)m->tiles, starts.p, flags.p); break;
        }
        const uint32_t pad = ntr * d - n;
        if (pad) {
            uint32_t h[2];
            CK(cudaMemcpyAsync(h, m->trp + ntr - 1, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (h[1] > h[0]) {
                const unsigned gp = std::min<unsigned>(cap, (h[1] - h[0] + 255) / 256);
                switch (word_bytes(d)) {
                    case 1: LAUNCH(k_check_pad_rows<uint8_t>, gp, 256, 0, s, h[0], h[1], d, pad, (const uint8_t *)m->tiles, flags.p); break;
                    case 2: LAUNCH(k_check_pad_rows<uint16_t>, gp, 256, 0, s, h[0], h[1], d, pad, (const uint16_t *)m->tiles, flags.p); break;
                    default: LAUNCH(k_check_pad_rows<uint32_t>, gp, 256, 0, s, h[0], h[1], d, pad, (const uint32_t *)m->tiles, flags.p); break;
                }
            }
        }
        f = read_scalar(flags.p, s);
    }
    return f;
}

static void throw_first(uint32_t f) {
    for (uint32_t bit = 1; bit <= V_PADCOL; bit <<= 1)
        if (f & bit) B2SR_THROW(B2SR_EFORMAT, "%s", violation_message(bit));
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

int b2sr_validate(const b2sr_matrix *m, void *stream) {
    API_BEGIN
    if (m->row0 != 0) B2SR_THROW(B2SR_EINVAL, "b2sr_validate needs a full matrix");
    throw_first(validate(m, (cudaStream_t)stream));
    API_END
}

int b2sr_from_host_checked(uint32_t n, uint32_t dim, const uint32_t *h_trp, const uint32_t *h_tci,
                           const void *h_tiles, uint64_t num_tiles, void *stream, b2sr_matrix **out) {
    API_BEGIN
    b2sr_matrix *m = nullptr;
    int rc = b2sr_from_host(n, dim, h_trp, h_tci, h_tiles, num_tiles, stream, &m);
    if (rc) return rc;
    try {
        throw_first(validate(m, (cudaStream_t)stream));
    } catch (...) {
        free_matrix(m);
        throw;
    }
    *out = m;
    API_END
}

}  // extern "C"
