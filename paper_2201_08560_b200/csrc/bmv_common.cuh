// Shared device helpers of the bin-SpMV family (bmv.cu, bmv_stream.cu, drivers.cu).
#pragma once

#include <algorithm>

#include "b2sr_internal.cuh"

namespace b2sr {

// Lane geometry of a 128-bit load over tiles of width D.
template <int D> struct Geo {
    static constexpr int WB = D == 32 ? 4 : (D == 16 ? 2 : 1);
    static constexpr int TB = D * WB;                    // tile bytes
    static constexpr int TPL = TB >= 16 ? 1 : 16 / TB;   // tiles per lane load
    static constexpr int LPT = TB >= 16 ? TB / 16 : 1;   // lanes per tile
    static constexpr int TPW = 32 * TPL / LPT;           // tiles per warp load
    static constexpr uint32_t CHUNK = 64 * TPW;          // tiles per work item
};

// d=4: bit r set when byte r of v is non-zero (bytes carry a low nibble only:
// byte + 0x0F sets bit 4 iff the byte is non-zero and never carries into the
// next byte; the multiply moves bits 4/12/20/28 to 28..31 without collisions)
__device__ __forceinline__ uint32_t nz_nibble_bytes(uint32_t v) {
    return (((v + 0x0F0F0F0Fu) & 0x10101010u) * 0x01020408u) >> 28;
}
// full-byte variant (d=8 rows): bit 7 of ((b & 0x7F) + 0x7F) | b is set iff
// b != 0; bits 7/15/23/31 -> 28..31
__device__ __forceinline__ uint32_t nz_bytes(uint32_t v) {
    return (((((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v) & 0x80808080u) * 0x00204081u) >> 28;
}
// per-byte popcounts packed in the bytes of a u32
__device__ __forceinline__ uint32_t popc_bytes(uint32_t v) {
    v = v - ((v >> 1) & 0x55555555u);
    v = (v & 0x33333333u) + ((v >> 2) & 0x33333333u);
    return (v + (v >> 4)) & 0x0F0F0F0Fu;
}

// Hit bits (positions within the tile-row word) of the 16 bytes a lane holds.
// xw[j] = x word of the j-th tile in the lane (0 for tiles outside the range).
template <int D>
__device__ __forceinline__ uint32_t hits16(uint4 v, const uint32_t *xw, uint32_t lane) {
    if constexpr (D == 4) {
        return nz_nibble_bytes(v.x & (xw[0] * 0x01010101u)) | nz_nibble_bytes(v.y & (xw[1] * 0x01010101u)) |
               nz_nibble_bytes(v.z & (xw[2] * 0x01010101u)) | nz_nibble_bytes(v.w & (xw[3] * 0x01010101u));
    } else if constexpr (D == 8) {
        uint32_t x0 = xw[0] * 0x01010101u, x1 = xw[1] * 0x01010101u;
        uint32_t lo = nz_bytes(v.x & x0) | nz_bytes(v.z & x1);
        uint32_t hi = nz_bytes(v.y & x0) | nz_bytes(v.w & x1);
        return lo | (hi << 4);
    } else if constexpr (D == 16) {
        uint32_t xr = xw[0] | (xw[0] << 16), w[4] = {v.x, v.y, v.z, v.w}, a = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            uint32_t y = w[i] & xr;
            a |= ((y & 0xFFFFu) ? 1u : 0u) << (2 * i);
            a |= ((y >> 16) ? 1u : 0u) << (2 * i + 1);
        }
        return a << (8 * (lane & 1));
    } else {
        uint32_t x = xw[0], a = 0;
        a |= (v.x & x) ? 1u : 0u;
        a |= (v.y & x) ? 2u : 0u;
        a |= (v.z & x) ? 4u : 0u;
        a |= (v.w & x) ? 8u : 0u;
        return a << (4 * (lane & 7));
    }
}

// Raise a kernel's dynamic shared-memory limit (idempotent, cheap).
void hot_smem_attr_raw(const void *kernel, size_t bytes);  // hot.cu: per-kernel, cached
template <typename K>
inline void hot_smem_attr(K kernel, size_t bytes) {
    hot_smem_attr_raw(reinterpret_cast<const void *>(kernel), bytes);
}

// x-word gathers used by the streaming kernels: plain global loads with a
// selectable cache policy, or the hot-column cache (hot.cu) in shared memory
template <int D>
struct XGlobal {
    const void *x;
    __device__ __forceinline__ uint32_t operator()(uint32_t c) const { return load_word<D>(x, c); }
};
// The hot words live in the kernel's dynamic shared memory; indexing the
// extern array directly lets ptxas address it with LDS immediates instead of
// re-deriving a generic->shared pointer for every gather.
__device__ __forceinline__ const uint8_t *hot_bytes() {
    extern __shared__ uint4 hot_dyn_smem[];
    return reinterpret_cast<const uint8_t *>(hot_dyn_smem);
}

template <int D>
struct XHot {
    uint32_t sbase;                        // shared-window address of the hot words
    const typename WordT<D>::T *xm;        // x - S: cold column c (>= S) reads xm[c]
    uint32_t S;
    __device__ __forceinline__ XHot(const void *x, uint32_t s)
        : xm(reinterpret_cast<const typename WordT<D>::T *>(x) - s), S(s) {
        // opaque to ptxas, so the base stays in a register instead of being
        // re-derived (S2R CgaCtaId + LEA) before every LDS
        asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(sbase) : "l"(hot_bytes()));
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t c) const {
        uint32_t v;
        if (c < S) {
            if constexpr (D == 4 && HOT_NIBBLES) {  // two 4-bit words per byte (hot.cu packs them)
                asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(sbase + (c >> 1)));
                // the other column's nibble may stay in bits 4-7: every consumer
                // ANDs with 4-wide tile bytes, whose high nibbles are clear
                return v >> ((c & 1u) * 4u);
            } else if constexpr (sizeof(typename WordT<D>::T) == 1) {
                asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(sbase + c));
            } else if constexpr (sizeof(typename WordT<D>::T) == 2) {
                unsigned short h;
                asm("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(sbase + 2 * c));
                v = h;
            } else {
                asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase + 4 * c));
            }
            return v;
        }
        if constexpr (sizeof(typename WordT<D>::T) == 1) {
            // cold column: one IMAD.WIDE (xm + c) and the load -- the plain
            // expression compiled to c - S, then a 64-bit add of x (4 instructions)
            unsigned long long a;
            asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(a) : "r"(c), "l"(reinterpret_cast<unsigned long long>(xm)));
            asm("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(a));
            return v;
        }
        return (uint32_t)__ldg(xm + c);
    }
};

// Copy the hot words (hot_fill output, 16-byte padded) into shared memory;
// all threads of the CTA take part, the caller syncs.
__device__ __forceinline__ void stage_hot(void *smem, const void *hx, uint32_t bytes16) {
    const uint4 *src = static_cast<const uint4 *>(hx);
    uint4 *dst = static_cast<uint4 *>(smem);
    const uint32_t n = bytes16 / 16;
    uint32_t i = threadIdx.x;
    for (; i + 3 * blockDim.x < n; i += 4 * blockDim.x) {
        uint4 a = __ldg(src + i), b = __ldg(src + i + blockDim.x), c = __ldg(src + i + 2 * blockDim.x),
              d = __ldg(src + i + 3 * blockDim.x);
        dst[i] = a;
        dst[i + blockDim.x] = b;
        dst[i + 2 * blockDim.x] = c;
        dst[i + 3 * blockDim.x] = d;
    }
    for (; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

}  // namespace b2sr
