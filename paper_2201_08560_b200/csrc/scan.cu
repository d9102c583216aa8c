// Device-wide exclusive prefix sums (reduce-then-scan, 4096 items per CTA).
// Used for tile_row_ptr (formats.py:457-459 bincount/cumsum), work-item
// offsets and CSR row pointers.
#include "b2sr_internal.cuh"

namespace b2sr {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ __forceinline__ uint64_t block_sum(uint64_t v, uint64_t *smem) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) smem[w] = v;
    __syncthreads();
    uint64_t t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < SCAN_THREADS / 32 ? smem[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;  // valid in warp 0
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const T *in, size_t n, uint64_t *partial) {
    __shared__ uint64_t sm[SCAN_THREADS / 32];
    size_t base = (size_t)blockIdx.x * SCAN_TILE;
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        size_t i = base + (size_t)j * SCAN_THREADS + threadIdx.x;
        if (i < n) acc += (uint64_t)in[i];
    }
    uint64_t t = block_sum<T>(acc, sm);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// Exclusive scan of one tile; `offset` (from the scanned partials) is added.
template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile(const T *in, size_t n, const uint64_t *offsets,
                                                             uint64_t *out) {
    __shared__ uint64_t sm[SCAN_THREADS / 32];
    size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    uint64_t v[SCAN_ITEMS];
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        size_t i = base + j;
        v[j] = i < n ? (uint64_t)in[i] : 0;
        acc += v[j];
    }
    // block exclusive scan of per-thread sums
    uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = acc;
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
    }
    if (lane == 31) sm[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint64_t s = lane < SCAN_THREADS / 32 ? sm[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= (uint32_t)o) s += y;
        }
        if (lane < SCAN_THREADS / 32) sm[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    uint64_t run = (offsets ? offsets[blockIdx.x] : 0) + (w ? sm[w - 1] : 0) + inc - acc;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        size_t i = base + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
    if (base <= n && n < base + SCAN_ITEMS) out[n] = run;  // total, written by the owner of slot n
}

template <typename T>
static void scan_impl(const T *in, uint64_t *out, size_t n, cudaStream_t s) {
    size_t blocks = (n + SCAN_TILE) / SCAN_TILE;  // +1 slot so out[n] has an owner
    if (blocks == 1) {
        LAUNCH(k_scan_tile<T>, 1, SCAN_THREADS, 0, s, in, n, (const uint64_t *)nullptr, out);
        return;
    }
    Buf<uint64_t> part(blocks, s), poff(blocks + 1, s);
    LAUNCH(k_scan_reduce<T>, (unsigned)blocks, SCAN_THREADS, 0, s, in, n, part.p);
    scan_impl<uint64_t>(part.p, poff.p, blocks, s);
    LAUNCH(k_scan_tile<T>, (unsigned)blocks, SCAN_THREADS, 0, s, in, n, (const uint64_t *)poff.p, out);
}

void exclusive_scan_u32_to_u64(const uint32_t *in, uint64_t *out, size_t n, cudaStream_t s) {
    scan_impl<uint32_t>(in, out, n, s);
}
void exclusive_scan_u64(const uint64_t *in, uint64_t *out, size_t n, cudaStream_t s) {
    scan_impl<uint64_t>(in, out, n, s);
}

}  // namespace b2sr
