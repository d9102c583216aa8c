// Internal helpers shared by the sm_100a translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <functional>
#include <mutex>
#include <string>

#include "b2sr_sm100.h"

namespace b2sr {

// ---------------------------------------------------------------- errors
struct Error {
    int code;
    std::string msg;
};

void set_error(int code, const char *fmt, ...);
void clear_error();

// Thrown only inside the library; every extern "C" entry point catches it
// (see API_BEGIN / API_END) and turns it into a status code.
#define B2SR_THROW(code, ...)                                  \
    do {                                                       \
        ::b2sr::set_error((code), __VA_ARGS__);                \
        throw ::b2sr::Error{(code), std::string()};            \
    } while (0)

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            int c_ = (e_ == cudaErrorMemoryAllocation) ? B2SR_ENOMEM : B2SR_ECUDA;             \
            B2SR_THROW(c_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,   \
                       __LINE__);                                                              \
        }                                                                                      \
    } while (0)

#define API_BEGIN \
    ::b2sr::clear_error(); \
    try {
#define API_END                                                                  \
    }                                                                            \
    catch (const ::b2sr::Error &e) {                                             \
        return e.code;                                                           \
    }                                                                            \
    catch (...) {                                                                \
        ::b2sr::set_error(B2SR_ECUDA, "unexpected C++ exception in b2sr");       \
        return B2SR_ECUDA;                                                       \
    }                                                                            \
    return B2SR_OK;

// ---------------------------------------------------------------- launches
extern std::atomic<uint64_t> g_launches;
// Programmatic dependent launch: the kernel may be scheduled while its
// predecessor in the stream drains (it must start with pdl_prologue(), which
// waits for the predecessor's completion and memory before anything is read).
// Used between the back-to-back kernels of the device-controlled BFS levels.
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
#define LAUNCH_PDL(pdl, kernel, grid, block, smem, strm_, ...)                                   \
    do {                                                                                          \
        if ((grid) > 0) {                                                                         \
            cudaLaunchConfig_t cfg_{};                                                            \
            cfg_.gridDim = dim3(grid);                                                            \
            cfg_.blockDim = dim3(block);                                                          \
            cfg_.dynamicSmemBytes = (smem);                                                       \
            cfg_.stream = (strm_);                                                                \
            cudaLaunchAttribute at_[1];                                                           \
            at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                       \
            at_[0].val.programmaticStreamSerializationAllowed = 1;                                \
            cfg_.attrs = at_;                                                                     \
            cfg_.numAttrs = (pdl) ? 1 : 0;                                                        \
            CK(cudaLaunchKernelEx(&cfg_, kernel, __VA_ARGS__));                                   \
            ::b2sr::g_launches.fetch_add(1, std::memory_order_relaxed);                           \
        }                                                                                         \
    } while (0)

#define LAUNCH(kernel, grid, block, smem, stream, ...)                     \
    do {                                                                   \
        if ((grid) > 0) {                                                  \
            kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);    \
            ::b2sr::g_launches.fetch_add(1, std::memory_order_relaxed);    \
            CK(cudaGetLastError());                                        \
        }                                                                  \
    } while (0)

// Per-thread CUDA-event bracket around one streaming kernel (b2sr_set_kernel_timing).
struct KernelTimer {
    bool on = false, recorded = false;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    void begin(cudaStream_t s);
    void end(cudaStream_t s);
};
KernelTimer &kernel_timer();

// ---------------------------------------------------------------- memory
void *dalloc(size_t bytes, cudaStream_t s);
void dfree(void *p, cudaStream_t s);

// Stream-ordered scratch buffer (freed on scope exit).
template <typename T>
struct Buf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    Buf() = default;
    Buf(size_t count, cudaStream_t st) : n(count), s(st) {
        p = static_cast<T *>(dalloc(count * sizeof(T) + 16, st));
    }
    Buf(const Buf &) = delete;
    Buf &operator=(const Buf &) = delete;
    Buf(Buf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; }
    Buf &operator=(Buf &&o) noexcept {
        reset();
        p = o.p; n = o.n; s = o.s; o.p = nullptr;
        return *this;
    }
    ~Buf() { reset(); }
    void reset() {
        if (p) dfree(p, s);
        p = nullptr;
    }
    T *release() {
        T *q = p;
        p = nullptr;
        return q;
    }
    T *get() const { return p; }
};

template <typename T>
T read_scalar(const T *dptr, cudaStream_t s) {
    T v;
    CK(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
}

// ---------------------------------------------------------------- matrix
struct WorkItem {      // one bin-SpMV work unit: tiles [t0, t1) of local tile row `row`
    uint32_t row;
    uint32_t t0;
    uint32_t t1;
    uint32_t split;    // 1 when the row is shared with other items (atomic store)
};

}  // namespace b2sr

struct b2sr_matrix {
    // lazily built per-matrix plans (items, stream, hot, bff, vlong, xperm,
    // live) are created under this lock: the C ABI is re-entrant and callers
    // may share a matrix across host threads
    std::recursive_mutex plan_mu;
    uint32_t n = 0;          // logical dimension (global)
    uint32_t dim = 0;        // tile width 4/8/16/32
    uint32_t ntr = 0;        // tile rows stored here (== ceil(n/dim) unless a row block)
    uint32_t row0 = 0;       // first global tile row (row blocks)
    uint64_t num_tiles = 0;
    uint32_t *trp = nullptr; // ntr + 1, local offsets starting at 0
    uint32_t *tci = nullptr; // num_tiles
    void *tiles = nullptr;   // num_tiles * dim words
    int device = 0;
    // cached bin-SpMV work partition (built lazily, immutable matrix)
    b2sr::WorkItem *items = nullptr;
    uint32_t n_items = 0;
    bool any_split = false;
    // cached row-liveness words (bit r of word I: bit-row I*dim+r holds any
    // set bit), same layout as a BitVector; BFS never needs to wait for a
    // vertex without in-edges
    void *live = nullptr;
    uint64_t live_tiles = 0;          // tiles in rows with a live bit (set with `live`)
    uint32_t *item_ofs = nullptr;     // ntr+1: first work item of each tile row (with `items`)
    void *vlong = nullptr;            // segmented plan for the very longest rows (bmv_vlong.cu)
    void *hot = nullptr;              // hot-column x cache plan (hot.cu)
    void *stream = nullptr;           // flat tile-stream row hints (bmv_stream.cu)
    void *bff = nullptr;              // float-gather row order (bmv_bff.cu)
    void *xperm = nullptr;            // hot-first x relabelling for the float gather (bmv_xperm.cu)
    void *csrplan = nullptr;          // CSR column lists for the wide-tile float gather (bmv_csr.cu)
};

namespace b2sr {

// The built-in add identity of a semiring (semirings.py:54-63): +inf for
// min-plus, 0 otherwise.  Public Semiring objects may carry any identity
// (b2sr_bmv_bff_ex passes it through).
inline double ring_identity(int ring) {
    return ring == B2SR_RING_MINPLUS ? __builtin_huge_val() : 0.0;
}

inline int word_bytes(int d) { return d == 32 ? 4 : (d == 16 ? 2 : 1); }
inline uint32_t tile_rows(uint32_t n, uint32_t d) { return (n + d - 1) / d; }
inline size_t padded_vec_bytes(uint32_t ntr, int d) { return ((size_t)ntr * word_bytes(d) + 3) / 4 * 4; }

b2sr_matrix *new_matrix(uint32_t n, uint32_t dim, uint32_t ntr, uint64_t T, cudaStream_t s);
void free_matrix(b2sr_matrix *m);
b2sr_matrix *transpose_device(const b2sr_matrix *m, cudaStream_t s);  // transpose.cu
void ensure_items(b2sr_matrix *m, cudaStream_t s);  // bin-SpMV work partition
int num_sms();
// host -> device copy; pageable sources are staged through page-locked
// chunks at the link rate (staging.cu)
void h2d(void *dst, const void *src, size_t bytes, cudaStream_t s);
// the arrays of a host B2SR matrix into m's device arrays in one staged upload
// (d = 4 tiles nibble-packed on the way; staging.cu)
void upload_b2sr(b2sr_matrix *m, const uint32_t *h_trp, const uint32_t *h_tci, const void *h_tiles, cudaStream_t s);
void launch_row_ids(const b2sr_matrix *m, uint32_t *rowid, cudaStream_t s);  // rowid[t] = tile row of t
void free_vlong(void *plan);
void *build_vlong(b2sr_matrix *m, uint32_t thresh, cudaStream_t s);
void launch_vlong(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                  cudaStream_t s, const std::function<void(cudaStream_t)> &overlap = {}, const uint32_t *gtci = nullptr);
// hot.cu: the S most referenced tile columns' x words live in shared memory
constexpr uint32_t HOT_SMEM_BYTES = 131072;  // 128 KB: the rest of the 228 KB stays L1 for the cold gathers and streams
constexpr bool HOT_NIBBLES = true;   // d=4: pack two 4-bit x words per byte (2x the slots, more ALU per gather)
struct HotView {
    uint32_t S;               // slots; tci2 values < S are slots, others S + column
    const uint32_t *cols;     // slot -> tile column (null: identity)
    const uint32_t *tci2;     // remapped tile-column indices
};
HotView hot_view(b2sr_matrix *m, cudaStream_t s);
void free_hot(void *plan);
size_t hot_fill_bytes(const HotView &hv, int dim);
void hot_fill(const HotView &hv, int dim, const void *x, void *hx, cudaStream_t s);
bool hot_enabled(int dim);
// bmv_stream.cu: flat tile-stream K4 (d = 4, 8)
bool stream_enabled(int dim);
// visited != null: BFS pull (y &= ~visited & live instead of keep)
// active_only (with visited): only the loads that hold a row with an unvisited live vertex
// K5 bbf (bmv.cu): y f64 per local row
void launch_bbf(b2sr_matrix *m, const void *x, const void *keep, double *y, cudaStream_t s);
void launch_bbb_stream(b2sr_matrix *m, const void *x, const void *keep, void *y, cudaStream_t s,
                       const void *visited = nullptr, bool active_only = false, bool lazy = false);
void free_stream(void *plan);
// bmv_bff.cu: float gather over the rows with <= thresh tiles
// gtci: the column array the gathers index x with (m->tci, or the relabelled
// one of bmv_xperm.cu with x relabelled to match)
void launch_bff_rows(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                     uint32_t thresh, cudaStream_t s, bool plan_only = false, const uint32_t *gtci = nullptr);
void free_bff(void *plan);
// bmv_csr.cu: the float gather at d = 16/32 over the matrix's cached CSR form
bool bff_csr_enabled(const b2sr_matrix *m);
void launch_bff_csr(b2sr_matrix *m, const double *x, int ring, double inc, double ident, const void *keep, double *y,
                    cudaStream_t s);
void free_csrplan(void *plan);
// bmv_xperm.cu: hot-first relabelling of x for the float gather
bool xperm_enabled(const b2sr_matrix *m);
const uint32_t *xperm_apply(b2sr_matrix *m, const double *x, double *xp, cudaStream_t s);
const uint32_t *xperm_apply_u32(b2sr_matrix *m, const uint32_t *x, uint32_t *xp, cudaStream_t s);  // d = 4, 8
void free_xperm(void *plan);
const uint4 *stream_desc(b2sr_matrix *m, cudaStream_t s, uint32_t *n_loads);  // per-load row descriptors
void launch_stream_sweep(b2sr_matrix *m, const uint32_t *list, const uint32_t *list_n, const void *hx, size_t hb,
                         const void *x, void *y, const int *gate, int want, cudaStream_t s, bool lazy = false);

// scan.cu
// out[i] = sum_{j<i} in[j] for i in [0, n]; out has n+1 entries (out[n] = total).
void exclusive_scan_u32_to_u64(const uint32_t *in, uint64_t *out, size_t n, cudaStream_t s);
void exclusive_scan_u64(const uint64_t *in, uint64_t *out, size_t n, cudaStream_t s);
// sort.cu: stable LSD radix sort over the low `bits` bits of keys (values optional).
size_t radix_sort_pairs_u32(uint32_t *keys, uint32_t *vals, size_t n, int bits, cudaStream_t s,
                            uint32_t **keys_out, uint32_t **vals_out, Buf<uint32_t> *kalt,
                            Buf<uint32_t> *valt);
// keys per CTA tile of the radix passes (sort.cu); counts0, when given, holds
// the first pass's per-tile digit counts (digit-major, RADIX_TILE keys per tile)
constexpr int RADIX_TILE = 2048;
void radix_sort_unpack4(uint64_t *keys, size_t n, int bits, uint32_t ntr, uint32_t *trp, uint32_t *tci,
                        uint32_t *tiles, cudaStream_t s, const uint32_t *counts0 = nullptr);
void radix_sort_ids(uint64_t *keys, uint32_t *vals, size_t n, int bits, cudaStream_t s, const uint32_t *counts0,
                    Buf<uint64_t> *kalt, Buf<uint32_t> *valt, uint64_t **kres, uint32_t **vres);
void radix_sort_unpack8(uint64_t *keys, uint64_t *vals, size_t n, int bits, uint32_t ntr, uint32_t *trp, uint32_t *tci,
                        uint64_t *tiles, cudaStream_t s, const uint32_t *counts0 = nullptr);
void radix_sort_keys_u64(uint64_t *keys, size_t n, int bits, cudaStream_t s, uint64_t **keys_out,
                         Buf<uint64_t> *kalt);

// ---------------------------------------------------------------- device helpers
template <int D> struct WordT;
template <> struct WordT<4> { using T = uint8_t; };
template <> struct WordT<8> { using T = uint8_t; };
template <> struct WordT<16> { using T = uint16_t; };
template <> struct WordT<32> { using T = uint32_t; };

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T ldg_nc(const T *p) { return __ldg(p); }

// Streaming 128-bit load that does not allocate in L1 (tiles are read once).
__device__ __forceinline__ uint4 ld_stream128(const void *p) {
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream32(const void *p) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// 32-bit shared-window addresses kept in registers: ptxas otherwise re-derives
// the base of every static __shared__ array (S2R CgaCtaId + LEA) inside hot
// loops.  The accessors are volatile with a memory clobber, so they stay
// ordered with barriers and with each other.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    uint32_t a;
    asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
    return a;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long lds_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}

#define B2SR_PLAN_LOCK(m) std::lock_guard<std::recursive_mutex> b2sr_plan_guard_((m)->plan_mu)

// Valid-bit mask of bit-vector word w (formats.py:433-441).
__device__ __forceinline__ uint32_t valid_mask(uint32_t w, uint32_t n, int d) {
    uint32_t full = d == 32 ? 0xFFFFFFFFu : ((1u << d) - 1u);
    uint64_t lo = (uint64_t)w * d;
    if (lo + d <= n) return full;
    if (lo >= n) return 0u;
    return (1u << (n - lo)) - 1u;
}

template <int D>
__device__ __forceinline__ uint32_t load_word(const void *v, uint32_t i) {
    return (uint32_t)(reinterpret_cast<const typename WordT<D>::T *>(v))[i];
}

// OR `val` into bit-vector word i of width D using a 32-bit atomic.
template <int D>
__device__ __forceinline__ void atomic_or_word(void *v, uint32_t i, uint32_t val) {
    constexpr int WB = D == 32 ? 4 : (D == 16 ? 2 : 1);
    size_t byte = (size_t)i * WB;
    uint32_t *base = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(v) + (byte & ~(size_t)3));
    atomicOr(base, val << (8 * (byte & 3)));
}

}  // namespace b2sr
