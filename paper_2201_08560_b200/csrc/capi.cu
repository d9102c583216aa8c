// Library plumbing: errors, memory, matrix lifecycle, host<->device copies.
// Replaces the host-side container logic of formats.py:228-329 for the
// device-resident B2srMatrix.
#include <mutex>
#include <vector>

#include "b2sr_internal.cuh"

namespace b2sr {

static thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};

KernelTimer &kernel_timer() {
    static thread_local KernelTimer t;
    return t;
}

void KernelTimer::begin(cudaStream_t s) {
    if (!on) return;
    if (!e0) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
    }
    CK(cudaEventRecord(e0, s));
}

void KernelTimer::end(cudaStream_t s) {
    if (!on) return;
    CK(cudaEventRecord(e1, s));
    recorded = true;
}

void set_error(int code, const char *fmt, ...) {
    (void)code;
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_err = buf;
}
void clear_error() { t_err.clear(); }

// Stream-ordered allocations from the device's default pool.  The release
// threshold is raised once per device so freed blocks are reused instead of
// being returned to the driver at every synchronisation.
static std::mutex g_pool_mu;
static bool g_pool_ready[64];

static void ensure_pool() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 64 && !g_pool_ready[dev]) {
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        g_pool_ready[dev] = true;
    }
}

void *dalloc(size_t bytes, cudaStream_t s) {
    ensure_pool();
    void *p = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        B2SR_THROW(B2SR_ENOMEM, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    }
    return p;
}

void dfree(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

int num_sms() {
    static int sms[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && sms[dev]) return sms[dev];
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) sms[dev] = v;
    return v;
}

b2sr_matrix *new_matrix(uint32_t n, uint32_t dim, uint32_t ntr, uint64_t T, cudaStream_t s) {
    b2sr_matrix *m = new b2sr_matrix();
    m->n = n;
    m->dim = dim;
    m->ntr = ntr;
    m->num_tiles = T;
    CK(cudaGetDevice(&m->device));
    try {
        m->trp = static_cast<uint32_t *>(dalloc(((size_t)ntr + 1) * 4, s));
        m->tci = static_cast<uint32_t *>(dalloc(T * 4 + 16, s));
        m->tiles = dalloc(T * (size_t)dim * word_bytes(dim) + 16, s);
    } catch (...) {
        free_matrix(m);
        throw;
    }
    return m;
}

void free_matrix(b2sr_matrix *m) {
    if (!m) return;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != m->device) cudaSetDevice(m->device);
    // Kernels reading this matrix may still be queued on a caller's
    // non-blocking stream, which the NULL-stream frees below are not ordered
    // after: wait for the device first (what a plain cudaFree would do).
    cudaDeviceSynchronize();
    dfree(m->trp, nullptr);
    dfree(m->tci, nullptr);
    dfree(m->tiles, nullptr);
    dfree(m->items, nullptr);
    dfree(m->live, nullptr);
    dfree(m->item_ofs, nullptr);
    free_vlong(m->vlong);
    free_hot(m->hot);
    free_stream(m->stream);
    free_bff(m->bff);
    free_xperm(m->xperm);
    free_csrplan(m->csrplan);
    // let the frees complete now: an allocation on another stream reuses
    // completed frees opportunistically, while pending ones made the pool map
    // fresh memory (s22 d = 32 conversions after a free: 77-101 vs 14 ms)
    cudaStreamSynchronize(nullptr);
    if (cur != m->device) cudaSetDevice(cur);
    delete m;
}

// ---------------------------------------------------------------- kernels
__global__ void k_compare_u32(const uint32_t *a, const uint32_t *b, size_t n, int *diff) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (a[i] != b[i]) { *diff = 1; return; }
}

__global__ void k_compare_bytes(const uint8_t *a, const uint8_t *b, size_t n, int *diff) {
    size_t n16 = n / 16;
    const uint4 *a4 = reinterpret_cast<const uint4 *>(a), *b4 = reinterpret_cast<const uint4 *>(b);
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        uint4 x = a4[i], y = b4[i];
        if (x.x != y.x || x.y != y.y || x.z != y.z || x.w != y.w) { *diff = 1; return; }
    }
    for (size_t i = n16 * 16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
        if (a[i] != b[i]) { *diff = 1; return; }
}

__global__ void k_rebase(const uint32_t *src, uint32_t *dst, uint32_t count, uint32_t base) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= count) dst[i] = src[i] - base;
}

}  // namespace b2sr

using namespace b2sr;

extern "C" {

const char *b2sr_last_error(void) { return t_err.c_str(); }
int b2sr_version(void) { return 100; }
uint64_t b2sr_launch_count(void) { return g_launches.load(); }

int b2sr_set_kernel_timing(int on) {
    API_BEGIN
    kernel_timer().on = on != 0;
    API_END
}

int b2sr_last_kernel_ms(float *ms) {
    API_BEGIN
    KernelTimer &t = kernel_timer();
    if (!t.recorded) B2SR_THROW(B2SR_EINVAL, "no timed kernel recorded (b2sr_set_kernel_timing(1) first)");
    CK(cudaEventSynchronize(t.e1));
    CK(cudaEventElapsedTime(ms, t.e0, t.e1));
    API_END
}

int b2sr_free(b2sr_matrix *m) {
    API_BEGIN
    free_matrix(m);
    API_END
}

int b2sr_info(const b2sr_matrix *m, uint32_t *n, uint32_t *dim, uint32_t *ntr, uint64_t *num_tiles) {
    API_BEGIN
    if (!m) B2SR_THROW(B2SR_EINVAL, "null matrix");
    if (n) *n = m->n;
    if (dim) *dim = m->dim;
    if (ntr) *ntr = m->ntr;
    if (num_tiles) *num_tiles = m->num_tiles;
    API_END
}

int b2sr_row_offset(const b2sr_matrix *m, uint32_t *tr_begin) {
    API_BEGIN
    if (!m) B2SR_THROW(B2SR_EINVAL, "null matrix");
    *tr_begin = m->row0;
    API_END
}

int b2sr_arrays(const b2sr_matrix *m, const uint32_t **trp, const uint32_t **tci, const void **tiles) {
    API_BEGIN
    if (!m) B2SR_THROW(B2SR_EINVAL, "null matrix");
    if (trp) *trp = m->trp;
    if (tci) *tci = m->tci;
    if (tiles) *tiles = m->tiles;
    API_END
}

int b2sr_from_host(uint32_t n, uint32_t dim, const uint32_t *h_trp, const uint32_t *h_tci, const void *h_tiles,
                   uint64_t num_tiles, void *stream, b2sr_matrix **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (dim != 4 && dim != 8 && dim != 16 && dim != 32) B2SR_THROW(B2SR_EINVAL, "tile dim must be 4/8/16/32");
    if (n == 0) B2SR_THROW(B2SR_EFORMAT, "matrix dimension must be positive");
    uint32_t ntr = tile_rows(n, dim);
    b2sr_matrix *m = new_matrix(n, dim, ntr, num_tiles, s);
    try {
        upload_b2sr(m, h_trp, h_tci, h_tiles, s);
    } catch (...) {
        free_matrix(m);
        throw;
    }
    *out = m;
    API_END
}

int b2sr_to_host(const b2sr_matrix *m, uint32_t *h_trp, uint32_t *h_tci, void *h_tiles, void *stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (h_trp) CK(cudaMemcpyAsync(h_trp, m->trp, ((size_t)m->ntr + 1) * 4, cudaMemcpyDeviceToHost, s));
    if (m->num_tiles) {
        if (h_tci) CK(cudaMemcpyAsync(h_tci, m->tci, m->num_tiles * 4, cudaMemcpyDeviceToHost, s));
        if (h_tiles)
            CK(cudaMemcpyAsync(h_tiles, m->tiles, m->num_tiles * m->dim * word_bytes(m->dim),
                               cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    API_END
}

int b2sr_equal(const b2sr_matrix *a, const b2sr_matrix *b, void *stream, int *equal) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    *equal = 0;
    if (a->n != b->n || a->dim != b->dim || a->ntr != b->ntr || a->num_tiles != b->num_tiles) return B2SR_OK;
    Buf<int> diff(1, s);
    CK(cudaMemsetAsync(diff.p, 0, sizeof(int), s));
    int g = num_sms() * 4;
    LAUNCH(k_compare_u32, g, 256, 0, s, a->trp, b->trp, (size_t)a->ntr + 1, diff.p);
    if (a->num_tiles) {
        LAUNCH(k_compare_u32, g, 256, 0, s, a->tci, b->tci, (size_t)a->num_tiles, diff.p);
        LAUNCH(k_compare_bytes, g, 256, 0, s, (const uint8_t *)a->tiles, (const uint8_t *)b->tiles,
               (size_t)a->num_tiles * a->dim * word_bytes(a->dim), diff.p);
    }
    *equal = read_scalar(diff.p, s) == 0;
    API_END
}

int b2sr_row_block(const b2sr_matrix *m, uint32_t tr_begin, uint32_t tr_end, void *stream, b2sr_matrix **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (tr_begin > tr_end || tr_end > m->ntr) B2SR_THROW(B2SR_EINVAL, "row block out of range");
    uint32_t h[2];
    CK(cudaMemcpyAsync(&h[0], m->trp + tr_begin, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h[1], m->trp + tr_end, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint32_t rows = tr_end - tr_begin;
    uint64_t T = h[1] - h[0];
    b2sr_matrix *r = new_matrix(m->n, m->dim, rows, T, s);
    r->row0 = m->row0 + tr_begin;
    LAUNCH(k_rebase, (rows + 256) / 256, 256, 0, s, m->trp + tr_begin, r->trp, rows, h[0]);
    if (T) {
        CK(cudaMemcpyAsync(r->tci, m->tci + h[0], T * 4, cudaMemcpyDeviceToDevice, s));
        size_t tb = (size_t)m->dim * word_bytes(m->dim);
        CK(cudaMemcpyAsync(r->tiles, (const char *)m->tiles + h[0] * tb, T * tb, cudaMemcpyDeviceToDevice, s));
    }
    *out = r;
    API_END
}

int b2sr_block_from_host(uint32_t n, uint32_t dim, uint32_t tr_begin, uint32_t tr_end, const uint32_t *h_trp,
                         const uint32_t *h_tci, const void *h_tiles, uint64_t num_tiles, void *stream,
                         b2sr_matrix **out) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    if (dim != 4 && dim != 8 && dim != 16 && dim != 32) B2SR_THROW(B2SR_EINVAL, "tile dim must be 4/8/16/32");
    if (n == 0) B2SR_THROW(B2SR_EFORMAT, "matrix dimension must be positive");
    if (tr_begin > tr_end || tr_end > tile_rows(n, dim)) B2SR_THROW(B2SR_EINVAL, "row block out of range");
    uint32_t rows = tr_end - tr_begin;
    b2sr_matrix *m = new_matrix(n, dim, rows, num_tiles, s);
    m->row0 = tr_begin;
    try {
        upload_b2sr(m, h_trp, h_tci, h_tiles, s);  // trp: rows + 1 entries (m->ntr = rows)
    } catch (...) {
        free_matrix(m);
        throw;
    }
    *out = m;
    API_END
}

}  // extern "C"
