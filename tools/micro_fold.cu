// Microbenchmark (tools only): cycles per term of one warp folding a long
// float64 region in order (the hub fold of K6), several feeding strategies.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fold_smem(const double *p, int nt, double *out, long long *cyc) {
    __shared__ double2 sb2[16];
    double *sb = reinterpret_cast<double *>(sb2);
    int lane = threadIdx.x;
    long long t0 = clock64();
    double acc = 0.0;
    double c0 = p[lane], c1 = p[32 + lane], c2 = p[64 + lane], c3 = p[96 + lane];
    for (int q = 0; q < nt; q += 32) {
        double c4 = q + 128 + lane < nt ? p[q + 128 + lane] : 0.0;
        __syncwarp();
        sb[lane] = c0;
        __syncwarp();
        double2 t[16];
#pragma unroll
        for (int j = 0; j < 16; j++) t[j] = sb2[j];
#pragma unroll
        for (int j = 0; j < 16; j++) { acc = __dadd_rn(acc, t[j].x); acc = __dadd_rn(acc, t[j].y); }
        c0 = c1; c1 = c2; c2 = c3; c3 = c4;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}

__global__ void fold_bcast(const double *p, int nt, double *out, long long *cyc) {
    // every lane loads the same 16-byte pairs (broadcast), two chunks in flight
    int lane = threadIdx.x;
    long long t0 = clock64();
    double acc = 0.0;
    const double2 *v = reinterpret_cast<const double2 *>(p);
    double2 a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = __ldg(v + j);
    for (int q = 0; q < nt / 2; q += 16) {
#pragma unroll
        for (int j = 0; j < 8; j++) b[j] = __ldg(v + q + 8 + j);
#pragma unroll
        for (int j = 0; j < 8; j++) { acc = __dadd_rn(acc, a[j].x); acc = __dadd_rn(acc, a[j].y); }
#pragma unroll
        for (int j = 0; j < 8; j++) a[j] = __ldg(v + q + 16 + j);
#pragma unroll
        for (int j = 0; j < 8; j++) { acc = __dadd_rn(acc, b[j].x); acc = __dadd_rn(acc, b[j].y); }
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}

__global__ void fold_shfl(const double *p, int nt, double *out, long long *cyc) {
    int lane = threadIdx.x;
    long long t0 = clock64();
    double acc = 0.0;
    double c0 = p[lane], c1 = p[32 + lane], c2 = p[64 + lane], c3 = p[96 + lane];
    for (int q = 0; q < nt; q += 32) {
        double c4 = q + 128 + lane < nt ? p[q + 128 + lane] : 0.0;
        double t[32];
#pragma unroll
        for (int j = 0; j < 32; j++) t[j] = __shfl_sync(0xffffffffu, c0, j);
#pragma unroll
        for (int j = 0; j < 32; j++) acc = __dadd_rn(acc, t[j]);
        c0 = c1; c1 = c2; c2 = c3; c3 = c4;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}

int main() {
    const int nt = 1 << 20;
    double *p, *o; long long *c, h;
    cudaMalloc(&p, (nt + 4096) * 8); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    cudaMemset(p, 0, (nt + 4096) * 8);
    auto run = [&](auto k, const char *name) {
        for (int i = 0; i < 2; i++) k<<<1, 32>>>(p, nt, o, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-12s %.2f cycles/term\n", name, (double)h / nt);
    };
    run(fold_smem, "smem");
    run(fold_bcast, "bcast-ldg");
    run(fold_shfl, "shfl");
    return 0;
}
