// Microbenchmark (tools only): dependent DADD chain latency on this GPU, and a
// shuffle-fed fold like k_vlong_fold.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double *x, double *out, int n, long long *cyc) {
    double acc = 0.0, a = x[0], b = x[1];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; i++) { acc = __dadd_rn(acc, a); a = __dadd_rn(a, b) * 0 + a; }
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
__global__ void chain2(const double *x, double *out, int n, long long *cyc) {
    double acc = 0.0, a = x[0];
    long long t0 = clock64();
#pragma unroll 32
    for (int i = 0; i < n; i++) acc = __dadd_rn(acc, a);
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
__global__ void fchain(const float *x, float *out, int n, long long *cyc) {
    float acc = 0.f, a = x[0];
    long long t0 = clock64();
#pragma unroll 32
    for (int i = 0; i < n; i++) acc = __fadd_rn(acc, a);
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
int main() {
    double *x, *o; float *fx, *fo; long long *c; long long h;
    cudaMalloc(&x, 64); cudaMalloc(&o, 64); cudaMalloc(&fx, 64); cudaMalloc(&fo, 64); cudaMalloc(&c, 8);
    double hx[2] = {1.0000001, 1e-300}; cudaMemcpy(x, hx, 16, cudaMemcpyHostToDevice);
    float hf[1] = {1.0001f}; cudaMemcpy(fx, hf, 4, cudaMemcpyHostToDevice);
    int n = 1 << 20;
    chain2<<<1, 1>>>(x, o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    chain2<<<1, 1>>>(x, o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent chain: %.2f cycles/add\n", (double)h / n);
    fchain<<<1, 1>>>(fx, fo, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    fchain<<<1, 1>>>(fx, fo, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FADD dependent chain: %.2f cycles/add\n", (double)h / n);
    return 0;
}
