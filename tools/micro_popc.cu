// Microbenchmark (tools only): AND+POPC throughput of the whole GPU (the unit
// of the TC masked SpGEMM).  Prints units/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned n, unsigned seed, unsigned *out) {
    unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b = seed * 11u + blockIdx.x;
    unsigned c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (unsigned i = 0; i < n; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            c0 += __popc(a0 & b); c1 += __popc(a1 & b); c2 += __popc(a2 & b); c3 += __popc(a3 & b);
            b = b * 1664525u + 1013904223u;
        }
    }
    if (c0 + c1 + c2 + c3 == 0x12345u) out[0] = 1;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *o; cudaMalloc(&o, 4);
    unsigned n = 4096; int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<blocks, threads>>>(n, 1, o);
    cudaEventRecord(a); k<<<blocks, threads>>>(n, 2, o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double units = (double)blocks * threads * n * 8 * 4;
    printf("{\"and_popc_units_per_s\": %.4g, \"ms\": %.3f, \"sms\": %d}\n", units / (ms * 1e-3), ms, sms);
    return 0;
}
