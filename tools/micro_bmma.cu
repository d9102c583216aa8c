// Microbenchmark (tools only): b1 tensor-core MMA (mma.sync m16n8k256 .and.popc)
// against the integer-pipe AND+POPC of tools/micro_popc.cu -- SURVEY.md north
// star item 3: is the b1 MMA a faster way to do the masked SpGEMM's AND+POPC?
// Reports 32-bit AND+POPC units/s (one mma = 16*8*256 bit products = 1024 units).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bmma(int (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__global__ void k(unsigned n, unsigned seed, int *out) {
    unsigned a[4] = {seed ^ threadIdx.x, seed * 3u, seed * 5u + threadIdx.x, seed * 7u};
    unsigned b0[2] = {seed * 11u + blockIdx.x, seed * 13u}, b1[2] = {seed * 17u, seed * 19u + threadIdx.x};
    int d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0}, d2[4] = {0, 0, 0, 0}, d3[4] = {0, 0, 0, 0};
    for (unsigned i = 0; i < n; i++) {
        bmma(d0, a, b0);
        bmma(d1, a, b1);
        bmma(d2, a, b0);
        bmma(d3, a, b1);
    }
    int s = 0;
    for (int j = 0; j < 4; j++) s += d0[j] + d1[j] + d2[j] + d3[j];
    if (s == 0x12345) out[0] = s;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int *o;
    cudaMalloc(&o, 4);
    unsigned n = 4096;
    int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<blocks, threads>>>(n, 1, o);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(n, 2, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double mmas = (double)blocks * (threads / 32) * n * 4;
    printf("{\"bmma_and_popc_units_per_s\": %.4g, \"mma_per_s\": %.4g, \"ms\": %.3f, \"sms\": %d, \"err\": \"%s\"}\n",
           mmas * 1024 / (ms * 1e-3), mmas / (ms * 1e-3), ms, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
