// Microbenchmark: same-address atomicAdd throughput on B200 (the appends of
// the raster setup) -- N warps each adding to one global counter, with the
// result used (returning atomics) or not (reductions).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ret(int* ctr, int* sink, int iters) {
    int acc = 0;
    for (int i = 0; i < iters; i++)
        if ((threadIdx.x & 31) == 0) acc += atomicAdd(ctr, 1);
    if (acc == -1) *sink = acc;
}
__global__ void k_spread(int* ctr, int* sink, int iters, int nctr) {
    int acc = 0;
    int c = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % nctr;
    for (int i = 0; i < iters; i++)
        if ((threadIdx.x & 31) == 0) acc += atomicAdd(ctr + 32 * c, 1);
    if (acc == -1) *sink = acc;
}

int main() {
    int *ctr, *sink;
    cudaMalloc(&ctr, 1 << 20);
    cudaMalloc(&sink, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks : {148, 592, 2368}) {
        const int iters = 16;
        cudaMemset(ctr, 0, 1 << 20);
        k_ret<<<blocks, 256>>>(ctr, sink, iters);
        cudaEventRecord(a);
        k_ret<<<blocks, 256>>>(ctr, sink, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long n = (long long)blocks * 8 * iters;
        printf("same address: %d blocks x 8 warps x %d = %lld warp atomics: %.1f us, %.2f ns each\n", blocks, iters, n,
               1000 * ms, 1e6 * ms / n);
        for (int nctr : {16, 148}) {
            k_spread<<<blocks, 256>>>(ctr, sink, iters, nctr);
            cudaEventRecord(a);
            k_spread<<<blocks, 256>>>(ctr, sink, iters, nctr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("  %3d counters: %.1f us, %.2f ns each\n", nctr, 1000 * ms, 1e6 * ms / n);
        }
    }
    return 0;
}
