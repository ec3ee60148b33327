// Microbenchmark: cost of a grid-wide barrier inside one cooperative kernel
// (cooperative_groups grid.sync vs a hand-rolled generation barrier), launched
// through a CUDA graph, against an empty-kernel chain of the same length.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_cg(int n, int* sink) {
    cg::grid_group g = cg::this_grid();
    int acc = 0;
    for (int i = 0; i < n; i++) {
        acc += threadIdx.x ^ i;
        g.sync();
    }
    if (acc == -1) *sink = acc;
}

__device__ unsigned int g_bar_count = 0, g_bar_gen = 0;
__device__ __forceinline__ void grid_barrier(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* genp = &g_bar_gen;
        unsigned gen = *genp;
        __threadfence();
        if (atomicAdd(&g_bar_count, 1) == nblocks - 1) {
            g_bar_count = 0;
            __threadfence();
            atomicAdd(&g_bar_gen, 1);
        } else {
            while (*genp == gen) { __nanosleep(20); }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_own(int n, int* sink) {
    int acc = 0;
    for (int i = 0; i < n; i++) {
        acc += threadIdx.x ^ i;
        grid_barrier(gridDim.x);
    }
    if (acc == -1) *sink = acc;
}

__global__ void k_empty(int* sink) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    // a dependent read-modify-write chain through global memory
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = sink[0] + 1;
}

__global__ void k_cg_dep(int n, int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < n; i++) {
        if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = sink[0] + 1;
        g.sync();
    }
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks : {148, 296}) {
        for (int threads : {256, 512}) {
            for (int mode = 0; mode < 3; mode++) {
                const int N = 20;
                cudaGraph_t g;
                cudaGraphExec_t ge;
                cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                if (mode == 2) {
                    for (int i = 0; i < N; i++) {
                        cudaLaunchConfig_t cfg = {};
                        cfg.gridDim = blocks; cfg.blockDim = threads; cfg.stream = s;
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                        at[0].val.programmaticStreamSerializationAllowed = 1;
                        cfg.attrs = at; cfg.numAttrs = 1;
                        cudaLaunchKernelEx(&cfg, k_empty, sink);
                    }
                } else {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = blocks; cfg.blockDim = threads; cfg.stream = s;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeCooperative;
                    at[0].val.cooperative = 1;
                    cfg.attrs = at; cfg.numAttrs = 1;
                    int n = N;
                    if (mode == 0) cudaLaunchKernelEx(&cfg, k_cg_dep, n, sink);
                    else cudaLaunchKernelEx(&cfg, k_own, n, sink);
                }
                cudaError_t ce = cudaStreamEndCapture(s, &g);
                if (ce != cudaSuccess) { printf("capture error %s\n", cudaGetErrorString(ce)); return 1; }
                cudaGraphInstantiate(&ge, g, 0);
                for (int w = 0; w < 5; w++) cudaGraphLaunch(ge, s);
                cudaEventRecord(e0, s);
                const int R = 50;
                for (int r = 0; r < R; r++) cudaGraphLaunch(ge, s);
                cudaEventRecord(e1, s);
                cudaError_t err = cudaStreamSynchronize(s);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("blocks %d threads %d %-10s : %.2f us per step (%s)\n", blocks, threads,
                       mode == 0 ? "cg.sync" : mode == 1 ? "own.sync" : "launches", 1000.f * ms / R / N,
                       cudaGetErrorString(err));
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(g);
            }
        }
    }
    return 0;
}
