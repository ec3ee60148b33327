// Microbenchmark: what a one-CTA, 1024-thread kernel costs on B200 (the
// order / select kernels of the frame): empty, barriers, an FP64 division
// chain, and large dynamic shared memory; chained in a graph with PDL.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(double* sink) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 9999) sink[0] = 1;
}
__global__ void k_bar(double* sink, int nb) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ int x[1024];
    int v = threadIdx.x;
    for (int i = 0; i < nb; i++) {
        x[threadIdx.x] = v;
        __syncthreads();
        v += x[(threadIdx.x + 1) & 1023];
        __syncthreads();
    }
    if (v == -1) sink[0] = v;
}
__global__ void k_fp64(double* sink, const double* in, int chain) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    double a = in[threadIdx.x], b = in[threadIdx.x + 1024];
    for (int i = 0; i < chain; i++) a = ceil(__dmul_rn(__ddiv_rn(__dsub_rn(a, b), 2.0), 1920.0)) + 1e-3;
    if (a == -1.0) sink[0] = a;
}
__global__ void k_smem(double* sink, int nb) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ int dyn[];
    int v = threadIdx.x;
    for (int i = 0; i < nb; i++) {
        dyn[threadIdx.x * 7 % 8000] = v;
        __syncthreads();
        v += dyn[(threadIdx.x + 1) & 1023];
        __syncthreads();
    }
    if (v == -1) sink[0] = v;
}

template <typename F>
float timed(cudaStream_t s, F launch) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal) != cudaSuccess) { printf("begin capture failed\n"); return -1.f; }
    for (int i = 0; i < 20; i++) launch();
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) { printf("capture: %s\n", cudaGetErrorString(e)); return -1.f; }
    e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) { printf("instantiate: %s\n", cudaGetErrorString(e)); return -1.f; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; w++) cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    for (int r = 0; r < 20; r++) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return 1000.f * ms / 400.f;
}

int main() {
    double *sink, *in;
    cudaMalloc(&sink, 64);
    cudaMalloc(&in, 4096 * 8);
    cudaMemset(in, 0, 4096 * 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    static cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    auto cfg = [&](int threads, size_t smem) {
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3(1); c.blockDim = dim3(threads); c.dynamicSmemBytes = smem; c.stream = s;
        c.attrs = at; c.numAttrs = 1;
        return c;
    };
    for (int threads : {256, 1024}) {
        printf("threads %d: empty %.2f us\n", threads, timed(s, [&] { auto c = cfg(threads, 0); cudaLaunchKernelEx(&c, k_empty, sink); }));
        for (int nb : {10, 40})
            printf("threads %d: %d barrier pairs %.2f us\n", threads, nb,
                   timed(s, [&] { auto c = cfg(threads, 0); cudaLaunchKernelEx(&c, k_bar, sink, nb); }));
        for (int ch : {5, 20})
            printf("threads %d: fp64 div chain %d %.2f us\n", threads, ch,
                   timed(s, [&] { auto c = cfg(threads, 0); cudaLaunchKernelEx(&c, k_fp64, sink, (const double*)in, ch); }));
        for (size_t kb : {32, 160})
            printf("threads %d: %zu KB dyn smem, 10 barrier pairs %.2f us\n", threads, kb,
                   timed(s, [&] { auto c = cfg(threads, kb * 1024); cudaLaunchKernelEx(&c, k_smem, sink, 10); }));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
