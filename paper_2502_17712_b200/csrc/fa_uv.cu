// fa_uv.cu — per-triangle atlas UVs (cli.py:424-450).
//
// One thread per visible triangle (ascending ids).  Each CTA stages its
// 256 x 6 UV values in shared memory and writes them back as 128-bit stores
// (the CTA's output slab starts at a multiple of 16 bytes).  Rows of
// triangles with a corner at or behind the camera plane (w <= W_EPSILON,
// cli.py:433-435) are NaN, as are rows of charts without a placement.
#include "fa_internal.h"

#define UV_THREADS 256

template <typename OutT>
__global__ void __launch_bounds__(UV_THREADS) k_uv(const double4* __restrict__ clip, const int* __restrict__ tris,
                                                   const int* __restrict__ vis_list, const int* __restrict__ label,
                                                   const int* __restrict__ cidx, const int* __restrict__ pinv,
                                                   const double* __restrict__ ndc, const int* __restrict__ px,
                                                   const long long* __restrict__ placements, int W, int H,
                                                   long long pad, OutT* __restrict__ uv,
                                                   const fa_dstat* __restrict__ st) {
    __shared__ __align__(16) OutT stage[UV_THREADS * 6];
    int n = st->n_vis;
    bool failed = (st->flags & (FA_DFLAG_PACK_FAILURE | FA_DFLAG_HEIGHT_OVERFLOW | FA_DFLAG_QUEUE_OVERFLOW)) != 0;
    for (int k0 = blockIdx.x * UV_THREADS; k0 < n; k0 += gridDim.x * UV_THREADS) {
        int k = k0 + threadIdx.x;
        double out[6];
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
        for (int i = 0; i < 6; i++) out[i] = qnan;
        if (k < n && !failed) {
            int t = vis_list[k];
            int c = cidx[label[t]];
            double4 v[3];
            bool behind = false;
#pragma unroll
            for (int i = 0; i < 3; i++) {
                v[i] = ldg4(clip + __ldg(tris + 3 * t + i));
                if (v[i].w <= FA_W_EPSILON) behind = true;
            }
            if (!behind) {
                int j = pinv[c];
                const long long* P = placements + 8 * (long long)j;
                long long cw = P[3] - 2 * pad, ch = P[4] - 2 * pad;
                double w_px = (double)px[2 * c], h_px = (double)px[2 * c + 1];
                double bx = (double)(P[1] + pad), by = (double)(P[2] + pad);
                double mnx = ndc[4 * c], mny = ndc[4 * c + 1];
                bool rot = P[5] != 0;
                double rx = rot ? __ddiv_rn((double)cw, h_px) : __ddiv_rn((double)cw, w_px);
                double ry = rot ? __ddiv_rn((double)ch, w_px) : __ddiv_rn((double)ch, h_px);
#pragma unroll
                for (int i = 0; i < 3; i++) {
                    double nx = __ddiv_rn(v[i].x, v[i].w), ny = __ddiv_rn(v[i].y, v[i].w);
                    double u = __dmul_rn(__dmul_rn(__dsub_rn(nx, mnx), 0.5), (double)W);
                    double vv = __dmul_rn(__dmul_rn(__dsub_rn(ny, mny), 0.5), (double)H);
                    out[2 * i] = __dadd_rn(bx, __dmul_rn(rot ? vv : u, rx));
                    out[2 * i + 1] = __dadd_rn(by, __dmul_rn(rot ? u : vv, ry));
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 6; i++) stage[threadIdx.x * 6 + i] = (OutT)out[i];
        __syncthreads();
        int cnt = min(UV_THREADS, n - k0);
        OutT* dst = uv + 6 * (long long)k0;
        int nelem = cnt * 6;
        const int per16 = 16 / sizeof(OutT);
        int nvec = nelem / per16;
        for (int i = threadIdx.x; i < nvec; i += UV_THREADS)
            reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(stage)[i];
        for (int i = nvec * per16 + threadIdx.x; i < nelem; i += UV_THREADS) dst[i] = stage[i];
        __syncthreads();
    }
}

void fa_launch_uv(const double4* clip, const int* tris, const int* vis_list, const int* label, const int* cidx,
                  const int* pinv, const double* ndc, const int* px, const long long* placements, int T, int W, int H,
                  long long pad, bool f64, void* uv, const fa_dstat* st, cudaStream_t s) {
    int grid = fa_grid(T, UV_THREADS, FA_NUM_SMS * 8);
    if (f64)
        k_uv<double><<<grid, UV_THREADS, 0, s>>>(clip, tris, vis_list, label, cidx, pinv, ndc, px, placements, W, H,
                                                 pad, (double*)uv, st);
    else
        k_uv<float><<<grid, UV_THREADS, 0, s>>>(clip, tris, vis_list, label, cidx, pinv, ndc, px, placements, W, H,
                                                pad, (float*)uv, st);
}
