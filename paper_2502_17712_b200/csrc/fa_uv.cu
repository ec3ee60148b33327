// fa_uv.cu — per-triangle atlas UVs (cli.py:424-450).
//
// One thread per visible triangle (ascending ids).  Each CTA stages its
// 256 x 6 UV values in shared memory and writes them back as 128-bit stores
// (the CTA's output slab starts at a multiple of 16 bytes).  Rows of
// triangles with a corner at or behind the camera plane (w <= W_EPSILON,
// cli.py:433-435) are NaN, as are rows of charts without a placement.
#define FA_TU_ID 6  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"

#define UV_THREADS 256

// Stretch of one (screen, atlas) triangle pair (metrics.py:58-111): the
// atlas->screen affine map M = Es * Ea^-1; area-weighted L2 needs only
// ||M||_F^2 = S1^2 + S2^2, Linf the larger singular value (closed form).
// Returns false for a degenerate atlas triangle (det == 0, skipped).
__device__ __forceinline__ bool tri_stretch(const double (&s)[6], const double (&a)[6], double& wterm, double& area,
                                            double& big) {
    double ea00 = a[2] - a[0], ea10 = a[3] - a[1], ea01 = a[4] - a[0], ea11 = a[5] - a[1];
    double es00 = s[2] - s[0], es10 = s[3] - s[1], es01 = s[4] - s[0], es11 = s[5] - s[1];
    double det = ea00 * ea11 - ea01 * ea10;
    if (det == 0.0) return false;
    double i00 = ea11 / det, i01 = -ea01 / det, i10 = -ea10 / det, i11 = ea00 / det;
    double m00 = es00 * i00 + es01 * i10, m01 = es00 * i01 + es01 * i11;
    double m10 = es10 * i00 + es11 * i10, m11 = es10 * i01 + es11 * i11;
    double f2 = m00 * m00 + m01 * m01 + m10 * m10 + m11 * m11;
    // stable 2x2 largest singular value: (|q| + |r|) / 2 with
    // q = (a + d, c - b), r = (a - d, c + b); no cancellation when S1 ~ S2
    double q = hypot(m00 + m11, m10 - m01), r = hypot(m00 - m11, m10 + m01);
    big = 0.5 * (q + r);
    area = fabs(es00 * es11 - es10 * es01) * 0.5;
    wterm = area * f2 * 0.5;
    return true;
}

#ifndef UV_MIN_BLOCKS
#define UV_MIN_BLOCKS 1  // minimum resident CTAs per SM (register cap)
#endif
template <typename OutT>
__global__ void __launch_bounds__(UV_THREADS, UV_MIN_BLOCKS) k_uv(const ClipSrc clip, const int* __restrict__ tris,
                                                   const int* __restrict__ vis_list, const int* __restrict__ label,
                                                   const int* __restrict__ cidx, const int* __restrict__ pinv,
                                                   const double* __restrict__ ndc, const int* __restrict__ px,
                                                   const long long* __restrict__ placements, int W, int H,
                                                   long long pad, OutT* __restrict__ uv,
                                                   int* __restrict__ vis_chart, const int* __restrict__ vis_cidx,
                                                   const int4* __restrict__ plc_c, const int4* __restrict__ vis_tris,
                                                   const int* __restrict__ vslot, float2* __restrict__ vuv,
                                                   fa_dstat* __restrict__ st, const double2* __restrict__ ndc2,
                                                   unsigned short* __restrict__ cidx16) {
    FA_PDL_PROLOGUE();
    __shared__ __align__(16) OutT stage[UV_THREADS * 6];
    __shared__ double red_w[UV_THREADS / 32], red_a[UV_THREADS / 32], red_m[UV_THREADS / 32];
    __shared__ int red_c[UV_THREADS / 32];
    double acc_w = 0.0, acc_a = 0.0, acc_m = 0.0;
    int acc_c = 0;
    int n = st->n_vis;
    bool failed = (st->flags & (FA_DFLAG_PACK_FAILURE | FA_DFLAG_HEIGHT_OVERFLOW | FA_DFLAG_QUEUE_OVERFLOW)) != 0;
    for (int k0 = blockIdx.x * UV_THREADS; k0 < n; k0 += gridDim.x * UV_THREADS) {
        int k = k0 + threadIdx.x;
        double out[6];
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
        for (int i = 0; i < 6; i++) out[i] = qnan;
        int4 vq = make_int4(0, 0, 0, -1);
        if (k < n && vis_tris) vq = vis_tris[k];
        if (k < n && vis_chart) vis_chart[k] = label[vis_tris ? vq.w : vis_list[k]];  // sparse chart_of_triangle
        // packed download format: the chart's index (roots[index] = its id),
        // 16 bits when the frame has < 2^16 charts (else the host takes vis_chart)
        if (k < n && cidx16 && vis_cidx && st->n_charts <= 65535) cidx16[k] = (unsigned short)vis_cidx[k];
        if (k < n && !failed) {
            int t = vis_tris ? vq.w : vis_list[k];
            // chart index and placement straight from the bounds / select
            // side outputs when present (two dependent loads instead of four)
            int c = vis_cidx ? vis_cidx[k] : cidx[label[t]];
            double nxs[3], nys[3];
            bool behind = false, fast = false;
            if (ndc2 && vis_tris) {
                // all three vertices strictly inside the frustum: their NDC
                // divisions were done once per vertex (vertex_ndc, same bits)
                const double2 n0 = __ldg(ndc2 + vq.x), n1 = __ldg(ndc2 + vq.y), n2 = __ldg(ndc2 + vq.z);
                fast = !isnan(n0.x) && !isnan(n1.x) && !isnan(n2.x);
                nxs[0] = n0.x; nxs[1] = n1.x; nxs[2] = n2.x;
                nys[0] = n0.y; nys[1] = n1.y; nys[2] = n2.y;
            }
            double4 v[3];
            if (!fast) {
#pragma unroll
                for (int i = 0; i < 3; i++) {
                    v[i] = clip(vis_tris ? (i == 0 ? vq.x : (i == 1 ? vq.y : vq.z)) : __ldg(tris + 3 * t + i));
                    if (v[i].w <= FA_W_EPSILON) behind = true;
                }
                if (!behind) {
#pragma unroll
                    for (int i = 0; i < 3; i++) {
                        nxs[i] = __ddiv_rn(v[i].x, v[i].w);
                        nys[i] = __ddiv_rn(v[i].y, v[i].w);
                    }
                }
            }
            if (behind && vuv) {
                // a vertex at or behind the camera plane makes every row it is
                // in NaN (cli.py:433-435): its compact UV is NaN
                const float qn = __int_as_float(0x7fc00000);
#pragma unroll
                for (int i = 0; i < 3; i++)
                    if (v[i].w <= FA_W_EPSILON)
                        vuv[vslot[i == 0 ? vq.x : (i == 1 ? vq.y : vq.z)]] = make_float2(qn, qn);
            }
            if (!behind) {
                long long px_, py_, pw_, ph_;
                bool rot;
                if (plc_c) {
                    const int4 a = plc_c[2 * c], b = plc_c[2 * c + 1];
                    px_ = a.x; py_ = a.y; pw_ = a.z; ph_ = a.w;
                    rot = b.x != 0;
                } else {
                    const long long* P = placements + 8 * (long long)pinv[c];
                    px_ = P[1]; py_ = P[2]; pw_ = P[3]; ph_ = P[4];
                    rot = P[5] != 0;
                }
                long long cw = pw_ - 2 * pad, ch = ph_ - 2 * pad;
                double w_px = (double)px[2 * c], h_px = (double)px[2 * c + 1];
                double bx = (double)(px_ + pad), by = (double)(py_ + pad);
                double mnx = ndc[4 * c], mny = ndc[4 * c + 1];
                double rx = rot ? __ddiv_rn((double)cw, h_px) : __ddiv_rn((double)cw, w_px);
                double ry = rot ? __ddiv_rn((double)ch, w_px) : __ddiv_rn((double)ch, h_px);
                double scr[6];
#pragma unroll
                for (int i = 0; i < 3; i++) {
                    const double nx = nxs[i], ny = nys[i];
                    double u = __dmul_rn(__dmul_rn(__dsub_rn(nx, mnx), 0.5), (double)W);
                    double vv = __dmul_rn(__dmul_rn(__dsub_rn(ny, mny), 0.5), (double)H);
                    out[2 * i] = __dadd_rn(bx, __dmul_rn(rot ? vv : u, rx));
                    out[2 * i + 1] = __dadd_rn(by, __dmul_rn(rot ? u : vv, ry));
                    scr[2 * i] = __dmul_rn(__dmul_rn(__dadd_rn(nx, 1.0), 0.5), (double)W);      // cli.py:437-439
                    scr[2 * i + 1] = __dmul_rn(__dmul_rn(__dadd_rn(ny, 1.0), 0.5), (double)H);
                }
                if (vuv) {
                    // compact format: one f32 pair per visible vertex (all of a
                    // vertex's triangles are in its chart and compute this value)
#pragma unroll
                    for (int i = 0; i < 3; i++) {
                        const int vtx = i == 0 ? vq.x : (i == 1 ? vq.y : vq.z);
                        vuv[vslot[vtx]] = make_float2((float)out[2 * i], (float)out[2 * i + 1]);
                    }
                }
                double wt, ar, big;
                if (tri_stretch(scr, out, wt, ar, big)) {
                    acc_w += wt;
                    acc_a += ar;
                    acc_m = big > acc_m ? big : acc_m;
                    acc_c++;
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
    // stretch sums: warp shuffles, then one set of atomics per block
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc_w += __shfl_xor_sync(0xffffffffu, acc_w, o);
        acc_a += __shfl_xor_sync(0xffffffffu, acc_a, o);
        acc_m = fmax(acc_m, __shfl_xor_sync(0xffffffffu, acc_m, o));
        acc_c += __shfl_xor_sync(0xffffffffu, acc_c, o);
    }
    int wid = threadIdx.x >> 5;
    if (lane_id() == 0) {
        red_w[wid] = acc_w;
        red_a[wid] = acc_a;
        red_m[wid] = acc_m;
        red_c[wid] = acc_c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double w = 0, a = 0, m = 0;
        int c = 0;
        for (int i = 0; i < UV_THREADS / 32; i++) {
            w += red_w[i];
            a += red_a[i];
            m = fmax(m, red_m[i]);
            c += red_c[i];
        }
        if (c) {
            // exact fixed-point sums (reproducible); the float sums are kept
            // for partials outside the fixed-point range
            if (!fx_add(st->stretch_fx[0], w) || !fx_add(st->stretch_fx[1], a))
                atomicOr(&st->flags, FA_DFLAG_STRETCH_RANGE);
            atomicAdd(&st->stretch_wsum, w);
            atomicAdd(&st->stretch_area, a);
            atomicMax(&st->stretch_linf_bits, (unsigned long long)__double_as_longlong(m));
            atomicAdd(&st->stretch_valid, c);
        }
    }
}

void fa_launch_uv(const ClipSrc clip, const int* tris, const int* vis_list, const int* label, const int* cidx,
                  const int* pinv, const double* ndc, const int* px, const long long* placements, int T, int W, int H,
                  long long pad, bool f64, void* uv, int* vis_chart, const int* vis_cidx, const int4* plc_c,
                  fa_dstat* st, cudaStream_t s, const int4* vis_tris, const int* vslot, float2* vuv,
                  const double2* ndc2, unsigned short* cidx16) {
    if (!vis_tris) vuv = nullptr;  // the compact UVs index vertices through vis_tris
    const long long nblk = ((long long)T + UV_THREADS - 1) / UV_THREADS;
    const int grid = f64 ? fa_wave_grid(k_uv<double>, UV_THREADS, 0, nblk, FA_NUM_SMS * 8)
                         : fa_wave_grid(k_uv<float>, UV_THREADS, 0, nblk, FA_NUM_SMS * 8);
    if (f64)
        fa_launch(k_uv<double>, grid, UV_THREADS, 0, s, clip, tris, vis_list, label, cidx, pinv, ndc, px, placements, W, H,
                                                 pad, (double*)uv, vis_chart, vis_cidx, plc_c, vis_tris, vslot, vuv, st, ndc2, cidx16);
    else
        fa_launch(k_uv<float>, grid, UV_THREADS, 0, s, clip, tris, vis_list, label, cidx, pinv, ndc, px, placements, W, H,
                                                pad, (float*)uv, vis_chart, vis_cidx, plc_c, vis_tris, vslot, vuv, st, ndc2, cidx16);
}

FA_TRACE_TU(uv)
