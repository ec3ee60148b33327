// fa_bounds.cu — conservative per-chart NDC boxes and target box dims.
//
// Reference: chart_bbox (geometry.py:281-322) with select_side_plane
// (geometry.py:257-278), _clip_poly_halfspace (geometry.py:203-220),
// blinn_clamped_ndc (geometry.py:185-200); viewport_box
// (geometry.py:352-362) and the prescale ceil (cli.py:379-384).
//
// One thread per visible triangle computes its box contribution; clipped
// polygons are streamed straight into the running min/max (no polygon is
// materialised — min/max are order independent).  Lanes holding the same
// chart form runs in the (ascending) visible list, so a segmented warp scan
// reduces each run and only the run tail issues the four u64 key atomics.
#define FA_TU_ID 4  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"

struct NBox {
    double mnx, mny, mxx, mxy;
};

// geometry.py:185-200
__device__ __forceinline__ void blinn_add(double x, double y, double w, NBox& b) {
    double aw = fabs(w);
    double cx, cy;
    if (aw == 0.0) {
        cx = x < 0 ? -1.0 : 1.0;
        cy = y < 0 ? -1.0 : 1.0;
    } else {
        double t = (-aw > x) ? -aw : x;
        t = (aw < t) ? aw : t;
        cx = __ddiv_rn(t, aw);
        t = (-aw > y) ? -aw : y;
        t = (aw < t) ? aw : t;
        cy = __ddiv_rn(t, aw);
    }
    if (cx < b.mnx) b.mnx = cx;
    if (cy < b.mny) b.mny = cy;
    if (cx > b.mxx) b.mxx = cx;
    if (cy > b.mxy) b.mxy = cy;
}

// geometry.py:203-220 (keep d > 0) streamed into a box
__device__ __forceinline__ void clip_gt_into(const double4 (&c)[3], const double (&d)[3], NBox& b) {
#pragma unroll
    for (int i = 0; i < 3; i++) {
        const int j = (i + 1) % 3;
        double da = d[i], db = d[j];
        if (da > 0) blinn_add(c[i].x, c[i].y, c[i].w, b);
        if ((da > 0) != (db > 0)) {
            double t = __ddiv_rn(da, __dsub_rn(da, db));
            double x = __dadd_rn(c[i].x, __dmul_rn(t, __dsub_rn(c[j].x, c[i].x)));
            double y = __dadd_rn(c[i].y, __dmul_rn(t, __dsub_rn(c[j].y, c[i].y)));
            double w = __dadd_rn(c[i].w, __dmul_rn(t, __dsub_rn(c[j].w, c[i].w)));
            blinn_add(x, y, w, b);
        }
    }
}

__device__ __forceinline__ void side_d(const double4 (&c)[3], int plane, double (&d)[3]) {
#pragma unroll
    for (int i = 0; i < 3; i++) {
        switch (plane) {
            case 0: d[i] = __dadd_rn(c[i].w, c[i].x); break;
            case 1: d[i] = __dsub_rn(c[i].w, c[i].x); break;
            case 2: d[i] = __dadd_rn(c[i].w, c[i].y); break;
            default: d[i] = __dsub_rn(c[i].w, c[i].y); break;
        }
    }
}

__device__ __forceinline__ NBox empty_box() {
    NBox b;
    b.mnx = b.mny = __longlong_as_double(0x7ff0000000000000ll);
    b.mxx = b.mxy = __longlong_as_double((long long)0xfff0000000000000ull);
    return b;
}

// select_side_plane (geometry.py:257-278): strict crossing, minimal
// Blinn-box area, ties to the lower plane index; -1 = None
__device__ __forceinline__ int select_plane(const double4 (&c)[3]) {
    int best = -1;
    double best_area = 0.0;
#pragma unroll
    for (int p = 0; p < 4; p++) {
        double sd[3];
        side_d(c, p, sd);
        bool pos = sd[0] > 0 || sd[1] > 0 || sd[2] > 0;
        bool neg = sd[0] < 0 || sd[1] < 0 || sd[2] < 0;
        if (pos && neg) {
            NBox cb = empty_box();
            clip_gt_into(c, sd, cb);
            double area = __dmul_rn(__dsub_rn(cb.mxx, cb.mnx), __dsub_rn(cb.mxy, cb.mny));
            if (best < 0 || area < best_area) { best = p; best_area = area; }
        }
    }
    return best;
}

// geometry.py:300-319 for one triangle; returns survived
__device__ __forceinline__ bool tri_box(const double4 (&c)[3], NBox& b) {
    double d[3];
    bool allp = true, anyp = false;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        d[i] = __dsub_rn(c[i].w, FA_W_EPSILON);
        if (d[i] > 0) anyp = true; else allp = false;
    }
    if (allp) {
        int best = select_plane(c);
        if (best < 0) {
#pragma unroll
            for (int i = 0; i < 3; i++) blinn_add(c[i].x, c[i].y, c[i].w, b);
        } else {
            double sd[3];
            side_d(c, best, sd);
            clip_gt_into(c, sd, b);
        }
        return true;
    }
    if (anyp) {
        clip_gt_into(c, d, b);
        return true;
    }
    return false;
}

// Root of t's set after the hooking: the frame's bounds run beside the
// flattening (k_compress, another stream), which only rewrites non-roots to
// their root, so every value read here is t's parent or its root -- both lead
// to the root.  L2 loads (not the read-only path: the array is being written).
__device__ __forceinline__ int uf_root(const int* label, int t) {
    int r = __ldcg(label + t);
    if (r == t) return t;
    for (;;) {
        const int p = __ldcg(label + r);
        if (p == r) return r;
        r = p;
    }
}

#ifndef BOUNDS_MIN_BLOCKS
#define BOUNDS_MIN_BLOCKS 1  // minimum resident CTAs per SM (register cap)
#endif
__global__ void __launch_bounds__(256, BOUNDS_MIN_BLOCKS) k_chart_bounds(const ClipSrc clip, const int* __restrict__ tris,
                                                      const int* __restrict__ vis_list, const int* label,
                                                      const int* __restrict__ cidx,
                                                      unsigned long long* __restrict__ keys,
                                                      int* __restrict__ survived, const fa_dstat* __restrict__ st,
                                                      int* __restrict__ vis_cidx, const int4* __restrict__ vis_tris,
                                                      const double2* __restrict__ ndc2) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int lane = lane_id();
    int stride = gridDim.x * blockDim.x;
    // the loop trip count is warp-uniform (all lanes share the same k base)
    for (int kb = blockIdx.x * blockDim.x + (threadIdx.x & ~31); kb < n; kb += stride) {
        int k = kb + lane;
        int c = -1;
        unsigned long long k0 = FA_KEY_POS_INF, k1 = FA_KEY_POS_INF, k2 = FA_KEY_NEG_INF, k3 = FA_KEY_NEG_INF;
        int surv = 0;
        if (k < n) {
            int t;
            NBox b = empty_box();
            bool got = false;
            if (vis_tris) {  // vertex indices next to the id: one dependent load fewer
                const int4 q = vis_tris[k];
                t = q.w;
                c = cidx[uf_root(label, t)];
                if (ndc2) {
                    // every vertex strictly inside the frustum (vertex_ndc not
                    // NaN): no side plane is crossed and the Blinn clamp is the
                    // plain division, so the box is the vertices' NDC, added in
                    // the same order and comparisons as tri_box's blinn_add
                    const double2 n0 = __ldg(ndc2 + q.x), n1 = __ldg(ndc2 + q.y), n2 = __ldg(ndc2 + q.z);
                    if (!isnan(n0.x) && !isnan(n1.x) && !isnan(n2.x)) {
                        const double2 nn[3] = {n0, n1, n2};
#pragma unroll
                        for (int i = 0; i < 3; i++) {
                            if (nn[i].x < b.mnx) b.mnx = nn[i].x;
                            if (nn[i].y < b.mny) b.mny = nn[i].y;
                            if (nn[i].x > b.mxx) b.mxx = nn[i].x;
                            if (nn[i].y > b.mxy) b.mxy = nn[i].y;
                        }
                        got = true;
                    }
                }
                if (!got) {
                    double4 cc[3] = {clip(q.x), clip(q.y), clip(q.z)};
                    got = tri_box(cc, b);
                }
            } else {
                t = vis_list[k];
                double4 cc[3];
#pragma unroll
                for (int j = 0; j < 3; j++) cc[j] = clip(__ldg(tris + 3 * t + j));
                c = cidx[uf_root(label, t)];
                got = tri_box(cc, b);
            }
            if (vis_cidx) vis_cidx[k] = c;  // k_uv's chart index (saves it two dependent loads)
            if (got) {
                surv = 1;
                k0 = f64_key(b.mnx);
                k1 = f64_key(b.mny);
                k2 = f64_key(b.mxx);
                k3 = f64_key(b.mxy);
            }
        }
        // segmented inclusive scan over runs of equal chart index
        int prev_c = __shfl_up_sync(0xffffffffu, c, 1);
        bool head = (lane == 0) || (prev_c != c);
        unsigned heads = __ballot_sync(0xffffffffu, head);
        int seg_start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long a0 = __shfl_up_sync(0xffffffffu, k0, o);
            unsigned long long a1 = __shfl_up_sync(0xffffffffu, k1, o);
            unsigned long long a2 = __shfl_up_sync(0xffffffffu, k2, o);
            unsigned long long a3 = __shfl_up_sync(0xffffffffu, k3, o);
            int as = __shfl_up_sync(0xffffffffu, surv, o);
            if (lane - o >= seg_start) {
                k0 = a0 < k0 ? a0 : k0;
                k1 = a1 < k1 ? a1 : k1;
                k2 = a2 > k2 ? a2 : k2;
                k3 = a3 > k3 ? a3 : k3;
                surv |= as;
            }
        }
        int next_c = __shfl_down_sync(0xffffffffu, c, 1);
        bool tail = (lane == 31) || (next_c != c);
        if (tail && c >= 0 && surv) {
            // fire-and-forget REDs (one set per chart run per warp); a
            // load-first check would add a round trip to every run
            unsigned long long* kk = keys + 4 * (long long)c;
            atomicMin(kk + 0, k0);
            atomicMin(kk + 1, k1);
            atomicMax(kk + 2, k2);
            atomicMax(kk + 3, k3);
            survived[c] = 1;
        }
    }
}

// viewport_box (geometry.py:352-362) + prescale (cli.py:379-381)
__global__ void k_box_dims(const unsigned long long* __restrict__ keys, const int* __restrict__ survived,
                           const int* __restrict__ roots, int W, int H, double prescale, double* __restrict__ ndc,
                           int* __restrict__ px, long long* __restrict__ target, long long* __restrict__ otw,
                           long long* __restrict__ oth, long long* __restrict__ cid, int cap,
                           fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    int n = st->n_charts;
    int stride = gridDim.x * blockDim.x;
    fa_box_dims_args a{keys, survived, roots, W, H, prescale, ndc, px, target, otw, oth, cid, cap};
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) fa_box_dims_one(a, j, st);
}

void fa_launch_chart_bounds(const ClipSrc clip, const int* tris, const int* vis_list, const int* label,
                            const int* cidx, int T, unsigned long long* ndc_keys, int* survived, const fa_dstat* st,
                            cudaStream_t s, int* vis_cidx, const int4* vis_tris, const double2* ndc2) {
    fa_launch(k_chart_bounds, fa_wave_grid(k_chart_bounds, 256, 0, ((long long)T + 255) / 256, FA_NUM_SMS * 8), 256, 0, s, clip, tris, vis_list, label, cidx, ndc_keys,
              survived, st, vis_cidx, vis_tris, vis_tris ? ndc2 : nullptr);
}

void fa_launch_box_dims(const unsigned long long* ndc_keys, const int* survived, const int* roots, int T, int W, int H,
                        double prescale, double* ndc, int* px, long long* target, long long* tw, long long* th,
                        long long* cid, int cap, fa_dstat* st, cudaStream_t s) {
    // grid-stride over the chart count; sized by the chart capacity, not T
    fa_launch(k_box_dims, fa_grid(cap < T ? cap : T, 256, FA_NUM_SMS * 4), 256, 0, s, ndc_keys, survived, roots, W, H,
              prescale, ndc, px, target, tw, th, cid, cap, st);
}

// ---- batched standalone API kernels -------------------------------------------
// blinn_clamped_ndc (geometry.py:185-200) over n homogeneous points
__global__ void k_blinn_points(const double* __restrict__ p4, int n, double* __restrict__ out) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        NBox b = empty_box();
        blinn_add(p4[4 * i], p4[4 * i + 1], p4[4 * i + 3], b);
        out[2 * i] = b.mnx;
        out[2 * i + 1] = b.mny;
    }
}

// select_side_plane over n homogeneous triangles (n,3,4)
__global__ void k_select_side_plane(const double* __restrict__ t12, int n, int* __restrict__ out) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double4 c[3];
#pragma unroll
        for (int j = 0; j < 3; j++)
            c[j] = make_double4(t12[12 * i + 4 * j], t12[12 * i + 4 * j + 1], t12[12 * i + 4 * j + 2],
                                t12[12 * i + 4 * j + 3]);
        out[i] = select_plane(c);
    }
}

// chart_bbox (geometry.py:281-322) over n world triangles (n,3,3)
__global__ void k_chart_bbox_world(const double* __restrict__ xyz, int n, const double* __restrict__ vp,
                                   unsigned long long* __restrict__ keys, int* __restrict__ surv) {
    FA_PDL_PROLOGUE();
    double m[16];
#pragma unroll
    for (int i = 0; i < 16; i++) m[i] = vp[i];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double4 c[3];
#pragma unroll
        for (int j = 0; j < 3; j++) c[j] = project_point(xyz[9 * i + 3 * j], xyz[9 * i + 3 * j + 1], xyz[9 * i + 3 * j + 2], m);
        NBox b = empty_box();
        if (tri_box(c, b)) {
            atomicMin(keys + 0, f64_key(b.mnx));
            atomicMin(keys + 1, f64_key(b.mny));
            atomicMax(keys + 2, f64_key(b.mxx));
            atomicMax(keys + 3, f64_key(b.mxy));
            *surv = 1;
        }
    }
}

__global__ void k_init_box_keys(unsigned long long* keys, int* surv) {
    FA_PDL_PROLOGUE();
    keys[0] = keys[1] = FA_KEY_POS_INF;
    keys[2] = keys[3] = FA_KEY_NEG_INF;
    *surv = 0;
}

__global__ void k_decode_box(const unsigned long long* keys, double* out) {
    FA_PDL_PROLOGUE();
    if (threadIdx.x < 4) out[threadIdx.x] = key_f64(keys[threadIdx.x]);
}

// viewport_box (geometry.py:352-362) over n boxes
__global__ void k_viewport_box(const double* __restrict__ box, int n, int W, int H, long long* __restrict__ out) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double fw = ceil(__dmul_rn(__ddiv_rn(__dsub_rn(box[4 * i + 2], box[4 * i]), 2.0), (double)W));
        double fh = ceil(__dmul_rn(__ddiv_rn(__dsub_rn(box[4 * i + 3], box[4 * i + 1]), 2.0), (double)H));
        out[2 * i] = fw < 1.0 ? 1 : (long long)fw;
        out[2 * i + 1] = fh < 1.0 ? 1 : (long long)fh;
    }
}

void fa_launch_blinn_points(const double* p4, int n, double* out, cudaStream_t s) {
    fa_launch(k_blinn_points, fa_grid(n, 256, FA_NUM_SMS * 4), 256, 0, s, p4, n, out);
}
void fa_launch_select_side_plane(const double* t12, int n, int* out, cudaStream_t s) {
    fa_launch(k_select_side_plane, fa_grid(n, 256, FA_NUM_SMS * 4), 256, 0, s, t12, n, out);
}
void fa_launch_chart_bbox_world(const double* xyz, int n, const double* vp, unsigned long long* keys, int* surv,
                                double* box_out, cudaStream_t s) {
    fa_launch(k_init_box_keys, 1, 1, 0, s, keys, surv);
    fa_launch(k_chart_bbox_world, fa_grid(n, 256, FA_NUM_SMS * 4), 256, 0, s, xyz, n, vp, keys, surv);
    fa_launch(k_decode_box, 1, 32, 0, s, keys, box_out);
}
void fa_launch_viewport_box(const double* box, int n, int W, int H, long long* out, cudaStream_t s) {
    fa_launch(k_viewport_box, fa_grid(n, 256, FA_NUM_SMS * 4), 256, 0, s, box, n, W, H, out);
}

FA_TRACE_TU(bounds)
