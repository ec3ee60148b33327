// fa_raster.cuh — per-triangle raster setup shared by the depth and
// visibility passes.  Restates charts.py:160-266 with identical float64
// operation order (compiled with -fmad=false).
#pragma once
#include "fa_common.cuh"

#define FA_SETUP_MAXV 12   // stored-setup polygon capacity (convex max is 10)

struct TriSetup {
    int tri;
    int n;
    int min_x, max_x, min_y, max_y;
    int use_plane;
    int incl_mask;
    double p0x, p0y, p0z, gx, gy, zmean;
    double ex[FA_SETUP_MAXV], ey[FA_SETUP_MAXV], edx[FA_SETUP_MAXV], edy[FA_SETUP_MAXV];
};

struct Poly4 {
    double v[FA_MAXV][4];
    int n;
};

// charts.py:178-189 — keep d >= 0; returns false on capacity overflow
__device__ __forceinline__ bool clip_halfspace_ge(const Poly4& in, const double* d, Poly4& out) {
    int n = in.n, m = 0;
    for (int i = 0; i < n; i++) {
        int j = (i + 1 == n) ? 0 : i + 1;
        double da = d[i], db = d[j];
        if (da >= 0) {
            if (m >= FA_MAXV) return false;
            out.v[m][0] = in.v[i][0]; out.v[m][1] = in.v[i][1];
            out.v[m][2] = in.v[i][2]; out.v[m][3] = in.v[i][3];
            m++;
        }
        if ((da >= 0) != (db >= 0)) {
            double t = __ddiv_rn(da, __dsub_rn(da, db));
            if (m >= FA_MAXV) return false;
#pragma unroll
            for (int k = 0; k < 4; k++)
                out.v[m][k] = __dadd_rn(in.v[i][k], __dmul_rn(t, __dsub_rn(in.v[j][k], in.v[i][k])));
            m++;
        }
    }
    out.n = m;
    return true;
}

// charts.py:160-175 (slow path: some plane clips).  Returns false on overflow.
static __device__ __noinline__ bool clip_triangle_frustum_slow(const double4 c0, const double4 c1, const double4 c2,
                                                        Poly4& out) {
    Poly4 tmp;
    double d[FA_MAXV];
    Poly4* cur = &out;
    Poly4* nxt = &tmp;
    cur->n = 3;
    cur->v[0][0] = c0.x; cur->v[0][1] = c0.y; cur->v[0][2] = c0.z; cur->v[0][3] = c0.w;
    cur->v[1][0] = c1.x; cur->v[1][1] = c1.y; cur->v[1][2] = c1.z; cur->v[1][3] = c1.w;
    cur->v[2][0] = c2.x; cur->v[2][1] = c2.y; cur->v[2][2] = c2.z; cur->v[2][3] = c2.w;
    bool any_pos = false, any_nonpos = false;
    for (int i = 0; i < 3; i++) {
        d[i] = __dsub_rn(cur->v[i][3], FA_W_EPSILON);
        if (d[i] > 0) any_pos = true;
        if (d[i] <= 0) any_nonpos = true;
    }
    if (!any_pos) { out.n = 0; return true; }
    if (any_nonpos) {
        if (!clip_halfspace_ge(*cur, d, *nxt)) return false;
        Poly4* t = cur; cur = nxt; nxt = t;
    }
    for (int p = 0; p < 6; p++) {
        if (cur->n == 0) break;
        int axis = p >> 1;
        bool neg = p & 1;
        bool all_ge = true;
        for (int i = 0; i < cur->n; i++) {
            double c = cur->v[i][axis];
            d[i] = neg ? __dsub_rn(cur->v[i][3], c) : __dadd_rn(cur->v[i][3], c);
            if (!(d[i] >= 0)) all_ge = false;
        }
        if (all_ge) continue;
        if (!clip_halfspace_ge(*cur, d, *nxt)) return false;
        Poly4* t = cur; cur = nxt; nxt = t;
    }
    if (cur != &out) {
        out.n = cur->n;
        for (int i = 0; i < cur->n; i++)
            for (int k = 0; k < 4; k++) out.v[i][k] = cur->v[i][k];
    }
    return true;
}

// OpenBLAS SkylakeX strided ddot (charts.py:253)
__device__ __forceinline__ double ddot_ob(const double* x, const double* y, int n) {
    double t1 = 0.0, t2 = 0.0;
    int i = 0, n1 = n & -4;
    for (; i < n1; i += 4) {
        double m3 = __dmul_rn(y[i + 2], x[i + 2]);
        double m4 = __dmul_rn(y[i + 3], x[i + 3]);
        t1 = __dadd_rn(t1, __fma_rn(y[i], x[i], m3));
        t2 = __dadd_rn(t2, __fma_rn(y[i + 1], x[i + 1], m4));
    }
    for (; i < n; i++) t1 = __fma_rn(y[i], x[i], t1);
    return __dadd_rn(t1, t2);
}

__device__ __forceinline__ double screen_x(double c, double w, int W) {
    double n = __ddiv_rn(c, w);
    return __dmul_rn(__dmul_rn(__dadd_rn(n, 1.0), 0.5), (double)W);
}

// Finish a setup from screen-space polygon (x,y,z arrays of n vertices):
// signed area / cull / flip, bbox, edges, depth plane.  charts.py:205-266.
// Returns 1 = samples possible, 0 = none, -1 = setup capacity overflow.
__device__ __forceinline__ int finish_setup(double* sx, double* sy, double* sz, int n, int W, int H,
                                            bool cull, TriSetup& s) {
    double ry[FA_MAXV], rx[FA_MAXV];
    for (int i = 0; i < n; i++) {
        int j = (i + 1 == n) ? 0 : i + 1;
        ry[i] = sy[j];
        rx[i] = sx[j];
    }
    double area2 = __dsub_rn(ddot_ob(sx, ry, n), ddot_ob(sy, rx, n));
    if (area2 == 0.0) return 0;
    if (area2 < 0.0) {
        if (cull) return 0;
        for (int i = 0; i < n / 2; i++) {
            double t;
            t = sx[i]; sx[i] = sx[n - 1 - i]; sx[n - 1 - i] = t;
            t = sy[i]; sy[i] = sy[n - 1 - i]; sy[n - 1 - i] = t;
            t = sz[i]; sz[i] = sz[n - 1 - i]; sz[n - 1 - i] = t;
        }
    }
    double mnx = sx[0], mxx = sx[0], mny = sy[0], mxy = sy[0];
    for (int i = 1; i < n; i++) {
        mnx = sx[i] < mnx ? sx[i] : mnx;
        mxx = sx[i] > mxx ? sx[i] : mxx;
        mny = sy[i] < mny ? sy[i] : mny;
        mxy = sy[i] > mxy ? sy[i] : mxy;
    }
    long long fx = (long long)floor(__dsub_rn(mnx, 0.5)), cx = (long long)ceil(mxx);
    long long fy = (long long)floor(__dsub_rn(mny, 0.5)), cy = (long long)ceil(mxy);
    s.min_x = fx > 0 ? (int)fx : 0;
    s.max_x = cx < W - 1 ? (int)cx : W - 1;
    s.min_y = fy > 0 ? (int)fy : 0;
    s.max_y = cy < H - 1 ? (int)cy : H - 1;
    if (s.min_x > s.max_x || s.min_y > s.max_y) return 0;
    if (n > FA_SETUP_MAXV) return -1;
    s.n = n;
    int mask = 0;
    for (int i = 0; i < n; i++) {
        int j = (i + 1 == n) ? 0 : i + 1;
        double dx = __dsub_rn(sx[j], sx[i]);
        double dy = __dsub_rn(sy[j], sy[i]);
        s.ex[i] = sx[i];
        s.ey[i] = sy[i];
        s.edx[i] = dx;
        s.edy[i] = dy;
        if (dy > 0 || (dy == 0 && dx < 0)) mask |= 1 << i;
    }
    s.incl_mask = mask;
    s.use_plane = 0;
    double p0x = sx[0], p0y = sy[0], p0z = sz[0];
    for (int j = 1; j < n - 1; j++) {
        double a1x = __dsub_rn(sx[j], p0x), a1y = __dsub_rn(sy[j], p0y), a1z = __dsub_rn(sz[j], p0z);
        double a2x = __dsub_rn(sx[j + 1], p0x), a2y = __dsub_rn(sy[j + 1], p0y), a2z = __dsub_rn(sz[j + 1], p0z);
        double det = __dsub_rn(__dmul_rn(a1x, a2y), __dmul_rn(a2x, a1y));
        if (fabs(det) > 1e-12) {
            s.gx = __ddiv_rn(__dsub_rn(__dmul_rn(a1z, a2y), __dmul_rn(a2z, a1y)), det);
            s.gy = __ddiv_rn(__dsub_rn(__dmul_rn(a2z, a1x), __dmul_rn(a1z, a2x)), det);
            s.p0x = p0x; s.p0y = p0y; s.p0z = p0z;
            s.use_plane = 1;
            break;
        }
    }
    if (!s.use_plane) {
        // numpy pairwise mean (charts.py:266)
        double res;
        if (n < 8) {
            res = -0.0;
            for (int i = 0; i < n; i++) res = __dadd_rn(res, sz[i]);
        } else {
            double r[8];
            int i;
            for (i = 0; i < 8; i++) r[i] = sz[i];
            for (i = 8; i < n - (n % 8); i += 8)
                for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], sz[i + k]);
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (; i < n; i++) res = __dadd_rn(res, sz[i]);
        }
        s.zmean = __ddiv_rn(res, (double)n);
    }
    return 1;
}

// Full per-triangle setup (charts.py:269-282 for one triangle).
// Returns 1 when the triangle yields a non-empty sample window, 0 otherwise,
// -1 on polygon-capacity overflow.
__device__ __forceinline__ int tri_setup(const double4* __restrict__ clip, const int* __restrict__ tris,
                                         int t, int W, int H, bool cull, TriSetup& s) {
    int ia = __ldg(tris + 3 * t), ib = __ldg(tris + 3 * t + 1), ic = __ldg(tris + 3 * t + 2);
    double4 c0 = ldg4(clip + ia), c1 = ldg4(clip + ib), c2 = ldg4(clip + ic);
    double sx[FA_MAXV], sy[FA_MAXV], sz[FA_MAXV];
    int n;
    // fast path: every vertex strictly in front and inside all six planes,
    // so _clip_triangle_frustum returns the triangle unchanged
    bool inside =
        __dsub_rn(c0.w, FA_W_EPSILON) > 0 && __dsub_rn(c1.w, FA_W_EPSILON) > 0 && __dsub_rn(c2.w, FA_W_EPSILON) > 0 &&
        __dadd_rn(c0.w, c0.x) >= 0 && __dsub_rn(c0.w, c0.x) >= 0 && __dadd_rn(c0.w, c0.y) >= 0 &&
        __dsub_rn(c0.w, c0.y) >= 0 && __dadd_rn(c0.w, c0.z) >= 0 && __dsub_rn(c0.w, c0.z) >= 0 &&
        __dadd_rn(c1.w, c1.x) >= 0 && __dsub_rn(c1.w, c1.x) >= 0 && __dadd_rn(c1.w, c1.y) >= 0 &&
        __dsub_rn(c1.w, c1.y) >= 0 && __dadd_rn(c1.w, c1.z) >= 0 && __dsub_rn(c1.w, c1.z) >= 0 &&
        __dadd_rn(c2.w, c2.x) >= 0 && __dsub_rn(c2.w, c2.x) >= 0 && __dadd_rn(c2.w, c2.y) >= 0 &&
        __dsub_rn(c2.w, c2.y) >= 0 && __dadd_rn(c2.w, c2.z) >= 0 && __dsub_rn(c2.w, c2.z) >= 0;
    if (inside) {
        n = 3;
        sx[0] = screen_x(c0.x, c0.w, W); sy[0] = screen_x(c0.y, c0.w, H); sz[0] = __ddiv_rn(c0.z, c0.w);
        sx[1] = screen_x(c1.x, c1.w, W); sy[1] = screen_x(c1.y, c1.w, H); sz[1] = __ddiv_rn(c1.z, c1.w);
        sx[2] = screen_x(c2.x, c2.w, W); sy[2] = screen_x(c2.y, c2.w, H); sz[2] = __ddiv_rn(c2.z, c2.w);
    } else {
        // reject early when no vertex is in front (charts.py:163-165)
        if (!(__dsub_rn(c0.w, FA_W_EPSILON) > 0 || __dsub_rn(c1.w, FA_W_EPSILON) > 0 ||
              __dsub_rn(c2.w, FA_W_EPSILON) > 0))
            return 0;
        Poly4 p;
        if (!clip_triangle_frustum_slow(c0, c1, c2, p)) return -1;
        if (p.n < 3) return 0;
        n = p.n;
        for (int i = 0; i < n; i++) {
            sx[i] = screen_x(p.v[i][0], p.v[i][3], W);
            sy[i] = screen_x(p.v[i][1], p.v[i][3], H);
            sz[i] = __ddiv_rn(p.v[i][2], p.v[i][3]);
        }
    }
    int r = finish_setup(sx, sy, sz, n, W, H, cull, s);
    if (r <= 0) return r;
    s.tri = t;
    return 1;
}

// ---- cluster culling (k_raster_setup) -------------------------------------
// Whole 32-triangle clusters of the setup order (fa_mesh.cu) whose triangles
// would all yield no samples are skipped before any vertex is gathered:
//  * outside: the bounding sphere lies beyond a frustum plane (or behind
//    w = W_EPSILON) by a margin far above the rounding of the reference's
//    clip coordinates, so every vertex fails that plane and clipping
//    (charts.py:160-189) leaves nothing -- clipped vertices are convex
//    combinations, still outside;
//  * back-facing (cull on, sphere strictly inside every plane, so no triangle
//    is clipped): for w_i > 0 the reference's shoelace is
//        area2 = W*H/4 * (-det3 * V) / (w0 w1 w2),  V = ((p1-p0) x (p2-p0)) . (C - p0),
//    C the projection centre, det3 = det of the x, y, w rows' 3x3 block.  The
//    normal cone and sphere bound sigma*V below by 2 * amin * g, g > 0, so
//    area2 < -area_k * 2 amin g / wmax^3; the cluster is culled only when that
//    bound exceeds tau (1e-6 px^2 + 1e-13 W H), far above the rounding of the
//    reference's area (charts.py:213-218 culls area2 < 0).
__device__ __forceinline__ bool cluster_culled(const fa_cluster& cl, const fa_view_consts& vc, bool cull) {
    const double cx = cl.c[0], cy = cl.c[1], cz = cl.c[2], r = cl.r;
    bool inside = true;
#pragma unroll
    for (int k = 0; k < 7; k++) {
        const double* P = vc.plane[k];
        const double dc = P[0] * cx + P[1] * cy + P[2] * cz + P[3];
        const double nr = vc.pn[k] * r;
        const double m = 1e-9 * (vc.pn[k] * (fabs(cx) + fabs(cy) + fabs(cz) + r) + fabs(P[3]));
        if (dc + nr < -m) return true;  // (NaN compares false: never culled)
        if (!(dc - nr > m)) inside = false;
    }
    if (!cull || !inside || !(cl.amin > 0) || vc.sigma == 0) return false;
    const double vx = vc.sigma * (vc.cam[0] - cx), vy = vc.sigma * (vc.cam[1] - cy), vz = vc.sigma * (vc.cam[2] - cz);
    const double vl = sqrt(vx * vx + vy * vy + vz * vz);
    if (!(vl > 0)) return false;
    const double cphi = (cl.a[0] * vx + cl.a[1] * vy + cl.a[2] * vz) / vl;
    const double sphi = sqrt(fmax(0.0, 1.0 - cphi * cphi));
    const double g = vl * (cphi * cl.cos_t - sphi * cl.sin_t) - r - 1e-9 * (vl + r);
    if (!(g > 0)) return false;
    const double* Pw = vc.plane[6];  // w - W_EPSILON
    const double wmax = Pw[0] * cx + Pw[1] * cy + Pw[2] * cz + Pw[3] + FA_W_EPSILON + vc.pn[6] * r;
    const double bound = vc.area_k * 2.0 * cl.amin * g / (wmax * wmax * wmax);
    return bound > vc.tau;
}

// view constants of the camera matrix m (row-major VP), screen W x H
__host__ __device__ inline void compute_view_consts(const double* m, int W, int H, fa_view_consts* vc) {
    const double* X = m;
    const double* Y = m + 4;
    const double* Z = m + 8;
    const double* Wr = m + 12;
    for (int k = 0; k < 4; k++) {
        vc->plane[0][k] = Wr[k] + X[k];
        vc->plane[1][k] = Wr[k] - X[k];
        vc->plane[2][k] = Wr[k] + Y[k];
        vc->plane[3][k] = Wr[k] - Y[k];
        vc->plane[4][k] = Wr[k] + Z[k];
        vc->plane[5][k] = Wr[k] - Z[k];
        vc->plane[6][k] = Wr[k];
    }
    vc->plane[6][3] = Wr[3] - FA_W_EPSILON;
    for (int q = 0; q < 7; q++)
        vc->pn[q] = sqrt(vc->plane[q][0] * vc->plane[q][0] + vc->plane[q][1] * vc->plane[q][1] +
                         vc->plane[q][2] * vc->plane[q][2]);
    // projection centre: X.C + X3 = Y.C + Y3 = W.C + W3 = 0 (Cramer)
    const double a00 = X[0], a01 = X[1], a02 = X[2], a10 = Y[0], a11 = Y[1], a12 = Y[2], a20 = Wr[0], a21 = Wr[1],
                 a22 = Wr[2];
    const double det3 = a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) + a02 * (a10 * a21 - a11 * a20);
    const double b0 = -X[3], b1 = -Y[3], b2 = -Wr[3];
    const double s = sqrt(a00 * a00 + a01 * a01 + a02 * a02) * sqrt(a10 * a10 + a11 * a11 + a12 * a12) *
                     sqrt(a20 * a20 + a21 * a21 + a22 * a22);
    if (!(fabs(det3) > 1e-9 * s)) {
        vc->sigma = 0.0;  // degenerate projection: no back-face culling
        vc->cam[0] = vc->cam[1] = vc->cam[2] = 0.0;
    } else {
        vc->sigma = det3 > 0 ? 1.0 : -1.0;
        vc->cam[0] = (b0 * (a11 * a22 - a12 * a21) - a01 * (b1 * a22 - a12 * b2) + a02 * (b1 * a21 - a11 * b2)) / det3;
        vc->cam[1] = (a00 * (b1 * a22 - a12 * b2) - b0 * (a10 * a22 - a12 * a20) + a02 * (a10 * b2 - b1 * a20)) / det3;
        vc->cam[2] = (a00 * (a11 * b2 - b1 * a21) - a01 * (a10 * b2 - b1 * a20) + b0 * (a10 * a21 - a11 * a20)) / det3;
    }
    vc->area_k = (double)W * (double)H * 0.25 * fabs(det3);
    vc->tau = 1e-6 + 1e-13 * (double)W * (double)H;
}

// ---- warp-parallel tri_setup (the clipping path) ---------------------------
// Same operations on the same values as tri_setup (so the same bits), with
// polygon vertex i on lane i: each Sutherland-Hodgman step (charts.py:
// 178-189) computes every output vertex -- kept vertex and/or edge crossing
// t = da / (da - db), a + t * (b - a) -- on the lane of its input vertex and
// places it by a warp prefix sum; the screen divides run one vertex per lane;
// lane 0 then finishes the setup (finish_setup: the OpenBLAS-order shoelace,
// cull / flip, bbox, edges, depth plane).  scratch: per-warp shared memory.
struct ClipScratch {
    double4 v[FA_MAXV];
    double sx[FA_MAXV], sy[FA_MAXV], sz[FA_MAXV];
};

// one clip step on the lanes' polygon (n vertices, vertex per lane, signed
// distances d): keeps d >= 0.  Returns false on capacity overflow.
__device__ __forceinline__ bool clip_step_warp(double4& v, int& n, double d, ClipScratch& cs) {
    const int lane = lane_id();
    const bool act = lane < n;
    const int j = (lane + 1 == n) ? 0 : lane + 1;
    const double db = __shfl_sync(0xffffffffu, d, j & 31);
    const double bx = __shfl_sync(0xffffffffu, v.x, j & 31), by = __shfl_sync(0xffffffffu, v.y, j & 31);
    const double bz = __shfl_sync(0xffffffffu, v.z, j & 31), bw = __shfl_sync(0xffffffffu, v.w, j & 31);
    const bool keep = act && d >= 0;
    const bool cross = act && ((d >= 0) != (db >= 0));
    const int cnt = (int)keep + (int)cross;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int m = __shfl_sync(0xffffffffu, incl, 31);
    if (m > FA_MAXV) return false;  // tri_setup fails adding the (FA_MAXV+1)-th vertex
    int pos = incl - cnt;
    __syncwarp();
    if (keep) cs.v[pos++] = v;
    if (cross) {
        const double t = __ddiv_rn(d, __dsub_rn(d, db));
        double4 o;
        o.x = __dadd_rn(v.x, __dmul_rn(t, __dsub_rn(bx, v.x)));
        o.y = __dadd_rn(v.y, __dmul_rn(t, __dsub_rn(by, v.y)));
        o.z = __dadd_rn(v.z, __dmul_rn(t, __dsub_rn(bz, v.z)));
        o.w = __dadd_rn(v.w, __dmul_rn(t, __dsub_rn(bw, v.w)));
        cs.v[pos] = o;
    }
    __syncwarp();
    n = m;
    if (lane < n) v = cs.v[lane];
    return true;
}

// 1 = setup filled (on every lane's return; `s` in shared memory), 0 = no
// samples, -1 = polygon capacity overflow.  Call with the whole warp.
static __device__ __noinline__ int tri_setup_warp(const ClipSrc clip, const int* __restrict__ tris, int t,
                                           int W, int H, bool cull, TriSetup& s, ClipScratch& cs) {
    const int lane = lane_id();
    int n = 3;
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    if (lane < 3) v = clip(__ldg(tris + 3 * t + lane));
    // charts.py:163-167: the w >= eps plane
    double d = __dsub_rn(v.w, FA_W_EPSILON);
    if (!__any_sync(0xffffffffu, lane < n && d > 0)) return 0;
    if (__any_sync(0xffffffffu, lane < n && d <= 0))
        if (!clip_step_warp(v, n, d, cs)) return -1;
    // charts.py:168-174: L, R, B, T, N, F, each skipped when every d >= 0
    for (int p = 0; p < 6; p++) {
        if (n == 0) break;
        const int axis = p >> 1;
        const double c = axis == 0 ? v.x : (axis == 1 ? v.y : v.z);
        d = (p & 1) ? __dsub_rn(v.w, c) : __dadd_rn(v.w, c);
        if (__all_sync(0xffffffffu, !(lane < n) || d >= 0)) continue;
        if (!clip_step_warp(v, n, d, cs)) return -1;
    }
    if (n < 3) return 0;
    if (lane < n) {
        cs.sx[lane] = screen_x(v.x, v.w, W);
        cs.sy[lane] = screen_x(v.y, v.w, H);
        cs.sz[lane] = __ddiv_rn(v.z, v.w);
    }
    __syncwarp();
    int r = 0;
    if (lane == 0) {
        r = finish_setup(cs.sx, cs.sy, cs.sz, n, W, H, cull, s);
        if (r > 0) s.tri = t;
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    __syncwarp();
    return r;
}

// ---- register-resident setup for unclipped triangles (the common case) ----
// Same arithmetic as tri_setup + finish_setup for n == 3, with every array
// indexed by compile-time constants so nothing lands in local memory.
struct Setup3 {
    double ax0, ay0, dx0, dy0, ax1, ay1, dx1, dy1, ax2, ay2, dx2, dy2;
    double p0x, p0y, p0z, gx, gy, zmean;
    int incl, use_plane;
    int min_x, max_x, min_y, max_y;
};

// ---- per-vertex screen record (written once per vertex by k_frame_init) ----
// {screen x, screen y, NDC z, outcode bits}: the divisions of the unclipped
// fast path depend only on the vertex, so they are done V times instead of
// 3T times (bit-identical: same operations on the same inputs).
// Outcode: bit 0 = !(w - 1e-9 > 0); bits 1-6 = !(d_p >= 0) and bits 7-12 =
// (d_p < 0) for the planes L,R,B,T,N,F (d = w+x, w-x, w+y, w-y, w+z, w-z),
// both kept so NaN coordinates classify exactly as the float tests do.
#define FA_OC_BEHIND 1u
#define FA_OC_NOTGE(p) (2u << (p))
#define FA_OC_LT(p) (0x80u << (p))

__device__ __forceinline__ double4 vertex_screen(double4 c, int W, int H) {
    unsigned code = __dsub_rn(c.w, FA_W_EPSILON) > 0 ? 0u : FA_OC_BEHIND;
    double d[6] = {__dadd_rn(c.w, c.x), __dsub_rn(c.w, c.x), __dadd_rn(c.w, c.y),
                   __dsub_rn(c.w, c.y), __dadd_rn(c.w, c.z), __dsub_rn(c.w, c.z)};
#pragma unroll
    for (int p = 0; p < 6; p++) {
        if (!(d[p] >= 0)) code |= FA_OC_NOTGE(p);
        if (d[p] < 0) code |= FA_OC_LT(p);
    }
    double4 o;
    if (code == 0) {
        o.x = __dmul_rn(__dmul_rn(__dadd_rn(__ddiv_rn(c.x, c.w), 1.0), 0.5), (double)W);
        o.y = __dmul_rn(__dmul_rn(__dadd_rn(__ddiv_rn(c.y, c.w), 1.0), 0.5), (double)H);
        o.z = __ddiv_rn(c.z, c.w);
    } else {
        o.x = o.y = o.z = 0.0;  // only read by the clipping path, which uses clip space
    }
    o.w = __longlong_as_double((long long)code);
    return o;
}

// Per-vertex NDC (x/w, y/w) of a vertex strictly inside every frustum plane
// (w - W_EPSILON > 0 and all six d >= 0), NaN otherwise.  For such a vertex
// the chart-bounds Blinn clamp (geometry.py:185-200) is the plain division
// and the UV emission's ndc (cli.py:436-439) is the same division, so both
// read these bits instead of dividing again per triangle.
__device__ __forceinline__ double2 vertex_ndc(double4 c) {
    const bool inside = __dsub_rn(c.w, FA_W_EPSILON) > 0 && __dadd_rn(c.w, c.x) >= 0 && __dsub_rn(c.w, c.x) >= 0 &&
                        __dadd_rn(c.w, c.y) >= 0 && __dsub_rn(c.w, c.y) >= 0 && __dadd_rn(c.w, c.z) >= 0 &&
                        __dsub_rn(c.w, c.z) >= 0;
    if (!inside) {
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        return make_double2(qnan, qnan);
    }
    return make_double2(__ddiv_rn(c.x, c.w), __ddiv_rn(c.y, c.w));
}

// 1 = Setup3 filled, 0 = no samples, 2 = needs the generic (clipping) path.
// Same decisions as tri_setup3 below, from the per-vertex screen records.
// ---- provably empty windows (no record for triangles that cover no sample) -
// About a quarter of the C2 small triangles cover no sample centre.  A sample
// the reference accepts (all three rounded edge values >= 0) lies within
// d < 1e-11 px of the triangle its rounded vertices and edge vectors define
// (the edge values' rounding over windows of a few hundred pixels); the
// vertices of that inflated triangle move by at most 2d / sin(min angle), and
// sin(min angle) >= area2 / Lmax^2.  So when area2 >= 1e-5 Lmax^2, every
// accepted sample centre is within 2e-6 px -- inside the margin m = 1e-4 -- of
// the vertices' bounding box:
//  * no centre within the box (+ m) in x or in y -> no sample;
//  * at most 4 centres there -> each is tested with the reference's own edge
//    arithmetic (sample_inside3); none inside -> no sample.
// Otherwise (slivers, NaN) the triangle keeps its record.
#ifndef FA_EMPTY_CULL
#define FA_EMPTY_CULL 1
#endif
#ifndef FA_EMPTY_MAXC
#define FA_EMPTY_MAXC 4  // candidate centres tested exactly (more: keep the record)
#endif
__device__ __forceinline__ bool sample_inside3(const Setup3& s, double px, double py);
__device__ __forceinline__ bool empty_window(const Setup3& s, double mnx, double mxx, double mny, double mxy,
                                             double area2) {
    const double l0 = s.dx0 * s.dx0 + s.dy0 * s.dy0, l1 = s.dx1 * s.dx1 + s.dy1 * s.dy1,
                 l2 = s.dx2 * s.dx2 + s.dy2 * s.dy2;
    const double lmax = fmax(l0, fmax(l1, l2));
    if (!(fabs(area2) >= 1e-5 * lmax)) return false;  // sliver (or NaN): keep
    const double m = 1e-4;
    const int xl = max(s.min_x, (int)ceil(mnx - m - 0.5)), xh = min(s.max_x, (int)floor(mxx + m - 0.5));
    const int yl = max(s.min_y, (int)ceil(mny - m - 0.5)), yh = min(s.max_y, (int)floor(mxy + m - 0.5));
    if (xl > xh || yl > yh) return true;
    if ((xh - xl + 1) * (yh - yl + 1) > FA_EMPTY_MAXC) return false;
    for (int iy = yl; iy <= yh; iy++)
        for (int ix = xl; ix <= xh; ix++)
            if (sample_inside3(s, (double)ix + 0.5, (double)iy + 0.5)) return false;
    return true;
}

__device__ __forceinline__ int tri_setup3s(const double4* __restrict__ scr, int ia, int ib, int ic, int W, int H,
                                           bool cull, Setup3& s) {
    double4 v0 = ldg4(scr + ia), v1 = ldg4(scr + ib), v2 = ldg4(scr + ic);
    unsigned c0 = (unsigned)__double_as_longlong(v0.w), c1 = (unsigned)__double_as_longlong(v1.w),
             c2 = (unsigned)__double_as_longlong(v2.w);
    unsigned any = c0 | c1 | c2;
    if (any) {
        unsigned all = c0 & c1 & c2;
        if (all & FA_OC_BEHIND) return 0;  // no vertex in front (charts.py:163-165)
        if (!(any & FA_OC_BEHIND)) {
            // exact trivial reject: first plane not passed by all vertices
#pragma unroll
            for (int p = 0; p < 6; p++) {
                if (!(any & FA_OC_NOTGE(p))) continue;
                if (all & FA_OC_LT(p)) return 0;
                break;
            }
        }
        return 2;
    }
    double x0 = v0.x, y0 = v0.y, z0 = v0.z;
    double x1 = v1.x, y1 = v1.y, z1 = v1.z;
    double x2 = v2.x, y2 = v2.y, z2 = v2.z;
    double A = __dadd_rn(__fma_rn(y0, x2, __fma_rn(y2, x1, __fma_rn(y1, x0, 0.0))), 0.0);
    double B = __dadd_rn(__fma_rn(x0, y2, __fma_rn(x2, y1, __fma_rn(x1, y0, 0.0))), 0.0);
    double area2 = __dsub_rn(A, B);
    if (area2 == 0.0) return 0;
    if (area2 < 0.0) {
        if (cull) return 0;
        double t;
        t = x0; x0 = x2; x2 = t;
        t = y0; y0 = y2; y2 = t;
        t = z0; z0 = z2; z2 = t;
    }
    double mnx = x0, mxx = x0, mny = y0, mxy = y0;
    mnx = x1 < mnx ? x1 : mnx; mxx = x1 > mxx ? x1 : mxx; mny = y1 < mny ? y1 : mny; mxy = y1 > mxy ? y1 : mxy;
    mnx = x2 < mnx ? x2 : mnx; mxx = x2 > mxx ? x2 : mxx; mny = y2 < mny ? y2 : mny; mxy = y2 > mxy ? y2 : mxy;
    long long fx = (long long)floor(__dsub_rn(mnx, 0.5)), cx = (long long)ceil(mxx);
    long long fy = (long long)floor(__dsub_rn(mny, 0.5)), cy = (long long)ceil(mxy);
    s.min_x = fx > 0 ? (int)fx : 0;
    s.max_x = cx < W - 1 ? (int)cx : W - 1;
    s.min_y = fy > 0 ? (int)fy : 0;
    s.max_y = cy < H - 1 ? (int)cy : H - 1;
    if (s.min_x > s.max_x || s.min_y > s.max_y) return 0;
    s.ax0 = x0; s.ay0 = y0; s.dx0 = __dsub_rn(x1, x0); s.dy0 = __dsub_rn(y1, y0);
    s.ax1 = x1; s.ay1 = y1; s.dx1 = __dsub_rn(x2, x1); s.dy1 = __dsub_rn(y2, y1);
    s.ax2 = x2; s.ay2 = y2; s.dx2 = __dsub_rn(x0, x2); s.dy2 = __dsub_rn(y0, y2);
    s.incl = ((s.dy0 > 0 || (s.dy0 == 0 && s.dx0 < 0)) ? 1 : 0) | ((s.dy1 > 0 || (s.dy1 == 0 && s.dx1 < 0)) ? 2 : 0) |
             ((s.dy2 > 0 || (s.dy2 == 0 && s.dx2 < 0)) ? 4 : 0);
#if FA_EMPTY_CULL
    if (empty_window(s, mnx, mxx, mny, mxy, area2)) return 0;
#endif
    double a1x = s.dx0, a1y = s.dy0, a1z = __dsub_rn(z1, z0);
    double a2x = __dsub_rn(x2, x0), a2y = __dsub_rn(y2, y0), a2z = __dsub_rn(z2, z0);
    double det = __dsub_rn(__dmul_rn(a1x, a2y), __dmul_rn(a2x, a1y));
    s.p0x = x0; s.p0y = y0; s.p0z = z0;
    if (fabs(det) > 1e-12) {
        s.gx = __ddiv_rn(__dsub_rn(__dmul_rn(a1z, a2y), __dmul_rn(a2z, a1y)), det);
        s.gy = __ddiv_rn(__dsub_rn(__dmul_rn(a2z, a1x), __dmul_rn(a1z, a2x)), det);
        s.use_plane = 1;
        s.zmean = 0.0;
    } else {
        s.use_plane = 0;
        s.gx = s.gy = 0.0;
        s.zmean = __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(-0.0, z0), z1), z2), 3.0);
    }
    return 1;
}

// 1 = Setup3 filled, 0 = no samples, 2 = needs the generic (clipping) path
__device__ __forceinline__ int tri_setup3(const double4* __restrict__ clip, const int* __restrict__ tris, int t,
                                          int W, int H, bool cull, Setup3& s) {
    int ia = __ldg(tris + 3 * t), ib = __ldg(tris + 3 * t + 1), ic = __ldg(tris + 3 * t + 2);
    double4 c0 = ldg4(clip + ia), c1 = ldg4(clip + ib), c2 = ldg4(clip + ic);
    bool inside =
        __dsub_rn(c0.w, FA_W_EPSILON) > 0 && __dsub_rn(c1.w, FA_W_EPSILON) > 0 && __dsub_rn(c2.w, FA_W_EPSILON) > 0 &&
        __dadd_rn(c0.w, c0.x) >= 0 && __dsub_rn(c0.w, c0.x) >= 0 && __dadd_rn(c0.w, c0.y) >= 0 &&
        __dsub_rn(c0.w, c0.y) >= 0 && __dadd_rn(c0.w, c0.z) >= 0 && __dsub_rn(c0.w, c0.z) >= 0 &&
        __dadd_rn(c1.w, c1.x) >= 0 && __dsub_rn(c1.w, c1.x) >= 0 && __dadd_rn(c1.w, c1.y) >= 0 &&
        __dsub_rn(c1.w, c1.y) >= 0 && __dadd_rn(c1.w, c1.z) >= 0 && __dsub_rn(c1.w, c1.z) >= 0 &&
        __dadd_rn(c2.w, c2.x) >= 0 && __dsub_rn(c2.w, c2.x) >= 0 && __dadd_rn(c2.w, c2.y) >= 0 &&
        __dsub_rn(c2.w, c2.y) >= 0 && __dadd_rn(c2.w, c2.z) >= 0 && __dsub_rn(c2.w, c2.z) >= 0;
    if (!inside) {
        bool f0 = __dsub_rn(c0.w, FA_W_EPSILON) > 0, f1 = __dsub_rn(c1.w, FA_W_EPSILON) > 0,
             f2 = __dsub_rn(c2.w, FA_W_EPSILON) > 0;
        if (!(f0 || f1 || f2)) return 0;
        if (f0 && f1 && f2) {
            // Exact trivial reject (charts.py:168-174): find the first plane in
            // L,R,B,T,N,F order that is not passed by all three vertices; every
            // earlier plane leaves the triangle untouched, so if all three
            // vertices fail this one, Sutherland-Hodgman returns an empty polygon.
            const double4 c[3] = {c0, c1, c2};
#pragma unroll
            for (int p = 0; p < 6; p++) {
                int ge = 0, lt = 0;
#pragma unroll
                for (int i = 0; i < 3; i++) {
                    double a = (p >> 1) == 0 ? c[i].x : ((p >> 1) == 1 ? c[i].y : c[i].z);
                    double d = (p & 1) ? __dsub_rn(c[i].w, a) : __dadd_rn(c[i].w, a);
                    ge += d >= 0;
                    lt += d < 0;
                }
                if (ge == 3) continue;
                if (lt == 3) return 0;
                break;
            }
        }
        return 2;
    }
    if (cull) {
        // Back-face pre-filter.  For w_i > 0 the screen shoelace sign equals
        // sign(D), D = det[x y w] of the clip vertices (screen area =
        // W*H/4 * D/(w0 w1 w2)).  Inside the frustum |x|,|y| <= w, so both D's
        // rounding error (~20 eps |w0w1w2|) and the reference shoelace's
        // (~1e-13 W*H) are far below the 1e-8 |w0w1w2| margin: a D under the
        // margin is certainly culled by the exact test (charts.py:213-218).
        double m0 = __dsub_rn(__dmul_rn(c1.y, c2.w), __dmul_rn(c2.y, c1.w));
        double m1 = __dsub_rn(__dmul_rn(c0.y, c2.w), __dmul_rn(c2.y, c0.w));
        double m2 = __dsub_rn(__dmul_rn(c0.y, c1.w), __dmul_rn(c1.y, c0.w));
        double D = __dadd_rn(__dsub_rn(__dmul_rn(c0.x, m0), __dmul_rn(c1.x, m1)), __dmul_rn(c2.x, m2));
        double wp = __dmul_rn(__dmul_rn(c0.w, c1.w), c2.w);
        if (D < -1e-8 * wp) return 0;
    }
    double x0 = screen_x(c0.x, c0.w, W), y0 = screen_x(c0.y, c0.w, H), z0 = __ddiv_rn(c0.z, c0.w);
    double x1 = screen_x(c1.x, c1.w, W), y1 = screen_x(c1.y, c1.w, H), z1 = __ddiv_rn(c1.z, c1.w);
    double x2 = screen_x(c2.x, c2.w, W), y2 = screen_x(c2.y, c2.w, H), z2 = __ddiv_rn(c2.z, c2.w);
    // OpenBLAS ddot tail (n = 3): t1 = fma(y_i, x_i, t1) from 0, then + t2 (= 0)
    double A = __dadd_rn(__fma_rn(y0, x2, __fma_rn(y2, x1, __fma_rn(y1, x0, 0.0))), 0.0);
    double B = __dadd_rn(__fma_rn(x0, y2, __fma_rn(x2, y1, __fma_rn(x1, y0, 0.0))), 0.0);
    double area2 = __dsub_rn(A, B);
    if (area2 == 0.0) return 0;
    if (area2 < 0.0) {
        if (cull) return 0;
        double t;
        t = x0; x0 = x2; x2 = t;
        t = y0; y0 = y2; y2 = t;
        t = z0; z0 = z2; z2 = t;
    }
    double mnx = x0, mxx = x0, mny = y0, mxy = y0;
    mnx = x1 < mnx ? x1 : mnx; mxx = x1 > mxx ? x1 : mxx; mny = y1 < mny ? y1 : mny; mxy = y1 > mxy ? y1 : mxy;
    mnx = x2 < mnx ? x2 : mnx; mxx = x2 > mxx ? x2 : mxx; mny = y2 < mny ? y2 : mny; mxy = y2 > mxy ? y2 : mxy;
    long long fx = (long long)floor(__dsub_rn(mnx, 0.5)), cx = (long long)ceil(mxx);
    long long fy = (long long)floor(__dsub_rn(mny, 0.5)), cy = (long long)ceil(mxy);
    s.min_x = fx > 0 ? (int)fx : 0;
    s.max_x = cx < W - 1 ? (int)cx : W - 1;
    s.min_y = fy > 0 ? (int)fy : 0;
    s.max_y = cy < H - 1 ? (int)cy : H - 1;
    if (s.min_x > s.max_x || s.min_y > s.max_y) return 0;
    s.ax0 = x0; s.ay0 = y0; s.dx0 = __dsub_rn(x1, x0); s.dy0 = __dsub_rn(y1, y0);
    s.ax1 = x1; s.ay1 = y1; s.dx1 = __dsub_rn(x2, x1); s.dy1 = __dsub_rn(y2, y1);
    s.ax2 = x2; s.ay2 = y2; s.dx2 = __dsub_rn(x0, x2); s.dy2 = __dsub_rn(y0, y2);
    s.incl = ((s.dy0 > 0 || (s.dy0 == 0 && s.dx0 < 0)) ? 1 : 0) | ((s.dy1 > 0 || (s.dy1 == 0 && s.dx1 < 0)) ? 2 : 0) |
             ((s.dy2 > 0 || (s.dy2 == 0 && s.dx2 < 0)) ? 4 : 0);
    double a1x = s.dx0, a1y = s.dy0, a1z = __dsub_rn(z1, z0);
    double a2x = __dsub_rn(x2, x0), a2y = __dsub_rn(y2, y0), a2z = __dsub_rn(z2, z0);
    double det = __dsub_rn(__dmul_rn(a1x, a2y), __dmul_rn(a2x, a1y));
    s.p0x = x0; s.p0y = y0; s.p0z = z0;
    if (fabs(det) > 1e-12) {
        s.gx = __ddiv_rn(__dsub_rn(__dmul_rn(a1z, a2y), __dmul_rn(a2z, a1y)), det);
        s.gy = __ddiv_rn(__dsub_rn(__dmul_rn(a2z, a1x), __dmul_rn(a1z, a2x)), det);
        s.use_plane = 1;
        s.zmean = 0.0;
    } else {
        s.use_plane = 0;
        s.gx = s.gy = 0.0;
        s.zmean = __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(-0.0, z0), z1), z2), 3.0);
    }
    return 1;
}

// Compact record of a covered small unclipped triangle, written by pass 1 so
// pass 2 never repeats the projection divides.  Edges are re-derived from the
// vertices with the same DSUBs, so the sample tests are bit-identical.
struct __align__(16) SmallRec {
    double x0, y0, x1, y1, x2, y2;  // screen vertices after the cull/flip
    double z0, g0, g1;              // plane (gx, gy) or (zmean, unused)
    int t;
    short min_x, max_x, min_y, max_y;
    int flags;                      // bits 0-2 incl, bit 3 use_plane
};

// triangle id of each small record, stored after the (T + 1) records
__device__ __forceinline__ int* small_ids(SmallRec* recs, int T) { return reinterpret_cast<int*>(recs + (T + 1)); }
__device__ __forceinline__ const int* small_ids(const SmallRec* recs, int T) {
    return reinterpret_cast<const int*>(recs + (T + 1));
}

__device__ __forceinline__ void store_rec(const Setup3& s, int t, SmallRec* r) {
    SmallRec q;
    q.x0 = s.ax0; q.y0 = s.ay0; q.x1 = s.ax1; q.y1 = s.ay1; q.x2 = s.ax2; q.y2 = s.ay2;
    q.z0 = s.p0z;
    q.g0 = s.use_plane ? s.gx : s.zmean;
    q.g1 = s.gy;
    q.t = t;
    q.min_x = (short)s.min_x; q.max_x = (short)s.max_x; q.min_y = (short)s.min_y; q.max_y = (short)s.max_y;
    q.flags = s.incl | (s.use_plane ? 8 : 0);
    *r = q;
}

__device__ __forceinline__ void load_rec(const SmallRec* __restrict__ r, Setup3& s, int& t) {
    SmallRec q = *r;
    s.ax0 = q.x0; s.ay0 = q.y0; s.ax1 = q.x1; s.ay1 = q.y1; s.ax2 = q.x2; s.ay2 = q.y2;
    s.dx0 = __dsub_rn(q.x1, q.x0); s.dy0 = __dsub_rn(q.y1, q.y0);
    s.dx1 = __dsub_rn(q.x2, q.x1); s.dy1 = __dsub_rn(q.y2, q.y1);
    s.dx2 = __dsub_rn(q.x0, q.x2); s.dy2 = __dsub_rn(q.y0, q.y2);
    s.incl = q.flags & 7;
    s.use_plane = (q.flags >> 3) & 1;
    s.p0x = q.x0; s.p0y = q.y0; s.p0z = q.z0;
    s.gx = q.g0; s.gy = q.g1; s.zmean = q.g0;
    s.min_x = q.min_x; s.max_x = q.max_x; s.min_y = q.min_y; s.max_y = q.max_y;
    t = q.t;
}

__device__ __forceinline__ bool edge_ok(double ax, double ay, double dx, double dy, bool incl, double px, double py) {
    double e = __dsub_rn(__dmul_rn(dx, __dsub_rn(py, ay)), __dmul_rn(dy, __dsub_rn(px, ax)));
    return incl ? (e >= 0) : (e > 0);
}

__device__ __forceinline__ bool sample_inside3(const Setup3& s, double px, double py) {
    return edge_ok(s.ax0, s.ay0, s.dx0, s.dy0, s.incl & 1, px, py) &&
           edge_ok(s.ax1, s.ay1, s.dx1, s.dy1, s.incl & 2, px, py) &&
           edge_ok(s.ax2, s.ay2, s.dx2, s.dy2, s.incl & 4, px, py);
}

__device__ __forceinline__ double sample_depth3(const Setup3& s, double px, double py) {
    if (s.use_plane)
        return __dadd_rn(__dadd_rn(s.p0z, __dmul_rn(s.gx, __dsub_rn(px, s.p0x))), __dmul_rn(s.gy, __dsub_rn(py, s.p0y)));
    return s.zmean;
}

// ---- hoisted sample evaluation -------------------------------------------
// e_i = dx_i*(py - ay_i) - dy_i*(px - ax_i) and z = (p0z + gx*(px - p0x)) +
// gy*(py - p0y) are evaluated with exactly the operations above; only the
// terms that depend on one coordinate are computed once per row (or per
// column) instead of once per sample, and the three edges are combined
// without short-circuiting so their DP chains overlap.
// Edge acceptance as one compare: incl ? e >= 0 : e > 0  ==  e >= thr with
// thr = 0 or the smallest positive subnormal (FP64 keeps subnormals; NaN
// fails both forms).
__device__ __forceinline__ double edge_thr(int incl_bit) { return incl_bit ? 0.0 : __longlong_as_double(1ll); }

struct RowTerms {
    double r0, r1, r2;  // dx_i * (py - ay_i)
    double zr;          // gy * (py - p0y)
    double t0, t1, t2;  // edge thresholds (edge_thr)
};

__device__ __forceinline__ RowTerms row_terms(const Setup3& s, double py) {
    RowTerms r;
    r.r0 = __dmul_rn(s.dx0, __dsub_rn(py, s.ay0));
    r.r1 = __dmul_rn(s.dx1, __dsub_rn(py, s.ay1));
    r.r2 = __dmul_rn(s.dx2, __dsub_rn(py, s.ay2));
    r.zr = __dmul_rn(s.gy, __dsub_rn(py, s.p0y));
    r.t0 = edge_thr(s.incl & 1);
    r.t1 = edge_thr(s.incl & 2);
    r.t2 = edge_thr(s.incl & 4);
    return r;
}

__device__ __forceinline__ bool inside_row(const Setup3& s, const RowTerms& r, double px) {
    double e0 = __dsub_rn(r.r0, __dmul_rn(s.dy0, __dsub_rn(px, s.ax0)));
    double e1 = __dsub_rn(r.r1, __dmul_rn(s.dy1, __dsub_rn(px, s.ax1)));
    double e2 = __dsub_rn(r.r2, __dmul_rn(s.dy2, __dsub_rn(px, s.ax2)));
    return (e0 >= r.t0) & (e1 >= r.t1) & (e2 >= r.t2);
}

__device__ __forceinline__ double depth_row(const Setup3& s, const RowTerms& r, double px) {
    if (s.use_plane) return __dadd_rn(__dadd_rn(s.p0z, __dmul_rn(s.gx, __dsub_rn(px, s.p0x))), r.zr);
    return s.zmean;
}

// ---- conservative row spans (sample pruning) -------------------------------
// Along a row, edge i's value is e_i(px) = r_i - dy_i*(px - ax_i), whose sign
// changes at x_i = ax_i + r_i/dy_i: dy_i > 0 bounds the covered samples from
// the right, dy_i < 0 from the left.  row_span() returns the pixel range
// whose samples lie within a margin M of [max left, min right]; every sample
// outside it fails the reference's exact test (charts.py:237-249), so only
// the range is tested -- exactly, with the operations above.
// Why skipping is exact, for any window: 1/dy_i comes from an FP32 MUFU
// reciprocal (relative error < 2^-22 after the FP32 rounding of dy_i) plus
// one FP64 Newton step (relative error < 2.5e-13 including its roundings),
// and is only used when |dy_i| >= 1e-3.  With |py - ay_i| <= rows + 3 (the
// unclipped vertices lie inside the screen and the window is their rounded
// bbox), the computed x_i is within
//     delta_i = 3e-13 * |dx_i| * |1/dy_i| * (rows + 3) + 1e-9
// px of the exact crossing of the reference's rounded r_i (the 1e-9 covers
// the final multiply-add's rounding for coordinates < 2^20).  The margin is
// M = FA_SPAN_MARGIN + max_i delta_i.  A sample more than M beyond the
// computed x_i is at least FA_SPAN_MARGIN = 1e-4 px beyond the exact one,
// so |r_i - dy_i (px - ax_i)| >= 1e-3 * 1e-4 = 1e-7 in the excluded
// direction, while the reference's rounded dy_i*(px - ax_i) is within
// 2.3e-16 |dy_i| (cols + 3) of exact -- below 1e-7 for windows < 10^8 px wide
// -- so its e_i has the excluded sign.  Edges with |dy_i| < 1e-3 give no
// bound (their samples are all tested exactly).  At C2 the margin stays
// below 1e-3 px.
#define FA_SPAN_MARGIN 1e-4
#define FA_SPAN_MIN_DY 1e-3

struct SpanEdges {
    double inv0, inv1, inv2;  // ~1/dy_i
    double margin;            // M above
    int kind;                 // 2 bits per edge: 1 right bound (dy > 0), 2 left bound (dy < 0), 0 none
};

__device__ __forceinline__ double approx_inv(double d) {
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)d));  // MUFU.RCP, rel. error < 2^-22
    double r = (double)rf;
    return __dmul_rn(r, __dsub_rn(2.0, __dmul_rn(d, r)));
}

__device__ __forceinline__ SpanEdges span_edges(const Setup3& f) {
    SpanEdges se;
    se.kind = 0;
    se.inv0 = se.inv1 = se.inv2 = 0.0;
    double q = 0.0;  // max |dx_i / dy_i| over the bounding edges
    if (fabs(f.dy0) >= FA_SPAN_MIN_DY) {
        se.inv0 = approx_inv(f.dy0);
        se.kind |= f.dy0 > 0 ? 1 : 2;
        q = fmax(q, fabs(f.dx0 * se.inv0));
    }
    if (fabs(f.dy1) >= FA_SPAN_MIN_DY) {
        se.inv1 = approx_inv(f.dy1);
        se.kind |= (f.dy1 > 0 ? 1 : 2) << 2;
        q = fmax(q, fabs(f.dx1 * se.inv1));
    }
    if (fabs(f.dy2) >= FA_SPAN_MIN_DY) {
        se.inv2 = approx_inv(f.dy2);
        se.kind |= (f.dy2 > 0 ? 1 : 2) << 4;
        q = fmax(q, fabs(f.dx2 * se.inv2));
    }
    // (1 + 1e-9) covers the rounding of q itself
    se.margin = FA_SPAN_MARGIN + 1e-9 + 3.0001e-13 * q * (double)(f.max_y - f.min_y + 4);
    return se;
}

__device__ __forceinline__ void span_edge(int k, double ax, double r, double inv, double& xl, double& xr) {
    if (k == 0) return;
    double x = ax + r * inv;
    if (k == 1) xr = fmin(xr, x);
    else xl = fmax(xl, x);
}

// pixel columns [lo, hi] of row terms rt that can hold covered samples
__device__ __forceinline__ void row_span(const Setup3& f, const RowTerms& rt, const SpanEdges& se, int& lo, int& hi) {
    double xl = (double)f.min_x, xr = (double)f.max_x + 1.0;
    span_edge(se.kind & 3, f.ax0, rt.r0, se.inv0, xl, xr);
    span_edge((se.kind >> 2) & 3, f.ax1, rt.r1, se.inv1, xl, xr);
    span_edge((se.kind >> 4) & 3, f.ax2, rt.r2, se.inv2, xl, xr);
    // sample px = ix + 0.5 is a candidate iff xl - M <= px <= xr + M
    // (clamped to the window so the conversions below stay in range)
    xl = fmin(xl, (double)f.max_x + 2.0);
    xr = fmax(xr, (double)f.min_x - 1.0);
    lo = max(f.min_x, (int)ceil(xl - 0.5 - se.margin));
    hi = min(f.max_x, (int)floor(xr - 0.5 + se.margin));
}

// Like row_span, plus the columns [clo, chi] whose samples certainly PASS the
// reference's edge test: the mirror of the exclusion argument above -- a
// sample more than M inside every edge's computed crossing has
// |r_i - dy_i (px - ax_i)| >= 1e-7 on the inside, far above the reference's
// rounding of e_i, so e_i > 0 (accepted with or without the top-left rule).
// Only when all three edges bound the row (|dy_i| >= 1e-3); otherwise the
// certified range is empty and every candidate is tested exactly.  Samples
// in [lo, hi] outside [clo, chi] (a crossing within M of a sample centre:
// rare) are tested exactly.
__device__ __forceinline__ void row_span_cert(const Setup3& f, const RowTerms& rt, const SpanEdges& se, int& lo,
                                              int& hi, int& clo, int& chi) {
    double xl = (double)f.min_x, xr = (double)f.max_x + 1.0;
    span_edge(se.kind & 3, f.ax0, rt.r0, se.inv0, xl, xr);
    span_edge((se.kind >> 2) & 3, f.ax1, rt.r1, se.inv1, xl, xr);
    span_edge((se.kind >> 4) & 3, f.ax2, rt.r2, se.inv2, xl, xr);
    xl = fmin(xl, (double)f.max_x + 2.0);
    xr = fmax(xr, (double)f.min_x - 1.0);
    lo = max(f.min_x, (int)ceil(xl - 0.5 - se.margin));
    hi = min(f.max_x, (int)floor(xr - 0.5 + se.margin));
    const bool all3 = (se.kind & 3) && ((se.kind >> 2) & 3) && ((se.kind >> 4) & 3);
    clo = all3 ? (int)ceil(xl - 0.5 + se.margin) : 1;
    chi = all3 ? (int)floor(xr - 0.5 - se.margin) : 0;
}

struct ColTerms {
    double c0, c1, c2;  // dy_i * (px - ax_i)
    double zc;          // p0z + gx * (px - p0x)
    double t0, t1, t2;  // edge thresholds (edge_thr)
};

__device__ __forceinline__ ColTerms col_terms(const Setup3& s, double px) {
    ColTerms c;
    c.c0 = __dmul_rn(s.dy0, __dsub_rn(px, s.ax0));
    c.c1 = __dmul_rn(s.dy1, __dsub_rn(px, s.ax1));
    c.c2 = __dmul_rn(s.dy2, __dsub_rn(px, s.ax2));
    c.zc = __dadd_rn(s.p0z, __dmul_rn(s.gx, __dsub_rn(px, s.p0x)));
    c.t0 = edge_thr(s.incl & 1);
    c.t1 = edge_thr(s.incl & 2);
    c.t2 = edge_thr(s.incl & 4);
    return c;
}

__device__ __forceinline__ bool inside_col(const Setup3& s, const ColTerms& c, double py) {
    double e0 = __dsub_rn(__dmul_rn(s.dx0, __dsub_rn(py, s.ay0)), c.c0);
    double e1 = __dsub_rn(__dmul_rn(s.dx1, __dsub_rn(py, s.ay1)), c.c1);
    double e2 = __dsub_rn(__dmul_rn(s.dx2, __dsub_rn(py, s.ay2)), c.c2);
    return (e0 >= c.t0) & (e1 >= c.t1) & (e2 >= c.t2);
}

__device__ __forceinline__ double depth_col(const Setup3& s, const ColTerms& c, double py) {
    if (s.use_plane) return __dadd_rn(c.zc, __dmul_rn(s.gy, __dsub_rn(py, s.p0y)));
    return s.zmean;
}

// ---- hierarchical-Z rejection for the visibility pass ----------------------
// Lower bound of the sampled depth over the pixel rectangle [xa,xb]x[ya,yb]:
// the plane is linear, so its minimum over the rectangle's sample positions is
// at a corner; the computed z (three roundings, charts.py:266 order) differs
// from the exact plane value by < 8 ulp of |p0z| + |gx dx| + |gy dy|, far below
// the 1e-12 relative margin subtracted here.
__device__ __forceinline__ double depth_lower_bound(const Setup3& f, int xa, int xb, int ya, int yb) {
    if (!f.use_plane) return f.zmean;
    double ta = f.gx * (((double)xa + 0.5) - f.p0x), tb = f.gx * (((double)xb + 0.5) - f.p0x);
    double ua = f.gy * (((double)ya + 0.5) - f.p0y), ub = f.gy * (((double)yb + 0.5) - f.p0y);
    double lo = f.p0z + fmin(ta, tb) + fmin(ua, ub);
    double mag = fabs(f.p0z) + fmax(fabs(ta), fabs(tb)) + fmax(fabs(ua), fabs(ub));
    return lo - 1e-12 * mag;
}

// True when no sample in the rectangle can pass z <= stored + 1e-6 max(1,|stored|)
// against the final depth: for every 8x8 tile it touches, zlb exceeds the
// threshold of the tile's largest stored depth (the threshold is monotone in
// the stored depth, so that bounds every pixel of the tile).  NaN never rejects.
__device__ __forceinline__ bool hiz_tile_rejects(unsigned long long k, double zlb) {
    if (k == 0) return true;  // no coverable pixel in this tile
    double stored = key_f64(k), a = fabs(stored);
    double thr = __dadd_rn(stored, __dmul_rn(FA_DEPTH_EPSILON, 1.0 > a ? 1.0 : a));  // as depth_passes
    return zlb > thr;
}

__device__ __forceinline__ bool hiz_rejects(const unsigned long long* __restrict__ hiz, int htx, int xa, int xb,
                                            int ya, int yb, double zlb) {
    for (int ty = ya / FA_HIZ; ty <= yb / FA_HIZ; ty++)
        for (int tx = xa / FA_HIZ; tx <= xb / FA_HIZ; tx++)
            if (!hiz_tile_rejects(__ldg(hiz + ty * htx + tx), zlb)) return false;
    return true;
}

__device__ __forceinline__ void setup3_to_generic(const Setup3& a, int t, TriSetup& s) {
    s.tri = t;
    s.n = 3;
    s.min_x = a.min_x; s.max_x = a.max_x; s.min_y = a.min_y; s.max_y = a.max_y;
    s.use_plane = a.use_plane;
    s.incl_mask = a.incl;
    s.p0x = a.p0x; s.p0y = a.p0y; s.p0z = a.p0z; s.gx = a.gx; s.gy = a.gy; s.zmean = a.zmean;
    s.ex[0] = a.ax0; s.ey[0] = a.ay0; s.edx[0] = a.dx0; s.edy[0] = a.dy0;
    s.ex[1] = a.ax1; s.ey[1] = a.ay1; s.edx[1] = a.dx1; s.edy[1] = a.dy1;
    s.ex[2] = a.ax2; s.ey[2] = a.ay2; s.edx[2] = a.dx2; s.edy[2] = a.dy2;
}

__device__ __forceinline__ bool sample_inside(const TriSetup& s, double px, double py) {
    for (int i = 0; i < s.n; i++) {
        double e = __dsub_rn(__dmul_rn(s.edx[i], __dsub_rn(py, s.ey[i])), __dmul_rn(s.edy[i], __dsub_rn(px, s.ex[i])));
        bool ok = ((s.incl_mask >> i) & 1) ? (e >= 0) : (e > 0);
        if (!ok) return false;
    }
    return true;
}

__device__ __forceinline__ double sample_depth(const TriSetup& s, double px, double py) {
    if (s.use_plane)
        return __dadd_rn(__dadd_rn(s.p0z, __dmul_rn(s.gx, __dsub_rn(px, s.p0x))), __dmul_rn(s.gy, __dsub_rn(py, s.p0y)));
    return s.zmean;
}

// charts.py:309-311: z <= stored + 1e-6 * max(1, |stored|)
__device__ __forceinline__ bool depth_passes(double z, double stored) {
    double a = fabs(stored);
    double slack = __dmul_rn(FA_DEPTH_EPSILON, 1.0 > a ? 1.0 : a);
    return z <= __dadd_rn(stored, slack);
}
