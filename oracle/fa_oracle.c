/*
 * fa_oracle.c — CPU restatement of the reference atlaspack per-frame path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2502_17712_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product path never links or calls it.
 *
 * Parity pinning: every function below follows the reference file:line it
 * cites, with the reference's exact IEEE-754 float64 operation order
 * (SURVEY.md §8.1).  The two places where the reference's arithmetic runs
 * inside OpenBLAS (numpy `@` and `np.dot`) are restated as the SkylakeX
 * kernels' FMA chains; both were checked bit-for-bit against numpy 2.3.5 /
 * scipy-openblas 0.3.30 in this container, and the whole oracle is pinned
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures, tests/test_oracle.py).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: no implicit FMA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define W_EPSILON 1e-9      /* geometry.py:19 */
#define DEPTH_EPSILON 1e-6  /* charts.py:26 */
#define MAX_POLY 64         /* clipped polygons stay far below this */
#define MAX_BOX_DIM (1LL << 23)  /* packing.py:25 */
#define SCALE_GRID_BITS 24       /* packing.py:29 */
#define DIRECTION_PERIOD 3       /* packing.py:32 */
#define MAX_OVERFLOW_ITERATIONS 8 /* packing.py:34 */

/* status codes shared with include/fastatlas.h */
#define ORC_OK 0
#define ORC_VALUE_ERROR 1
#define ORC_PACK_FAILURE 2
#define ORC_NOTHING_VISIBLE 3
#define ORC_HEIGHT_OVERFLOW 4
#define ORC_INTERNAL -100

/* ------------------------------------------------------------------------ */
/* projection: charts.py:273-274, geometry.py:301, cli.py:422-423            */
/* homo @ vp.T through OpenBLAS dgemm: acc = x*m0; fma(y,m1); fma(z,m2);      */
/* fma(1,m3)                                                   */
/* ------------------------------------------------------------------------ */
static void project_one(const double *p, const double *vp, double out[4])
{
    for (int r = 0; r < 4; r++) {
        double a = p[0] * vp[r * 4 + 0];
        a = fma(p[1], vp[r * 4 + 1], a);
        a = fma(p[2], vp[r * 4 + 2], a);
        a = fma(1.0, vp[r * 4 + 3], a);
        out[r] = a;
    }
}

void orc_project(const double *pos, int64_t V, const double *vp, double *clip)
{
    for (int64_t v = 0; v < V; v++) project_one(pos + 3 * v, vp, clip + 4 * v);
}

/* ------------------------------------------------------------------------ */
/* rasterization (charts.py:150-282)                                          */
/* ------------------------------------------------------------------------ */
typedef struct { double v[MAX_POLY][4]; int n; } poly4;

/* charts.py:178-189: keep d >= 0, interpolate a + t*(b-a), t = da/(da-db) */
static int clip_halfspace_ge(const poly4 *in, const double *d, poly4 *out)
{
    int n = in->n, m = 0;
    for (int i = 0; i < n; i++) {
        int j = (i + 1) % n;
        double da = d[i], db = d[j];
        if (da >= 0) {
            if (m >= MAX_POLY) return -1;
            memcpy(out->v[m++], in->v[i], sizeof(double) * 4);
        }
        if ((da >= 0) != (db >= 0)) {
            double t = da / (da - db);
            if (m >= MAX_POLY) return -1;
            for (int k = 0; k < 4; k++) out->v[m][k] = in->v[i][k] + t * (in->v[j][k] - in->v[i][k]);
            m++;
        }
    }
    out->n = m;
    return 0;
}

/* charts.py:150-157 plane list, charts.py:160-175 the clip */
static int clip_triangle_frustum(const double c[3][4], poly4 *out)
{
    static const int axis[6] = {0, 0, 1, 1, 2, 2};
    static const double sgn[6] = {1.0, -1.0, 1.0, -1.0, 1.0, -1.0};
    poly4 a, b;
    double d[MAX_POLY];
    a.n = 3;
    for (int i = 0; i < 3; i++) memcpy(a.v[i], c[i], sizeof(double) * 4);
    int any_pos = 0, any_nonpos = 0;
    for (int i = 0; i < 3; i++) {
        d[i] = c[i][3] - W_EPSILON;
        if (d[i] > 0) any_pos = 1;
        if (d[i] <= 0) any_nonpos = 1;
    }
    if (!any_pos) { out->n = 0; return 0; }
    poly4 *cur = &a, *nxt = &b;
    if (any_nonpos) {
        if (clip_halfspace_ge(cur, d, nxt)) return -1;
        poly4 *t = cur; cur = nxt; nxt = t;
    }
    for (int p = 0; p < 6; p++) {
        if (cur->n == 0) break;
        int all_ge = 1;
        for (int i = 0; i < cur->n; i++) {
            d[i] = cur->v[i][3] + sgn[p] * cur->v[i][axis[p]];
            if (!(d[i] >= 0)) all_ge = 0;
        }
        if (all_ge) continue;
        if (clip_halfspace_ge(cur, d, nxt)) return -1;
        poly4 *t = cur; cur = nxt; nxt = t;
    }
    *out = *cur;
    return 0;
}

/* OpenBLAS SkylakeX strided ddot (np.dot at charts.py:253) */
static double ddot_strided(const double *x, const double *y, int n)
{
    double t1 = 0.0, t2 = 0.0;
    int i = 0, n1 = n & -4;
    for (; i < n1; i += 4) {
        double m3 = y[i + 2] * x[i + 2];
        double m4 = y[i + 3] * x[i + 3];
        t1 += fma(y[i], x[i], m3);
        t2 += fma(y[i + 1], x[i + 1], m4);
    }
    for (; i < n; i++) t1 = fma(y[i], x[i], t1);
    return t1 + t2;
}

typedef struct {
    double x[MAX_POLY], y[MAX_POLY], z[MAX_POLY];
    int n;
} spoly;

/* charts.py:192-202 */
static void polygon_to_screen(const poly4 *p, int W, int H, spoly *s)
{
    s->n = p->n;
    for (int i = 0; i < p->n; i++) {
        double nx = p->v[i][0] / p->v[i][3];
        double ny = p->v[i][1] / p->v[i][3];
        double nz = p->v[i][2] / p->v[i][3];
        s->x[i] = (nx + 1.0) * 0.5 * (double)W;
        s->y[i] = (ny + 1.0) * 0.5 * (double)H;
        s->z[i] = nz;
    }
}

/* charts.py:251-253 */
static double signed_area2(const spoly *s)
{
    double ry[MAX_POLY], rx[MAX_POLY];
    int n = s->n;
    for (int i = 0; i < n; i++) { ry[i] = s->y[(i + 1) % n]; rx[i] = s->x[(i + 1) % n]; }
    return ddot_strided(s->x, ry, n) - ddot_strided(s->y, rx, n);
}

/* exported for the host-arithmetic probe (tests/test_host_arithmetic.py):
 * _signed_area2 of an n-gon given as x[n], y[n] (charts.py:251-253) */
double orc_signed_area2(const double *x, const double *y, int n)
{
    spoly s;
    if (n < 1 || n > MAX_POLY) return 0.0;
    s.n = n;
    for (int i = 0; i < n; i++) { s.x[i] = x[i]; s.y[i] = y[i]; s.z[i] = 0.0; }
    return signed_area2(&s);
}

/* numpy pairwise sum used by poly[:,2].mean() (charts.py:266) */
static double np_mean(const double *a, int n)
{
    double res;
    if (n < 8) {
        res = -0.0;
        for (int i = 0; i < n; i++) res += a[i];
    } else {
        double r[8];
        int i;
        for (i = 0; i < 8; i++) r[i] = a[i];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += a[i + k];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
    }
    return res / (double)n;
}

typedef struct {
    int ok;            /* 0 -> no samples */
    int n;
    double ex[MAX_POLY], ey[MAX_POLY], edx[MAX_POLY], edy[MAX_POLY];
    int incl[MAX_POLY];
    int min_x, max_x, min_y, max_y;
    int use_plane;
    double p0x, p0y, p0z, gx, gy, zmean;
} raster_setup;

/* charts.py:205-248 setup + charts.py:256-266 depth plane */
static void raster_prepare(spoly *s, int W, int H, int cull, raster_setup *rs)
{
    rs->ok = 0;
    double area2 = signed_area2(s);
    if (area2 == 0.0) return;
    int n = s->n;
    if (area2 < 0.0) {
        if (cull) return;
        for (int i = 0; i < n / 2; i++) {
            double t;
            t = s->x[i]; s->x[i] = s->x[n - 1 - i]; s->x[n - 1 - i] = t;
            t = s->y[i]; s->y[i] = s->y[n - 1 - i]; s->y[n - 1 - i] = t;
            t = s->z[i]; s->z[i] = s->z[n - 1 - i]; s->z[n - 1 - i] = t;
        }
    }
    double mnx = s->x[0], mxx = s->x[0], mny = s->y[0], mxy = s->y[0];
    for (int i = 1; i < n; i++) {
        if (s->x[i] < mnx) mnx = s->x[i];
        if (s->x[i] > mxx) mxx = s->x[i];
        if (s->y[i] < mny) mny = s->y[i];
        if (s->y[i] > mxy) mxy = s->y[i];
    }
    long fx = (long)floor(mnx - 0.5), cx = (long)ceil(mxx);
    long fy = (long)floor(mny - 0.5), cy = (long)ceil(mxy);
    rs->min_x = fx > 0 ? (int)fx : 0;
    rs->max_x = cx < W - 1 ? (int)cx : W - 1;
    rs->min_y = fy > 0 ? (int)fy : 0;
    rs->max_y = cy < H - 1 ? (int)cy : H - 1;
    if (rs->min_x > rs->max_x || rs->min_y > rs->max_y) return;
    rs->n = n;
    for (int i = 0; i < n; i++) {
        int j = (i + 1) % n;
        double ax = s->x[i], ay = s->y[i], bx = s->x[j], by = s->y[j];
        rs->ex[i] = ax; rs->ey[i] = ay;
        rs->edx[i] = bx - ax; rs->edy[i] = by - ay;
        double dy = by - ay;
        rs->incl[i] = (dy > 0 || (dy == 0 && bx - ax < 0));
    }
    /* _interp_depth: first fan triangle with |det| > 1e-12 */
    rs->use_plane = 0;
    double p0x = s->x[0], p0y = s->y[0], p0z = s->z[0];
    for (int j = 1; j < n - 1; j++) {
        double p1x = s->x[j], p1y = s->y[j], p1z = s->z[j];
        double p2x = s->x[j + 1], p2y = s->y[j + 1], p2z = s->z[j + 1];
        double det = (p1x - p0x) * (p2y - p0y) - (p2x - p0x) * (p1y - p0y);
        if (fabs(det) > 1e-12) {
            rs->gx = ((p1z - p0z) * (p2y - p0y) - (p2z - p0z) * (p1y - p0y)) / det;
            rs->gy = ((p2z - p0z) * (p1x - p0x) - (p1z - p0z) * (p2x - p0x)) / det;
            rs->p0x = p0x; rs->p0y = p0y; rs->p0z = p0z;
            rs->use_plane = 1;
            break;
        }
    }
    if (!rs->use_plane) rs->zmean = np_mean(s->z, n);
    rs->ok = 1;
}

static inline int sample_inside(const raster_setup *rs, double px, double py)
{
    for (int i = 0; i < rs->n; i++) {
        double e = rs->edx[i] * (py - rs->ey[i]) - rs->edy[i] * (px - rs->ex[i]);
        if (rs->incl[i]) { if (!(e >= 0)) return 0; }
        else { if (!(e > 0)) return 0; }
    }
    return 1;
}

static inline double sample_depth(const raster_setup *rs, double px, double py)
{
    if (rs->use_plane) return rs->p0z + rs->gx * (px - rs->p0x) + rs->gy * (py - rs->p0y);
    return rs->zmean;
}

/* charts.py:269-282 for one triangle: returns 1 with rs filled when it yields samples */
static int triangle_setup(const double *clip, const int64_t *tri, int W, int H, int cull,
                          raster_setup *rs, int *err)
{
    double c[3][4];
    for (int k = 0; k < 3; k++) memcpy(c[k], clip + 4 * tri[k], sizeof(double) * 4);
    poly4 p;
    if (clip_triangle_frustum(c, &p)) { *err = 1; return 0; }
    if (p.n < 3) return 0;
    spoly s;
    polygon_to_screen(&p, W, H, &s);
    raster_prepare(&s, W, H, cull, rs);
    return rs->ok;
}

/* charts.py:285-299 ; depth is (H, W) row-major, +inf when uncovered */
int orc_depth_prepass(const double *pos, int64_t V, const int64_t *tris, int64_t T,
                      const double *vp, int W, int H, int cull, double *depth)
{
    if (W < 1 || H < 1) return ORC_VALUE_ERROR;
    for (int64_t i = 0; i < (int64_t)W * H; i++) depth[i] = INFINITY;
    double *clip = (double *)malloc(sizeof(double) * 4 * (V > 0 ? V : 1));
    orc_project(pos, V, vp, clip);
    int err = 0;
    raster_setup rs;
    for (int64_t t = 0; t < T; t++) {
        if (!triangle_setup(clip, tris + 3 * t, W, H, cull, &rs, &err)) continue;
        for (int iy = rs.min_y; iy <= rs.max_y; iy++) {
            double py = (double)iy + 0.5;
            for (int ix = rs.min_x; ix <= rs.max_x; ix++) {
                double px = (double)ix + 0.5;
                if (!sample_inside(&rs, px, py)) continue;
                double z = sample_depth(&rs, px, py);
                double *d = depth + (int64_t)iy * W + ix;
                if (z < *d || isnan(z)) *d = z; /* np.minimum */
            }
        }
    }
    free(clip);
    return err ? ORC_INTERNAL : ORC_OK;
}

/* charts.py:302-313 */
int orc_mark_visible(const double *pos, int64_t V, const int64_t *tris, int64_t T,
                     const double *vp, const double *depth, int W, int H, int cull, uint8_t *flags)
{
    double *clip = (double *)malloc(sizeof(double) * 4 * (V > 0 ? V : 1));
    orc_project(pos, V, vp, clip);
    int err = 0;
    raster_setup rs;
    for (int64_t t = 0; t < T; t++) {
        flags[t] = 0;
        if (!triangle_setup(clip, tris + 3 * t, W, H, cull, &rs, &err)) continue;
        for (int iy = rs.min_y; iy <= rs.max_y && !flags[t]; iy++) {
            double py = (double)iy + 0.5;
            for (int ix = rs.min_x; ix <= rs.max_x; ix++) {
                double px = (double)ix + 0.5;
                if (!sample_inside(&rs, px, py)) continue;
                double z = sample_depth(&rs, px, py);
                double stored = depth[(int64_t)iy * W + ix];
                double a = fabs(stored);
                double slack = DEPTH_EPSILON * (1.0 > a ? 1.0 : a);
                if (z <= stored + slack) { flags[t] = 1; break; }
            }
        }
    }
    free(clip);
    return err ? ORC_INTERNAL : ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* chartification (charts.py:64-77, 319-406)                                  */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t u, v, t, e; } edge_rec;

static int edge_cmp(const void *a, const void *b)
{
    const edge_rec *x = (const edge_rec *)a, *y = (const edge_rec *)b;
    if (x->u != y->u) return x->u < y->u ? -1 : 1;
    if (x->v != y->v) return x->v < y->v ? -1 : 1;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    return (x->e > y->e) - (x->e < y->e);
}

/* charts.py:64-77: link only edges used by exactly two (t, e) slots */
void orc_build_adjacency(const int64_t *tris, int64_t T, int64_t *adj)
{
    edge_rec *E = (edge_rec *)malloc(sizeof(edge_rec) * 3 * (T > 0 ? T : 1));
    for (int64_t t = 0; t < T; t++) {
        for (int e = 0; e < 3; e++) {
            int64_t a = tris[3 * t + e], b = tris[3 * t + (e + 1) % 3];
            edge_rec *r = &E[3 * t + e];
            r->u = a < b ? a : b; r->v = a < b ? b : a; r->t = t; r->e = e;
            adj[3 * t + e] = -1;
        }
    }
    int64_t n = 3 * T;
    qsort(E, (size_t)n, sizeof(edge_rec), edge_cmp);
    for (int64_t i = 0; i < n;) {
        int64_t j = i + 1;
        while (j < n && E[j].u == E[i].u && E[j].v == E[i].v) j++;
        if (j - i == 2) {
            adj[3 * E[i].t + E[i].e] = E[i + 1].t;
            adj[3 * E[i + 1].t + E[i + 1].e] = E[i].t;
        }
        i = j;
    }
    free(E);
}

/* charts.py:319-340 */
static int64_t ds_find(int64_t *parent, int64_t a)
{
    int64_t root = a;
    while (parent[root] != root) root = parent[root];
    while (parent[a] != root) { int64_t nx = parent[a]; parent[a] = root; a = nx; }
    return root;
}

static void ds_union(int64_t *parent, int64_t a, int64_t b)
{
    int64_t ra = ds_find(parent, a), rb = ds_find(parent, b);
    if (ra != rb) {
        if (ra < rb) parent[rb] = ra; else parent[ra] = rb;
    }
}

/* charts.py:389-406 (labels only; canonical label = min member of each root) */
static void labels_from_roots(int64_t *parent, const uint8_t *vis, int64_t T, int64_t *labels)
{
    int64_t *canon = (int64_t *)malloc(sizeof(int64_t) * (T > 0 ? T : 1));
    for (int64_t t = 0; t < T; t++) canon[t] = -1;
    for (int64_t t = 0; t < T; t++) {
        if (!vis[t]) continue;
        int64_t r = ds_find(parent, t);
        if (canon[r] < 0 || t < canon[r]) canon[r] = t;
    }
    for (int64_t t = 0; t < T; t++) labels[t] = vis[t] ? canon[ds_find(parent, t)] : -1;
    free(canon);
}

/* charts.py:343-359 */
void orc_connected_charts(const int64_t *adj, const uint8_t *flags, int64_t T, int64_t *labels)
{
    int64_t *parent = (int64_t *)malloc(sizeof(int64_t) * (T > 0 ? T : 1));
    for (int64_t t = 0; t < T; t++) parent[t] = t;
    for (int64_t t = 0; t < T; t++) {
        if (!flags[t]) continue;
        for (int e = 0; e < 3; e++) {
            int64_t nb = adj[3 * t + e];
            if (nb >= 0 && flags[nb]) ds_union(parent, t, nb);
        }
    }
    labels_from_roots(parent, flags, T, labels);
    free(parent);
}

/* charts.py:362-386; v2c[v] = chart of vertex v or -1 */
void orc_merge_shared_vertices(const int64_t *tris, int64_t T, int64_t V, const int64_t *labels_in,
                               int64_t *labels_out, int64_t *v2c)
{
    int64_t *parent = (int64_t *)malloc(sizeof(int64_t) * (T > 0 ? T : 1));
    int64_t *first = (int64_t *)malloc(sizeof(int64_t) * (V > 0 ? V : 1));
    uint8_t *vis = (uint8_t *)calloc((size_t)(T > 0 ? T : 1), 1);
    for (int64_t t = 0; t < T; t++) { parent[t] = t; vis[t] = labels_in[t] >= 0; }
    for (int64_t v = 0; v < V; v++) first[v] = -1;
    /* union(root, t) for every member: members of a chart share its label */
    for (int64_t t = 0; t < T; t++)
        if (vis[t]) ds_union(parent, labels_in[t], t);
    for (int64_t t = 0; t < T; t++) {
        if (!vis[t]) continue;
        for (int k = 0; k < 3; k++) {
            int64_t v = tris[3 * t + k];
            if (first[v] < 0) first[v] = t;
            else if (first[v] != t) ds_union(parent, t, first[v]);
        }
    }
    labels_from_roots(parent, vis, T, labels_out);
    for (int64_t v = 0; v < V; v++) v2c[v] = first[v] >= 0 ? labels_out[first[v]] : -1;
    free(parent); free(first); free(vis);
}

/* ------------------------------------------------------------------------ */
/* chart bounds (geometry.py:185-322, 352-362; cli.py:374-384)                */
/* ------------------------------------------------------------------------ */
/* geometry.py:185-200 */
static void blinn_clamped_ndc(const double *p, double *cx, double *cy)
{
    double x = p[0], y = p[1], w = p[3];
    double aw = fabs(w);
    if (aw == 0.0) {
        *cx = x < 0 ? -1.0 : 1.0;
        *cy = y < 0 ? -1.0 : 1.0;
        return;
    }
    double t;
    t = (-aw > x) ? -aw : x;  /* max(x, -aw) */
    t = (aw < t) ? aw : t;    /* min(., aw)  */
    *cx = t / aw;
    t = (-aw > y) ? -aw : y;
    t = (aw < t) ? aw : t;
    *cy = t / aw;
}

/* geometry.py:203-220: keep d > 0 */
static int clip_poly_halfspace_gt(const poly4 *in, const double *d, poly4 *out)
{
    int n = in->n, m = 0;
    for (int i = 0; i < n; i++) {
        int j = (i + 1) % n;
        double da = d[i], db = d[j];
        if (da > 0) {
            if (m >= MAX_POLY) return -1;
            memcpy(out->v[m++], in->v[i], sizeof(double) * 4);
        }
        if ((da > 0) != (db > 0)) {
            double t = da / (da - db);
            if (m >= MAX_POLY) return -1;
            for (int k = 0; k < 4; k++) out->v[m][k] = in->v[i][k] + t * (in->v[j][k] - in->v[i][k]);
            m++;
        }
    }
    out->n = m;
    return 0;
}

/* geometry.py:239-247 */
static void side_dists(const poly4 *p, int plane, double *d)
{
    for (int i = 0; i < p->n; i++) {
        const double *v = p->v[i];
        switch (plane) {
        case 0: d[i] = v[3] + v[0]; break;
        case 1: d[i] = v[3] - v[0]; break;
        case 2: d[i] = v[3] + v[1]; break;
        default: d[i] = v[3] - v[1]; break;
        }
    }
}

/* geometry.py:250-254 + NdcBox.area (geometry.py:140-142) */
static double blinn_box_area(const poly4 *p)
{
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int i = 0; i < p->n; i++) {
        double cx, cy;
        blinn_clamped_ndc(p->v[i], &cx, &cy);
        /* python min()/max() over lists: first extreme wins */
        if (i == 0) { mnx = mxx = cx; mny = mxy = cy; continue; }
        if (cx < mnx) mnx = cx;
        if (cx > mxx) mxx = cx;
        if (cy < mny) mny = cy;
        if (cy > mxy) mxy = cy;
    }
    return (mxx - mnx) * (mxy - mny);
}

/* geometry.py:257-278: returns -1 for None */
static int select_side_plane(const poly4 *tri, int *err)
{
    double best_area = 0;
    int best = -1;
    double d[MAX_POLY];
    for (int idx = 0; idx < 4; idx++) {
        side_dists(tri, idx, d);
        int anyp = 0, anyn = 0;
        for (int i = 0; i < tri->n; i++) { if (d[i] > 0) anyp = 1; if (d[i] < 0) anyn = 1; }
        if (!(anyp && anyn)) continue;
        poly4 c;
        if (clip_poly_halfspace_gt(tri, d, &c)) { *err = 1; return -1; }
        double area = blinn_box_area(&c);
        /* key (area, idx) < best: idx ascending, so strict area compare */
        if (best < 0 || area < best_area) { best = idx; best_area = area; }
    }
    return best;
}

/* geometry.py:281-322 per-triangle contribution; returns 1 if it survived */
static int tri_bbox_contrib(const double c[3][4], double box[4], int *err)
{
    poly4 tri, poly;
    tri.n = 3;
    for (int i = 0; i < 3; i++) memcpy(tri.v[i], c[i], sizeof(double) * 4);
    double d[MAX_POLY];
    int allp = 1, anyp = 0;
    for (int i = 0; i < 3; i++) {
        d[i] = c[i][3] - W_EPSILON;
        if (d[i] > 0) anyp = 1; else allp = 0;
    }
    if (allp) {
        int plane = select_side_plane(&tri, err);
        if (plane < 0) poly = tri;
        else {
            side_dists(&tri, plane, d);
            if (clip_poly_halfspace_gt(&tri, d, &poly)) { *err = 1; return 0; }
        }
    } else if (anyp) {
        if (clip_poly_halfspace_gt(&tri, d, &poly)) { *err = 1; return 0; }
    } else {
        return 0;
    }
    for (int i = 0; i < poly.n; i++) {
        double cx, cy;
        blinn_clamped_ndc(poly.v[i], &cx, &cy);
        if (cx < box[0]) box[0] = cx;  /* min(min_x, cx) */
        if (cy < box[1]) box[1] = cy;
        if (cx > box[2]) box[2] = cx;
        if (cy > box[3]) box[3] = cy;
    }
    return 1;
}

/* chart_bbox over an explicit list of world triangles (n,3,3); returns 1 on
 * success, 0 for DegenerateChart.  box = (min_x, min_y, max_x, max_y). */
int orc_chart_bbox(const double *tris_xyz, int64_t n, const double *vp, double *box)
{
    box[0] = box[1] = INFINITY;
    box[2] = box[3] = -INFINITY;
    int survived = 0, err = 0;
    for (int64_t i = 0; i < n; i++) {
        double c[3][4];
        for (int k = 0; k < 3; k++) project_one(tris_xyz + 9 * i + 3 * k, vp, c[k]);
        if (tri_bbox_contrib(c, box, &err)) survived = 1;
    }
    if (err) return ORC_INTERNAL;
    return survived;
}

/* geometry.py:352-362 */
static void viewport_box(const double box[4], int W, int H, int64_t *w, int64_t *h)
{
    double fw = ceil((box[2] - box[0]) / 2.0 * (double)W);
    double fh = ceil((box[3] - box[1]) / 2.0 * (double)H);
    *w = fw < 1 ? 1 : (int64_t)fw;
    *h = fh < 1 ? 1 : (int64_t)fh;
}

void orc_viewport_box(const double *box, int W, int H, int64_t *wh)
{
    viewport_box(box, W, H, &wh[0], &wh[1]);
}

/* cli.py:371-384: per chart (ascending roots) box, pixel dims, target dims.
 * labels: merged chart_of_triangle (-1 invisible).  Outputs sized >= #charts.
 * Returns number of charts written (degenerate charts skipped, see
 * cli.py:377-378), or negative status. */
int64_t orc_chart_boxes(const double *pos, int64_t V, const int64_t *tris, int64_t T,
                        const double *vp, const int64_t *labels, int W, int H, double prescale,
                        int64_t *roots, double *ndc, int64_t *px, int64_t *target)
{
    double *clip = (double *)malloc(sizeof(double) * 4 * (V > 0 ? V : 1));
    orc_project(pos, V, vp, clip);
    int64_t *cidx = (int64_t *)malloc(sizeof(int64_t) * (T > 0 ? T : 1));
    int64_t C = 0;
    for (int64_t t = 0; t < T; t++) {
        cidx[t] = -1;
        if (labels[t] == t) cidx[t] = C++;
    }
    double *bx = (double *)malloc(sizeof(double) * 4 * (C > 0 ? C : 1));
    uint8_t *surv = (uint8_t *)calloc((size_t)(C > 0 ? C : 1), 1);
    for (int64_t c = 0; c < C; c++) {
        bx[4 * c + 0] = bx[4 * c + 1] = INFINITY;
        bx[4 * c + 2] = bx[4 * c + 3] = -INFINITY;
    }
    int err = 0;
    for (int64_t t = 0; t < T; t++) {
        if (labels[t] < 0) continue;
        int64_t c = cidx[labels[t]];
        double cc[3][4];
        for (int k = 0; k < 3; k++) memcpy(cc[k], clip + 4 * tris[3 * t + k], sizeof(double) * 4);
        if (tri_bbox_contrib(cc, bx + 4 * c, &err)) surv[c] = 1;
    }
    int64_t out = 0;
    for (int64_t t = 0; t < T; t++) {
        if (cidx[t] < 0) continue;
        int64_t c = cidx[t];
        if (!surv[c]) continue;
        int64_t w, h;
        viewport_box(bx + 4 * c, W, H, &w, &h);
        double tw = ceil(prescale * (double)w), th = ceil(prescale * (double)h);
        roots[out] = t;
        memcpy(ndc + 4 * out, bx + 4 * c, sizeof(double) * 4);
        px[2 * out] = w; px[2 * out + 1] = h;
        target[2 * out] = tw < 1 ? 1 : (int64_t)tw;
        target[2 * out + 1] = th < 1 ? 1 : (int64_t)th;
        out++;
    }
    free(clip); free(cidx); free(bx); free(surv);
    return err ? ORC_INTERNAL : out;
}

/* ------------------------------------------------------------------------ */
/* packing (packing.py:109-362)                                               */
/* ------------------------------------------------------------------------ */
static int check_omega(int64_t omega) { return omega >= 1 && (omega & (omega - 1)) == 0; }

static int ilog2(int64_t omega) { int k = 0; while ((1LL << (k + 1)) <= omega) k++; return k; }

/* packing.py:348-350: -((-num*t)//den), max(min_dim) + 2*pad */
static int64_t scaled_dim(int64_t t, int64_t num, int64_t den, int64_t min_dim, int64_t pad)
{
    __int128 p = (__int128)num * t;
    __int128 q = p / den;
    if (q * den != p) q += 1; /* ceil for non-negative p */
    int64_t s = (int64_t)q;
    if (s < min_dim) s = min_dim;
    return s + 2 * pad;
}

static int64_t gcd64(int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a < 0 ? -a : a; }

/* packing.py:353-362: floor(num*grid/den) over grid, reduced */
static void snap_scale(__int128 num, __int128 den, int64_t *on, int64_t *od)
{
    __int128 grid = (__int128)1 << SCALE_GRID_BITS;
    __int128 f = (num * grid) / den;
    int64_t n = (int64_t)f, d = (int64_t)grid;
    if (n == 0) { *on = 0; *od = 1; return; }
    int64_t g = gcd64(n, d);
    *on = n / g; *od = d / g;
}

/* packing.py:133-158 */
int orc_fold(const int64_t *w, int64_t n, int64_t omega, int64_t *rows, int64_t *xs, int64_t *m_out)
{
    if (!check_omega(omega) || n <= 0) return ORC_VALUE_ERROR;
    for (int64_t i = 0; i < n; i++) if (w[i] < 1 || w[i] > omega) return ORC_VALUE_ERROR;
    int k = ilog2(omega);
    int64_t p = 0, m = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t r = p >> k, q = p & (omega - 1);
        rows[i] = r;
        xs[i] = (r % DIRECTION_PERIOD == 0) ? q : omega - q - w[i];
        int64_t over = q + w[i] - omega;
        if (i == 0 || over > m) m = over;
        p += w[i];
    }
    *m_out = m > 0 ? m : 0;
    return ORC_OK;
}

/* packing.py:170-215 (m == 0 precondition checked by caller) */
int orc_push_up(const int64_t *rows, const int64_t *xs, const int64_t *w, const int64_t *h, int64_t n,
                int64_t omega, int64_t *y, int64_t *used)
{
    int64_t *front = (int64_t *)calloc((size_t)omega + 1, sizeof(int64_t));
    if (!front) return ORC_INTERNAL;
    int64_t i = 0;
    while (i < n) {
        int64_t j = i;
        while (j < n && rows[j] == rows[i]) j++;
        /* read phase: every box against the pre-row frontline */
        for (int64_t b = i; b < j; b++) {
            int64_t rest = front[xs[b]];
            for (int64_t c = xs[b] + 1; c < xs[b] + w[b]; c++) if (front[c] > rest) rest = front[c];
            y[b] = rest;
        }
        for (int64_t b = i; b < j; b++)
            for (int64_t c = xs[b]; c < xs[b] + w[b]; c++) front[c] = y[b] + h[b];
        i = j;
    }
    int64_t mx = front[0];
    for (int64_t c = 1; c <= omega; c++) if (front[c] > mx) mx = front[c];
    *used = mx;
    free(front);
    return ORC_OK;
}

/* packing.py:245-292.  ow/oh: ordered oriented target dims.  On accept
 * returns 1 and fills x, y, w, h (per ordered box) and the reduced scale. */
int orc_pack_arrays(const int64_t *ow, const int64_t *oh, int64_t n, int64_t num, int64_t den,
                    int64_t omega, int64_t min_dim, int64_t pad,
                    int64_t *x, int64_t *y, int64_t *wd, int64_t *ht, int64_t *snum, int64_t *sden)
{
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * n);
    int have_fold = 0;
    int64_t m = 0;
    for (int it = 0; it < MAX_OVERFLOW_ITERATIONS + 1; it++) {
        int64_t wmax = 0;
        for (int64_t i = 0; i < n; i++) {
            wd[i] = scaled_dim(ow[i], num, den, min_dim, pad);
            ht[i] = scaled_dim(oh[i], num, den, min_dim, pad);
            if (i == 0 || wd[i] > wmax) wmax = wd[i];
        }
        if (wmax > omega) {
            m = wmax - omega;
            have_fold = 0;
        } else {
            orc_fold(wd, n, omega, rows, x, &m);
            have_fold = 1;
        }
        if (m == 0) break;
        have_fold = 0;
        snap_scale((__int128)num * omega, (__int128)den * (omega + m), &num, &den);
    }
    int ok = 0;
    if (have_fold && m == 0) {
        uint64_t area = 0; /* np.sum of int64 wraps */
        for (int64_t i = 0; i < n; i++) area += (uint64_t)wd[i] * (uint64_t)ht[i];
        if (!((int64_t)area > omega * omega)) {
            int64_t used;
            orc_push_up(rows, x, wd, ht, n, omega, y, &used);
            if (used <= omega) {
                ok = 1;
                int64_t g = gcd64(num, den);
                if (g == 0) g = 1;
                *snum = num / g; *sden = den / g;
            }
        }
    }
    free(rows);
    return ok;
}

/* packing.py:109-130: orient + stable order by (-h, min_tri).  perm[i] =
 * index into the input of the i-th ordered box. */
static int i64_cmp(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static const int64_t *g_key_h, *g_key_mt;
static int order_cmp(const void *a, const void *b)
{
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    if (g_key_h[i] != g_key_h[j]) return g_key_h[i] > g_key_h[j] ? -1 : 1;
    if (g_key_mt[i] != g_key_mt[j]) return g_key_mt[i] < g_key_mt[j] ? -1 : 1;
    return (i > j) - (i < j);
}

int orc_orient_order(const int64_t *tw, const int64_t *th, const int64_t *min_tri, int64_t n,
                     int64_t max_h, int64_t *perm, int64_t *ow, int64_t *oh, uint8_t *rot)
{
    int64_t *w = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *h = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; i++) {
        int r = tw[i] > th[i];
        w[i] = r ? th[i] : tw[i];
        h[i] = r ? tw[i] : th[i];
        if (h[i] > max_h) { free(w); free(h); return ORC_HEIGHT_OVERFLOW; }
        perm[i] = i;
    }
    g_key_h = h; g_key_mt = min_tri;
    qsort(perm, (size_t)n, sizeof(int64_t), order_cmp);
    for (int64_t i = 0; i < n; i++) {
        int64_t s = perm[i];
        ow[i] = w[s]; oh[i] = h[s]; rot[i] = tw[s] > th[s];
    }
    free(w); free(h);
    return ORC_OK;
}

/* packing.py:295-345.  Inputs in caller order; placements out in packing
 * order as 8 int64 each: chart_id x y w h rotated target_w target_h.
 * accept_mask (n_scales bytes, optional) receives the accept vector. */
int orc_pack(const int64_t *tw, const int64_t *th, const int64_t *chart_id, const int64_t *min_tri,
             int64_t n, int64_t omega, int64_t n_scales, int64_t min_dim, int64_t pad,
             int64_t *placements, int64_t *snum, int64_t *sden, uint8_t *accept_mask)
{
    if (!check_omega(omega)) return ORC_VALUE_ERROR;
    if (!(1 <= n_scales && n_scales <= (1 << 20))) return ORC_VALUE_ERROR;
    if (n == 0) { *snum = 1; *sden = 1; return ORC_OK; }
    {   /* packing.py:319-323 duplicate min_tri -> ValueError */
        int64_t *s = (int64_t *)malloc(sizeof(int64_t) * n);
        memcpy(s, min_tri, sizeof(int64_t) * n);
        qsort(s, (size_t)n, sizeof(int64_t), i64_cmp);
        for (int64_t i = 1; i < n; i++)
            if (s[i] == s[i - 1]) { free(s); return ORC_VALUE_ERROR; }
        free(s);
    }
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *ow = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *oh = (int64_t *)malloc(sizeof(int64_t) * n);
    uint8_t *rot = (uint8_t *)malloc((size_t)n);
    int st = orc_orient_order(tw, th, min_tri, n, MAX_BOX_DIM, perm, ow, oh, rot);
    if (st) { free(perm); free(ow); free(oh); free(rot); return st; }
    int64_t fmax = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t f = scaled_dim(ow[i], 1, n_scales, min_dim, pad);
        if (i == 0 || f > fmax) fmax = f;
    }
    int status = ORC_PACK_FAILURE;
    if (fmax <= omega) {
        int64_t *x = (int64_t *)malloc(sizeof(int64_t) * n), *y = (int64_t *)malloc(sizeof(int64_t) * n);
        int64_t *wd = (int64_t *)malloc(sizeof(int64_t) * n), *ht = (int64_t *)malloc(sizeof(int64_t) * n);
        int found = 0;
        for (int64_t i = n_scales; i >= 1; i--) {
            int64_t g = gcd64(i, n_scales);
            int64_t a, b;
            int ok = orc_pack_arrays(ow, oh, n, i / g, n_scales / g, omega, min_dim, pad,
                                     x, y, wd, ht, &a, &b);
            if (accept_mask) accept_mask[i - 1] = (uint8_t)ok;
            if (ok && !found) {
                found = 1;
                *snum = a; *sden = b;
                for (int64_t k = 0; k < n; k++) {
                    int64_t s = perm[k];
                    int64_t *P = placements + 8 * k;
                    P[0] = chart_id[s]; P[1] = x[k]; P[2] = y[k]; P[3] = wd[k]; P[4] = ht[k];
                    P[5] = rot[k]; P[6] = tw[s]; P[7] = th[s];
                }
                if (!accept_mask) break;
            }
        }
        if (found) status = ORC_OK;
        free(x); free(y); free(wd); free(ht);
    }
    free(perm); free(ow); free(oh); free(rot);
    return status;
}

/* ------------------------------------------------------------------------ */
/* UV emission (cli.py:409-450).  For every visible triangle t (ascending)   */
/* whose chart has a placement: uv[6*k..] = atlas (x,y) of its 3 corners;    */
/* NaN when any corner has w <= W_EPSILON (cli.py:433-435).                  */
/* placement_of_root: per chart (ascending-root index) 8 ints, ndc per chart */
/* ------------------------------------------------------------------------ */
void orc_uv(const double *pos, int64_t V, const int64_t *tris, const double *vp,
            const int64_t *vis_list, int64_t nvis, const int64_t *chart_of_vis,
            const double *ndc, const int64_t *px, const int64_t *plc, int W, int H, int64_t pad,
            double *uv)
{
    for (int64_t k = 0; k < nvis; k++) {
        int64_t t = vis_list[k];
        int64_t c = chart_of_vis[k];
        double *o = uv + 6 * k;
        if (c < 0) { for (int i = 0; i < 6; i++) o[i] = NAN; continue; }
        double v[3][4];
        int behind = 0;
        for (int i = 0; i < 3; i++) {
            project_one(pos + 3 * tris[3 * t + i], vp, v[i]);
            if (v[i][3] <= W_EPSILON) behind = 1;
        }
        if (behind) { for (int i = 0; i < 6; i++) o[i] = NAN; continue; }
        const int64_t *P = plc + 8 * c;
        int64_t cw = P[3] - 2 * pad, ch = P[4] - 2 * pad;
        double w_px = (double)px[2 * c], h_px = (double)px[2 * c + 1];
        double bx = (double)(P[1] + pad), by = (double)(P[2] + pad);
        for (int i = 0; i < 3; i++) {
            double nx = v[i][0] / v[i][3], ny = v[i][1] / v[i][3];
            double u = (nx - ndc[4 * c + 0]) * 0.5 * (double)W;
            double vv = (ny - ndc[4 * c + 1]) * 0.5 * (double)H;
            if (P[5]) {
                o[2 * i] = bx + vv * ((double)cw / h_px);
                o[2 * i + 1] = by + u * ((double)ch / w_px);
            } else {
                o[2 * i] = bx + u * ((double)cw / w_px);
                o[2 * i + 1] = by + vv * ((double)ch / h_px);
            }
        }
    }
}
