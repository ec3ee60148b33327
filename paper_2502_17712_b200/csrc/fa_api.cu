// fa_api.cu — C ABI (include/fastatlas.h): contexts, per-stage entry
// points and the whole-frame pipeline (run_scene_pipeline, cli.py:360-406).
//
// The frame is a fixed sequence of kernels whose work sizes are read from a
// device status block (fa_dstat), so the whole frame needs no host round
// trip and is captured once per shape into a CUDA graph; per frame only the
// 128-byte camera matrix is uploaded before the graph launch.
#include <math.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#define FA_TU_ID 1  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"
#include <cuda_profiler_api.h>
#include "fa_raster.cuh"

static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) return set_err(FA_CUDA_ERROR, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

#define CKL()                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = cudaGetLastError();                                                     \
        if (e_ != cudaSuccess) return set_err(FA_CUDA_ERROR, "launch: %s", cudaGetErrorString(e_)); \
    } while (0)

size_t fa_trisetup_bytes() { return sizeof(TriSetup); }

bool fa_ensure(fa_ctx* ctx, fa_buf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return true;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t alloc = bytes + bytes / 4 + 256;
    if (cudaMalloc(&b.p, alloc) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    b.bytes = alloc;
    ctx->gen++;
    return true;
}

// value of a fixed-point digit accumulator (fx_add), rounded to double
static double fx_value(const unsigned long long (&acc)[FA_FX_DIGITS]) {
    double v = 0.0;
    for (int k = FA_FX_DIGITS - 1; k >= 0; k--) v += ldexp((double)acc[k], 32 * k - 80);
    return v;
}

#define ENSURE(buf, n)                                                                     \
    do {                                                                                   \
        if (!fa_ensure(ctx, ctx->buf, (size_t)(n)))                                        \
            return set_err(FA_CUDA_ERROR, "out of device memory allocating " #buf " (%zu B)", (size_t)(n)); \
    } while (0)

template <typename T>
static T* P(const fa_buf& b) {
    return reinterpret_cast<T*>(b.p);
}

static void free_buf(fa_buf& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

extern "C" {

int fa_abi_version(void) { return FA_ABI_VERSION; }
const char* fa_last_error(void) { return g_err.c_str(); }

int fa_create(fa_ctx** out, int device) {
    if (!out) return set_err(FA_VALUE_ERROR, "null output pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return set_err(FA_CUDA_ERROR, "no CUDA device: %s", cudaGetErrorString(e));
    if (device < 0 || device >= n) return set_err(FA_VALUE_ERROR, "bad device %d", device);
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return set_err(FA_CUDA_ERROR, "device %s is sm_%d%d; this library is built for sm_100a", prop.name,
                       prop.major, prop.minor);
    fa_ctx* c = new fa_ctx();
    c->device = device;
    c->max_large = 1 << 16;
    c->max_tiles = 1 << 18;
    // test knob: tiny initial work queues, so frames take the overflow ->
    // grow -> rerun path (tests/test_gpu_parity.py::test_queue_overflow_reruns)
    c->queue_init = fa_env_int("FASTATLAS_QUEUE_INIT", 0);
    if (c->queue_init > 0) c->max_large = c->max_tiles = c->queue_init;
    c->pack_batch = 148;
    if (cudaMallocHost(&c->hstat, sizeof(fa_dstat)) != cudaSuccess ||
        cudaMallocHost(&c->hvp, fa_ctx::kVpSlots * FA_VP_DOUBLES * sizeof(double)) != cudaSuccess) {
        delete c;
        return set_err(FA_CUDA_ERROR, "cudaMallocHost failed");
    }
    memset(c->hstat, 0, sizeof(fa_dstat));
    *out = c;
    return FA_OK;
}

void fa_destroy(fa_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    fa_buf* bufs[] = {&c->small_rec, &c->clip, &c->depth_keys, &c->depth_f64, &c->flags, &c->vis_list, &c->large,
                      &c->tiles, &c->label, &c->vmin, &c->v2c, &c->cidx, &c->roots, &c->ndc_keys, &c->ndc, &c->px,
                      &c->target, &c->survived, &c->okey, &c->oidx, &c->ow, &c->oh, &c->orot, &c->sortk, &c->sortv,
                      &c->pinv, &c->cand, &c->cand_p, &c->cand_w, &c->cand_h, &c->cand_y, &c->rowstart,
                      &c->placements, &c->uv, &c->vp_dev, &c->blocks, &c->dstat, &c->aux, &c->in_tw, &c->in_th,
                      &c->in_cid, &c->in_mt, &c->scr, &c->clip_list, &c->hiz, &c->wid, &c->vis_chart, &c->vis_cidx, &c->plc_c, &c->pos_perm, &c->tris_perm, &c->vperm_buf, &c->vis_tris, &c->vslot, &c->vlist, &c->vuv, &c->vblocks, &c->pstat, &c->tperm_buf, &c->tris_sorted_buf, &c->clusters_buf, &c->live_buf, &c->mesh_first, &c->mesh_scratch, &c->mesh_sort, &c->mesh_tris_s, &c->ord_tw, &c->ord_th, &c->ord_cid, &c->ndc2, &c->vis_mask, &c->vvis_mask, &c->cidx16, &c->slots4_buf};
    for (fa_buf* b : bufs) free_buf(*b);
    for (cudaEvent_t e : c->fj)
        if (e) cudaEventDestroy(e);
    if (c->copy_done) cudaEventDestroy(c->copy_done);
    for (cudaEvent_t e : c->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->vp_ev)
        if (e) cudaEventDestroy(e);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->side2) cudaStreamDestroy(c->side2);
    if (c->hstat) cudaFreeHost(c->hstat);
    if (c->hvp) cudaFreeHost(c->hvp);
    delete c;
}

int fa_set_mesh(fa_ctx* ctx, const double* positions, int64_t n_vertices, const int32_t* triangles,
                int64_t n_triangles) {
    if (!ctx) return set_err(FA_VALUE_ERROR, "null context");
    if (n_vertices < 0 || n_triangles < 0 || n_vertices >= (1ll << 31) - 1 || n_triangles >= (1ll << 31) / 4)
        return set_err(FA_VALUE_ERROR, "mesh too large for 32-bit indices");
    if ((n_vertices > 0 && !positions) || (n_triangles > 0 && !triangles))
        return set_err(FA_VALUE_ERROR, "null mesh buffer");
    // The context is rebound only once the new mesh is known to be valid: a
    // failed call leaves no mesh bound (T = V = 0), never an invalid one.
    ctx->pos = ctx->pos_user = nullptr;
    ctx->tris = nullptr;
    ctx->vperm = nullptr;
    ctx->tperm = nullptr;
    ctx->tris_sorted = nullptr;
    ctx->clusters = nullptr;
    ctx->V = ctx->T = 0;
    ctx->gen++;  // any captured frame graph refers to the previous mesh
    if (n_triangles > 0) {
        // On the device (fa_mesh.cu): the index range check (Mesh.__post_init__,
        // charts.py:45-48); the raster setup's triangle order (Morton order of
        // the centroids, FASTATLAS_TRI_ORDER=0: the given order); the vertices
        // renumbered in order of first use along that order
        // (FASTATLAS_VERTEX_ORDER=0: kept); the per-cluster culling data.
        CK(cudaSetDevice(ctx->device));
        const bool renumber = fa_env_int("FASTATLAS_VERTEX_ORDER", 1) != 0;
        const bool order = fa_env_int("FASTATLAS_TRI_ORDER", 1) != 0;
        const long long T = n_triangles;
        const int V = (int)n_vertices;
        // scratch kept by the context (grow-only): a rebind allocates nothing
        fa_buf& first = ctx->mesh_first;
        fa_buf& scratch = ctx->mesh_scratch;
        fa_buf& sort_scratch = ctx->mesh_sort;
        fa_buf& tris_s = ctx->mesh_tris_s;
        const size_t vb = (size_t)(n_vertices > 0 ? n_vertices : 1) * 4;
        bool ok = fa_ensure(ctx, first, vb) &&
                  fa_ensure(ctx, scratch, (size_t)fa_mesh_scratch_ints(n_vertices, T) * 4 + vb + 16) &&
                  fa_ensure(ctx, ctx->clusters_buf, (size_t)((T + FA_CLUSTER - 1) / FA_CLUSTER) * sizeof(fa_cluster)) &&
                  fa_ensure(ctx, ctx->tris_sorted_buf, (size_t)T * 12) && fa_ensure(ctx, ctx->tperm_buf, (size_t)T * 4) &&
                  fa_ensure(ctx, ctx->slots4_buf, (size_t)T * 16);
        if (ok && order) ok = fa_ensure(ctx, sort_scratch, fa_mesh_sort_scratch_bytes(T)) && fa_ensure(ctx, tris_s, (size_t)T * 12);
        if (ok && renumber) {
            ok = fa_ensure(ctx, ctx->tris_perm, (size_t)T * 12) && fa_ensure(ctx, ctx->vperm_buf, vb) &&
                 fa_ensure(ctx, ctx->pos_perm, (size_t)n_vertices * 24 + 8);
        }
        if (!ok) return set_err(FA_CUDA_ERROR, "out of device memory binding the mesh");
        cudaStream_t s = nullptr;
        int* bad = P<int>(scratch);
        int* newidx = P<int>(scratch) + 1 + fa_mesh_scratch_ints(n_vertices, T);
        fa_launch_mesh_validate(triangles, T, V, P<int>(first), bad, s);
        int hbad = 0;
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && !hbad) {
            // setup order: sorted slot -> triangle (user vertex ids)
            const int* tri_src = triangles;  // triangles in setup order
            if (order) {
                fa_launch_mesh_order(positions, triangles, (int)T, V, sort_scratch.p, P<int>(ctx->tperm_buf),
                                     P<int>(tris_s), s);
                tri_src = P<int>(tris_s);
            }
            const double* pos_k = positions;
            if (renumber) {
                // first use along the setup order, then both triangle arrays remapped
                fa_launch_mesh_validate(tri_src, T, V, P<int>(first), bad, s);
                fa_launch_mesh_renumber(positions, tri_src, T, V, P<int>(first), bad + 1, newidx,
                                        P<int>(ctx->tris_sorted_buf), P<int>(ctx->vperm_buf), P<double>(ctx->pos_perm),
                                        s);
                fa_launch_mesh_remap(triangles, T, newidx, P<int>(ctx->tris_perm), s);
                pos_k = P<double>(ctx->pos_perm);
            } else {
                cudaMemcpyAsync(ctx->tris_sorted_buf.p, tri_src, (size_t)T * 12, cudaMemcpyDeviceToDevice, s);
            }
            fa_launch_cluster_build(pos_k, P<int>(ctx->tris_sorted_buf), (int)T, P<fa_cluster>(ctx->clusters_buf), s);
            fa_launch_make_slots4(P<int>(ctx->tris_sorted_buf), order ? P<int>(ctx->tperm_buf) : nullptr, (int)T,
                                  P<int4>(ctx->slots4_buf), s);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        }
        if (e != cudaSuccess) return set_err(FA_CUDA_ERROR, "fa_set_mesh: %s", cudaGetErrorString(e));
        if (hbad) return set_err(FA_VALUE_ERROR, "triangle index out of range");
        if (renumber) {
            ctx->pos = P<double>(ctx->pos_perm);
            ctx->tris = P<int>(ctx->tris_perm);
            ctx->vperm = P<int>(ctx->vperm_buf);
        }
        ctx->tperm = order ? P<int>(ctx->tperm_buf) : nullptr;
        ctx->tris_sorted = P<int>(ctx->tris_sorted_buf);
        ctx->clusters = P<fa_cluster>(ctx->clusters_buf);
    }
    if (!ctx->tris) {
        ctx->pos = positions;
        ctx->tris = triangles;
    }
    ctx->pos_user = positions;
    ctx->V = n_vertices;
    ctx->T = n_triangles;
    return FA_OK;
}

}  // extern "C"

// integer tuning knob from the environment (read once per name)
int fa_env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

float fa_grid_cap_scale() {
    static float f = -1.f;
    if (f < 0.f) {
        const char* e = getenv("FASTATLAS_GRID_CAP");
        f = e ? (float)atof(e) : 1.f;
        if (!(f > 0.f)) f = 1.f;
    }
    return f;
}

bool fa_pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("FASTATLAS_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on != 0;
}

// ---------------------------------------------------------------------------
// internal helpers
// ---------------------------------------------------------------------------
static int ensure_raster(fa_ctx* ctx, int W, int H, bool depth) {
    int64_t T = ctx->T, V = ctx->V;
    ENSURE(clip, (V > 0 ? V : 1) * sizeof(double4));
    ENSURE(scr, (V > 0 ? V : 1) * sizeof(double4));
    ENSURE(ndc2, (V > 0 ? V : 1) * sizeof(double2));
    if (depth) ENSURE(depth_keys, (size_t)W * H * 8);
    if (depth && T < (1 << 24)) ENSURE(wid, (size_t)W * H * 8);
    ENSURE(hiz, (size_t)fa_hiz_dim(W) * fa_hiz_dim(H) * 8);
    ENSURE(flags, ((T + 15) / 16 + 1) * 16);
    ENSURE(clip_list, (T + 1) * 4);
    ENSURE(small_rec, (T + 1) * sizeof(SmallRec) + (T + 1) * 4);  // records + their triangle ids
    // tile descriptors: 16 B each; a queue overflow costs a rerun of the
    // frame, so start at one descriptor per 8 pixels (C2 views use up to ~1/30)
    long long want_tiles = ctx->queue_init > 0 ? 0 : (long long)W * H / 8;
    if (want_tiles > ctx->max_tiles) ctx->max_tiles = (int)(want_tiles < (1ll << 30) ? want_tiles : (1 << 30));
    ENSURE(large, (size_t)ctx->max_large * sizeof(TriSetup));
    ENSURE(tiles, (size_t)ctx->max_tiles * sizeof(int4));
    ENSURE(dstat, sizeof(fa_dstat));
    ENSURE(vp_dev, FA_VP_DOUBLES * sizeof(double));
    ENSURE(live_buf, (size_t)((T + FA_CLUSTER - 1) / FA_CLUSTER + 1) * 4);
    return FA_OK;
}

static int ensure_charts(fa_ctx* ctx) {
    int64_t T = ctx->T, V = ctx->V;
    ENSURE(vis_list, (T + 1) * 4);
    ENSURE(vis_tris, (T + 1) * 16);
    ENSURE(label, (T + 1) * 4);
    ENSURE(vmin, (V + 1) * 4);
    ENSURE(v2c, (V + 1) * 4);
    ENSURE(cidx, (T + 1) * 4);
    ENSURE(aux, (T + 1) * 4);
    ENSURE(roots, (T + 1) * 4);
    ENSURE(ndc_keys, (T + 1) * 32);
    ENSURE(survived, (T + 1) * 4);
    ENSURE(ndc, (T + 1) * 32);
    ENSURE(px, (T + 1) * 8);
    ENSURE(target, (T + 1) * 16);
    ENSURE(blocks, (size_t)fa_compact_blocks(T + 1) * 4 + 64);
    return FA_OK;
}

// pack scratch for n_cap boxes, batch candidates, n_scales records
static int ensure_pack(fa_ctx* ctx, int64_t n_cap, int64_t n_scales, int64_t omega, int batch) {
    int64_t n = n_cap > 0 ? n_cap : 1;
    if (n < ctx->pack_cap) n = ctx->pack_cap;  // never shrink the capacity
    ctx->pack_cap = n;
    ENSURE(in_tw, n * 8);
    ENSURE(in_th, n * 8);
    ENSURE(in_cid, n * 8);
    ENSURE(ow, n * 8);
    ENSURE(oh, n * 8);
    ENSURE(orot, n + 16);
    ENSURE(oidx, n * 4);  // perm
    ENSURE(pinv, n * 4);
    ENSURE(sortk, 2 * n * 8);
    ENSURE(sortv, 2 * n * 4);
    ENSURE(cand, (size_t)n_scales * FA_CAND_REC * 8);
    ENSURE(cand_p, (size_t)batch * n * 8);
    ENSURE(cand_w, (size_t)batch * n * 4);
    ENSURE(cand_h, (size_t)batch * n * 4);
    ENSURE(cand_y, (size_t)batch * n * 4);
    ENSURE(rowstart, (size_t)batch * n * 4);
    ENSURE(placements, n * 64);
    ENSURE(ord_tw, n * 8);
    ENSURE(ord_th, n * 8);
    ENSURE(ord_cid, n * 8);
    ENSURE(plc_c, n * 32);
    if (!fa_front_in_smem(omega)) ENSURE(okey, (size_t)batch * (omega + 1) * 4);
    return FA_OK;
}

static fa_pack_bufs pack_bufs(fa_ctx* ctx, const long long* tw, const long long* th, const long long* cid,
                              long long* placements, unsigned char* accept_out) {
    fa_pack_bufs b;
    b.tw = tw;
    b.th = th;
    b.chart_id = cid;
    b.ow = P<long long>(ctx->ow);
    b.oh = P<long long>(ctx->oh);
    b.rot = P<unsigned char>(ctx->orot);
    b.perm = P<int>(ctx->oidx);
    b.pinv = P<int>(ctx->pinv);
    b.sortk = P<unsigned long long>(ctx->sortk);
    b.sortv = P<int>(ctx->sortv);
    b.cand = P<long long>(ctx->cand);
    b.cand_p = P<long long>(ctx->cand_p);
    b.cand_w = P<int>(ctx->cand_w);
    b.cand_h = P<int>(ctx->cand_h);
    b.cand_y = P<int>(ctx->cand_y);
    b.rowstart = P<int>(ctx->rowstart);
    b.placements = placements;
    b.plc_by_src = nullptr;
    b.accept_out = accept_out;
    b.gfront = P<int>(ctx->okey);
    return b;
}

static int check_omega(int64_t omega) {
    if (omega < 1 || (omega & (omega - 1)) != 0) return set_err(FA_VALUE_ERROR, "omega must be a power of two >= 1");
    if (omega > (1ll << 30)) return set_err(FA_VALUE_ERROR, "omega above 2^30 is not supported");
    return FA_OK;
}

static int status_from_flags(const fa_dstat* h) {
    if (h->flags & FA_DFLAG_POLY_OVERFLOW) return set_err(FA_INTERNAL_ERROR, "clipped polygon exceeded capacity");
    if (h->flags & FA_DFLAG_QUEUE_OVERFLOW) return set_err(FA_INTERNAL_ERROR, "work queue overflow");
    if (h->flags & FA_DFLAG_KEY_RANGE) return set_err(FA_VALUE_ERROR, "box key range exceeds 64 bits");
    if (h->flags & FA_DFLAG_DUPLICATE_MIN_TRI) return set_err(FA_VALUE_ERROR, "duplicate min_tri in pack request");
    if (h->flags & FA_DFLAG_HEIGHT_OVERFLOW) return set_err(FA_HEIGHT_OVERFLOW, "box height exceeds capacity");
    return FA_OK;
}

static void grow_queues(fa_ctx* ctx, const fa_dstat* h) {
    if (h->n_large > ctx->max_large) ctx->max_large = h->n_large + h->n_large / 2;
    long long nt = (long long)h->n_tiles + h->n_tiles_clip;
    if (nt > ctx->max_tiles) ctx->max_tiles = (int)(nt + nt / 2 < (1ll << 30) ? nt + nt / 2 : (1 << 30));
}

static int read_stat(fa_ctx* ctx, cudaStream_t s) {
    CK(cudaMemcpyAsync(ctx->hstat, ctx->dstat.p, sizeof(fa_dstat), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return FA_OK;
}

static_assert(FA_VC_OFF * 8 + sizeof(fa_view_consts) <= FA_VP_DOUBLES * 8, "camera slot too small");
static int upload_vp(fa_ctx* ctx, const double* vp_host, cudaStream_t s, int W = 0, int H = 0) {
    // The 16 doubles are copied into a context-owned pinned slot before the
    // call returns, so the caller may reuse or refill its matrix at once (a
    // pinned caller buffer would otherwise be read asynchronously).  A slot
    // is reused only after the copy that read it has executed.
    const int k = ctx->vp_next;
    ctx->vp_next = (k + 1) % fa_ctx::kVpSlots;
    if (!ctx->vp_ev[k]) CK(cudaEventCreateWithFlags(&ctx->vp_ev[k], cudaEventDisableTiming));
    else CK(cudaEventSynchronize(ctx->vp_ev[k]));
    double* slot = ctx->hvp + FA_VP_DOUBLES * k;
    memcpy(slot, vp_host, 16 * sizeof(double));
    // the cluster culling's view constants, computed here once per frame
    // (the culling's margins dwarf any host/device rounding difference)
    compute_view_consts(slot, W, H, reinterpret_cast<fa_view_consts*>(slot + FA_VC_OFF));
    CK(cudaMemcpyAsync(ctx->vp_dev.p, slot, FA_VP_DOUBLES * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(ctx->vp_ev[k], s));
    return FA_OK;
}

// the setup order + cluster culling of the bound mesh (vc: the view
// constants k_frame_init writes each frame)
static fa_setup_order setup_order(fa_ctx* ctx) {
    fa_setup_order o{};
    o.tperm = ctx->tperm;
    o.tris_sorted = ctx->tris_sorted;
    o.slots4 = ctx->tris_sorted && ctx->slots4_buf.p ? P<int4>(ctx->slots4_buf) : nullptr;
    if (ctx->clusters && ctx->live_buf.p && fa_env_int("FASTATLAS_CLUSTER_CULL", 1)) {
        o.live = P<int>(ctx->live_buf);
        o.n_live = &P<fa_dstat>(ctx->dstat)->n_live;
    }
    return o;
}

// k_frame_init's cluster culling for setup_order's live list
static fa_cull_args cull_args(fa_ctx* ctx, int cull) {
    fa_cull_args c{};
    if (ctx->clusters && ctx->live_buf.p && fa_env_int("FASTATLAS_CLUSTER_CULL", 1)) {
        c.clusters = ctx->clusters;
        c.n_clusters = (int)((ctx->T + FA_CLUSTER - 1) / FA_CLUSTER);
        c.cull = cull;
        c.live = P<int>(ctx->live_buf);
        c.st = P<fa_dstat>(ctx->dstat);
    }
    return c;
}

// clip-space vertices: the array k_frame_init wrote (the standalone entry
// points), or recomputed from the positions where needed (the frame, whose
// k_frame_init skips the (V,4) array)
static ClipSrc clip_stored(fa_ctx* ctx) { return ClipSrc{P<double4>(ctx->clip), nullptr, nullptr}; }
static ClipSrc clip_recomputed(fa_ctx* ctx) { return ClipSrc{nullptr, ctx->pos, P<double>(ctx->vp_dev)}; }

// depth pass (shared by fa_depth_prepass and the frame)
static int launch_depth(fa_ctx* ctx, int W, int H, int cull, unsigned char* flags_out, cudaStream_t s, int& nl) {
    int T = (int)ctx->T, V = (int)ctx->V;
    const fa_setup_order ord = setup_order(ctx);
    fa_launch_cluster_cull(P<double>(ctx->vp_dev), W, H, cull_args(ctx, cull), s);
    fa_launch_frame_init(ctx->pos, V, P<double>(ctx->vp_dev), P<double4>(ctx->clip), P<double4>(ctx->scr), W, H,
                         P<int>(ctx->vmin), P<unsigned long long>(ctx->depth_keys), nullptr, (long long)W * H,
                         flags_out, T, s);
    if (ord.live) nl += 1;
    nl += 1 + fa_launch_depth_pass(true, clip_stored(ctx), P<double4>(ctx->scr), ctx->tris, T, W, H, cull,
                                   P<unsigned long long>(ctx->depth_keys), nullptr, P<SmallRec>(ctx->small_rec),
                                   P<int>(ctx->clip_list), P<TriSetup>(ctx->large), ctx->max_large,
                                   P<int4>(ctx->tiles), ctx->max_tiles, P<fa_dstat>(ctx->dstat), s, nullptr, nullptr,
                                   nullptr, nullptr, nullptr, nullptr, ord);
    return FA_OK;
}

// side stream and fork/join events (created on first use)
static int ensure_side(fa_ctx* ctx) {
    if (!ctx->side) CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    if (!ctx->side2) CK(cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking));
    for (cudaEvent_t& e : ctx->fj)
        if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!ctx->copy_done) CK(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
    return FA_OK;
}

// ---------------------------------------------------------------------------
// comparison packers (shared by their entry points and the frame's packer
// dispatch).  Boxes are device arrays, n >= 1; `stat` is the status block the
// packer may clobber (the frame passes its own scratch, not the frame status).
// ---------------------------------------------------------------------------
static int seq_search_core(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h, const int64_t* chart_id,
                           const int64_t* min_tri, int64_t n, int64_t omega, int64_t n_scales, int64_t min_dim,
                           int64_t padding, int64_t* placements_out, int64_t* scale_host, fa_buf& stat,
                           cudaStream_t s) {
    int batch = (int)(n_scales < ctx->pack_batch ? n_scales : ctx->pack_batch);
    int r = ensure_pack(ctx, n, n_scales, omega, batch);
    if (r) return r;
    ENSURE(aux, 64);
    CK(cudaMemsetAsync(stat.p, 0, sizeof(fa_dstat), s));
    CK(cudaMemsetAsync(ctx->cand.p, 0, (size_t)n_scales * FA_CAND_REC * 8, s));
    fa_dstat* st = P<fa_dstat>(stat);
    int nn = (int)n;
    fa_launch_orient_sort_mt((const long long*)target_w, (const long long*)target_h, (const long long*)min_tri, nn,
                             FA_MAX_BOX_DIM, P<long long>(ctx->ow), P<long long>(ctx->oh), P<unsigned char>(ctx->orot),
                             P<int>(ctx->oidx), P<int>(ctx->pinv), P<unsigned long long>(ctx->sortk),
                             P<int>(ctx->sortv), 0, st, s);
    fa_launch_seq_search(P<long long>(ctx->ow), P<long long>(ctx->oh), nn, omega, n_scales, min_dim, padding, batch,
                         P<int>(ctx->cand_w), P<int>(ctx->cand_h), P<int>(ctx->cand_p), P<int>(ctx->cand_y),
                         P<int>(ctx->rowstart), fa_front_in_smem(omega) ? nullptr : P<int>(ctx->okey),
                         P<long long>(ctx->cand), &st->done, s);
    fa_launch_seq_select((const long long*)target_w, (const long long*)target_h, (const long long*)chart_id,
                         P<unsigned char>(ctx->orot), P<int>(ctx->oidx), nn, n_scales, P<long long>(ctx->cand),
                         P<int>(ctx->cand_w), P<int>(ctx->cand_h), P<int>(ctx->cand_p), P<int>(ctx->cand_y),
                         (long long*)placements_out, P<long long>(ctx->aux), s);
    CKL();
    fa_dstat hs;
    long long best = 0;
    CK(cudaMemcpyAsync(&hs, stat.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&best, ctx->aux.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    r = status_from_flags(&hs);
    if (r) return r;
    if (best == 0) return set_err(FA_PACK_FAILURE, "every candidate scale was rejected");
    if (scale_host) {
        long long g = best, b = n_scales;
        while (b) { long long t = g % b; g = b; b = t; }
        scale_host[0] = best / g;
        scale_host[1] = n_scales / g;
    }
    return FA_OK;
}

static int check_superblock(int64_t omega, int64_t block_size) {
    int r = check_omega(omega);
    if (r) return r;
    if (block_size < 1 || (block_size & (block_size - 1)))
        return set_err(FA_VALUE_ERROR, "block_size must be a power of two");
    if (block_size > omega) return set_err(FA_VALUE_ERROR, "block_size must not exceed omega");
    if (omega % block_size) return set_err(FA_VALUE_ERROR, "omega must be divisible by block_size");
    return FA_OK;
}

static int superblock_core(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h, const int64_t* chart_id,
                           const int64_t* min_tri, int64_t n, int64_t omega, int64_t block_size, int halving_enabled,
                           int64_t* placements_out, int64_t* scale_host, int64_t* block_used_host, fa_buf& stat,
                           cudaStream_t s) {
    int n_levels = 1;
    if (halving_enabled)
        while ((block_size >> n_levels) >= 16) n_levels++;
    int r = ensure_pack(ctx, n, 1, omega, 1);
    if (r) return r;
    CK(cudaMemsetAsync(stat.p, 0, sizeof(fa_dstat), s));
    fa_dstat* st = P<fa_dstat>(stat);
    int nn = (int)n;
    fa_launch_orient_sort_mt((const long long*)target_w, (const long long*)target_h, (const long long*)min_tri, nn,
                             FA_MAX_BOX_DIM, P<long long>(ctx->ow), P<long long>(ctx->oh), P<unsigned char>(ctx->orot),
                             P<int>(ctx->oidx), P<int>(ctx->pinv), P<unsigned long long>(ctx->sortk),
                             P<int>(ctx->sortv), 0, st, s);
    // per level: used_h[nb] + nsh[nb] + 3 * nb * block shelf arrays (largest at the smallest block)
    long long smallest = block_size >> (n_levels - 1);
    long long nb_max = (omega / smallest) * (omega / smallest);
    size_t state_stride = (size_t)(2 * nb_max + 3 * nb_max * smallest);
    size_t out_stride = (size_t)4 * nn;
    fa_buf state, xywh, lvl, out;
    bool ok = fa_ensure(ctx, state, state_stride * n_levels * 4) && fa_ensure(ctx, xywh, out_stride * n_levels * 4) &&
              fa_ensure(ctx, lvl, 64 * 4) && fa_ensure(ctx, out, 64);
    if (ok) {
        fa_launch_superblock(P<long long>(ctx->ow), P<long long>(ctx->oh), (const long long*)target_w,
                             (const long long*)target_h, (const long long*)chart_id, P<unsigned char>(ctx->orot),
                             P<int>(ctx->oidx), nn, omega, (int)block_size, n_levels, P<int>(state), state_stride,
                             P<int>(xywh), out_stride, P<int>(lvl), (long long*)placements_out, P<long long>(out), s);
        r = FA_OK;
        cudaError_t e = cudaGetLastError();
        long long res[3] = {-1, 1, 1};
        fa_dstat hs;
        if (e == cudaSuccess) e = cudaMemcpyAsync(res, out.p, sizeof(res), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&hs, stat.p, sizeof(hs), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            r = set_err(FA_CUDA_ERROR, "superblock: %s", cudaGetErrorString(e));
        } else if ((r = status_from_flags(&hs)) != FA_OK) {
        } else if (res[0] < 0) {
            r = set_err(FA_PACK_FAILURE, "superblock allocation failed at the halving floor");
        } else {
            long long g = res[1], b = res[2];
            while (b) { long long t = g % b; g = b; b = t; }
            if (scale_host) { scale_host[0] = res[1] / g; scale_host[1] = res[2] / g; }
            if (block_used_host) *block_used_host = block_size >> res[0];
        }
    } else {
        r = set_err(FA_CUDA_ERROR, "out of device memory for superblock state");
    }
    free_buf(state);
    free_buf(xywh);
    free_buf(lvl);
    free_buf(out);
    return r;
}

extern "C" {

int fa_project(fa_ctx* ctx, const double* vp_host, double* clip_out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !vp_host || (!clip_out && ctx->V)) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    ENSURE(vp_dev, FA_VP_DOUBLES * sizeof(double));
    int r = upload_vp(ctx, vp_host, s);
    if (r) return r;
    fa_launch_frame_init(ctx->pos_user, (int)ctx->V, P<double>(ctx->vp_dev), (double4*)clip_out, nullptr, 0, 0, nullptr,
                         nullptr, nullptr, 0, nullptr, 0, s);
    CKL();
    return FA_OK;
}

int fa_depth_prepass(fa_ctx* ctx, const double* vp_host, int width, int height, int backface_cull, double* depth_out,
                     void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !vp_host) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (width < 1 || height < 1) return set_err(FA_VALUE_ERROR, "resolution must be at least 1x1");
    CK(cudaSetDevice(ctx->device));
    for (int attempt = 0; attempt < 4; attempt++) {
        int r = ensure_raster(ctx, width, height, true);
        if (!r) r = ensure_charts(ctx);
        if (r) return r;
        CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
        r = upload_vp(ctx, vp_host, s, width, height);
        if (r) return r;
        int nl = 0;
        launch_depth(ctx, width, height, backface_cull, nullptr, s, nl);
        fa_launch_decode_depth(P<unsigned long long>(ctx->depth_keys), depth_out, (long long)width * height, s);
        CKL();
        r = read_stat(ctx, s);
        if (r) return r;
        if (ctx->hstat->flags & FA_DFLAG_QUEUE_OVERFLOW) {
            grow_queues(ctx, ctx->hstat);
            continue;
        }
        return status_from_flags(ctx->hstat);
    }
    return set_err(FA_INTERNAL_ERROR, "raster queue kept overflowing");
}

int fa_mark_visible(fa_ctx* ctx, const double* vp_host, const double* depth, int width, int height,
                    int backface_cull, uint8_t* flags_out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !vp_host || !depth) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (width < 1 || height < 1) return set_err(FA_VALUE_ERROR, "resolution must be at least 1x1");
    CK(cudaSetDevice(ctx->device));
    int T = (int)ctx->T, V = (int)ctx->V;
    for (int attempt = 0; attempt < 4; attempt++) {
        int r = ensure_raster(ctx, width, height, true);
        if (!r) r = ensure_charts(ctx);
        if (r) return r;
        CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
        r = upload_vp(ctx, vp_host, s, width, height);
        if (r) return r;
        const fa_setup_order ord = setup_order(ctx);
        fa_launch_cluster_cull(P<double>(ctx->vp_dev), width, height, cull_args(ctx, backface_cull), s);
        fa_launch_frame_init(ctx->pos, V, P<double>(ctx->vp_dev), P<double4>(ctx->clip), P<double4>(ctx->scr), width,
                             height, nullptr, nullptr, nullptr, 0, P<unsigned char>(ctx->flags), T, s);
        fa_launch_encode_depth(depth, P<unsigned long long>(ctx->depth_keys), (long long)width * height, s);
        fa_launch_depth_pass(false, clip_stored(ctx), P<double4>(ctx->scr), ctx->tris, T, width, height,
                             backface_cull, nullptr, nullptr, P<SmallRec>(ctx->small_rec), P<int>(ctx->clip_list),
                             P<TriSetup>(ctx->large), ctx->max_large, P<int4>(ctx->tiles), ctx->max_tiles,
                             P<fa_dstat>(ctx->dstat), s, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ord);
        fa_launch_depth_hiz(P<unsigned long long>(ctx->depth_keys), nullptr, width, height,
                            P<unsigned long long>(ctx->hiz), nullptr, nullptr, s);
        fa_launch_raster_vis(P<SmallRec>(ctx->small_rec), P<TriSetup>(ctx->large), P<int4>(ctx->tiles),
                             ctx->max_tiles, ctx->max_large, T, width, P<unsigned long long>(ctx->depth_keys),
                             P<unsigned long long>(ctx->hiz), P<unsigned char>(ctx->flags), P<int>(ctx->clip_list),
                             P<fa_dstat>(ctx->dstat), s, nullptr, nullptr, nullptr);
        CKL();
        r = read_stat(ctx, s);
        if (r) return r;
        if (ctx->hstat->flags & FA_DFLAG_QUEUE_OVERFLOW) {
            grow_queues(ctx, ctx->hstat);
            continue;
        }
        if (T) CK(cudaMemcpyAsync(flags_out, ctx->flags.p, T, cudaMemcpyDeviceToDevice, s));
        return status_from_flags(ctx->hstat);
    }
    return set_err(FA_INTERNAL_ERROR, "raster queue kept overflowing");
}

int fa_build_adjacency(fa_ctx* ctx, int32_t* adjacency_out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || (ctx->T && !adjacency_out)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (ctx->T == 0) return FA_OK;
    CK(cudaSetDevice(ctx->device));
    unsigned long long n = 3ull * (unsigned long long)ctx->T, size = 1;
    while (size < 2 * n) size <<= 1;  // load factor <= 1/2
    fa_buf keys, cnt, c0, c1;
    bool ok = fa_ensure(ctx, keys, size * 8) && fa_ensure(ctx, cnt, size * 4) && fa_ensure(ctx, c0, size * 4) &&
              fa_ensure(ctx, c1, size * 4);
    int r = FA_OK;
    if (!ok) {
        r = set_err(FA_CUDA_ERROR, "out of device memory for the edge table");
    } else {
        fa_launch_build_adjacency(ctx->tris, (int)ctx->T, P<unsigned long long>(keys), P<int>(cnt), P<int>(c0),
                                  P<int>(c1), size, adjacency_out, s);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) r = set_err(FA_CUDA_ERROR, "build_adjacency: %s", cudaGetErrorString(e));
    }
    free_buf(keys);
    free_buf(cnt);
    free_buf(c0);
    free_buf(c1);
    return r;
}

int fa_connected_charts(fa_ctx* ctx, const int32_t* adjacency, const uint8_t* flags, int32_t* labels_out,
                        void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || (ctx->T && (!adjacency || !flags || !labels_out))) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    int T = (int)ctx->T;
    int r = ensure_charts(ctx);
    if (r) return r;
    ENSURE(dstat, sizeof(fa_dstat));
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    fa_dstat* st = P<fa_dstat>(ctx->dstat);
    // flags may not be 16-byte padded: stage a padded copy
    ENSURE(flags, ((T + 15) / 16 + 1) * 16);
    if (T) CK(cudaMemcpyAsync(ctx->flags.p, flags, T, cudaMemcpyDeviceToDevice, s));
    fa_launch_compact_visible(P<unsigned char>(ctx->flags), T, P<int>(ctx->blocks), P<int>(ctx->vis_list), labels_out,
                              st, s);
    fa_launch_uf_edges(adjacency, P<unsigned char>(ctx->flags), P<int>(ctx->vis_list), labels_out, T, st, s);
    fa_launch_uf_compress(P<int>(ctx->vis_list), labels_out, T, st, s);
    CKL();
    return FA_OK;
}

int fa_merge_shared_vertices(fa_ctx* ctx, const int32_t* labels_in, int32_t* labels_out, int32_t* v2c_out,
                             void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || (ctx->T && (!labels_in || !labels_out))) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    int T = (int)ctx->T, V = (int)ctx->V;
    int r = ensure_charts(ctx);
    if (r) return r;
    ENSURE(dstat, sizeof(fa_dstat));
    ENSURE(flags, ((T + 15) / 16 + 1) * 16);
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    fa_dstat* st = P<fa_dstat>(ctx->dstat);
    unsigned char* fl = P<unsigned char>(ctx->flags);
    fa_launch_flags_from_labels(labels_in, fl, T, s);
    fa_launch_compact_visible(fl, T, P<int>(ctx->blocks), P<int>(ctx->vis_list), labels_out, st, s);
    // general chart sets: every node starts as its own root (charts.py:371)
    fa_launch_iota(labels_out, T, s);
    fa_launch_fill(P<int>(ctx->vmin), V, 0x7fffffff, s);
    fa_launch_uf_vertex(ctx->tris, P<int>(ctx->vis_list), P<int>(ctx->vmin), labels_out, T, st, s);
    fa_launch_uf_labels(labels_in, P<int>(ctx->vis_list), labels_out, T, st, s);
    fa_launch_uf_compress(P<int>(ctx->vis_list), labels_out, T, st, s);
    fa_launch_canonicalize(P<int>(ctx->vis_list), labels_out, P<int>(ctx->aux), T, st, s);
    fa_launch_canon_apply(fl, labels_out, P<int>(ctx->aux), T, s);
    if (v2c_out) fa_launch_v2c(P<int>(ctx->vmin), labels_out, v2c_out, V, s, ctx->vperm);
    CKL();
    return FA_OK;
}

int fa_chart_boxes(fa_ctx* ctx, const double* vp_host, const int32_t* labels, int width, int height, double prescale,
                   int32_t* roots_out, double* ndc_out, int32_t* px_out, int64_t* target_out, int64_t* n_charts_host,
                   void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !vp_host || (ctx->T && !labels)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (width < 1 || height < 1) return set_err(FA_VALUE_ERROR, "screen dimensions must be >= 1");
    CK(cudaSetDevice(ctx->device));
    int T = (int)ctx->T, V = (int)ctx->V;
    int r = ensure_charts(ctx);
    if (!r) r = ensure_raster(ctx, 1, 1, false);
    if (!r) r = ensure_pack(ctx, T, 1, 1, 1);
    if (r) return r;
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    r = upload_vp(ctx, vp_host, s);
    if (r) return r;
    fa_dstat* st = P<fa_dstat>(ctx->dstat);
    unsigned char* fl = P<unsigned char>(ctx->flags);
    fa_launch_frame_init(ctx->pos, V, P<double>(ctx->vp_dev), P<double4>(ctx->clip), nullptr, 0, 0, nullptr, nullptr,
                         nullptr, 0, nullptr, 0, s);
    fa_launch_flags_from_labels(labels, fl, T, s);
    fa_launch_compact_visible(fl, T, P<int>(ctx->blocks), P<int>(ctx->vis_list), P<int>(ctx->aux), st, s);
    fa_launch_compact_roots(P<int>(ctx->vis_list), labels, T, P<int>(ctx->blocks), P<int>(ctx->roots),
                            P<int>(ctx->cidx), P<unsigned long long>(ctx->ndc_keys), P<int>(ctx->survived), st, s);
    fa_launch_chart_bounds(clip_stored(ctx), ctx->tris, P<int>(ctx->vis_list), labels, P<int>(ctx->cidx), T,
                           P<unsigned long long>(ctx->ndc_keys), P<int>(ctx->survived), st, s);
    fa_launch_box_dims(P<unsigned long long>(ctx->ndc_keys), P<int>(ctx->survived), P<int>(ctx->roots), T, width,
                       height, prescale, P<double>(ctx->ndc), P<int>(ctx->px), P<long long>(ctx->target),
                       P<long long>(ctx->in_tw), P<long long>(ctx->in_th), P<long long>(ctx->in_cid),
                       (int)ctx->pack_cap, st, s);
    CKL();
    r = read_stat(ctx, s);
    if (r) return r;
    int C = ctx->hstat->n_charts;
    if (ctx->hstat->flags & FA_DFLAG_DEGENERATE_CHART)
        return set_err(FA_DEGENERATE_CHART, "a chart has no triangle surviving clipping");
    if (C) {
        CK(cudaMemcpyAsync(roots_out, ctx->roots.p, (size_t)C * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ndc_out, ctx->ndc.p, (size_t)C * 32, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(px_out, ctx->px.p, (size_t)C * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(target_out, ctx->target.p, (size_t)C * 16, cudaMemcpyDeviceToDevice, s));
    }
    if (n_charts_host) *n_charts_host = C;
    CK(cudaStreamSynchronize(s));
    return FA_OK;
}

int fa_orient_order(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h, const int64_t* min_tri, int64_t n,
                    int64_t max_h, int32_t* perm_out, int64_t* ow_out, int64_t* oh_out, uint8_t* rot_out,
                    void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || n < 0 || n >= (1ll << 30)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (n == 0) return FA_OK;
    CK(cudaSetDevice(ctx->device));
    int r = ensure_pack(ctx, n, 1, 1, 1);
    if (r) return r;
    ENSURE(dstat, sizeof(fa_dstat));
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    fa_launch_orient_sort_mt((const long long*)target_w, (const long long*)target_h, (const long long*)min_tri, (int)n,
                             max_h, (long long*)ow_out, (long long*)oh_out, rot_out, perm_out, P<int>(ctx->pinv),
                             P<unsigned long long>(ctx->sortk), P<int>(ctx->sortv), 0, P<fa_dstat>(ctx->dstat), s);
    CKL();
    r = read_stat(ctx, s);
    if (r) return r;
    return status_from_flags(ctx->hstat);
}

int fa_fold(fa_ctx* ctx, const int64_t* widths, int64_t n, int64_t omega, int64_t* rows_out, int64_t* x_out,
            int64_t* m_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || n <= 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "fold requires a non-empty width sequence");
    int r = check_omega(omega);
    if (r) return r;
    CK(cudaSetDevice(ctx->device));
    ENSURE(aux, 64);
    fa_launch_fold((const long long*)widths, (int)n, omega, (long long*)rows_out, (long long*)x_out,
                   P<long long>(ctx->aux), s);
    CKL();
    long long m = 0;
    CK(cudaMemcpyAsync(&m, ctx->aux.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (m < 0) return set_err(FA_VALUE_ERROR, "widths must be in [1, omega]");
    if (m_host) *m_host = m;
    return FA_OK;
}

int fa_push_up(fa_ctx* ctx, const int64_t* rows, const int64_t* x, const int64_t* widths, const int64_t* heights,
               int64_t n, int64_t omega, int64_t* y_out, int64_t* used_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || n < 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "bad arguments");
    int r = check_omega(omega);
    if (r) return r;
    CK(cudaSetDevice(ctx->device));
    if (n == 0) {
        if (used_host) *used_host = 0;
        return FA_OK;
    }
    ENSURE(rowstart, (size_t)n * 4 + 64);
    ENSURE(aux, 64);
    int* gfront = nullptr;
    if (!fa_front_in_smem(omega)) {
        ENSURE(okey, (size_t)(omega + 1) * 4);
        gfront = P<int>(ctx->okey);
    }
    fa_launch_push_up_impl((const long long*)rows, (const long long*)x, (const long long*)widths,
                           (const long long*)heights, (int)n, omega, P<int>(ctx->rowstart), (long long*)y_out,
                           P<long long>(ctx->aux), gfront, s);
    CKL();
    long long used = 0;
    CK(cudaMemcpyAsync(&used, ctx->aux.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (used_host) *used_host = used;
    return FA_OK;
}

int fa_pack_at_scale(fa_ctx* ctx, const int64_t* ow, const int64_t* oh, int64_t n, int64_t num, int64_t den,
                     int64_t omega, int64_t min_dim, int64_t padding, int64_t* xywh_out, int64_t* scale_host,
                     int* accepted_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int r = check_omega(omega);
    if (r) return r;
    if (!ctx || n < 0 || n >= (1ll << 30)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (!(num > 0 && den > 0 && num <= den)) return set_err(FA_VALUE_ERROR, "scale must be in (0, 1]");
    if (min_dim < 1 || padding < 0 || min_dim > (1 << 28) || padding > (1 << 28))
        return set_err(FA_VALUE_ERROR, "min_dim must be >= 1 and padding >= 0");
    CK(cudaSetDevice(ctx->device));
    if (n == 0) {
        long long g = num, b = den;
        while (b) { long long t = g % b; g = b; b = t; }
        if (scale_host) { scale_host[0] = num / g; scale_host[1] = den / g; }
        if (accepted_host) *accepted_host = 1;
        return FA_OK;
    }
    r = ensure_pack(ctx, n, 1, omega, 1);
    if (r) return r;
    CK(cudaMemsetAsync(ctx->cand.p, 0, FA_CAND_REC * 8, s));
    fa_launch_pack_at_scale((const long long*)ow, (const long long*)oh, (int)n, num, den, omega, min_dim, padding,
                            P<long long>(ctx->cand), P<long long>(ctx->cand_p), P<int>(ctx->cand_w),
                            P<int>(ctx->cand_h), P<int>(ctx->cand_y), P<int>(ctx->rowstart), P<int>(ctx->okey), s);
    fa_launch_xywh(P<long long>(ctx->cand), P<long long>(ctx->cand_p), P<int>(ctx->cand_w), P<int>(ctx->cand_h),
                   P<int>(ctx->cand_y), (int)n, omega, (long long*)xywh_out, s);
    CKL();
    long long rec[FA_CAND_REC];
    CK(cudaMemcpyAsync(rec, ctx->cand.p, sizeof(rec), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (accepted_host) *accepted_host = (int)rec[0];
    if (scale_host && rec[0]) {
        scale_host[0] = rec[1];
        scale_host[1] = rec[2];
    }
    return FA_OK;
}

int fa_pack(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h, const int64_t* chart_id,
            const int64_t* min_tri, int64_t n, int64_t omega, int64_t n_scales, int64_t min_dim, int64_t padding,
            int64_t* placements_out, int64_t* scale_host, uint8_t* accept_out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int r = check_omega(omega);
    if (r) return r;
    if (!ctx) return set_err(FA_VALUE_ERROR, "null context");
    if (!(1 <= n_scales && n_scales <= (1 << 20))) return set_err(FA_VALUE_ERROR, "n_scales must be in [1, 2^20]");
    if (min_dim < 1 || padding < 0 || min_dim > (1 << 28) || padding > (1 << 28))
        return set_err(FA_VALUE_ERROR, "min_dim must be >= 1 and padding >= 0");
    if (n < 0 || n >= (1ll << 30)) return set_err(FA_VALUE_ERROR, "bad box count");
    if (n == 0) {
        if (scale_host) { scale_host[0] = 1; scale_host[1] = 1; }
        return FA_OK;
    }
    CK(cudaSetDevice(ctx->device));
    int batch = (int)(n_scales < ctx->pack_batch ? n_scales : ctx->pack_batch);
    r = ensure_pack(ctx, n, n_scales, omega, batch);
    if (r) return r;
    ENSURE(dstat, sizeof(fa_dstat));
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    CK(cudaMemsetAsync(ctx->cand.p, 0, (size_t)n_scales * FA_CAND_REC * 8, s));
    fa_dstat* st = P<fa_dstat>(ctx->dstat);
    fa_launch_orient_sort_mt((const long long*)target_w, (const long long*)target_h, (const long long*)min_tri, (int)n,
                             FA_MAX_BOX_DIM, P<long long>(ctx->ow), P<long long>(ctx->oh), P<unsigned char>(ctx->orot),
                             P<int>(ctx->oidx), P<int>(ctx->pinv), P<unsigned long long>(ctx->sortk),
                             P<int>(ctx->sortv), 1, st, s);
    fa_pack_bufs b = pack_bufs(ctx, (const long long*)target_w, (const long long*)target_h,
                               (const long long*)chart_id, (long long*)placements_out, accept_out);
    fa_launch_pack(b, (int)n, nullptr, omega, n_scales, min_dim, padding, batch, st, s);
    CKL();
    r = read_stat(ctx, s);
    if (r) return r;
    r = status_from_flags(ctx->hstat);
    if (r) return r;
    if (ctx->hstat->flags & FA_DFLAG_PACK_FAILURE) return set_err(FA_PACK_FAILURE, "every candidate scale was rejected");
    if (scale_host) {
        scale_host[0] = ctx->hstat->scale_num;
        scale_host[1] = ctx->hstat->scale_den;
    }
    return FA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// whole frame
// ---------------------------------------------------------------------------
// The comparison packers of make_packer (cli.py:318-339) inside the frame.
// Runs outside graph capture: the frame so far (boxes in in_tw / in_th /
// in_cid, ascending roots) is synchronised once, the packer runs on the box
// count it reads, and the frame status receives the layout's scale and
// texel count.  k_uv then reads the placements in packing order through
// pinv (written by the packer's own orient + order, packing.py:109-130).
static int frame_external_pack(fa_ctx* ctx, const fa_frame_params* p, cudaStream_t s, int& nl) {
    int r = read_stat(ctx, s);
    if (r) return r;
    fa_dstat* h = ctx->hstat;
    int64_t n = h->n_charts;
    // any earlier failure (or a box count beyond the scratch, which
    // fa_frame_finish grows and reruns) is reported by fa_frame_finish; the
    // pack-failure flag keeps k_uv from reading placements
    if (h->flags || h->n_vis == 0 || n > ctx->pack_cap) {
        h->flags |= FA_DFLAG_PACK_FAILURE;
        CK(cudaMemcpyAsync(ctx->dstat.p, h, sizeof(fa_dstat), cudaMemcpyHostToDevice, s));
        return FA_OK;
    }
    ENSURE(pstat, sizeof(fa_dstat));
    const int64_t* tw = P<int64_t>(ctx->in_tw);
    const int64_t* th = P<int64_t>(ctx->in_th);
    const int64_t* cid = P<int64_t>(ctx->in_cid);
    int64_t* plc = P<int64_t>(ctx->placements);
    int64_t scale[2] = {1, 1};
    if (p->packer == FA_PACKER_SEQUENTIAL) {
        if (n > 0) {
            if (p->n_scales < 1) r = set_err(FA_PACK_FAILURE, "every candidate scale was rejected");
            else r = seq_search_core(ctx, tw, th, cid, cid, n, p->omega, p->n_scales, p->min_dim, p->padding, plc,
                                     scale, ctx->pstat, s);
            nl += 3;
        }
    } else if (p->packer == FA_PACKER_SUPERBLOCK) {
        // SuperblockConfig(block_size or default_block_size(omega)), halving on (cli.py:331-333)
        int64_t bs = p->block_size;
        if (bs == 0) bs = std::max<int64_t>(16, std::min<int64_t>(p->omega, p->omega / 8));
        r = check_superblock(p->omega, bs);
        if (!r && n > 0) {
            r = superblock_core(ctx, tw, th, cid, cid, n, p->omega, bs, 1, plc, scale, nullptr, ctx->pstat, s);
            nl += 3;
        }
    } else {
        return set_err(FA_VALUE_ERROR, "unknown packer '%d' (choose from fastatlas, sequential, superblock)",
                       p->packer);
    }
    if (r == FA_PACK_FAILURE) {
        h->flags |= FA_DFLAG_PACK_FAILURE;
    } else if (r) {
        return r;
    } else {
        // texels_allocated (cli.py:391-393) over the placements
        std::vector<long long> hp((size_t)n * 8);
        if (n) CK(cudaMemcpy(hp.data(), plc, (size_t)n * 64, cudaMemcpyDeviceToHost));
        long long tex = 0;
        for (int64_t j = 0; j < n; j++) {
            long long cw = hp[8 * j + 3] - 2 * p->padding, ch = hp[8 * j + 4] - 2 * p->padding;
            tex += (cw > 0 ? cw : 0) * (ch > 0 ? ch : 0);
        }
        h->scale_num = scale[0];
        h->scale_den = scale[1];
        h->texels_allocated = tex;
        h->best = 1;
    }
    CK(cudaMemcpyAsync(ctx->dstat.p, h, sizeof(fa_dstat), cudaMemcpyHostToDevice, s));
    return FA_OK;
}

static int frame_sequence(fa_ctx* ctx, const fa_frame_params* p, cudaStream_t s, int& nl) {
    int T = (int)ctx->T, V = (int)ctx->V, W = p->width, H = p->height;
    fa_dstat* st = P<fa_dstat>(ctx->dstat);
    int64_t n_cap = ctx->pack_cap;
    int batch = (int)(p->n_scales < ctx->pack_batch ? p->n_scales : ctx->pack_batch);
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    CK(cudaMemsetAsync(ctx->cand.p, 0, (size_t)p->n_scales * FA_CAND_REC * 8, s));
    nl = 0;
    bool prof = p->profile && !p->use_graph;
    ctx->n_stage_marks = 0;
    // debug knob for ncu range replay (tools/frame_traffic.py):
    // FASTATLAS_PROFILE_STAGE=k brackets stage k (between marks k and k + 1
    // below) of the FASTATLAS_PROFILE_FRAME-th non-graph frame (default 4)
    // with cudaProfilerStart/Stop
    static const int prof_stage = fa_env_int("FASTATLAS_PROFILE_STAGE", -1);
    static const int prof_frame = fa_env_int("FASTATLAS_PROFILE_FRAME", 4);
    static int frame_no = 0;
    const bool prof_this = prof_stage >= 0 && !p->use_graph && frame_no++ == prof_frame;
    int n_marks = 0;
    auto mark = [&]() -> int {
        if (prof_this) {
            if (n_marks == prof_stage) cudaProfilerStart();
            if (n_marks == prof_stage + 1) cudaProfilerStop();
        }
        n_marks++;
        if (!prof) return FA_OK;
        if (!ctx->ev[ctx->n_stage_marks]) CK(cudaEventCreate(&ctx->ev[ctx->n_stage_marks]));
        CK(cudaEventRecord(ctx->ev[ctx->n_stage_marks], s));
        ctx->n_stage_marks++;
        return FA_OK;
    };
    unsigned char* flags = P<unsigned char>(ctx->flags);
    // pixel-winner buffer: triangle ids must fit the low FA_WID_BITS (24) bits
    unsigned long long* wid = T < (1 << 24) ? P<unsigned long long>(ctx->wid) : nullptr;
    mark();  // 0: start
    // The depth/winner clears (33 MB at C2, HBM-bound) run on the side
    // stream beside the projection and the setup, which never touch them.
    int r = ensure_side(ctx);
    if (r) return r;
    CK(cudaEventRecord(ctx->fj[9], s));
    CK(cudaStreamWaitEvent(ctx->side, ctx->fj[9], 0));
    fa_launch_frame_init(nullptr, 0, nullptr, nullptr, nullptr, W, H, nullptr, P<unsigned long long>(ctx->depth_keys), wid,
                         (long long)W * H, nullptr, T, ctx->side,
                         fa_env_int("FASTATLAS_CLEAR_BLOCKS", FA_NUM_SMS));  // a slice of the GPU: the setup keeps the rest
    CK(cudaEventRecord(ctx->fj[10], ctx->side));
    const fa_setup_order ord = setup_order(ctx);
    // the cluster culling runs in the projection's launch (its first blocks):
    // beside it, with no launch or join of its own
    const fa_cull_args cua = cull_args(ctx, p->backface_cull);
    fa_launch_frame_init(ctx->pos, V, P<double>(ctx->vp_dev), nullptr, P<double4>(ctx->scr), W, H,
                         P<int>(ctx->vmin), nullptr, nullptr, 0, flags, T, s, 0, P<double2>(ctx->ndc2), &cua);
    nl += 2;
    mark();  // 1: project + clears
    nl += fa_launch_depth_pass(true, clip_recomputed(ctx), P<double4>(ctx->scr), ctx->tris, T, W, H,
                               p->backface_cull, P<unsigned long long>(ctx->depth_keys), wid,
                               P<SmallRec>(ctx->small_rec), P<int>(ctx->clip_list), P<TriSetup>(ctx->large),
                               ctx->max_large, P<int4>(ctx->tiles), ctx->max_tiles, st, s,
                               fa_env_int("FASTATLAS_DEPTH_BRANCHES", 3) >= 2 ? ctx->side : nullptr,
                               fa_env_int("FASTATLAS_DEPTH_BRANCHES", 3) >= 3 ? ctx->side2 : nullptr,
                               ctx->fj[0], ctx->fj[1], ctx->fj[7], ctx->fj[10], ord);
    fa_launch_depth_hiz(P<unsigned long long>(ctx->depth_keys), wid, W, H, P<unsigned long long>(ctx->hiz), flags, st,
                        s);
    nl += 1;
    mark();  // 2: depth pass
    nl += fa_launch_raster_vis(P<SmallRec>(ctx->small_rec), P<TriSetup>(ctx->large), P<int4>(ctx->tiles),
                               ctx->max_tiles, ctx->max_large, T, W, P<unsigned long long>(ctx->depth_keys),
                               P<unsigned long long>(ctx->hiz), flags, P<int>(ctx->clip_list), st, s, ctx->side,
                               ctx->fj[2], ctx->fj[3]);
    mark();  // 3: visibility pass
    // the previous frame's downloads must be done before this frame rewrites
    // the downloaded buffers (the compaction is the first writer; in a graph
    // an external event-wait node)
    {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(s, &cs));
        static const bool no_wait = fa_env_int("FASTATLAS_DEBUG_NO_COPY_WAIT", 0) != 0;  // (tests only)
        if (!no_wait)
            CK(cudaStreamWaitEvent(s, ctx->copy_done, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
    }
    // the compaction also lowers vmin (frame_init filled it with INT_MAX)
    fa_launch_compact_visible(flags, T, P<int>(ctx->blocks), P<int>(ctx->vis_list), P<int>(ctx->label), st, s,
                              ctx->tris, P<int>(ctx->vmin), P<int4>(ctx->vis_tris), P<unsigned int>(ctx->vis_mask));
    nl += 2;
    mark();  // 4: visible compaction
    // debug knob (results invalid): end the frame after the raster passes
    // and the visible compaction,
    // to measure what the rest of the frame costs the pipelined throughput
    static const int dbg_stop = fa_env_int("FASTATLAS_DEBUG_STOP_AFTER_RASTER", 0);
    if (dbg_stop) {
        CK(cudaMemcpyAsync(ctx->hstat, ctx->dstat.p, sizeof(fa_dstat), cudaMemcpyDeviceToHost, s));
        return FA_OK;
    }
    nl += fa_launch_uf_vertex(ctx->tris, P<int>(ctx->vis_list), P<int>(ctx->vmin), P<int>(ctx->label), T, st, s,
                              true, P<int4>(ctx->vis_tris));
    mark();  // 5: union-find charts (hooking)
    // Roots are the nodes with label[t] == t after hooking, which flattening
    // never changes (it only rewrites non-roots to their root, also != t), so
    // the roots compaction (s) and the flatten + vertex map (side) overlap.
    CK(cudaEventRecord(ctx->fj[4], s));
    CK(cudaStreamWaitEvent(ctx->side, ctx->fj[4], 0));
    fa_launch_uf_compress(P<int>(ctx->vis_list), P<int>(ctx->label), T, st, ctx->side);
    fa_launch_v2c(P<int>(ctx->vmin), P<int>(ctx->label), P<int>(ctx->v2c), V, ctx->side, ctx->vperm);
    fa_launch_visible_vertices(P<int>(ctx->vmin), V, ctx->vperm, P<int>(ctx->vblocks), P<int>(ctx->vslot),
                               P<int>(ctx->vlist), st, ctx->side, P<float2>(ctx->vuv), P<unsigned int>(ctx->vvis_mask));
    CK(cudaEventRecord(ctx->fj[6], ctx->side));
    nl += 4;
    fa_launch_compact_roots(P<int>(ctx->vis_list), P<int>(ctx->label), T, P<int>(ctx->blocks), P<int>(ctx->roots),
                            P<int>(ctx->cidx), P<unsigned long long>(ctx->ndc_keys), P<int>(ctx->survived), st, s);
    nl += 2;
    // (the bounds find each triangle's root themselves, beside the flattening)
    mark();  // 6: chart roots (+ flatten)
    fa_launch_chart_bounds(clip_recomputed(ctx), ctx->tris, P<int>(ctx->vis_list), P<int>(ctx->label),
                           P<int>(ctx->cidx), T, P<unsigned long long>(ctx->ndc_keys), P<int>(ctx->survived), st, s,
                           P<int>(ctx->vis_cidx), P<int4>(ctx->vis_tris), P<double2>(ctx->ndc2));
    nl += 1;
    mark();  // 7: chart bounds (the box dims run at the head of the order kernel)
    fa_pack_bufs b = pack_bufs(ctx, P<long long>(ctx->in_tw), P<long long>(ctx->in_th), P<long long>(ctx->in_cid),
                               P<long long>(ctx->placements), nullptr);
    b.plc_by_src = P<int4>(ctx->plc_c);
    b.ord_tw = P<long long>(ctx->ord_tw);
    b.ord_th = P<long long>(ctx->ord_th);
    b.ord_cid = P<long long>(ctx->ord_cid);
    b.ord_written = fa_env_int("FASTATLAS_ORDER_ONCHIP", 1) != 0;
    const fa_box_dims_args bd{P<unsigned long long>(ctx->ndc_keys), P<int>(ctx->survived), P<int>(ctx->roots), W, H,
                              p->prescale, P<double>(ctx->ndc), P<int>(ctx->px), P<long long>(ctx->target),
                              P<long long>(ctx->in_tw), P<long long>(ctx->in_th), P<long long>(ctx->in_cid),
                              (int)n_cap};
    fa_launch_orient_sort(b, (int)n_cap, &st->n_charts, FA_MAX_BOX_DIM, st, s, &bd);
    nl += 1;
    mark();  // 8: orient + radix order
    if (p->packer == FA_PACKER_FASTATLAS) {
        nl += fa_launch_pack(b, (int)n_cap, &st->n_charts, p->omega, p->n_scales, p->min_dim, p->padding, batch, st, s);
    } else {
        r = frame_external_pack(ctx, p, s, nl);
        if (r) return r;
    }
    mark();  // 9: candidate pack + select
    CK(cudaStreamWaitEvent(s, ctx->fj[6], 0));  // vertex -> chart map and the visible-vertex slots
    fa_launch_uv(clip_recomputed(ctx), ctx->tris, P<int>(ctx->vis_list), P<int>(ctx->label), P<int>(ctx->cidx),
                 P<int>(ctx->pinv), P<double>(ctx->ndc), P<int>(ctx->px), P<long long>(ctx->placements), T, W, H,
                 p->padding, p->uv_f64 != 0, ctx->uv.p, P<int>(ctx->vis_chart), P<int>(ctx->vis_cidx),
                 p->packer == FA_PACKER_FASTATLAS ? P<int4>(ctx->plc_c) : nullptr, st, s, P<int4>(ctx->vis_tris),
                 P<int>(ctx->vslot), P<float2>(ctx->vuv), P<double2>(ctx->ndc2), P<unsigned short>(ctx->cidx16));
    nl += 1;
    mark();  // 10: uv
    if (p->want_depth) {
        fa_launch_decode_depth(P<unsigned long long>(ctx->depth_keys), P<double>(ctx->depth_f64), (long long)W * H, s);
        nl += 1;
    }

    CK(cudaMemcpyAsync(ctx->hstat, ctx->dstat.p, sizeof(fa_dstat), cudaMemcpyDeviceToHost, s));
    CKL();
    return FA_OK;
}

static int frame_prepare(fa_ctx* ctx, const fa_frame_params* p) {
    if (p->width < 1 || p->height < 1) return set_err(FA_VALUE_ERROR, "screen must be at least 1x1");
    int r = check_omega(p->omega);
    if (r) return r;
    if (!(1 <= p->n_scales && p->n_scales <= (1 << 20))) return set_err(FA_VALUE_ERROR, "n_scales must be in [1, 2^20]");
    if (p->min_dim < 1 || p->padding < 0 || p->min_dim > (1 << 28) || p->padding > (1 << 28))
        return set_err(FA_VALUE_ERROR, "min_dim must be >= 1 and padding >= 0");
    if (!(p->prescale > 0)) return set_err(FA_VALUE_ERROR, "prescale must be positive");
    if (ctx->T > 0 && (!ctx->pos || !ctx->tris)) return set_err(FA_VALUE_ERROR, "no mesh bound");
    r = ensure_raster(ctx, p->width, p->height, true);
    if (!r) r = ensure_charts(ctx);
    if (r) return r;
    int64_t cap = ctx->pack_cap;
    if (cap < 16384) cap = 16384;
    if (cap > ctx->T + 1) cap = ctx->T + 1;
    int batch = (int)(p->n_scales < ctx->pack_batch ? p->n_scales : ctx->pack_batch);
    r = ensure_pack(ctx, cap, p->n_scales, p->omega, batch);
    if (r) return r;
    ENSURE(uv, (size_t)(ctx->T + 1) * 6 * (p->uv_f64 ? 8 : 4));
    ENSURE(vis_chart, (size_t)(ctx->T + 1) * 4);
    ENSURE(vis_cidx, (size_t)(ctx->T + 1) * 4);
    ENSURE(vis_mask, (size_t)(ctx->T / 32 + 1) * 4);
    ENSURE(vvis_mask, (size_t)(ctx->V / 32 + 1) * 4);
    ENSURE(cidx16, (size_t)(ctx->T + 1) * 2);
    ENSURE(vslot, (size_t)(ctx->V + 1) * 4);
    ENSURE(vlist, (size_t)(ctx->V + 1) * 4);
    ENSURE(vuv, (size_t)(ctx->V + 1) * 8);
    ENSURE(vblocks, (size_t)fa_vertex_blocks(ctx->V + 1) * 4 + 64);
    if (p->want_depth) ENSURE(depth_f64, (size_t)p->width * p->height * 8);
    return FA_OK;
}

extern "C" {

int fa_frame_launch(fa_ctx* ctx, const double* vp_host, const fa_frame_params* p, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !vp_host || !p) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    int r = frame_prepare(ctx, p);
    if (r) return r;
    ctx->last_params = *p;
    r = upload_vp(ctx, vp_host, s, p->width, p->height);
    if (r) return r;
    if (!p->use_graph || p->profile || p->packer != FA_PACKER_FASTATLAS) {
        fa_frame_params q = *p;
        q.use_graph = 0;
        p = &q;
        int nl = 0;
        r = frame_sequence(ctx, p, s, nl);
        ctx->last_launches = nl;
        return r;
    }
    fa_graph_key key;
    key.width = p->width;
    key.height = p->height;
    key.cull = p->backface_cull;
    key.uv_f64 = p->uv_f64;
    key.want_depth = p->want_depth;
    key.omega = p->omega;
    key.n_scales = p->n_scales;
    key.min_dim = p->min_dim;
    key.padding = p->padding;
    key.prescale = p->prescale;
    key.T = ctx->T;
    key.V = ctx->V;
    key.pos = ctx->pos;
    key.tris = ctx->tris;
    key.gen = ctx->gen;
    if (!ctx->graph_exec || !(key == ctx->graph_key)) {
        if (ctx->graph_exec) {
            cudaGraphExecDestroy(ctx->graph_exec);
            ctx->graph_exec = nullptr;
        }
        cudaStream_t cap;
        CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        int nl = 0;
        int rr = frame_sequence(ctx, p, cap, nl);
        cudaGraph_t g;
        cudaError_t e = cudaStreamEndCapture(cap, &g);
        cudaStreamDestroy(cap);
        if (rr) return rr;
        if (e != cudaSuccess) return set_err(FA_CUDA_ERROR, "graph capture: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&ctx->graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return set_err(FA_CUDA_ERROR, "graph instantiate: %s", cudaGetErrorString(e));
        ctx->graph_key = key;
        ctx->last_launches = nl;
        static const int dbg_cap = fa_env_int("FASTATLAS_DEBUG_CAPTURE", 0);
        if (dbg_cap) fprintf(stderr, "fastatlas: frame graph captured (ctx %p, gen %llu)\n", (void*)ctx,
                             (unsigned long long)ctx->gen);
    }
    CK(cudaGraphLaunch(ctx->graph_exec, s));
    return FA_OK;
}

int fa_frame_finish(fa_ctx* ctx, fa_frame_result* out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !out) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(s));
    const fa_dstat* h = ctx->hstat;
    memset(out, 0, sizeof(*out));
    out->n_visible = h->n_vis;
    out->n_charts = h->n_charts;
    out->scale_num = h->scale_num;
    out->scale_den = h->scale_den;
    out->screen_fragments = h->screen_fragments;
    out->texels_allocated = h->texels_allocated;
    out->stretch_count = h->stretch_valid;
    {
        double linf;
        memcpy(&linf, &h->stretch_linf_bits, sizeof(linf));
        out->stretch_linf = h->stretch_valid ? linf : 0.0;
        double wsum = h->stretch_wsum, area = h->stretch_area;
        if (!(h->flags & FA_DFLAG_STRETCH_RANGE)) {
            wsum = fx_value(h->stretch_fx[0]);
            area = fx_value(h->stretch_fx[1]);
        }
        out->stretch_l2 = (h->stretch_valid && area > 0) ? sqrt(wsum / area) : 0.0;
    }
    out->depth = ctx->last_params.want_depth ? P<double>(ctx->depth_f64) : nullptr;
    out->flags = P<uint8_t>(ctx->flags);
    out->visible = P<int32_t>(ctx->vis_list);
    out->chart_of_triangle = P<int32_t>(ctx->label);
    out->vertex_to_chart = P<int32_t>(ctx->v2c);
    out->roots = P<int32_t>(ctx->roots);
    out->ndc = P<double>(ctx->ndc);
    out->px = P<int32_t>(ctx->px);
    out->target = P<int64_t>(ctx->target);
    out->placements = P<int64_t>(ctx->placements);
    out->uv = ctx->uv.p;
    out->visible_chart = P<int32_t>(ctx->vis_chart);
    out->n_visible_vertices = h->n_vis_vertices;
    out->visible_vertices = P<int32_t>(ctx->vlist);
    out->vertex_uv = P<float>(ctx->vuv);
    int64_t n_cap = ctx->pack_cap;
    ctx->needs_rerun = false;
    if (h->flags & FA_DFLAG_QUEUE_OVERFLOW || h->n_charts > n_cap) {
        grow_queues(ctx, h);
        if (h->n_charts > n_cap) {
            int batch = (int)(ctx->last_params.n_scales < ctx->pack_batch ? ctx->last_params.n_scales : ctx->pack_batch);
            int r = ensure_pack(ctx, (int64_t)h->n_charts * 2, ctx->last_params.n_scales, ctx->last_params.omega, batch);
            if (r) return r;
        }
        out->status = FA_INTERNAL_ERROR;
        ctx->needs_rerun = true;
        return set_err(FA_INTERNAL_ERROR, "work queue overflow (capacity grown; rerun the frame)");
    }
    int r = status_from_flags(h);
    if (r) {
        out->status = r;
        return r;
    }
    if (h->n_vis == 0) {
        out->status = FA_NOTHING_VISIBLE;
        return set_err(FA_NOTHING_VISIBLE, "no triangle covers a depth-passing sample");
    }
    if (h->flags & FA_DFLAG_DEGENERATE_CHART) {
        out->status = FA_DEGENERATE_CHART;
        return set_err(FA_DEGENERATE_CHART, "a visible chart has no surviving triangle");
    }
    if (h->flags & FA_DFLAG_PACK_FAILURE) {
        out->status = FA_PACK_FAILURE;
        return set_err(FA_PACK_FAILURE, "every candidate scale was rejected");
    }
    out->status = FA_OK;
    return FA_OK;
}

int fa_frame(fa_ctx* ctx, const double* vp_host, const fa_frame_params* p, fa_frame_result* out, void* stream) {
    for (int attempt = 0; attempt < 4; attempt++) {
        int r = fa_frame_launch(ctx, vp_host, p, stream);
        if (r) return r;
        r = fa_frame_finish(ctx, out, stream);
        if (r == FA_INTERNAL_ERROR && ctx->needs_rerun) continue;
        return r;
    }
    return set_err(FA_INTERNAL_ERROR, "frame kept overflowing its work queues");
}

int fa_frame_download(fa_ctx* ctx, const fa_frame_result* res, int32_t* chart_of_triangle, int32_t* visible,
                      void* uv, int64_t* placements, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !res) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (res->status != FA_OK) return set_err(FA_VALUE_ERROR, "frame result has no outputs (status %d)", res->status);
    CK(cudaSetDevice(ctx->device));
    size_t nv = (size_t)res->n_visible, C = (size_t)res->n_charts;
    size_t uv_elem = ctx->last_params.uv_f64 ? 8 : 4;
    if (chart_of_triangle && ctx->T)
        CK(cudaMemcpyAsync(chart_of_triangle, res->chart_of_triangle, (size_t)ctx->T * 4, cudaMemcpyDefault, s));
    if (visible && nv) CK(cudaMemcpyAsync(visible, res->visible, nv * 4, cudaMemcpyDefault, s));
    if (uv && nv) CK(cudaMemcpyAsync(uv, res->uv, nv * 6 * uv_elem, cudaMemcpyDefault, s));
    if (placements && C) CK(cudaMemcpyAsync(placements, res->placements, C * 64, cudaMemcpyDefault, s));
    if (ctx->copy_done) CK(cudaEventRecord(ctx->copy_done, s));
    return FA_OK;
}

int fa_frame_download_compact(fa_ctx* ctx, const fa_frame_result* res, int32_t* visible, int32_t* visible_chart,
                              int32_t* visible_vertices, float* vertex_uv, int64_t* placements, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !res) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (res->status != FA_OK) return set_err(FA_VALUE_ERROR, "frame result has no outputs (status %d)", res->status);
    CK(cudaSetDevice(ctx->device));
    size_t nv = (size_t)res->n_visible, C = (size_t)res->n_charts, nvv = (size_t)res->n_visible_vertices;
    if (visible && nv) CK(cudaMemcpyAsync(visible, res->visible, nv * 4, cudaMemcpyDefault, s));
    if (visible_chart && nv) CK(cudaMemcpyAsync(visible_chart, res->visible_chart, nv * 4, cudaMemcpyDefault, s));
    if (visible_vertices && nvv)
        CK(cudaMemcpyAsync(visible_vertices, res->visible_vertices, nvv * 4, cudaMemcpyDefault, s));
    if (vertex_uv && nvv) CK(cudaMemcpyAsync(vertex_uv, res->vertex_uv, nvv * 8, cudaMemcpyDefault, s));
    if (placements && C) CK(cudaMemcpyAsync(placements, res->placements, C * 64, cudaMemcpyDefault, s));
    if (ctx->copy_done) CK(cudaEventRecord(ctx->copy_done, s));
    return FA_OK;
}

// debug knob (tests/test_pipeline.py): FASTATLAS_DEBUG_COPY_DELAY=us spins on
// the download stream before the copies, so a missing copy_done wait in the
// next frame would let it overwrite the buffers first
__global__ void k_debug_spin(long long ns) {
    long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

int fa_frame_download_packed(fa_ctx* ctx, const fa_frame_result* res, uint32_t* visible_mask,
                             uint16_t* visible_cidx, int32_t* roots, uint32_t* vertex_mask, float* vertex_uv,
                             int64_t* placements, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !res) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (res->status != FA_OK) return set_err(FA_VALUE_ERROR, "frame result has no outputs (status %d)", res->status);
    if (res->n_charts > 65535) return set_err(FA_VALUE_ERROR, "more than 65535 charts: use fa_frame_download_compact");
    if (!ctx->vis_mask.p || !ctx->cidx16.p) return set_err(FA_VALUE_ERROR, "no frame outputs");
    CK(cudaSetDevice(ctx->device));
    static const int dbg_delay = fa_env_int("FASTATLAS_DEBUG_COPY_DELAY", 0);
    if (dbg_delay > 0) k_debug_spin<<<1, 1, 0, s>>>((long long)dbg_delay * 1000);
    size_t nv = (size_t)res->n_visible, C = (size_t)res->n_charts, nvv = (size_t)res->n_visible_vertices;
    if (visible_mask && ctx->T)
        CK(cudaMemcpyAsync(visible_mask, ctx->vis_mask.p, (size_t)((ctx->T + 31) / 32) * 4, cudaMemcpyDefault, s));
    if (visible_cidx && nv) CK(cudaMemcpyAsync(visible_cidx, ctx->cidx16.p, nv * 2, cudaMemcpyDefault, s));
    if (roots && C) CK(cudaMemcpyAsync(roots, res->roots, C * 4, cudaMemcpyDefault, s));
    if (vertex_mask && ctx->V)
        CK(cudaMemcpyAsync(vertex_mask, ctx->vvis_mask.p, (size_t)((ctx->V + 31) / 32) * 4, cudaMemcpyDefault, s));
    if (vertex_uv && nvv) CK(cudaMemcpyAsync(vertex_uv, res->vertex_uv, nvv * 8, cudaMemcpyDefault, s));
    if (placements && C) CK(cudaMemcpyAsync(placements, res->placements, C * 64, cudaMemcpyDefault, s));
    if (ctx->copy_done) CK(cudaEventRecord(ctx->copy_done, s));
    return FA_OK;
}

int fa_vertex_order(fa_ctx* ctx, int32_t* out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !out) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    if (ctx->vperm) {
        CK(cudaMemcpyAsync(out, ctx->vperm, (size_t)ctx->V * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } else {
        for (int64_t v = 0; v < ctx->V; v++) out[v] = (int32_t)v;
    }
    return FA_OK;
}

int fa_frame_download_visible(fa_ctx* ctx, const fa_frame_result* res, int32_t* visible, int32_t* visible_chart,
                              void* uv, int64_t* placements, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !res) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (res->status != FA_OK) return set_err(FA_VALUE_ERROR, "frame result has no outputs (status %d)", res->status);
    CK(cudaSetDevice(ctx->device));
    size_t nv = (size_t)res->n_visible, C = (size_t)res->n_charts;
    size_t uv_elem = ctx->last_params.uv_f64 ? 8 : 4;
    if (visible && nv) CK(cudaMemcpyAsync(visible, res->visible, nv * 4, cudaMemcpyDefault, s));
    if (visible_chart && nv)
        CK(cudaMemcpyAsync(visible_chart, res->visible_chart, nv * 4, cudaMemcpyDefault, s));
    if (uv && nv) CK(cudaMemcpyAsync(uv, res->uv, nv * 6 * uv_elem, cudaMemcpyDefault, s));
    if (placements && C) CK(cudaMemcpyAsync(placements, res->placements, C * 64, cudaMemcpyDefault, s));
    if (ctx->copy_done) CK(cudaEventRecord(ctx->copy_done, s));
    return FA_OK;
}

int fa_last_launch_count(fa_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

int fa_frame_counters(fa_ctx* ctx, int64_t* out, int max) {
    if (!ctx || !out || !ctx->hstat) return 0;
    const fa_dstat* h = ctx->hstat;
    const int64_t v[9] = {h->n_small3, h->n_large3, h->n_clip, h->n_large, h->n_tiles, h->n_vis, h->n_charts,
                          h->screen_fragments, h->n_live};
    int n = max < 9 ? max : 9;
    for (int i = 0; i < n; i++) out[i] = v[i];
    return n;
}

static const char* kStageNames[] = {"project+clear", "depth pass",   "visibility pass", "visible compaction",
                                    "union-find",    "chart roots",  "bounds+dims",     "order",
                                    "pack+select",   "uv"};

const char* fa_stage_name(int i) {
    return (i >= 0 && i < (int)(sizeof(kStageNames) / sizeof(kStageNames[0]))) ? kStageNames[i] : "";
}

int fa_stage_times(fa_ctx* ctx, float* ms_out, int max, void* stream) {
    if (!ctx || !ms_out) return 0;
    cudaStreamSynchronize((cudaStream_t)stream);
    int n = ctx->n_stage_marks - 1;
    if (n < 0) n = 0;
    if (n > max) n = max;
    for (int i = 0; i < n; i++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]);
        ms_out[i] = ms;
    }
    return n;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// batched geometry helpers backing the scalar reference API
// ---------------------------------------------------------------------------
extern "C" {

int fa_blinn_clamped_ndc(fa_ctx* ctx, const double* points4, int64_t n, double* out2, void* stream) {
    if (!ctx || n < 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (n == 0) return FA_OK;
    CK(cudaSetDevice(ctx->device));
    fa_launch_blinn_points(points4, (int)n, out2, (cudaStream_t)stream);
    CKL();
    return FA_OK;
}

int fa_select_side_plane(fa_ctx* ctx, const double* tris12, int64_t n, int32_t* out, void* stream) {
    if (!ctx || n < 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (n == 0) return FA_OK;
    CK(cudaSetDevice(ctx->device));
    fa_launch_select_side_plane(tris12, (int)n, out, (cudaStream_t)stream);
    CKL();
    return FA_OK;
}

int fa_chart_bbox(fa_ctx* ctx, const double* vp_host, const double* tris_xyz, int64_t n, double* box_host,
                  void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !vp_host || n < 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (n == 0) return set_err(FA_DEGENERATE_CHART, "chart has no triangles");
    CK(cudaSetDevice(ctx->device));
    ENSURE(vp_dev, FA_VP_DOUBLES * sizeof(double));
    ENSURE(aux, 128);
    int r = upload_vp(ctx, vp_host, s);
    if (r) return r;
    unsigned long long* keys = P<unsigned long long>(ctx->aux);
    int* surv = reinterpret_cast<int*>(keys + 4);
    double* box = reinterpret_cast<double*>(keys + 6);
    fa_launch_chart_bbox_world(tris_xyz, (int)n, P<double>(ctx->vp_dev), keys, surv, box, s);
    CKL();
    double hb[4];
    int hs = 0;
    CK(cudaMemcpyAsync(hb, box, 32, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs, surv, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!hs) return set_err(FA_DEGENERATE_CHART, "no triangle survives clipping");
    memcpy(box_host, hb, sizeof(hb));
    return FA_OK;
}

int fa_viewport_box(fa_ctx* ctx, const double* boxes4, int64_t n, int width, int height, int64_t* out2,
                    void* stream) {
    if (!ctx || n < 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (width < 1 || height < 1) return set_err(FA_VALUE_ERROR, "screen dimensions must be >= 1");
    if (n == 0) return FA_OK;
    CK(cudaSetDevice(ctx->device));
    fa_launch_viewport_box(boxes4, (int)n, width, height, (long long*)out2, (cudaStream_t)stream);
    CKL();
    return FA_OK;
}

int fa_sequential_scale_search(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h,
                               const int64_t* chart_id, const int64_t* min_tri, int64_t n, int64_t omega,
                               int64_t n_scales, int64_t min_dim, int64_t padding, int64_t* placements_out,
                               int64_t* scale_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int r = check_omega(omega);
    if (r) return r;
    if (!ctx || n < 0 || n >= (1ll << 30) || n_scales > (1 << 20)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (n > 0 && n_scales < 1) return set_err(FA_PACK_FAILURE, "every candidate scale was rejected");
    if (min_dim < 1 || padding < 0 || min_dim > (1 << 28) || padding > (1 << 28))
        return set_err(FA_VALUE_ERROR, "min_dim must be >= 1 and padding >= 0");
    if (n == 0) {
        if (scale_host) { scale_host[0] = 1; scale_host[1] = 1; }
        return FA_OK;
    }
    CK(cudaSetDevice(ctx->device));
    ENSURE(dstat, sizeof(fa_dstat));
    return seq_search_core(ctx, target_w, target_h, chart_id, min_tri, n, omega, n_scales, min_dim, padding,
                           placements_out, scale_host, ctx->dstat, s);
}

int fa_sequential_pack(fa_ctx* ctx, const int64_t* widths, const int64_t* heights, int64_t n, int64_t omega,
                       int64_t* rows_out, int64_t* x_out, int64_t* y_out, int64_t* used_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int r = check_omega(omega);
    if (r) return r;
    if (!ctx || n < 1 || n >= (1ll << 30)) return set_err(FA_VALUE_ERROR, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    r = ensure_pack(ctx, n, 1, omega, 1);
    if (r) return r;
    ENSURE(dstat, sizeof(fa_dstat));
    CK(cudaMemsetAsync(ctx->dstat.p, 0, sizeof(fa_dstat), s));
    CK(cudaMemsetAsync(ctx->cand.p, 0, FA_CAND_REC * 8, s));
    fa_launch_seq_single((const long long*)widths, (const long long*)heights, (int)n, omega, P<int>(ctx->cand_w),
                         P<int>(ctx->cand_h), P<int>(ctx->cand_p), P<int>(ctx->cand_y), P<int>(ctx->rowstart),
                         P<int>(ctx->oidx), fa_front_in_smem(omega) ? nullptr : P<int>(ctx->okey),
                         P<long long>(ctx->cand), &P<fa_dstat>(ctx->dstat)->done, (long long*)rows_out,
                         (long long*)x_out, (long long*)y_out, s);
    CKL();
    long long rec[3];
    CK(cudaMemcpyAsync(rec, ctx->cand.p, sizeof(rec), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (used_host) *used_host = rec[1];
    return FA_OK;
}

int fa_superblock_pack(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h, const int64_t* chart_id,
                       const int64_t* min_tri, int64_t n, int64_t omega, int64_t block_size, int halving_enabled,
                       int64_t* placements_out, int64_t* scale_host, int64_t* block_used_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || n < 0 || n >= (1ll << 30)) return set_err(FA_VALUE_ERROR, "bad arguments");
    int r = check_superblock(omega, block_size);
    if (r) return r;
    if (n == 0) {
        if (scale_host) { scale_host[0] = 1; scale_host[1] = 1; }
        if (block_used_host) *block_used_host = block_size;
        return FA_OK;
    }
    CK(cudaSetDevice(ctx->device));
    ENSURE(dstat, sizeof(fa_dstat));
    return superblock_core(ctx, target_w, target_h, chart_id, min_tri, n, omega, block_size, halving_enabled,
                           placements_out, scale_host, block_used_host, ctx->dstat, s);
}

int fa_orient(fa_ctx* ctx, const int64_t* target_w, const int64_t* target_h, int64_t n, int64_t* ow_out,
              int64_t* oh_out, uint8_t* rot_out, void* stream) {
    if (!ctx || n < 0 || n >= (1ll << 31)) return set_err(FA_VALUE_ERROR, "bad arguments");
    if (n == 0) return FA_OK;
    CK(cudaSetDevice(ctx->device));
    fa_launch_orient((const long long*)target_w, (const long long*)target_h, (int)n, (long long*)ow_out,
                     (long long*)oh_out, rot_out, (cudaStream_t)stream);
    CKL();
    return FA_OK;
}

}  // extern "C"

FA_TRACE_TU(api)

#ifdef FA_TRACE
// ---- debug trace (FA_TRACE builds): per-kernel device timestamps ------------
void fa_trace_bind_raster(void*);
void fa_trace_bind_charts(void*);
void fa_trace_bind_bounds(void*);
void fa_trace_bind_pack(void*);
void fa_trace_bind_uv(void*);
void fa_trace_bind_baselines(void*);
void fa_trace_bind_mesh(void*);
static fa_trace_rec* g_trace_dev = nullptr;

extern "C" int fa_debug_trace_reset(void) {
    if (!g_trace_dev && cudaMalloc(&g_trace_dev, 128 * sizeof(fa_trace_rec)) != cudaSuccess) return -1;
    fa_trace_rec init[128];
    for (auto& r : init) r = {0ull, ~0ull, 0ull, 0ull};
    cudaMemcpy(g_trace_dev, init, sizeof(init), cudaMemcpyHostToDevice);
    void* p = g_trace_dev;
    fa_trace_bind_raster(p); fa_trace_bind_charts(p); fa_trace_bind_bounds(p); fa_trace_bind_pack(p);
    fa_trace_bind_uv(p); fa_trace_bind_baselines(p); fa_trace_bind_mesh(p); fa_trace_bind_api(p);
    return 0;
}

// n records: kernel key (decimal string, names[64*i]), first start, last end (ns), launches
extern "C" int fa_debug_trace_read(char* names, unsigned long long* start, unsigned long long* end,
                                   unsigned long long* hits, int max) {
    if (!g_trace_dev) return 0;
    cudaDeviceSynchronize();
    fa_trace_rec rec[128];
    cudaMemcpy(rec, g_trace_dev, sizeof(rec), cudaMemcpyDeviceToHost);
    int n = 0;
    for (int i = 0; i < 128 && n < max; i++) {
        if (!rec[i].name) continue;
        char buf[64] = {0};
        snprintf(buf, sizeof(buf), "%llu", rec[i].name);
        memcpy(names + 64 * n, buf, 64);
        start[n] = rec[i].start;
        end[n] = rec[i].end;
        hits[n] = rec[i].hits;
        n++;
    }
    return n;
}
#endif
