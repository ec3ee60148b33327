// fa_internal.h — context layout and kernel launchers (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fastatlas.h"
#include "fa_common.cuh"

struct TriSetup;
struct SmallRec;

// Culling data of 32 consecutive triangles of the setup order (fa_mesh.cu)
struct fa_cluster {
    double c[3], r;        // bounding sphere
    double a[3];           // normal cone axis (unit)
    double cos_t, sin_t;   // cone half angle (widened for rounding)
    double amin;           // smallest triangle area (0: never back-face culled)
};

// The raster setup's triangle order and cluster culling data (fa_set_mesh);
// all null: the given order, no culling
struct fa_setup_order {
    const int* tperm;
    const int* tris_sorted;
    const int4* slots4;  // (a, b, c, triangle id) per setup slot: one 16-byte load (or null)
    const int* live;    // live clusters (k_frame_init), or null: every slot
    const int* n_live;
};

// k_frame_init's cluster culling (clusters null: none)
struct fa_cull_args {
    const fa_cluster* clusters;
    int n_clusters;
    int cull;
    int* live;
    fa_dstat* st;
};

// Per-frame view constants derived from the camera matrix (k_frame_init)
struct fa_view_consts {  // (FA_VP_DOUBLES - FA_VC_OFF doubles at most)
    double plane[7][4];    // L, R, B, T, N, F (w +- x, y, z) and w - W_EPSILON, as rows over (x, y, z, 1)
    double pn[7];          // |plane normal|
    double cam[3];         // projection centre (x = y = w = 0)
    double sigma;          // sign of det([VP_x; VP_y; VP_w] 3x3); 0 disables back-face culling
    double area_k;         // W * H / 4 * |det3|
    double tau;            // screen area (px^2) above any rounding of the reference's shoelace
};

// growable device buffer
struct fa_buf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct fa_graph_key {
    int width = 0, height = 0, cull = 0, uv_f64 = 0, want_depth = 0;
    long long omega = 0, n_scales = 0, min_dim = 0, padding = 0;
    double prescale = 0;
    long long T = 0, V = 0;
    const void* pos = nullptr;
    const void* tris = nullptr;
    size_t gen = 0;  // buffer generation (graph invalid after any regrow)
    bool operator==(const fa_graph_key& o) const {
        return width == o.width && height == o.height && cull == o.cull && uv_f64 == o.uv_f64 &&
               want_depth == o.want_depth && omega == o.omega && n_scales == o.n_scales && min_dim == o.min_dim &&
               padding == o.padding && prescale == o.prescale && T == o.T && V == o.V && pos == o.pos &&
               tris == o.tris && gen == o.gen;
    }
};

struct fa_ctx {
    int device = 0;
    // resident mesh.  pos/tris are what the kernels read: the context's own
    // copy with vertices renumbered in order of first use (fa_set_mesh), so
    // the three vertices of consecutive triangles share cache lines; the
    // caller's arrays stay untouched (pos_user feeds per-vertex outputs in
    // the caller's numbering, vperm maps new -> caller vertex index).
    const double* pos = nullptr;
    const int* tris = nullptr;
    const double* pos_user = nullptr;
    const int* vperm = nullptr;
    int64_t V = 0, T = 0;
    fa_buf pos_perm, tris_perm, vperm_buf;
    // the raster setup's order: Morton order of the triangle centroids
    // (tperm[slot] = triangle id, tris_sorted = its renumbered vertex
    // indices) and the culling data of each 32-slot cluster
    const int* tperm = nullptr;
    const int* tris_sorted = nullptr;
    const fa_cluster* clusters = nullptr;
    fa_buf tperm_buf, tris_sorted_buf, clusters_buf, live_buf, slots4_buf;
    fa_buf mesh_first, mesh_scratch, mesh_sort, mesh_tris_s;  // fa_set_mesh scratch
    fa_buf ord_tw, ord_th, ord_cid;  // per packing position (k_order_frame -> k_select)
    fa_buf ndc2;                     // per-vertex NDC of the inside vertices (vertex_ndc), for bounds and UVs

    // scratch (grown on demand)
    fa_buf small_rec, clip, depth_keys, depth_f64, flags, vis_list, large, tiles, label, vmin, v2c, cidx;
    fa_buf roots, ndc_keys, ndc, px, target, survived, okey, oidx, ow, oh, orot, sortk, sortv, pinv;
    fa_buf cand, cand_p, cand_w, cand_h, cand_y, rowstart, placements, uv, vp_dev, blocks, dstat, aux;
    fa_buf in_tw, in_th, in_cid, in_mt;
    fa_buf pstat;           // comparison packers' status block inside a frame (the frame keeps dstat)
    fa_buf scr, clip_list;  // per-vertex screen records; generic-path triangle list
    fa_buf hiz;             // 8x8 hierarchical-Z max keys of the final depth
    fa_buf wid;             // pass-1 pixel winners (truncated key | triangle id)
    fa_buf vis_chart;       // chart id of each visible triangle (written by k_uv)
    fa_buf vis_mask;        // packed download format: visibility bit per triangle (k_scatter_visible)
    fa_buf vvis_mask;       //   bit per vertex in the context's order (k_vert_scatter)
    fa_buf cidx16;          //   16-bit chart index per visible triangle (k_uv)
    fa_buf vis_cidx;        // chart index of each visible triangle (written by k_chart_bounds, read by k_uv)
    fa_buf plc_c;           // placements by chart index (2 x int4 each; written by k_select, read by k_uv)
    fa_buf vis_tris;        // (a, b, c, t) of each visible triangle (written by the compaction)
    fa_buf vslot, vlist, vuv, vblocks;  // visible vertices: slot per vertex, caller ids, f32 UV pairs, block counts
    size_t gen = 0;
    int max_large = 0, max_tiles = 0;
    int queue_init = 0;  // FASTATLAS_QUEUE_INIT (tests): initial large/tile queue capacity
    int pack_batch = 0;  // candidates per pack launch
    int64_t pack_cap = 0;  // boxes the pack scratch holds
    bool needs_rerun = false;

    fa_dstat* hstat = nullptr;  // pinned mirror of the device status
    // pinned camera staging: a ring of 16-double slots, each reused only
    // after the event recorded behind its upload has completed
    static const int kVpSlots = 8;
    double* hvp = nullptr;      // kVpSlots x FA_VP_DOUBLES doubles
    cudaEvent_t vp_ev[kVpSlots] = {};
    int vp_next = 0;
    fa_frame_params last_params{};
    int last_launches = 0;

    // CUDA graph per frame shape
    cudaGraphExec_t graph_exec = nullptr;
    fa_graph_key graph_key{};

    // stage timing (params.profile)
    static const int kMaxStages = 12;
    cudaEvent_t ev[kMaxStages + 1] = {};
    int n_stage_marks = 0;

    // side stream + fork/join events for the independent raster branches
    cudaStream_t side = nullptr, side2 = nullptr;
    cudaEvent_t fj[12] = {};
    // recorded after a frame's downloads (fa_frame_download*): the next frame
    // waits on it before its first write to a downloaded buffer, so the copies
    // may run on another stream, overlapping the next frame's start
    cudaEvent_t copy_done = nullptr;
};

// growth helper: ensures buf has >= bytes; returns false on allocation failure
bool fa_ensure(fa_ctx* ctx, fa_buf& b, size_t bytes);

// ---- raster (fa_raster.cu) ------------------------------------------------
// wid (may be null): pass-1 winner buffer, cleared to all ones with depth
void fa_launch_frame_init(const double* pos, int V, const double* vp, double4* clip, double4* scr, int W, int H,
                          int* vmin, unsigned long long* depth, unsigned long long* wid, long long npx,
                          unsigned char* flags, int T, cudaStream_t s, int max_blocks = 0,
                          double2* ndc2 = nullptr,
                          const fa_cull_args* cull = nullptr);
// the setup's live-cluster list (no-op when cu.clusters is null)
void fa_launch_cluster_cull(const double* vp, int W, int H, const fa_cull_args& cu, cudaStream_t s);
// side == nullptr: everything on s; otherwise fork/join through the events.
// Both return the number of kernels launched.  wid: see depth_min (may be null).
int fa_launch_depth_pass(bool write_depth, const ClipSrc clip, const double4* scr, const int* tris, int T, int W,
                         int H, int cull, unsigned long long* depth, unsigned long long* wid, SmallRec* small_rec,
                         int* clip_list, TriSetup* large, int max_large, int4* tiles, int max_tiles, fa_dstat* st,
                         cudaStream_t s, cudaStream_t side, cudaStream_t side2, cudaEvent_t ev_fork,
                         cudaEvent_t ev_join, cudaEvent_t ev_join2, cudaEvent_t ev_clear = nullptr,
                         fa_setup_order ord = fa_setup_order{});
int fa_launch_raster_vis(const SmallRec* small_rec, const TriSetup* large, const int4* tiles, int max_tiles,
                         int max_large, int T, int W, const unsigned long long* depth, const unsigned long long* hiz,
                         unsigned char* flags, int* vis_queue, fa_dstat* st, cudaStream_t s, cudaStream_t side,
                         cudaEvent_t ev_fork, cudaEvent_t ev_join);
void fa_launch_decode_depth(const unsigned long long* keys, double* out, long long n, cudaStream_t s);
// screen_fragments (st may be null) + 8x8 hierarchical-Z max keys + flags of
// the pass-1 pixel winners (wid may be null)
void fa_launch_depth_hiz(const unsigned long long* depth, const unsigned long long* wid, int W, int H,
                         unsigned long long* hiz, unsigned char* flags, fa_dstat* st, cudaStream_t s);
static inline int fa_hiz_dim(int n) { return (n + FA_HIZ - 1) / FA_HIZ; }
void fa_launch_encode_depth(const double* in, unsigned long long* keys, long long n, cudaStream_t s);
size_t fa_trisetup_bytes();

// ---- charts (fa_charts.cu) -----------------------------------------------
// ordered compaction of flags -> vis list; label[t] = flag ? t : -1
// with tris + vmin (vmin pre-filled with INT_MAX) it also computes vmin
// with tris: also vis_tris[k] = (a, b, c, t) of each visible triangle (when
// non-null) and vmin lowering (when non-null)
void fa_launch_compact_visible(const unsigned char* flags, int T, int* blocks, int* vis_list, int* label,
                               fa_dstat* st, cudaStream_t s, const int* tris = nullptr, int* vmin = nullptr,
                               int4* vis_tris = nullptr,
                               unsigned int* vis_mask = nullptr);
int fa_compact_blocks(long long n);
// vmin_ready: vmin already holds the per-vertex minima (computed by the
// visible compaction); otherwise it must hold INT_MAX and is computed here
int fa_launch_uf_vertex(const int* tris, const int* vis_list, int* vmin, int* label, int T, const fa_dstat* st,
                         cudaStream_t s, bool vmin_ready = false, const int4* vis_tris = nullptr);
void fa_launch_uf_edges(const int* adjacency, const unsigned char* flags, const int* vis_list, int* label, int T,
                        const fa_dstat* st, cudaStream_t s);
void fa_launch_uf_labels(const int* labels_in, const int* vis_list, int* label, int T, const fa_dstat* st,
                         cudaStream_t s);
void fa_launch_iota(int* label, int T, cudaStream_t s);
void fa_launch_build_adjacency(const int* tris, int T, unsigned long long* keys, int* cnt, int* c0, int* c1,
                               unsigned long long table_size, int* adj, cudaStream_t s);
void fa_launch_uf_compress(const int* vis_list, int* label, int T, const fa_dstat* st, cudaStream_t s);
void fa_launch_canonicalize(const int* vis_list, int* label, int* tmp, int T, const fa_dstat* st, cudaStream_t s);
void fa_launch_v2c(const int* vmin, const int* label, int* v2c, int V, cudaStream_t s, const int* vperm = nullptr);
// visible vertices: vslot (V,) slot or -1, vlist (n,) caller ids, st->n_vis_vertices;
// blocks holds fa_vertex_blocks(V) ints
int fa_vertex_blocks(long long V);
void fa_launch_visible_vertices(const int* vmin, int V, const int* vperm, int* blocks, int* vslot, int* vlist,
                                fa_dstat* st, cudaStream_t s, float2* vuv = nullptr,
                                unsigned int* vvis_mask = nullptr);
// out[v] = pos[vperm[v]] (3 doubles each)
void fa_launch_permute_pos(const double* pos, const int* vperm, double* out, int V, cudaStream_t s);
void fa_launch_flags_from_labels(const int* labels, unsigned char* flags, int T, cudaStream_t s);
// ordered compaction of roots (label[t]==t over the vis list) -> roots, cidx, chart init
void fa_launch_compact_roots(const int* vis_list, const int* label, int T, int* blocks, int* roots, int* cidx,
                             unsigned long long* ndc_keys, int* survived, fa_dstat* st, cudaStream_t s);
void fa_launch_canon_apply(const unsigned char* flags, int* label, const int* tmp, int T, cudaStream_t s);
void fa_launch_fill(int* a, int n, int v, cudaStream_t s);

// ---- mesh binding (fa_mesh.cu) ----------------------------------------------
int fa_mesh_scratch_ints(long long V, long long T);
void fa_launch_mesh_validate(const int* tris, long long T, int V, int* first, int* bad, cudaStream_t s);
void fa_launch_mesh_renumber(const double* pos, const int* tris, long long T, int V, const int* first, int* scratch,
                             int* newidx, int* tris_out, int* perm, double* pos_out, cudaStream_t s);

size_t fa_mesh_sort_scratch_bytes(long long T);
void fa_launch_mesh_order(const double* pos, const int* tris, int T, int V, void* scratch, int* order,
                          int* tris_sorted, cudaStream_t s);
void fa_launch_mesh_remap(const int* tris, long long T, const int* newidx, int* out, cudaStream_t s);
void fa_launch_make_slots4(const int* tris_sorted, const int* tperm, int T, int4* out, cudaStream_t s);
void fa_launch_cluster_build(const double* pos, const int* tris_sorted, int T, fa_cluster* out, cudaStream_t s);

// ---- bounds (fa_bounds.cu) -----------------------------------------------
void fa_launch_chart_bounds(const ClipSrc clip, const int* tris, const int* vis_list, const int* label,
                            const int* cidx, int T, unsigned long long* ndc_keys, int* survived, const fa_dstat* st,
                            cudaStream_t s, int* vis_cidx = nullptr, const int4* vis_tris = nullptr, const double2* ndc2 = nullptr);
void fa_launch_box_dims(const unsigned long long* ndc_keys, const int* survived, const int* roots, int T, int W, int H,
                        double prescale, double* ndc, int* px, long long* target, long long* tw, long long* th,
                        long long* cid, int cap, fa_dstat* st, cudaStream_t s);

// ---- pack (fa_pack.cu) ---------------------------------------------------
struct fa_pack_bufs {
    const long long* tw;       // target dims, input order
    const long long* th;
    const long long* chart_id; // per input box
    long long* ow;             // ordered oriented dims
    long long* oh;
    unsigned char* rot;        // ordered rotated flag
    int* perm;                 // ordered -> input index
    int* pinv;                 // input index -> ordered position
    unsigned long long* sortk; // radix ping-pong
    int* sortv;
    long long* cand;           // per-candidate results (4 x int64 each)
    long long* cand_p;         // per-candidate prefix sums (n each)
    int* cand_w;
    int* cand_h;
    int* cand_y;
    int* rowstart;             // per-candidate row starts (n each)
    long long* placements;     // (n,8) packing order
    int4* plc_by_src;          // optional (n,2) int4 per input box: {x, y, w, h}, {rot, 0, 0, 0}
    unsigned char* accept_out; // optional
    int* gfront;               // global frontline (batch x (omega+1)) when omega is too big for smem
    // frame path: target dims / chart id per packing position (k_order_frame
    // writes them when ord_written, k_select reads them without perm)
    long long* ord_tw = nullptr;
    long long* ord_th = nullptr;
    long long* ord_cid = nullptr;
    bool ord_written = false;
};
// bd (optional): compute the per-chart box dims (k_box_dims' work) first, in the same launch
void fa_launch_orient_sort(const fa_pack_bufs& b, int n_max, const int* n_dev, long long max_h, fa_dstat* st,
                           cudaStream_t s, const fa_box_dims_args* bd = nullptr);
int fa_launch_pack(const fa_pack_bufs& b, int n_max, const int* n_dev, long long omega, long long n_scales,
                   long long min_dim, long long pad, int batch, fa_dstat* st, cudaStream_t s);
void fa_launch_orient_sort_mt(const long long* tw, const long long* th, const long long* mt, int n, long long max_h,
                              long long* ow, long long* oh, unsigned char* rot, int* perm, int* pinv,
                              unsigned long long* sk, int* sv, int reject_dups, fa_dstat* st, cudaStream_t s);
void fa_launch_pack_at_scale(const long long* ow, const long long* oh, int n, long long num, long long den,
                             long long omega, long long min_dim, long long pad, long long* cand, long long* cand_p,
                             int* cand_w, int* cand_h, int* cand_y, int* rowstart, int* gfront, cudaStream_t s);
void fa_launch_xywh(const long long* cand, const long long* cand_p, const int* cand_w, const int* cand_h,
                    const int* cand_y, int n, long long omega, long long* out, cudaStream_t s);
void fa_launch_push_up_impl(const long long* rows, const long long* x, const long long* w, const long long* h, int n,
                            long long omega, int* rowstart, long long* y, long long* used, int* gfront,
                            cudaStream_t s);
bool fa_front_in_smem(long long omega);
#define FA_CAND_REC 5
void fa_launch_fold(const long long* w, int n, long long omega, long long* rows, long long* x, long long* m,
                    cudaStream_t s);

// ---- uv (fa_uv.cu) -------------------------------------------------------
void fa_launch_uv(const ClipSrc clip, const int* tris, const int* vis_list, const int* label, const int* cidx,
                  const int* pinv, const double* ndc, const int* px, const long long* placements, int T, int W, int H,
                  long long pad, bool f64, void* uv, int* vis_chart, const int* vis_cidx, const int4* plc_c,
                  fa_dstat* st, cudaStream_t s, const int4* vis_tris = nullptr, const int* vslot = nullptr,
                  float2* vuv = nullptr, const double2* ndc2 = nullptr, unsigned short* cidx16 = nullptr);

// ---- comparison packers (fa_baselines.cu) -----------------------------------
void fa_launch_seq_search(const long long* ow, const long long* oh, int n, long long omega, long long n_scales,
                          long long min_dim, long long pad, int batch, int* cw, int* ch, int* cx, int* cy,
                          int* rowstart, int* gfront, long long* cand, unsigned* done, cudaStream_t s);
void fa_launch_seq_single(const long long* w, const long long* h, int n, long long omega, int* cw, int* ch, int* cx,
                          int* cy, int* rowstart, int* rows, int* gfront, long long* cand, const unsigned* done_zero,
                          long long* rows_out, long long* x_out, long long* y_out, cudaStream_t s);
void fa_launch_seq_select(const long long* tw, const long long* th, const long long* cid, const unsigned char* rot,
                          const int* perm, int n, long long n_scales, const long long* cand, const int* cw,
                          const int* ch, const int* cx, const int* cy, long long* placements, long long* out,
                          cudaStream_t s);
void fa_launch_superblock(const long long* ow, const long long* oh, const long long* tw, const long long* th,
                          const long long* cid, const unsigned char* rot, const int* perm, int n, long long omega,
                          int block0, int n_levels, int* state, size_t state_stride, int* xywh, size_t out_stride,
                          int* level_ok, long long* placements, long long* out, cudaStream_t s);

// ---- standalone helpers (fa_bounds.cu / fa_pack.cu) -------------------------
void fa_launch_blinn_points(const double* p4, int n, double* out, cudaStream_t s);
void fa_launch_select_side_plane(const double* t12, int n, int* out, cudaStream_t s);
void fa_launch_chart_bbox_world(const double* xyz, int n, const double* vp, unsigned long long* keys, int* surv,
                                double* box_out, cudaStream_t s);
void fa_launch_viewport_box(const double* box, int n, int W, int H, long long* out, cudaStream_t s);
void fa_launch_orient(const long long* tw, const long long* th, int n, long long* ow, long long* oh,
                      unsigned char* rot, cudaStream_t s);
