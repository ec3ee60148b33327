/*
 * fastatlas.h — C ABI of the B200 (sm_100a) per-frame atlasing library.
 *
 * The reference (`atlaspack`, pure Python/numpy) has no FFI; its boundary is
 * the Python API re-exported by /root/reference/pkg/src/atlaspack/__init__.py:3-64
 * plus `run_scene_pipeline` (cli.py:360-406).  Each entry point below replaces
 * one reference function on the per-frame path; the comment names it.  The
 * Python mirror (paper_2502_17712_b200/) binds these through ctypes, exactly
 * as INTEGRATION.md shows for the reference package.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers unless the parameter says host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - A context is bound to one device, owns its scratch and frame outputs
 *     (valid until the next call on the same context) and is not thread safe.
 *   - Return value: FA_OK or one of the status codes, which map 1:1 onto the
 *     reference's exceptions (ValueError, PackFailure, NothingVisible,
 *     HeightOverflow, DegenerateChart); negative codes are CUDA / internal
 *     errors.  fa_last_error() gives a message.
 *   - Triangles are int32 (T,3) row-major; positions float64 (V,3) row-major;
 *     camera matrices are the 16 row-major float64 of CameraFrame.view_proj
 *     (geometry.py:90-92), passed by HOST pointer.
 */
#ifndef FASTATLAS_H
#define FASTATLAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FA_ABI_VERSION 2

enum fa_status {
    FA_OK = 0,
    FA_VALUE_ERROR = 1,       /* ValueError (packing.py:313-323,365-367, charts.py:294-295, ...) */
    FA_PACK_FAILURE = 2,      /* PackFailure (packing.py:328-332,345) */
    FA_NOTHING_VISIBLE = 3,   /* NothingVisible (cli.py:366-368) */
    FA_HEIGHT_OVERFLOW = 4,   /* HeightOverflow (packing.py:127-129) */
    FA_DEGENERATE_CHART = 5,  /* DegenerateChart (geometry.py:320-321) */
    FA_CUDA_ERROR = -1,
    FA_INTERNAL_ERROR = -2
};

typedef struct fa_ctx fa_ctx;

/* ---- context ---------------------------------------------------------- */
int fa_abi_version(void);
const char *fa_last_error(void);
int fa_create(fa_ctx **out, int device);
void fa_destroy(fa_ctx *ctx);

/* Bind a resident mesh (Mesh, charts.py:29-61): device pointers, positions
 * (V,3) float64 and triangles (T,3) int32.  The context keeps its own copy
 * with the vertices renumbered in order of first use (better locality for
 * the per-vertex gathers; triangle order and every output are unchanged,
 * per-vertex outputs come back in the caller's numbering), so call it again
 * after modifying the caller's arrays.  ValueError on an index outside
 * [0, V).  `positions` must stay valid for fa_project, which reads it. */
int fa_set_mesh(fa_ctx *ctx, const double *positions, int64_t n_vertices,
                const int32_t *triangles, int64_t n_triangles);

/* ---- per-stage entry points (reference functions) ----------------------- */

/* homo @ view_proj.T for every vertex (charts.py:273-274); clip_out is (V,4). */
int fa_project(fa_ctx *ctx, const double *vp_host, double *clip_out, void *stream);

/* depth_prepass (charts.py:285-299): depth_out (H,W) float64, +inf uncovered. */
int fa_depth_prepass(fa_ctx *ctx, const double *vp_host, int width, int height, int backface_cull,
                     double *depth_out, void *stream);

/* mark_visible (charts.py:302-313): flags_out (T,) uint8. */
int fa_mark_visible(fa_ctx *ctx, const double *vp_host, const double *depth, int width, int height,
                    int backface_cull, uint8_t *flags_out, void *stream);

/* build_adjacency (charts.py:64-77) of the bound mesh: adjacency_out (T,3)
 * int32, the triangle sharing edge e of t, or -1 unless exactly two (t, e)
 * slots use that edge.  Synchronises the stream (per mesh, not per frame). */
int fa_build_adjacency(fa_ctx *ctx, int32_t *adjacency_out, void *stream);

/* connected_charts (charts.py:343-359): labels_out (T,) int32, -1 invisible. */
int fa_connected_charts(fa_ctx *ctx, const int32_t *adjacency, const uint8_t *flags,
                        int32_t *labels_out, void *stream);

/* merge_shared_vertices (charts.py:362-386): labels_out (T,), vertex_to_chart_out (V,) int32. */
int fa_merge_shared_vertices(fa_ctx *ctx, const int32_t *labels_in, int32_t *labels_out,
                             int32_t *vertex_to_chart_out, void *stream);

/* Per-chart chart_bbox (geometry.py:281-322) + viewport_box (geometry.py:352-362)
 * + prescale (cli.py:379-384) for every chart of `labels` in ascending-root
 * order.  Outputs are sized for the worst case (T charts); *n_charts_host
 * receives the count (synchronises the stream). */
int fa_chart_boxes(fa_ctx *ctx, const double *vp_host, const int32_t *labels, int width, int height,
                   double prescale, int32_t *roots_out, double *ndc_out, int32_t *px_out,
                   int64_t *target_out, int64_t *n_charts_host, void *stream);

/* Batched forms of the scalar geometry helpers on the chart_bbox path:
 * blinn_clamped_ndc (geometry.py:185-200) over (n,4) points -> (n,2);
 * select_side_plane (geometry.py:257-278) over (n,3,4) clip triangles ->
 * plane index 0..3 (left, right, bottom, top) or -1 for None;
 * chart_bbox (geometry.py:281-322) of (n,3,3) world triangles -> box_host[4]
 * (FA_DEGENERATE_CHART when nothing survives);
 * viewport_box (geometry.py:352-362) over (n,4) boxes -> (n,2) int64. */
int fa_blinn_clamped_ndc(fa_ctx *ctx, const double *points4, int64_t n, double *out2, void *stream);
int fa_select_side_plane(fa_ctx *ctx, const double *tris12, int64_t n, int32_t *out, void *stream);
int fa_chart_bbox(fa_ctx *ctx, const double *vp_host, const double *tris_xyz, int64_t n, double *box_host,
                  void *stream);
int fa_viewport_box(fa_ctx *ctx, const double *boxes4, int64_t n, int width, int height, int64_t *out2,
                    void *stream);

/* orient (packing.py:109-117): rotate boxes wider than tall. */
int fa_orient(fa_ctx *ctx, const int64_t *target_w, const int64_t *target_h, int64_t n, int64_t *ow_out,
              int64_t *oh_out, uint8_t *rot_out, void *stream);

/* orient + order (packing.py:109-130): perm_out[i] = input index of the i-th
 * ordered box; ow/oh oriented dims, rot rotated flag. */
int fa_orient_order(fa_ctx *ctx, const int64_t *target_w, const int64_t *target_h,
                    const int64_t *min_tri, int64_t n, int64_t max_h, int32_t *perm_out,
                    int64_t *ow_out, int64_t *oh_out, uint8_t *rot_out, void *stream);

/* fold (packing.py:133-158). *m_host receives overflow_m (synchronises). */
int fa_fold(fa_ctx *ctx, const int64_t *widths, int64_t n, int64_t omega, int64_t *rows_out,
            int64_t *x_out, int64_t *m_host, void *stream);

/* push_up (packing.py:170-215). *used_host receives the frontline maximum. */
int fa_push_up(fa_ctx *ctx, const int64_t *rows, const int64_t *x, const int64_t *widths,
               const int64_t *heights, int64_t n, int64_t omega, int64_t *y_out, int64_t *used_host,
               void *stream);

/* pack_at_scale / _pack_arrays (packing.py:218-292) on ordered oriented
 * boxes.  *accepted_host = 1 and xywh_out (n,4), scale_host[2] on accept. */
int fa_pack_at_scale(fa_ctx *ctx, const int64_t *ow, const int64_t *oh, int64_t n, int64_t num,
                     int64_t den, int64_t omega, int64_t min_dim, int64_t padding, int64_t *xywh_out,
                     int64_t *scale_host, int *accepted_host, void *stream);

/* pack (packing.py:295-345).  placements_out (n,8) int64 in packing order:
 * chart_id x y w h rotated target_w target_h.  scale_host[2] = num, den.
 * accept_out (optional, n_scales bytes, device) receives the accept vector. */
int fa_pack(fa_ctx *ctx, const int64_t *target_w, const int64_t *target_h, const int64_t *chart_id,
            const int64_t *min_tri, int64_t n, int64_t omega, int64_t n_scales, int64_t min_dim,
            int64_t padding, int64_t *placements_out, int64_t *scale_host, uint8_t *accept_out,
            void *stream);

/* ---- comparison packers (atlaspack.baselines, used by `compare`) -------- */

/* sequential_scale_search (baselines.py:110-141): placements_out (n,8) in
 * packing order, scale_host[2]; FA_PACK_FAILURE when no candidate fits. */
int fa_sequential_scale_search(fa_ctx *ctx, const int64_t *target_w, const int64_t *target_h,
                               const int64_t *chart_id, const int64_t *min_tri, int64_t n, int64_t omega,
                               int64_t n_scales, int64_t min_dim, int64_t padding, int64_t *placements_out,
                               int64_t *scale_host, void *stream);

/* sequential_fold + sequential_pack (baselines.py:53-107) on the caller's
 * order at the stated dims (widths must be in [1, omega]): rows/x/y (n) int64
 * and the used height; the layout is accepted iff *used_host <= omega. */
int fa_sequential_pack(fa_ctx *ctx, const int64_t *widths, const int64_t *heights, int64_t n, int64_t omega,
                       int64_t *rows_out, int64_t *x_out, int64_t *y_out, int64_t *used_host, void *stream);

/* superblock_pack (baselines.py:187-261): placements_out (n,8), scale_host[2]
 * = worst per-box downscale, *block_used_host = block size that succeeded;
 * FA_PACK_FAILURE when even the halving floor fails (reference returns None). */
int fa_superblock_pack(fa_ctx *ctx, const int64_t *target_w, const int64_t *target_h, const int64_t *chart_id,
                       const int64_t *min_tri, int64_t n, int64_t omega, int64_t block_size, int halving_enabled,
                       int64_t *placements_out, int64_t *scale_host, int64_t *block_used_host, void *stream);

/* ---- whole frame: run_scene_pipeline (cli.py:360-406) -------------------- */

/* fa_frame_params.packer: the packer registry of cli.py:318-339 (make_packer).
 * FASTATLAS runs inside the frame's CUDA graph; the comparison packers run
 * the frame without a graph, with one host synchronisation after the chart
 * boxes (their box count sizes the launches).  Any other value fails with
 * FA_VALUE_ERROR after the NothingVisible check, where the reference's
 * make_packer raises InputError (cli.py:339, called at :386). */
#define FA_PACKER_FASTATLAS 0   /* pack (packing.py:295-345) */
#define FA_PACKER_SEQUENTIAL 1  /* sequential_scale_search (baselines.py:110-141) */
#define FA_PACKER_SUPERBLOCK 2  /* superblock_pack (baselines.py:187-261); None -> FA_PACK_FAILURE (cli.py:333-335) */

typedef struct fa_frame_params {
    int width, height;       /* SceneConfig.screen */
    int64_t omega;           /* SceneConfig.omega (power of two) */
    int64_t n_scales;        /* SceneConfig.n_scales */
    int64_t min_dim;         /* SceneConfig.min_dim */
    int64_t padding;         /* SceneConfig.padding */
    double prescale;         /* SceneConfig.prescale */
    int backface_cull;       /* SceneConfig.backface_cull */
    int uv_f64;              /* 1: emit float64 UVs (bit-exact), 0: float32 */
    int want_depth;          /* 1: decode the depth buffer into float64 */
    int use_graph;           /* 1: replay a captured CUDA graph per shape */
    int profile;             /* 1: record CUDA events between stages (implies use_graph = 0) */
    int packer;              /* FA_PACKER_* (run_scene_pipeline's `packer`, cli.py:360) */
    int64_t block_size;      /* superblock block size; 0 = default_block_size(omega) (cli.py:313-314) */
} fa_frame_params;

typedef struct fa_frame_result {
    int status;                   /* fa_status of the frame */
    int32_t n_visible;            /* visible triangles */
    int32_t n_charts;             /* charts (= boxes = placements) */
    int64_t scale_num, scale_den; /* AtlasLayout.scale */
    int64_t screen_fragments;     /* cli.py:390 */
    int64_t texels_allocated;     /* cli.py:391-393 */
    double stretch_l2;            /* scene_stretch L2 (metrics.py:84-111, via cli.py:409-454) */
    double stretch_linf;          /* scene_stretch Linf */
    int64_t stretch_count;        /* triangle pairs in the stretch sums; 0 -> stretch is None */
    /* device pointers owned by the context, valid until its next frame */
    const double *depth;            /* (H,W) float64 when want_depth */
    const uint8_t *flags;           /* (T,) visibility */
    const int32_t *visible;         /* (n_visible,) ascending triangle ids */
    const int32_t *chart_of_triangle; /* (T,) -1 invisible */
    const int32_t *vertex_to_chart; /* (V,) -1 unmapped */
    const int32_t *roots;           /* (n_charts,) ascending chart ids */
    const double *ndc;              /* (n_charts,4) min_x min_y max_x max_y */
    const int32_t *px;              /* (n_charts,2) viewport w_px h_px */
    const int64_t *target;          /* (n_charts,2) target_w target_h */
    const int64_t *placements;      /* (n_charts,8) packing order */
    const void *uv;                 /* (n_visible,6) float32 or float64, NaN = no UV */
    const int32_t *visible_chart;   /* (n_visible,) chart id of each visible triangle (sparse chart_of_triangle) */
    int64_t n_visible_vertices;     /* vertices touched by a visible triangle */
    const int32_t *visible_vertices; /* (n_visible_vertices,) their ids, ascending, caller's numbering */
    const float *vertex_uv;         /* (n_visible_vertices,2) float32 UV of each (NaN: at/behind the camera plane, or in no UV row) */
} fa_frame_result;

/* Enqueue a whole frame on `stream` (no host synchronisation). */
int fa_frame_launch(fa_ctx *ctx, const double *vp_host, const fa_frame_params *params, void *stream);
/* Wait for the frame and fill `out` (synchronises the stream). */
int fa_frame_finish(fa_ctx *ctx, fa_frame_result *out, void *stream);
/* launch + finish */
int fa_frame(fa_ctx *ctx, const double *vp_host, const fa_frame_params *params, fa_frame_result *out,
             void *stream);

/* Enqueue (asynchronously, on `stream`) the device->host copies of a
 * finished frame's results into caller buffers (pinned host memory for
 * overlap, or device memory: the copies use cudaMemcpyDefault); any pointer
 * may be NULL to skip that output.  Sizes come from `res`:
 * chart_of_triangle T int32, visible n_visible int32, uv n_visible x 6
 * (float32, or float64 when the frame ran with uv_f64), placements n_charts
 * x 8 int64.  The caller synchronises `stream` before reading.  Replaces the
 * per-array `.cpu()` reads of SceneResult (reference cli.py:404-406).
 * Every fa_frame_download* call records a context event after its copies, and
 * the context's next frame waits for it on the device before it rewrites any
 * downloaded buffer -- so the copies may run on another stream, overlapping
 * the start of the next frame (FramePipeline does this). */
int fa_frame_download(fa_ctx *ctx, const fa_frame_result *res, int32_t *chart_of_triangle, int32_t *visible,
                      void *uv, int64_t *placements, void *stream);

/* Sparse form of fa_frame_download for streaming clients: the chart ids of
 * the visible triangles only (visible_chart, n_visible int32; every other
 * triangle's chart id is -1), so chart_of_triangle[visible[i]] =
 * visible_chart[i] is rebuilt on the host without copying the (T,) array.
 * Same conventions as fa_frame_download. */
int fa_frame_download_visible(fa_ctx *ctx, const fa_frame_result *res, int32_t *visible, int32_t *visible_chart,
                              void *uv, int64_t *placements, void *stream);

/* Compact wire format for streaming clients: fa_frame_download_visible
 * without the (n_visible,6) UV rows, plus the UV of each visible vertex
 * (visible_vertices n_visible_vertices int32, vertex_uv n_visible_vertices x 2
 * float32).  Every triangle of a vertex's chart computes the same UV for it
 * (cli.py:436-449 depends on the vertex and its chart only), so a visible
 * triangle's float32 row is (vertex_uv of its 3 vertices), NaN when any of
 * them is NaN -- bit-identical to the frame's float32 `uv` rows. */
int fa_frame_download_compact(fa_ctx *ctx, const fa_frame_result *res, int32_t *visible, int32_t *visible_chart,
                              int32_t *visible_vertices, float *vertex_uv, int64_t *placements, void *stream);

/* Packed wire format (about half the bytes of the compact one, for the
 * same information):
 *   visible_mask  ceil(T/32) uint32: bit t % 32 of word t / 32 set for each
 *                 visible triangle (the reference's mark_visible flags,
 *                 charts.py:302-313, packed; visible = flatnonzero),
 *   visible_cidx  n_visible uint16: the index of each visible triangle's
 *                 chart in `roots` (chart id = roots[visible_cidx[i]]),
 *   roots         n_charts int32: the chart ids (root triangle ids, ascending),
 *   vertex_mask   ceil(V/32) uint32: bit i set for the i-th vertex of the
 *                 context's vertex order (fa_vertex_order) that a visible
 *                 triangle touches, and
 *   vertex_uv     n_visible_vertices x 2 float32 in that same order (as in
 *                 fa_frame_download_compact), placements as above.
 * FA_VALUE_ERROR when the frame has more than 65535 charts (use
 * fa_frame_download_compact).  Same conventions as fa_frame_download. */
int fa_frame_download_packed(fa_ctx *ctx, const fa_frame_result *res, uint32_t *visible_mask,
                             uint16_t *visible_cidx, int32_t *roots, uint32_t *vertex_mask, float *vertex_uv,
                             int64_t *placements, void *stream);

/* The context's vertex order (V int32 caller vertex ids; the identity when the
 * mesh was bound without renumbering): entry i is the caller id of the i-th
 * bit of fa_frame_download_packed's vertex_mask.  Changes only with
 * fa_set_mesh.  Synchronises `stream`. */
int fa_vertex_order(fa_ctx *ctx, int32_t *out, void *stream);

/* Number of kernels the last fa_frame_launch enqueued (benchmark accounting). */
int fa_last_launch_count(fa_ctx *ctx);

/* Per-stage device times (ms, CUDA events on the frame stream) of the last
 * frame launched with params.profile = 1; returns the stage count (<= max).
 * Synchronises the stream.  fa_stage_name(i) names stage i. */
int fa_stage_times(fa_ctx *ctx, float *ms_out, int max, void *stream);
const char *fa_stage_name(int i);

/* Work-queue counters of the last finished frame (diagnostics; valid after
 * fa_frame_finish): [small records, large records, clipped triangles,
 * generic setups, large-raster tiles, visible, charts, screen fragments,
 * 32-triangle clusters the setup processed (the rest culled as a whole)].
 * Returns the number written (<= max). */
int fa_frame_counters(fa_ctx *ctx, int64_t *out, int max);

#ifdef __cplusplus
}
#endif
#endif /* FASTATLAS_H */
