// fa_raster.cu — projection, depth pre-pass and visibility pass on sm_100a.
//
// Reference: charts.py:269-313 (depth_prepass / mark_visible) over the
// per-triangle clip + raster of charts.py:160-266.
//
// Work split (load balance): k_raster_setup builds one exact setup per
// triangle from the per-vertex screen records and emits 96-byte records —
// small windows (<= FA_SMALL_PX pixels) for the warp-cooperative sampler,
// large ones with their 16x8 tiles for a warp per tile — and lists the
// clipped triangles for a warp each (k_raster_clipped).  The depth buffer
// holds order-preserving u64 keys of the float64 NDC depth, so the per-pixel
// minimum is one fire-and-forget 64-bit RED.MIN in L2; a second RED keeps the
// pixel winner.  Pass 2 (visibility) skips the winners, rejects occluded
// records with an 8x8 hierarchical Z, and replays the stored records.
// DESIGN.md §2.1 has the full picture.
#define FA_TU_ID 2  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"
#include "fa_raster.cuh"

#ifndef FA_VIS_WARP_PX
#define FA_VIS_WARP_PX 48  // pass-2 survivors with larger windows are sampled a warp per record
#endif
#ifndef FA_SMALL_PX
#define FA_SMALL_PX 96
#endif
#define TILE_W 16
#define TILE_H 8

#ifdef FA_COOP_STATS
// debug builds only (tools/debug_coopstats.py): small records by window size
// (<=4, <=9, <=16, <=48, more) x (no / some covered sample)
__device__ unsigned long long g_coop_stats[5][2];
extern "C" void fa_debug_coop_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_coop_stats, sizeof(g_coop_stats));
    if (reset) {
        unsigned long long z[10] = {};
        cudaMemcpyToSymbol(g_coop_stats, z, sizeof(z));
    }
}
#endif
#ifdef FA_HIZ_STATS
// debug build only: [small records rejected by the hierarchical Z, small
// records sampled, tiles tested, tiles rejected, tiles skipped (visible)]
__device__ unsigned long long g_hiz_stats[6];
extern "C" void fa_debug_hiz_stats(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_hiz_stats, sizeof(g_hiz_stats));
    unsigned long long z[6] = {0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_hiz_stats, z, sizeof(z));
}
#endif

// Pass-1 depth write.  Besides the exact order-preserving key minimum, when a
// winner buffer is bound it keeps min((key & ~0xFFFFFF) | t): the triangle it
// names at a pixel has a key equal to the final minimum in its top 40 bits
// (sign, exponent, 28 mantissa bits), i.e. a depth within 2^-27 relative of
// it — far inside the visibility slack of 1e-6 (charts.py:309-311), so that
// triangle is visible and k_depth_hiz can flag it without a second raster.
// `check` skips both atomics when the stored key is already <= key: the
// triangle that first lowers a pixel to its final key always executes them.
#define FA_WID_BITS 24
__device__ __forceinline__ void depth_min(unsigned long long* __restrict__ depth, unsigned long long* __restrict__ wid,
                                          long long off, unsigned long long key, int t, bool check) {
    unsigned long long* d = depth + off;
    if (check && !(key < *d)) return;
    atomicMin(d, key);
    if (wid) atomicMin(wid + off, (key & ~((1ull << FA_WID_BITS) - 1)) | (unsigned long long)t);
}

// warp-aggregated single-slot append among the currently active lanes
__device__ __forceinline__ int active_append1(int* counter) {
    unsigned mask = __activemask();
    int lane = lane_id();
    int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(mask & ((1u << lane) - 1u));
}

// ---- frame init: projection + buffer clears ------------------------------
// the live-cluster list: one thread per cluster, warp-aggregated appends.
// `vc` (shared memory) holds the frame's view constants, uploaded with the
// camera (compute_view_consts on the host).
__device__ __forceinline__ void cull_clusters(const fa_view_consts& vc, const fa_cull_args& cu, long long t0,
                                              long long stride) {
    const long long n_pad = ((long long)cu.n_clusters + 31) & ~31ll;
    for (long long c = t0; c < n_pad; c += stride) {
        const bool live = c < cu.n_clusters && !cluster_culled(cu.clusters[c], vc, cu.cull != 0);
        const unsigned mk = __ballot_sync(0xffffffffu, live);
        int base = 0;
        if (lane_id() == 0 && mk) base = atomicAdd(&cu.st->n_live, __popc(mk));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (live) cu.live[base + __popc(mk & ((1u << lane_id()) - 1u))] = (int)c;
    }
}

__device__ __forceinline__ void load_view_consts(const double* vp_dev, fa_view_consts* s_vc) {
    const double* src = vp_dev + FA_VC_OFF;
    double* dst = reinterpret_cast<double*>(s_vc);
    for (int i = threadIdx.x; i < (int)(sizeof(fa_view_consts) / 8); i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
}

// Blocks [0, cull_blocks) cull the clusters (k_cluster_cull's work, so the
// culling runs beside the projection with no extra launch or join); the rest
// project the vertices / clear.
__global__ void __launch_bounds__(256, 4) k_frame_init(const double* __restrict__ pos, int V,
                                                       const double* __restrict__ vp_dev,
                                                       double4* __restrict__ clip, double4* __restrict__ scr, int W,
                                                       int H, int* __restrict__ vmin,
                                                       unsigned long long* __restrict__ depth,
                                                       unsigned long long* __restrict__ wid, long long npx,
                                                       unsigned int* __restrict__ flags32, int nflag32,
                                                       double2* __restrict__ ndc2, fa_cull_args cu, int cull_blocks) {
    FA_PDL_PROLOGUE();
    if ((int)blockIdx.x < cull_blocks) {
        __shared__ fa_view_consts s_vc;
        load_view_consts(vp_dev, &s_vc);
        cull_clusters(s_vc, cu, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)cull_blocks * blockDim.x);
        return;
    }
    long long stride = (long long)(gridDim.x - cull_blocks) * blockDim.x;
    long long i0 = (long long)(blockIdx.x - cull_blocks) * blockDim.x + threadIdx.x;
    double m[16];
#pragma unroll
    for (int i = 0; i < 16; i++) m[i] = V > 0 ? __ldg(vp_dev + i) : 0.0;  // (clear-only launches pass no matrix)
    for (long long v = i0; v < V; v += stride) {
        double x = pos[3 * v], y = pos[3 * v + 1], z = pos[3 * v + 2];
        double4 c = project_point(x, y, z, m);
        if (clip) clip[v] = c;
        if (ndc2) ndc2[v] = vertex_ndc(c);
        if (scr) scr[v] = vertex_screen(c, W, H);
        if (vmin) vmin[v] = 0x7fffffff;
    }
    if (depth) {
        ulonglong2* d2 = reinterpret_cast<ulonglong2*>(depth);
        long long n2 = npx >> 1;
        for (long long i = i0; i < n2; i += stride) d2[i] = make_ulonglong2(FA_KEY_POS_INF, FA_KEY_POS_INF);
        if ((npx & 1) && i0 == 0) depth[npx - 1] = FA_KEY_POS_INF;
    }
    if (wid) {
        ulonglong2* w2 = reinterpret_cast<ulonglong2*>(wid);
        long long n2 = npx >> 1;
        for (long long i = i0; i < n2; i += stride) w2[i] = make_ulonglong2(~0ull, ~0ull);
        if ((npx & 1) && i0 == 0) wid[npx - 1] = ~0ull;
    }
    if (flags32)
        for (long long i = i0; i < nflag32; i += stride) flags32[i] = 0u;
}

// The setup's live clusters: those not culled as a whole (cluster_culled:
// outside the frustum or facing away -> no samples).  Their order does not
// matter (every output is keyed by triangle id).  Independent of the
// projection, so it runs beside it.
__global__ void __launch_bounds__(256) k_cluster_cull(const double* __restrict__ vp_dev, int W, int H, fa_cull_args cu) {
    FA_PDL_PROLOGUE();
    __shared__ fa_view_consts s_vc;
    load_view_consts(vp_dev, &s_vc);
    cull_clusters(s_vc, cu, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
}

void fa_launch_cluster_cull(const double* vp, int W, int H, const fa_cull_args& cu, cudaStream_t s) {
    if (!cu.clusters) return;
    fa_launch(k_cluster_cull, fa_grid(cu.n_clusters, 256, FA_NUM_SMS), 256, 0, s, vp, W, H, cu);
}

// keys -> float64 depth (debug / standalone depth_prepass output)
__global__ void k_decode_depth(const unsigned long long* __restrict__ keys, double* __restrict__ out, long long n) {
    FA_PDL_PROLOGUE();
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = key_f64(keys[i]);
}

// float64 depth -> keys (standalone mark_visible input)
__global__ void k_encode_depth(const double* __restrict__ in, unsigned long long* __restrict__ keys, long long n) {
    FA_PDL_PROLOGUE();
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) keys[i] = f64_key(in[i]);
}

// ---- pass 1: setup + record / tile enqueue --------------------------------
// One warp per 32 consecutive triangles (block-uniform loop; appends are
// aggregated per block step).  Per triangle: 3 index loads, 3 gathers of
// the per-vertex screen records, the exact cull / bbox / edge / plane setup
// (tri_setup3s), then
//   small unclipped  -> 96-byte record at the front of `recs` (k_small_coop),
//   large unclipped  -> record at the back of `recs` + its 16x8 tiles, whose
//                       descriptors the warp writes together,
//   anything else    -> index into `clip_list` for k_raster_clipped.
// Nothing is rasterized here, so no lane waits on another's pixels.
#ifndef SETUP_WARPS
#define SETUP_WARPS 8
#endif
#ifndef SETUP_DEFER
#define SETUP_DEFER 1
#endif
#ifndef SETUP_MIN_BLOCKS
#define SETUP_MIN_BLOCKS (32 / SETUP_WARPS)
#endif
__global__ void __launch_bounds__(SETUP_WARPS * 32, SETUP_MIN_BLOCKS) k_raster_setup(const double4* __restrict__ scr,
                                                      const int* __restrict__ tris,
                                                      int T, int W, int H, int cull,
                                                      SmallRec* __restrict__ recs, int* __restrict__ clip_list,
                                                      int4* __restrict__ tiles, int max_tiles,
                                                      fa_dstat* __restrict__ st, fa_setup_order ord) {
    FA_PDL_PROLOGUE();
    // per-warp counts -> per-warp bases; one atomic per counter per block step
    // (a same-address atomic per warp serialises ~30K times in the L2)
    __shared__ int s_cnt[2][4][SETUP_WARPS];
    __shared__ int s_base[2][4][SETUP_WARPS];
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const bool rec_ok = W <= 32767 && H <= 32767;
    const unsigned lt_mask = (1u << lane) - 1u;
    // the next step's vertex indices are loaded one step ahead, so each step
    // waits for one round trip (the screen-record gathers), not two
    // slots walk the setup order (fa_mesh.cu: Morton order of the centroids,
    // 32-slot clusters); t is the slot's triangle id
    // With a live-cluster list (k_frame_init: clusters outside the frustum
    // or facing away dropped) a warp step is one live cluster; otherwise 32
    // consecutive slots.  t is the slot's triangle id.
    const int* ts = ord.tris_sorted ? ord.tris_sorted : tris;
    const int* live = ord.live;
    // warp items of 32 slots: 32 / FA_CLUSTER live clusters, or 32 consecutive slots
    constexpr int CPW = 32 / FA_CLUSTER;
    const int n_items = live ? (*ord.n_live + CPW - 1) / CPW : (T + 31) >> 5;
    const int n_live_c = live ? *ord.n_live : 0;
    const int istep = gridDim.x * SETUP_WARPS;
    auto slot_of = [&](int item) -> int {
        if (item >= n_items) return T;
        if (!live) return item * 32 + lane;
        const int ci = item * CPW + lane / FA_CLUSTER;
        return ci < n_live_c ? __ldg(live + ci) * FA_CLUSTER + (lane % FA_CLUSTER) : T;
    };
    const int4* __restrict__ s4 = ord.slots4;
    auto load_slot = [&](int sl, int& a, int& b, int& c, int& id) {
        if (s4) {
            const int4 q = __ldg(s4 + sl);
            a = q.x, b = q.y, c = q.z, id = q.w;
        } else {
            a = __ldg(ts + 3 * sl), b = __ldg(ts + 3 * sl + 1), c = __ldg(ts + 3 * sl + 2);
            id = ord.tperm ? __ldg(ord.tperm + sl) : sl;
        }
    };
    int nslot = slot_of(blockIdx.x * SETUP_WARPS + warp);
    int na = 0, nb = 0, nc = 0, nt_id = T;
    if (nslot < T) load_slot(nslot, na, nb, nc, nt_id);
#if SETUP_DEFER
    // deferred publication (see the loop): the records of a step wait in
    // shared memory until the next step's barrier has published their bases
    __shared__ SmallRec s_stage[SETUP_WARPS][32];
    static_assert(SETUP_WARPS * 32 * sizeof(SmallRec) <= 40 * 1024,
                  "SETUP_DEFER stages 3 KB per warp in static shared memory: at most 13 warps per block");
    int step = 0, resv = 0;
    unsigned pm1 = 0, pm2 = 0, pm3 = 0;
    int p_kind = 0, p_t = 0, p_nt = 0, p_incl = 0, p_total = 0;
    // leader thread c: per-warp bases of counter c for the step of parity q
    auto publish_bases = [&](int q, int b) {
        const int c = threadIdx.x;
        for (int w = 0; w < SETUP_WARPS; w++) {
            s_base[q][c][w] = b;
            b += s_cnt[q][c][w];
        }
    };
    // write out the warp's staged step (parity q): small records to
    // [sb, sb + n1), large ones downward from T - lb, their ids, clip list
    // entries and tile descriptors
    auto flush = [&](int q) {
        const int sb = s_base[q][0][warp], lb = s_base[q][1][warp], cb = s_base[q][2][warp],
                  tb = s_base[q][3][warp];
        const int n1 = __popc(pm1), n2 = __popc(pm2);
        const int4* src = reinterpret_cast<const int4*>(s_stage[warp]);
        constexpr int C16 = sizeof(SmallRec) / 16;
        for (int j = lane; j < (n1 + n2) * C16; j += 32) {
            const int r = j / C16, c = j - r * C16;
            SmallRec* dst = r < n1 ? recs + sb + r : recs + (T - (lb + (r - n1)));
            reinterpret_cast<int4*>(dst)[c] = src[j];
        }
        if (p_kind == 1) small_ids(recs, T)[sb + __popc(pm1 & lt_mask)] = p_t;
        if (p_kind == 3) clip_list[cb + __popc(pm3 & lt_mask)] = p_t;
        if (pm2) {
            const int ri = T - (lb + __popc(pm2 & lt_mask));
            if (tb + p_total > max_tiles && lane == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
            unsigned m = pm2;
            while (m) {
                int srcl = __ffs(m) - 1;
                m &= m - 1;
                int r_src = __shfl_sync(0xffffffffu, ri, srcl);
                int n_src = __shfl_sync(0xffffffffu, p_nt, srcl);
                int t_src = __shfl_sync(0xffffffffu, p_t, srcl);
                int e_src = tb + __shfl_sync(0xffffffffu, p_incl, srcl) - n_src;
                for (int k = lane; k < n_src; k += 32)
                    if (e_src + k < max_tiles) tiles[e_src + k] = make_int4(r_src, k, t_src, 0);
            }
        }
    };
#endif
    for (int ibase = blockIdx.x * SETUP_WARPS; ibase < n_items; ibase += istep) {
        const int slot = nslot;
        const int ia = na, ib = nb, ic = nc, t = nt_id;
        nslot = slot_of(ibase + istep + warp);
        if (nslot < T) load_slot(nslot, na, nb, nc, nt_id);
        Setup3 f;
        int kind = 0;  // 0 none, 1 small record, 2 large record, 3 generic path
        int nt = 0;
        if (slot < T) {
            int r3 = tri_setup3s(scr, ia, ib, ic, W, H, cull != 0, f);
            if (r3 == 2 || (r3 == 1 && !rec_ok)) {
                kind = 3;
            } else if (r3 == 1) {
                int bw = f.max_x - f.min_x + 1, bh = f.max_y - f.min_y + 1;
                if (bw * bh <= FA_SMALL_PX) {
                    kind = 1;
                } else {
                    kind = 2;
                    nt = ((bw + TILE_W - 1) / TILE_W) * ((bh + TILE_H - 1) / TILE_H);
                }
            }
        }
        const unsigned m1 = __ballot_sync(0xffffffffu, kind == 1);
        const unsigned m2 = __ballot_sync(0xffffffffu, kind == 2);
        const unsigned m3 = __ballot_sync(0xffffffffu, kind == 3);
        int incl = nt;  // inclusive scan of the warp's tile counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
#if SETUP_DEFER
        // One barrier per step.  The counts of this step are published; the
        // leader threads then (1) write the PREVIOUS step's per-warp bases
        // from the global reservation they issued one step ago -- so the
        // atomic's round trip overlaps a whole step of setup work -- and (2)
        // issue this step's reservation.  Each warp stages this step's
        // records in shared memory and writes them out (coalesced) one step
        // later, once their bases are known.
        const int par = step & 1;
        if (lane == 0) {
            s_cnt[par][0][warp] = __popc(m1);
            s_cnt[par][1][warp] = __popc(m2);
            s_cnt[par][2][warp] = __popc(m3);
            s_cnt[par][3][warp] = total;
        }
        if (step > 0 && threadIdx.x < 4) publish_bases(par ^ 1, resv);
        __syncthreads();
        if (threadIdx.x < 4) {
            const int c = threadIdx.x;
            int sum = 0;
            for (int w = 0; w < SETUP_WARPS; w++) sum += s_cnt[par][c][w];
            int* ctr = c == 0 ? &st->n_small3 : c == 1 ? &st->n_large3 : c == 2 ? &st->n_clip : &st->n_tiles;
            resv = sum ? atomicAdd(ctr, sum) : 0;  // consumed at the next step's publish
        }
        if (step > 0) flush(par ^ 1);
        // stage this step (the flush above read the staging area: same warp)
        __syncwarp();
        if (kind == 1) store_rec(f, t, s_stage[warp] + __popc(m1 & lt_mask));
        else if (kind == 2) store_rec(f, t, s_stage[warp] + __popc(m1) + __popc(m2 & lt_mask));
        __syncwarp();
        pm1 = m1, pm2 = m2, pm3 = m3, p_kind = kind, p_t = t, p_nt = nt, p_incl = incl, p_total = total;
        step++;
    }
    if (step > 0) {
        if (threadIdx.x < 4) publish_bases((step - 1) & 1, resv);
        __syncthreads();
        flush((step - 1) & 1);
    }
#else
        if (lane == 0) {
            s_cnt[0][0][warp] = __popc(m1);
            s_cnt[0][1][warp] = __popc(m2);
            s_cnt[0][2][warp] = __popc(m3);
            s_cnt[0][3][warp] = total;
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            const int c = threadIdx.x;
            int sum = 0;
            for (int w = 0; w < SETUP_WARPS; w++) sum += s_cnt[0][c][w];
            int* ctr = c == 0 ? &st->n_small3 : c == 1 ? &st->n_large3 : c == 2 ? &st->n_clip : &st->n_tiles;
            int b = sum ? atomicAdd(ctr, sum) : 0;
            for (int w = 0; w < SETUP_WARPS; w++) {
                s_base[0][c][w] = b;
                b += s_cnt[0][c][w];
            }
        }
        __syncthreads();
        if (m1 && kind == 1) {
            const int idx = s_base[0][0][warp] + __popc(m1 & lt_mask);
            store_rec(f, t, recs + idx);
            small_ids(recs, T)[idx] = t;  // lets the visibility filter skip flagged records unread
        }
        if (m3 && kind == 3) clip_list[s_base[0][2][warp] + __popc(m3 & lt_mask)] = t;
        if (m2) {
            // large records are stored downward from index T (small + large
            // records <= T, so the two ends never meet)
            const int rb = s_base[0][1][warp], tb = s_base[0][3][warp];
            int ri = T - (rb + __popc(m2 & lt_mask));
            if (kind == 2) store_rec(f, t, recs + ri);
            if (tb + total > max_tiles && lane == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
            // the warp writes every large lane's tile descriptors, coalesced
            unsigned m = m2;
            while (m) {
                int src = __ffs(m) - 1;
                m &= m - 1;
                int r_src = __shfl_sync(0xffffffffu, ri, src);
                int n_src = __shfl_sync(0xffffffffu, nt, src);
                int t_src = __shfl_sync(0xffffffffu, t, src);
                int e_src = tb + __shfl_sync(0xffffffffu, incl, src) - n_src;
                for (int k = lane; k < n_src; k += 32)
                    if (e_src + k < max_tiles) tiles[e_src + k] = make_int4(r_src, k, t_src, 0);
            }
        }
    }
#endif
}

// ---- pass 1, generic path: clipped polygons (and oversize screens) --------
// One warp per listed triangle: the warp clips (tri_setup_warp, a vertex per
// lane) and builds the TriSetup in shared memory, then stores it to the `large`
// queue and either samples the whole window (<= FA_SMALL_PX pixels, depth
// pass only) or writes the descriptors of its 16x8 tiles (negative ids).
// The visibility pass finds every stored setup through the queue.
template <bool WRITE_DEPTH>
__global__ void __launch_bounds__(256) k_raster_clipped(const ClipSrc clip, const int* __restrict__ tris,
                                                        int W, int H, int cull, const int* __restrict__ clip_list,
                                                        unsigned long long* __restrict__ depth,
                                                        unsigned long long* __restrict__ wid,
                                                        TriSetup* __restrict__ large, int max_large,
                                                        int4* __restrict__ tiles, int max_tiles,
                                                        fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    __shared__ TriSetup sm[8];
    __shared__ ClipScratch cs[8];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int nwarps = gridDim.x * 8;
    const int n = st->n_clip;
    for (int w = blockIdx.x * 8 + warp; w < n; w += nwarps) {
        const int t = clip_list[w];
        __syncwarp();
        const int r = tri_setup_warp(clip, tris, t, W, H, cull != 0, sm[warp], cs[warp]);
        if (r < 0) {
            if (lane == 0) atomicOr(&st->flags, FA_DFLAG_POLY_OVERFLOW);
            continue;
        }
        if (r == 0) continue;
        const TriSetup& s = sm[warp];
        int slot = 0;
        if (lane == 0) slot = atomicAdd(&st->n_large, 1);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= max_large) {
            if (lane == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
            continue;
        }
        {
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&s);
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(large + slot);
            for (int i = lane; i < (int)(sizeof(TriSetup) / 8); i += 32) dst[i] = src[i];
        }
        const int bw = s.max_x - s.min_x + 1, bh = s.max_y - s.min_y + 1;
        if (bw * bh <= FA_SMALL_PX) {
            if (WRITE_DEPTH) {
                for (int k = lane; k < bw * bh; k += 32) {
                    int dy = k / bw;
                    int iy = s.min_y + dy, ix = s.min_x + (k - dy * bw);
                    double px = (double)ix + 0.5, py = (double)iy + 0.5;
                    if (!sample_inside(s, px, py)) continue;
                    depth_min(depth, wid, (long long)iy * W + ix, f64_key(sample_depth(s, px, py)), t, true);
                }
            }
        } else {
            // tiles of generic setups are stored downward from max_tiles - 1
            // (k_raster_setup's unclipped tiles fill the front, and were all
            // counted before this kernel started)
            const int nt = ((bw + TILE_W - 1) / TILE_W) * ((bh + TILE_H - 1) / TILE_H);
            const int room = max_tiles - min(st->n_tiles, max_tiles);
            int base = 0;
            if (lane == 0) base = atomicAdd(&st->n_tiles_clip, nt);
            base = __shfl_sync(0xffffffffu, base, 0);
            // on overflow write the part that fits and flag the frame; the
            // host grows the queue and reruns
            if (base + nt > room && lane == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
            for (int k = lane; k < nt; k += 32)
                if (base + k < room) tiles[max_tiles - 1 - (base + k)] = make_int4(-slot - 1, k, t, 0);
        }
    }
}

// One pass over the final depth keys, one thread per 8x8 pixel tile:
//  * screen_fragments = #finite depth samples (cli.py:390), and
//  * the hierarchical-Z buffer for the visibility pass: per tile the largest
//    key in [key(-inf), key(+inf)) — +inf (empty) and NaN pixels can never make
//    a sample pass (charts.py:309-311), so they are left out — or 0 when the
//    tile has none (nothing can be covered there).
//  * with a winner buffer (depth_min), the flag of every pixel's winner at a
//    finite final depth — those triangles are visible (see depth_min), so the
//    visibility pass skips them.  (At -inf the slack test is NaN: no flag.)
__global__ void __launch_bounds__(256) k_depth_hiz(const unsigned long long* __restrict__ depth,
                                                   const unsigned long long* __restrict__ wid, int W, int H,
                                                   unsigned long long* __restrict__ hiz, int htx, int hty,
                                                   unsigned char* __restrict__ flags, fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    // one thread per pixel column of a tile row (8 pixels tall): the loads of
    // a warp are 32 consecutive pixels of one image row; 8 consecutive lanes
    // form one tile and reduce its maximum with shuffles
    long long c = 0;
    const int rowlen = htx * FA_HIZ;
    const int n = rowlen * hty;
    const int n_pad = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += gridDim.x * blockDim.x) {
        const int ty = i / rowlen, x = i - ty * rowlen;
        const int y0 = ty * FA_HIZ, y1 = min(y0 + FA_HIZ, H);
        unsigned long long mx = 0;
        if (i < n && x < W) {
            // all loads of the strip first (one round trip), then the tests
            unsigned long long dv[FA_HIZ], wv[FA_HIZ];
#pragma unroll
            for (int k = 0; k < FA_HIZ; k++) {
                const long long p = (long long)(y0 + k) * W + x;
                const bool in = y0 + k < y1;
                dv[k] = in ? depth[p] : FA_KEY_POS_INF;
                wv[k] = (in && wid) ? wid[p] : ~0ull;
            }
            int last = -1;
#pragma unroll
            for (int k = 0; k < FA_HIZ; k++) {
                const unsigned long long v = dv[k];
                bool fin = v > FA_KEY_NEG_INF && v < FA_KEY_POS_INF;
                c += fin;
                if (v >= FA_KEY_NEG_INF && v < FA_KEY_POS_INF && v > mx) mx = v;
                if (wid && fin) {
                    // the winner is only trusted when its truncated key is the
                    // final key's (so any subset of writers may skip the RED)
                    const unsigned long long hi = ~((1ull << FA_WID_BITS) - 1);
                    if ((wv[k] & hi) == (v & hi)) {
                        int id = (int)(wv[k] & ~hi);
                        if (id != last) flags[id] = 1;
                        last = id;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 1; o < FA_HIZ; o <<= 1) {
            unsigned long long m = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = m > mx ? m : mx;
        }
        if (i < n && (x & (FA_HIZ - 1)) == 0) hiz[ty * htx + x / FA_HIZ] = mx;
    }
    c = warp_sum(c);
    if (st && lane_id() == 0 && c) atomicAdd((unsigned long long*)&st->screen_fragments, (unsigned long long)c);
}

// copy one TriSetup into warp-private shared memory
__device__ __forceinline__ void load_setup_warp(const TriSetup* __restrict__ g, TriSetup* sm) {
    const int nwords = sizeof(TriSetup) / 8;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(g);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(sm);
    for (int i = lane_id(); i < nwords; i += 32) dst[i] = __ldg(src + i);
    __syncwarp();
}

// tile (ti) of a bbox -> this lane's pixel column x and first row y0
// (16 columns x 2 rows per step; 4 steps cover the 16x8 tile)
__device__ __forceinline__ void tile_lane_origin(int min_x, int max_x, int min_y, int ti, int& x, int& y0) {
    int tx = (max_x - min_x + 1 + TILE_W - 1) / TILE_W;
    int lane = lane_id();
    x = min_x + (ti % tx) * TILE_W + (lane & 15);
    y0 = min_y + (ti / tx) * TILE_H + (lane >> 4);
}


// ---- pass 1 large: one warp per 16x8 tile --------------------------------
// Tile records: x >= 0 indexes a compact unclipped record (every lane loads
// the same 96 bytes — one broadcast transaction per LDG — and rebuilds the
// edge functions in registers); x < 0 is a generic clipped setup, staged in
// warp-private shared memory.
__global__ void __launch_bounds__(256) k_raster_depth_tiles(const SmallRec* __restrict__ recs,
                                                            const TriSetup* __restrict__ large,
                                                            const int4* __restrict__ tiles, int W,
                                                            unsigned long long* __restrict__ depth,
                                                            unsigned long long* __restrict__ wid,
                                                            fa_dstat* __restrict__ st, int max_tiles, int check,
                                                            int tile_wid, int from_back) {
    FA_PDL_PROLOGUE();
    __shared__ TriSetup sm[8];
    int warp = threadIdx.x >> 5, lane = lane_id();
    int nwarps = gridDim.x * 8;
    // front: the unclipped tiles of k_raster_setup; back: the clipped
    // (generic) setups' tiles of k_raster_clipped, stored downward
    const int n_front = min(st->n_tiles, max_tiles);
    const int n_tiles = from_back ? min(st->n_tiles_clip, max_tiles - n_front) : n_front;
    const int4* tl = from_back ? tiles + (max_tiles - 1) : tiles;
    const int dir = from_back ? -1 : 1;
    // Pipeline: the next tile's 96-byte record streams into shared memory
    // (cp.async, lanes 0-5) while this tile samples, and descriptors are read
    // two steps ahead, so a step waits for neither.
    __shared__ __align__(16) SmallRec srec[8][2];
    const int w0 = (int)blockIdx.x * 8 + warp;
    int4 cur = make_int4(-1, 0, 0, 0), nxt = make_int4(-1, 0, 0, 0);
    if (w0 < n_tiles) cur = tl[dir * w0];
    if (w0 + nwarps < n_tiles) nxt = tl[dir * (w0 + nwarps)];
    auto fetch = [&](const int4& d, int b) {
        if (d.x >= 0 && lane < (int)(sizeof(SmallRec) / 16))
            cp_async16(reinterpret_cast<char*>(&srec[warp][b]) + 16 * lane,
                       reinterpret_cast<const char*>(recs + d.x) + 16 * lane);
    };
    if (w0 < n_tiles) fetch(cur, 0);
    cp_async_commit();
    int buf = 0;
    for (int w = w0; w < n_tiles; w += nwarps, buf ^= 1) {
        int4 rec = cur;
        cur = nxt;
        if (w + 2 * nwarps < n_tiles) nxt = tl[dir * (w + 2 * nwarps)];
        if (w + nwarps < n_tiles) fetch(cur, buf ^ 1);
        cp_async_commit();
        cp_async_wait1();
        __syncwarp();
        if (rec.x >= 0) {
            Setup3 f;
            int t;
            load_rec(&srec[warp][buf], f, t);
            int x, y0;
            tile_lane_origin(f.min_x, f.max_x, f.min_y, rec.y, x, y0);
            if (x <= f.max_x) {
                const ColTerms ct = col_terms(f, (double)x + 0.5);
#pragma unroll
                for (int k = 0; k < TILE_H / 2; k++) {
                    int y = y0 + 2 * k;
                    if (y > f.max_y) break;
                    double py = (double)y + 0.5;
                    if (!inside_col(f, ct, py)) continue;
                    depth_min(depth, tile_wid ? wid : nullptr, (long long)y * W + x, f64_key(depth_col(f, ct, py)), t,
                              check != 0);
                }
            }
            __syncwarp();  // this buffer is refilled by the next step's prefetch
            continue;
        }
        rec.x = -rec.x - 1;
        __syncwarp();
        load_setup_warp(large + rec.x, &sm[warp]);
        const TriSetup& s = sm[warp];
        int bw = s.max_x - s.min_x + 1;
        int tx = (bw + TILE_W - 1) / TILE_W;
        int x = s.min_x + (rec.y % tx) * TILE_W + (lane & 15);
        int y0 = s.min_y + (rec.y / tx) * TILE_H + (lane >> 4);
        if (x <= s.max_x) {
            double px = (double)x + 0.5;
            for (int k = 0; k < TILE_H / 2; k++) {
                int y = y0 + 2 * k;
                if (y > s.max_y) break;
                double py = (double)y + 0.5;
                if (!sample_inside(s, px, py)) continue;
                depth_min(depth, wid, (long long)y * W + x, f64_key(sample_depth(s, px, py)), s.tri, check != 0);
            }
        }
        __syncwarp();
    }
}

// ---- small unclipped triangles: warp-cooperative sampling ------------------
// A warp stages 32 records in shared memory, prefix-sums their window ROW
// counts, and gives every lane one contiguous, equal chunk of the combined
// rows, so per-triangle size differences no longer diverge the warp.  Per row
// only the conservative span (row_span) is tested exactly: a small record's
// window averages ~20 samples for ~1.5 covered ones.  Depth pass only
// (RED.MIN.64 per covered sample).
#define COOP_WARPS 4
#ifndef COOP_GRID_MULT
#define COOP_GRID_MULT 5  // one wave: the resident CTAs loop (persistent)
#endif
#ifndef COOP_UNROLL
#define COOP_UNROLL 2  // samples of a row span in flight per lane
#endif
#ifndef COOP_MIN_BLOCKS
#define COOP_MIN_BLOCKS 5
#endif
struct __align__(16) CoopWarp {
    SmallRec rec[2][32];  // double buffer: the next 32 records stream in (one bulk copy) during the current ones
    unsigned long long bar[2];  // bulk-copy completion, one mbarrier per buffer
    int prefix[33];
    SpanEdges se[32];     // each record's span reciprocals, computed once by the lane that owns it
};


// records [base, base + 32) (clipped to n) -> dst: one bulk copy by lane 0
__device__ __forceinline__ void coop_issue(const SmallRec* __restrict__ recs, int base, int n, SmallRec* dst,
                                           unsigned long long* bar) {
    if (lane_id() == 0 && base < n)
        bulk_g2s(dst, recs + base, (unsigned)(min(32, n - base) * sizeof(SmallRec)), bar);
}

__global__ void __launch_bounds__(COOP_WARPS * 32, COOP_MIN_BLOCKS) k_small_coop(const SmallRec* __restrict__ recs, int W,
                                                                   unsigned long long* __restrict__ depth,
                                                                   unsigned long long* __restrict__ wid,
                                                                   const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    __shared__ CoopWarp sh[COOP_WARPS];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    CoopWarp& cw = sh[warp];
    const int n = st->n_small3;
#ifdef FA_COOP_STATS
    __shared__ int cw_cov[COOP_WARPS][32];
    cw_cov[warp][lane] = 0;
    __syncwarp();
#endif
    const int stride = gridDim.x * COOP_WARPS * 32;
    int base = ((int)blockIdx.x * COOP_WARPS + warp) * 32;
    int buf = 0;
    if (lane == 0) {
        mbar_init(&cw.bar[0], 1);
        mbar_init(&cw.bar[1], 1);
        fence_async_shared();
    }
    __syncwarp();
    coop_issue(recs, base, n, cw.rec[0], &cw.bar[0]);
    for (int it = 0; base < n; base += stride, buf ^= 1, it++) {
        coop_issue(recs, base + stride, n, cw.rec[buf ^ 1], &cw.bar[buf ^ 1]);
        mbar_wait(&cw.bar[buf], (it >> 1) & 1);  // use it>>1 of this buffer
        const SmallRec* rb = cw.rec[buf];
        const int cnt = min(32, n - base);
        int np = 0;
        if (lane < cnt) {
            np = rb[lane].max_y - rb[lane].min_y + 1;
            Setup3 fo;
            int to;
            load_rec(&rb[lane], fo, to);
            cw.se[lane] = span_edges(fo);
        }
        int incl = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        cw.prefix[lane + 1] = incl;
        if (lane == 0) cw.prefix[0] = 0;
        __syncwarp();
        const int S = __shfl_sync(0xffffffffu, incl, 31);
        const int chunk = (S + 31) >> 5;
        int s = lane * chunk;
        const int s_end = min(S, s + chunk);
        if (s < s_end) {
            // record holding row s: largest r with prefix[r] <= s
            int lo = 0, hi = cnt - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (cw.prefix[mid] <= s) lo = mid; else hi = mid - 1;
            }
            int r = lo;
            Setup3 f;
            int t;
            load_rec(&rb[r], f, t);
            SpanEdges se = cw.se[r];
            int pe = cw.prefix[r + 1];
            int iy = f.min_y + (s - cw.prefix[r]);
            for (; s < s_end; s++, iy++) {
                if (s >= pe) {
                    do {
                        r++;
                        pe = cw.prefix[r + 1];
                    } while (s >= pe);
                    load_rec(&rb[r], f, t);
                    se = cw.se[r];
                    iy = f.min_y;
                }
                const RowTerms rt = row_terms(f, (double)iy + 0.5);
                int xa, xb, ca, cb;
                row_span_cert(f, rt, se, xa, xb, ca, cb);
                const long long rowoff = (long long)iy * W;
                double px = (double)xa + 0.5;  // px += 1 below is exact (half-integers < 2^52)
                constexpr int kUnroll = COOP_UNROLL;
#pragma unroll kUnroll
                for (int ix = xa; ix <= xb; ix++, px += 1.0) {
                    // the edge test only near a crossing (row_span_cert)
                    const double z = depth_row(f, rt, px);
                    if ((ix >= ca && ix <= cb) || inside_row(f, rt, px)) {
                        depth_min(depth, wid, rowoff + ix, f64_key(z), t, false);
#ifdef FA_COOP_STATS
                        cw_cov[warp][r] = 1;
#endif
                    }
                }
            }
        }
        __syncwarp();
#ifdef FA_COOP_STATS
        if (lane < cnt) {
            const SmallRec& q = rb[lane];
            const int area = (q.max_x - q.min_x + 1) * (q.max_y - q.min_y + 1);
            const int bucket = area <= 4 ? 0 : area <= 9 ? 1 : area <= 16 ? 2 : area <= 48 ? 3 : 4;
            atomicAdd(&g_coop_stats[bucket][cw_cov[warp][lane]], 1ull);
            cw_cov[warp][lane] = 0;
        }
        __syncwarp();
#endif
    }
}

// ---- pass 2 small: filter, then sample the survivors densely ---------------
// One thread per stored record.  One round trip decides most records without
// sampling: the flag (set by k_depth_hiz for the pixel winners of pass 1) and
// the record's 8x8 hierarchical-Z tiles (when its window spans at most 2x2 of
// them).  The ~20% that survive are appended (one atomic per block step) to a
// queue that k_vis_small_sample walks one thread per survivor, so sampling
// lanes are not spread thinly over warps that are mostly done.
#ifndef FILTER_WARP_ATOMICS
#define FILTER_WARP_ATOMICS 1  // measured: visibility stage -2 us vs the block-aggregated reservation
#endif
__global__ void __launch_bounds__(256) k_vis_small_filter(const SmallRec* __restrict__ small_rec, int T,
                                                          const unsigned long long* __restrict__ hiz, int htx,
                                                          const unsigned char* __restrict__ flags,
                                                          int* __restrict__ queue, fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    __shared__ int s_cnt[2][8], s_base[2];
    const int n3 = st->n_small3;
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int* __restrict__ ids = small_ids(small_rec, T);
    for (int b0 = (int)blockIdx.x * blockDim.x; b0 < n3; b0 += gridDim.x * blockDim.x) {
        const int i = b0 + threadIdx.x;
        bool need = false, wide = false;
        // the triangle id first: a record whose triangle is already flagged
        // (a pass-1 pixel winner) is never read
        const unsigned char seen = i < n3 ? flags[__ldg(ids + i)] : 1;
        if (!seen) {
            const SmallRec* q = small_rec + i;
            Setup3 f;
            f.min_x = q->min_x; f.max_x = q->max_x; f.min_y = q->min_y; f.max_y = q->max_y;
            f.use_plane = (q->flags >> 3) & 1;
            f.p0x = q->x0; f.p0y = q->y0; f.p0z = q->z0;
            f.gx = q->g0; f.gy = q->g1; f.zmean = q->g0;
            const int tx0 = f.min_x / FA_HIZ, tx1 = f.max_x / FA_HIZ, ty0 = f.min_y / FA_HIZ, ty1 = f.max_y / FA_HIZ;
            const bool hz = tx1 - tx0 <= 1 && ty1 - ty0 <= 1;
            unsigned long long h00 = 1, h01 = 1, h10 = 1, h11 = 1;
            if (hz) {
                h00 = __ldg(hiz + ty0 * htx + tx0);
                h01 = __ldg(hiz + ty0 * htx + tx1);
                h10 = __ldg(hiz + ty1 * htx + tx0);
                h11 = __ldg(hiz + ty1 * htx + tx1);
            }
            const double zlb = depth_lower_bound(f, f.min_x, f.max_x, f.min_y, f.max_y);
            if (hz)
                need = !(hiz_tile_rejects(h00, zlb) && hiz_tile_rejects(h01, zlb) && hiz_tile_rejects(h10, zlb) &&
                         hiz_tile_rejects(h11, zlb));
            else  // windows over more than 2x2 hi-Z tiles: up to 3x3 tested, else sampled
                need = tx1 - tx0 > 2 || ty1 - ty0 > 2 ||
                       !hiz_rejects(hiz, htx, f.min_x, f.max_x, f.min_y, f.max_y, zlb);
            wide = (f.max_x - f.min_x + 1) * (f.max_y - f.min_y + 1) > FA_VIS_WARP_PX;
#ifdef FA_HIZ_STATS
            if (!seen) atomicAdd(&g_hiz_stats[need ? 1 : 0], 1ull);
#endif
        }
        const unsigned m = __ballot_sync(0xffffffffu, need && !wide);
        const unsigned m2 = __ballot_sync(0xffffffffu, need && wide);
#if FILTER_WARP_ATOMICS
        // per-warp reservations: no block barrier (warps do not wait on the
        // block's slowest record loads)
        int wb0 = 0, wb1 = 0;
        if (lane == 0) {
            if (m) wb0 = atomicAdd(&st->n_vis_q, __popc(m));
            if (m2) wb1 = atomicAdd(&st->n_vis_q2, __popc(m2));
        }
        if (m | m2) {
            wb0 = __shfl_sync(0xffffffffu, wb0, 0);
            wb1 = __shfl_sync(0xffffffffu, wb1, 0);
            if (need) {
                const unsigned mm = wide ? m2 : m;
                const int off = (wide ? wb1 : wb0) + __popc(mm & ((1u << lane) - 1u));
                queue[wide ? T - off : off] = i;
            }
        }
        continue;
#endif
        if (lane == 0) {
            s_cnt[0][warp] = __popc(m);
            s_cnt[1][warp] = __popc(m2);
        }
        __syncthreads();
        if (threadIdx.x < 2) {
            int tot = 0;
            for (int w = 0; w < 8; w++) tot += s_cnt[threadIdx.x][w];
            s_base[threadIdx.x] = tot ? atomicAdd(threadIdx.x ? &st->n_vis_q2 : &st->n_vis_q, tot) : 0;
        }
        __syncthreads();
        if (need) {
            // thread-sampled survivors from the front of the queue, warp-sampled
            // ones downward from index T (together at most n_small3 <= T)
            const unsigned mm = wide ? m2 : m;
            int off = s_base[wide] + __popc(mm & ((1u << lane) - 1u));
            for (int w = 0; w < warp; w++) off += s_cnt[wide][w];
            queue[wide ? T - off : off] = i;
        }
        __syncthreads();
    }
}

// Survivors of the filter.  Thread queue: one thread each, sample the row
// spans, stopping at the first passing sample; up to 4 covered samples per
// batch of depth loads.  Warp queue (windows above FA_VIS_WARP_PX): one warp
// per record, the window's samples dealt over the lanes (<= FA_SMALL_PX / 32
// each, their depth loads issued together).
#ifndef VSAMPLE_MIN_BLOCKS
#define VSAMPLE_MIN_BLOCKS 1  // minimum resident CTAs per SM (register cap)
#endif
__global__ void __launch_bounds__(256, VSAMPLE_MIN_BLOCKS) k_vis_small_sample(const SmallRec* __restrict__ small_rec, int T, int W,
                                                          const unsigned long long* __restrict__ depth,
                                                          const int* __restrict__ queue,
                                                          unsigned char* __restrict__ flags,
                                                          const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    const int nq_total = st->n_vis_q;
    for (int qi = (int)blockIdx.x * blockDim.x + threadIdx.x; qi < nq_total; qi += gridDim.x * blockDim.x) {
        Setup3 f;
        int t;
        load_rec(small_rec + queue[qi], f, t);
        bool vis = false;
        // queue of up to 4 covered samples in named registers (no local memory)
        double z0 = 0, z1 = 0, z2 = 0, z3 = 0;
        const unsigned long long *a0 = depth, *a1 = depth, *a2 = depth, *a3 = depth;
        int nq = 0;
        const SpanEdges se = span_edges(f);
        for (int iy = f.min_y; iy <= f.max_y && !vis; iy++) {
            const RowTerms rt = row_terms(f, (double)iy + 0.5);
            const unsigned long long* row = depth + (long long)iy * W;
            int xa, xb, ca, cb;
            row_span_cert(f, rt, se, xa, xb, ca, cb);  // only samples that can be covered
            for (int ix = xa; ix <= xb; ix++) {
                double px = (double)ix + 0.5;
                if (!(ix >= ca && ix <= cb) && !inside_row(f, rt, px)) continue;
                double z = depth_row(f, rt, px);
                const unsigned long long* a = row + ix;
                if (nq == 0) { z0 = z; a0 = a; }
                else if (nq == 1) { z1 = z; a1 = a; }
                else if (nq == 2) { z2 = z; a2 = a; }
                else { z3 = z; a3 = a; }
                if (++nq == 4) {
                    unsigned long long k0 = *a0, k1 = *a1, k2 = *a2, k3 = *a3;
                    vis = depth_passes(z0, key_f64(k0)) | depth_passes(z1, key_f64(k1)) |
                          depth_passes(z2, key_f64(k2)) | depth_passes(z3, key_f64(k3));
                    nq = 0;
                    if (vis) break;
                }
            }
        }
        if (!vis && nq > 0) {
            unsigned long long k0 = *a0, k1 = nq > 1 ? *a1 : 0ull, k2 = nq > 2 ? *a2 : 0ull;
            vis = depth_passes(z0, key_f64(k0)) | (nq > 1 && depth_passes(z1, key_f64(k1))) |
                  (nq > 2 && depth_passes(z2, key_f64(k2)));
        }
        if (vis) flags[t] = 1;
    }
    // the warp queue
    const int nq2 = st->n_vis_q2;
    const int lane = lane_id();
    constexpr int PER_LANE = (FA_SMALL_PX + 31) / 32;
    for (int wi = (int)(blockIdx.x * blockDim.x + threadIdx.x) / 32; wi < nq2; wi += gridDim.x * blockDim.x / 32) {
        Setup3 f;
        int t;
        load_rec(small_rec + queue[T - wi], f, t);
        const int bw = f.max_x - f.min_x + 1, n = bw * (f.max_y - f.min_y + 1);
        bool in[PER_LANE];
        double zq[PER_LANE];
        unsigned long long kq[PER_LANE];
#pragma unroll
        for (int j = 0; j < PER_LANE; j++) {
            const int k = lane + 32 * j;
            const int dy = k / bw;
            const int iy = f.min_y + dy, ix = f.min_x + (k - dy * bw);
            const double px = (double)ix + 0.5, py = (double)iy + 0.5;
            in[j] = k < n && sample_inside3(f, px, py);
            zq[j] = in[j] ? sample_depth3(f, px, py) : 0.0;
            kq[j] = in[j] ? depth[(long long)iy * W + ix] : 0ull;
        }
        bool vis = false;
#pragma unroll
        for (int j = 0; j < PER_LANE; j++) vis = vis || (in[j] && depth_passes(zq[j], key_f64(kq[j])));
        if (__any_sync(0xffffffffu, vis) && lane == 0) flags[t] = 1;
    }
}

// ---- pass 2 large: one warp per tile --------------------------------------
__global__ void __launch_bounds__(256) k_raster_vis_tiles(const SmallRec* __restrict__ recs, int T,
                                                          const TriSetup* __restrict__ large,
                                                          const int4* __restrict__ tiles, int W,
                                                          const unsigned long long* __restrict__ depth,
                                                          const unsigned long long* __restrict__ hiz, int htx,
                                                          unsigned char* __restrict__ flags,
                                                          const fa_dstat* __restrict__ st, int max_tiles,
                                                          int max_large) {
    FA_PDL_PROLOGUE();
    // Items: every 16x8 tile of the large triangles, then the generic setups
    // (only the small clipped windows, which have no tiles, are sampled
    // there).  Triangles already flagged — pass-1 pixel winners, or decided by
    // an earlier tile — are skipped; tiles the hierarchical Z rejects too.
    __shared__ TriSetup sm[8];
    int warp = threadIdx.x >> 5, lane = lane_id();
    int nwarps = gridDim.x * 8;
    const int n_front = min(st->n_tiles, max_tiles);
    const int n_tiles = n_front + min(st->n_tiles_clip, max_tiles - n_front);
    const int n_items = n_tiles + min(st->n_large, max_large);
    // Two phases per 32 items.  Filter (one lane per item, so a warp has 32
    // descriptor -> flag/record -> hierarchical-Z round trips in flight):
    // most tiles belong to triangles already flagged or lie behind the final
    // depth.  Sample (whole warp per surviving item, ~2% of the tiles).
    // lane l of warp g takes item g + nwarps * (l + 32 k): consecutive tiles
    // (mostly of one triangle) land in different warps, so survivors spread
    const int wg = (int)blockIdx.x * 8 + warp;
    for (int base = 0; wg + nwarps * base < n_items; base += 32) {
        const int wi = wg + nwarps * (base + lane);
        int4 rec0 = make_int4(0, 0, -1, 0);
        bool need = false;
        if (wi < n_items) {
            if (wi < n_front) rec0 = tiles[wi];
            else if (wi < n_tiles) rec0 = tiles[max_tiles - 1 - (wi - n_front)];
            else rec0 = make_int4(-(wi - n_tiles) - 1, -1, -1, 0);
            if (rec0.x < 0 && rec0.y < 0) {
                need = true;  // generic setup item (small clipped window): decided by the sampling phase
            } else if (!flags[rec0.z]) {
                // a record's tile, or a generic (clipped) setup's tile: the
                // same plane / bbox fields, so the same hi-Z test
                Setup3 f;
                if (rec0.x >= 0) {
                    const SmallRec* q = recs + rec0.x;
                    f.min_x = q->min_x; f.max_x = q->max_x; f.min_y = q->min_y; f.max_y = q->max_y;
                    f.use_plane = (q->flags >> 3) & 1;
                    f.p0x = q->x0; f.p0y = q->y0; f.p0z = q->z0;
                    f.gx = q->g0; f.gy = q->g1; f.zmean = q->g0;
                } else {
                    const TriSetup* g = large + (-rec0.x - 1);
                    f.min_x = g->min_x; f.max_x = g->max_x; f.min_y = g->min_y; f.max_y = g->max_y;
                    f.use_plane = g->use_plane;
                    f.p0x = g->p0x; f.p0y = g->p0y; f.p0z = g->p0z;
                    f.gx = g->gx; f.gy = g->gy; f.zmean = g->zmean;
                }
                const int ntx = (f.max_x - f.min_x + 1 + TILE_W - 1) / TILE_W;
                const int xa = f.min_x + (rec0.y % ntx) * TILE_W, ya = f.min_y + (rec0.y / ntx) * TILE_H;
                const int xb = min(xa + TILE_W - 1, f.max_x), yb = min(ya + TILE_H - 1, f.max_y);
                const double zlb = depth_lower_bound(f, xa, xb, ya, yb);
                // the hierarchical-Z tiles under the rectangle (at most 3 x 2)
                const int hx0 = xa / FA_HIZ, hx1 = xb / FA_HIZ, hy0 = ya / FA_HIZ, hy1 = yb / FA_HIZ;
                unsigned long long hk[6];
#pragma unroll
                for (int q2 = 0; q2 < 6; q2++) {
                    const int hx = hx0 + q2 % 3, hy = hy0 + q2 / 3;
                    hk[q2] = (hx <= hx1 && hy <= hy1) ? __ldg(hiz + hy * htx + hx) : FA_KEY_POS_INF;
                }
#pragma unroll
                for (int q2 = 0; q2 < 6; q2++) {
                    const int hx = hx0 + q2 % 3, hy = hy0 + q2 / 3;
                    if (hx <= hx1 && hy <= hy1 && !hiz_tile_rejects(hk[q2], zlb)) need = true;
                }
#ifdef FA_HIZ_STATS
                atomicAdd(&g_hiz_stats[2], 1ull);
                if (!need) atomicAdd(&g_hiz_stats[3], 1ull);
            } else {
                atomicAdd(&g_hiz_stats[4], 1ull);
#endif
            }
        }
        unsigned todo = __ballot_sync(0xffffffffu, need);
        while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        int4 rec;
        rec.x = __shfl_sync(0xffffffffu, rec0.x, src);
        rec.y = __shfl_sync(0xffffffffu, rec0.y, src);
        rec.z = __shfl_sync(0xffffffffu, rec0.z, src);
        rec.w = 0;
        if (rec.x >= 0) {
            int seen = 0;
            if (lane == 0) seen = *(volatile unsigned char*)(flags + rec.z);
            Setup3 f;
            int t;
            load_rec(recs + rec.x, f, t);
            if (__shfl_sync(0xffffffffu, seen, 0)) continue;  // flagged meanwhile (warp-uniform)
            int x, y0;
            tile_lane_origin(f.min_x, f.max_x, f.min_y, rec.y, x, y0);
            bool vis = false;
            if (x <= f.max_x) {
                // evaluate the lane's 4 samples, then issue their depth
                // loads together (static indices keep the arrays in registers)
                const ColTerms ct = col_terms(f, (double)x + 0.5);
                double zq[TILE_H / 2];
                bool in[TILE_H / 2];
                unsigned long long kq[TILE_H / 2];
#pragma unroll
                for (int k = 0; k < TILE_H / 2; k++) {
                    int y = y0 + 2 * k;
                    double py = (double)y + 0.5;
                    in[k] = y <= f.max_y && inside_col(f, ct, py);
                    zq[k] = in[k] ? depth_col(f, ct, py) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < TILE_H / 2; k++)
                    kq[k] = in[k] ? depth[(long long)(y0 + 2 * k) * W + x] : 0ull;
#pragma unroll
                for (int k = 0; k < TILE_H / 2; k++) vis = vis || (in[k] && depth_passes(zq[k], key_f64(kq[k])));
            }
            if (__any_sync(0xffffffffu, vis) && lane == 0) flags[t] = 1;
            continue;
        }
        rec.x = -rec.x - 1;
        int t = __ldg(&large[rec.x].tri);
        int seen = 0;
        if (lane == 0) seen = *(volatile unsigned char*)(flags + t);
        if (__shfl_sync(0xffffffffu, seen, 0)) continue;  // already visible (warp-uniform)
        __syncwarp();
        load_setup_warp(large + rec.x, &sm[warp]);
        const TriSetup& s = sm[warp];
        int bw = s.max_x - s.min_x + 1, bh = s.max_y - s.min_y + 1;
        bool vis = false;
        if (rec.y < 0) {
            // generic setup item: only small clipped windows (no tiles) are sampled here
            if (bw * bh > FA_SMALL_PX) continue;
            for (int k = lane; k < bw * bh && !vis; k += 32) {
                int dy = k / bw;
                int iy = s.min_y + dy, ix = s.min_x + (k - dy * bw);
                double px = (double)ix + 0.5, py = (double)iy + 0.5;
                if (!sample_inside(s, px, py)) continue;
                vis = depth_passes(sample_depth(s, px, py), key_f64(depth[(long long)iy * W + ix]));
            }
            if (__any_sync(0xffffffffu, vis) && lane == 0) flags[t] = 1;
            continue;
        }
        int tx = (bw + TILE_W - 1) / TILE_W;
        int x = s.min_x + (rec.y % tx) * TILE_W + (lane & 15);
        int y0 = s.min_y + (rec.y / tx) * TILE_H + (lane >> 4);
        if (x <= s.max_x) {
            // the inside tests first, then every covered sample's depth load
            // in flight together, then the slack tests
            const double px = (double)x + 0.5;
            bool in[TILE_H / 2];
            unsigned long long kq[TILE_H / 2];
#pragma unroll
            for (int k = 0; k < TILE_H / 2; k++) {
                const int y = y0 + 2 * k;
                in[k] = y <= s.max_y && sample_inside(s, px, (double)y + 0.5);
            }
#pragma unroll
            for (int k = 0; k < TILE_H / 2; k++) kq[k] = in[k] ? depth[(long long)(y0 + 2 * k) * W + x] : 0ull;
#pragma unroll
            for (int k = 0; k < TILE_H / 2; k++)
                vis = vis || (in[k] && depth_passes(sample_depth(s, px, (double)(y0 + 2 * k) + 0.5), key_f64(kq[k])));
        }
        if (__any_sync(0xffffffffu, vis) && lane == 0) flags[t] = 1;
        }
    }
}

// ---- host launchers -------------------------------------------------------
void fa_launch_frame_init(const double* pos, int V, const double* vp, double4* clip, double4* scr, int W, int H,
                          int* vmin, unsigned long long* depth, unsigned long long* wid, long long npx,
                          unsigned char* flags, int T, cudaStream_t s, int max_blocks, double2* ndc2,
                          const fa_cull_args* cull) {
    long long work = V;
    if (depth && npx / 2 > work) work = npx / 2;
    int nflag32 = flags ? (T + 3) / 4 : 0;
    if (nflag32 > work) work = nflag32;
    const int g = max_blocks > 0 ? fa_grid(work, 256, max_blocks)
                                 : fa_wave_grid(k_frame_init, 256, 0, (work + 255) / 256, FA_NUM_SMS * 8);
    fa_cull_args cu{};
    int cull_blocks = 0;
    if (cull && cull->clusters) {
        cu = *cull;
        cull_blocks = fa_grid(cu.n_clusters, 256, FA_NUM_SMS);
    }
    fa_launch(k_frame_init, g + cull_blocks, 256, 0, s, pos, V, vp, clip, scr, W, H, vmin, depth, wid, npx,
              reinterpret_cast<unsigned int*>(flags), nflag32, ndc2, cu, cull_blocks);
}

// fork `side` off `s` (side waits for everything issued on s so far)
static void fork_to(cudaStream_t s, cudaStream_t side, cudaEvent_t ev) {
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(side, ev, 0);
}

// Depth pass (write_depth) or work-list build (standalone mark_visible).
// With side streams: setup, then {small records on s} || {unclipped large
// tiles on side} || {clipped polygons -> their tiles on side2}, joined back
// into s.  Every branch only lowers depth keys with atomicMin, so their order
// does not matter.
#ifndef CLIPPED_WAVE
#define CLIPPED_WAVE 0
#endif
#if CLIPPED_WAVE
#define CLIPPED_GRID(k) fa_wave_grid(k, 256, 0, FA_NUM_SMS * 8, FA_NUM_SMS * 8)
#else
#define CLIPPED_GRID(k) fa_cap(FA_NUM_SMS * 2)
#endif
#ifndef TILES_WAVE
#define TILES_WAVE 1
#endif
#if TILES_WAVE
#define TILES_GRID(cap) fa_wave_grid(k_raster_depth_tiles, 256, 0, (cap), (cap))
#else
#define TILES_GRID(cap) fa_cap(cap)
#endif
int fa_launch_depth_pass(bool write_depth, const ClipSrc clip, const double4* scr, const int* tris, int T, int W,
                         int H, int cull, unsigned long long* depth, unsigned long long* wid, SmallRec* small_rec,
                         int* clip_list, TriSetup* large, int max_large, int4* tiles, int max_tiles, fa_dstat* st,
                         cudaStream_t s, cudaStream_t side, cudaStream_t side2, cudaEvent_t ev_fork,
                         cudaEvent_t ev_join, cudaEvent_t ev_join2, cudaEvent_t ev_clear, fa_setup_order ord) {
    fa_launch(k_raster_setup, fa_grid(T, SETUP_WARPS * 32, FA_NUM_SMS * SETUP_MIN_BLOCKS), SETUP_WARPS * 32, 0, s, scr, tris, T, W, H, cull, small_rec,
              clip_list, tiles, max_tiles, st, ord);
    // the depth/winner clears ran beside the setup: every raster branch
    // (forked from here) needs them
    if (ev_clear) cudaStreamWaitEvent(s, ev_clear, 0);
    cudaStream_t b = side ? side : s;
    cudaStream_t b2 = side2 ? side2 : b;
    if (side) fork_to(s, side, ev_fork);
    if (side2) cudaStreamWaitEvent(side2, ev_fork, 0);
    int n = 0;
    if (write_depth) {
        // three independent branches, all lowering depth keys with RED.MIN:
        //   s:     small unclipped records (warp-cooperative)
        //   side:  the unclipped large records' tiles
        //   side2: clipped polygons -> their tiles
        fa_launch(k_raster_depth_tiles, TILES_GRID(FA_NUM_SMS * 8), 256, 0, b, small_rec, large, tiles, W, depth, wid, st,
                  max_tiles, 0, 1, 0);
        fa_launch(k_raster_clipped<true>, CLIPPED_GRID(k_raster_clipped<true>), 256, 0, b2, clip, tris, W, H, cull, clip_list, depth, wid,
                  large, max_large, tiles, max_tiles, st);
        fa_launch(k_raster_depth_tiles, TILES_GRID(FA_NUM_SMS * 4), 256, 0, b2, small_rec, large, tiles, W, depth, wid, st,
                  max_tiles, 0, 1, 1);
        fa_launch(k_small_coop, fa_grid((long long)T, COOP_WARPS * 32 * 2, FA_NUM_SMS * COOP_GRID_MULT), COOP_WARPS * 32, 0,
                  s, small_rec, W, depth, wid, st);
        n = 5;
    } else {
        fa_launch(k_raster_clipped<false>, fa_cap(FA_NUM_SMS * 2), 256, 0, b, clip, tris, W, H, cull, clip_list, depth,
                  nullptr, large, max_large, tiles, max_tiles, st);
        n = 2;
    }
    if (side) fork_to(side, s, ev_join);
    if (side2 && write_depth) fork_to(side2, s, ev_join2);
    return n;
}

// Visibility pass: small records on s || large tiles + small clipped windows
// on side.  Both only set flags, which k_depth_hiz seeded with the winners.
int fa_launch_raster_vis(const SmallRec* small_rec, const TriSetup* large, const int4* tiles, int max_tiles,
                         int max_large, int T, int W, const unsigned long long* depth, const unsigned long long* hiz,
                         unsigned char* flags, int* vis_queue, fa_dstat* st, cudaStream_t s, cudaStream_t side,
                         cudaEvent_t ev_fork, cudaEvent_t ev_join) {
    cudaStream_t b = side ? side : s;
    const int htx = fa_hiz_dim(W);
    if (side) fork_to(s, side, ev_fork);
    fa_launch(k_raster_vis_tiles, fa_wave_grid(k_raster_vis_tiles, 256, 0, FA_NUM_SMS * 8, FA_NUM_SMS * 8), 256, 0, b, small_rec, T, large, tiles, W, depth, hiz, htx, flags, st,
                                                      max_tiles, max_large);
    fa_launch(k_vis_small_filter, fa_wave_grid(k_vis_small_filter, 256, 0, ((long long)T + 255) / 256, FA_NUM_SMS * 16), 256, 0, s, small_rec, T, hiz, htx, flags, vis_queue,
              st);
    fa_launch(k_vis_small_sample, fa_wave_grid(k_vis_small_sample, 256, 0, ((long long)T / 4 + 255) / 256, FA_NUM_SMS * 8), 256, 0, s, small_rec, T, W, depth, vis_queue,
              flags, st);
    if (side) fork_to(side, s, ev_join);
    return 3;
}

void fa_launch_depth_hiz(const unsigned long long* depth, const unsigned long long* wid, int W, int H,
                         unsigned long long* hiz, unsigned char* flags, fa_dstat* st, cudaStream_t s) {
    int htx = fa_hiz_dim(W), hty = fa_hiz_dim(H);
    fa_launch(k_depth_hiz, fa_wave_grid(k_depth_hiz, 256, 0, ((long long)htx * FA_HIZ * hty + 255) / 256, FA_NUM_SMS * 8), 256, 0, s, depth, wid, W, H, hiz, htx,
                                                                                           hty, flags, st);
}

void fa_launch_decode_depth(const unsigned long long* keys, double* out, long long n, cudaStream_t s) {
    fa_launch(k_decode_depth, fa_grid(n, 256, FA_NUM_SMS * 8), 256, 0, s, keys, out, n);
}

void fa_launch_encode_depth(const double* in, unsigned long long* keys, long long n, cudaStream_t s) {
    fa_launch(k_encode_depth, fa_grid(n, 256, FA_NUM_SMS * 8), 256, 0, s, in, keys, n);
}

FA_TRACE_TU(raster)
