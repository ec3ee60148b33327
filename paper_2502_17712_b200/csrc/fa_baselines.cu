// fa_baselines.cu — the comparison packers of atlaspack.baselines on sm_100a
// (used by `compare`, cli.py:619-674).
//
// * sequential_scale_search (baselines.py:110-141): one CTA per candidate
//   scale i/n (all candidates concurrently instead of n..1 in turn).  Each CTA
//   computes the scaled dims, rejects when a box is wider than the atlas,
//   walks the ordered boxes once to assign rows (sequential_fold,
//   baselines.py:53-76; one thread, it is a serial recurrence), then runs the
//   shared push-up (packing.py:170-215) with thread groups per row box.  The
//   result is the largest accepted candidate, which is exactly the first
//   success of the reference's descending scan.
// * superblock_pack (baselines.py:187-261): the halving levels are
//   independent, so each level runs in its own CTA; inside a level one warp
//   places boxes in order, its lanes testing 32 blocks at a time for the
//   first-fit block (ballot), the winning lane updating that block's shelves.
//   The result is the first (largest-block) level that places every box.
#define FA_TU_ID 7  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"
#include "fa_pack.cuh"

#define BL_THREADS 256
#define SB_FLOOR 16  // baselines.py:31

// shared push-up of rows with explicit x; returns max top (saturated at omega + 1)
__device__ long long cta_push_up_x(const int* __restrict__ xs, const int* __restrict__ w, const int* __restrict__ h,
                                   const int* __restrict__ rowstart, int n_rows, int n, long long omega, int* front,
                                   int* y, long long* red) {
    int tid = threadIdx.x;
    for (int c = tid; c <= omega; c += blockDim.x) front[c] = 0;
    __syncthreads();
    long long used = 0;
    for (int r = 0; r < n_rows; r++) {
        int b0 = rowstart[r];
        int b1 = (r + 1 < n_rows) ? rowstart[r + 1] : n;
        int nb = b1 - b0;
        int G = 32;
        while (G > 1 && G * nb > (int)blockDim.x) G >>= 1;
        int groups = blockDim.x / G;
        int g = tid / G, gl = tid % G;
        for (int gbase = 0; gbase < nb; gbase += groups) {
            int gb = gbase + g;
            bool act = gb < nb;
            int b = b0 + (act ? gb : 0);
            int x = xs[b], wb = act ? w[b] : 0;
            int rest = 0;
            for (int c = x + gl; c < x + wb; c += G) rest = max(rest, front[c]);
            for (int o = G >> 1; o > 0; o >>= 1) rest = max(rest, __shfl_xor_sync(0xffffffffu, rest, o, G));
            long long top64 = (long long)rest + h[b];
            int top = top64 > omega ? (int)(omega + 1) : (int)top64;
            if (act) {
                for (int c = x + gl; c < x + wb; c += G) front[c] = top;
                if (gl == 0) y[b] = rest;
                used = top > used ? top : used;
            }
        }
        __syncthreads();
    }
    return block_max_ll(used, red);
}

// cand record: [accept, used, slot]
#define SEQ_REC 3

__global__ void __launch_bounds__(BL_THREADS) k_seq_candidates(const long long* __restrict__ ow,
                                                               const long long* __restrict__ oh, int n, long long omega,
                                                               long long n_scales, long long first, long long min_dim,
                                                               long long pad, int* __restrict__ cw, int* __restrict__ ch,
                                                               int* __restrict__ cx, int* __restrict__ cy,
                                                               int* __restrict__ rowstart, int* __restrict__ gfront,
                                                               long long* __restrict__ cand,
                                                               const unsigned* __restrict__ done,
                                                               int* __restrict__ rows_out) {
    FA_PDL_PROLOGUE();
    extern __shared__ int dyn_front[];
    __shared__ long long red[33];
    __shared__ int s_rows;
    long long i = first - blockIdx.x;
    if (i < 1 || *done) return;
    size_t slot = blockIdx.x;
    int* w = cw + slot * n;
    int* h = ch + slot * n;
    int* x = cx + slot * n;
    int* y = cy + slot * n;
    int* rs = rowstart + slot * n;
    int* front = gfront ? gfront + slot * (size_t)(omega + 1) : dyn_front;
    long long wmax = 0;
    for (int b = threadIdx.x; b < n; b += blockDim.x) {
        long long wb = scaled_dim(ow[b], i, n_scales, min_dim, pad);
        w[b] = (int)wb;
        h[b] = (int)scaled_dim(oh[b], i, n_scales, min_dim, pad);
        wmax = wb > wmax ? wb : wmax;
    }
    wmax = block_max_ll(wmax, red);
    long long* rec = cand + SEQ_REC * (i - 1);
    if (wmax > omega) {  // baselines.py:130-131
        if (threadIdx.x == 0) { rec[0] = 0; rec[1] = 0; rec[2] = (long long)slot; }
        return;
    }
    if (threadIdx.x == 0) {
        // sequential_fold (baselines.py:53-76): a box that would cross the
        // atlas edge starts the next row
        int row = 0;
        long long used = 0;
        rs[0] = 0;
        for (int b = 0; b < n; b++) {
            int wb = w[b];
            if (used + wb > omega) {
                row++;
                used = 0;
                rs[row] = b;
            }
            x[b] = (row % FA_DIRECTION_PERIOD == 0) ? (int)used : (int)(omega - used - wb);
            if (rows_out) rows_out[b] = row;
            used += wb;
        }
        s_rows = row + 1;
    }
    __syncthreads();
    long long used = cta_push_up_x(x, w, h, rs, s_rows, n, omega, front, y, red);
    if (threadIdx.x == 0) {
        rec[0] = used <= omega;
        rec[1] = used;
        rec[2] = (long long)slot;
    }
}

__global__ void k_seq_batch_done(const long long* __restrict__ cand, long long lo, long long hi, unsigned* done) {
    FA_PDL_PROLOGUE();
    bool any = false;
    for (long long i = lo + threadIdx.x; i <= hi; i += blockDim.x) any |= cand[SEQ_REC * (i - 1)] != 0;
    if (__syncthreads_or(any) && threadIdx.x == 0) *done = 1;
}

__global__ void __launch_bounds__(1024) k_seq_select(const long long* __restrict__ tw, const long long* __restrict__ th,
                                                     const long long* __restrict__ chart_id,
                                                     const unsigned char* __restrict__ rot, const int* __restrict__ perm,
                                                     int n, long long n_scales, const long long* __restrict__ cand,
                                                     const int* __restrict__ cw, const int* __restrict__ ch,
                                                     const int* __restrict__ cx, const int* __restrict__ cy,
                                                     long long* __restrict__ placements, long long* __restrict__ out) {
    FA_PDL_PROLOGUE();
    __shared__ long long red[33];
    long long best = 0;
    for (long long i = threadIdx.x + 1; i <= n_scales; i += blockDim.x)
        if (cand[SEQ_REC * (i - 1)] != 0 && i > best) best = i;
    best = block_max_ll(best, red);
    if (threadIdx.x == 0) out[0] = best;
    if (best == 0) return;
    size_t slot = (size_t)cand[SEQ_REC * (best - 1) + 2];
    const int *w = cw + slot * n, *h = ch + slot * n, *x = cx + slot * n, *y = cy + slot * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        int src = perm[j];
        long long* P = placements + 8 * (long long)j;
        P[0] = chart_id[src];
        P[1] = x[j];
        P[2] = y[j];
        P[3] = w[j];
        P[4] = h[j];
        P[5] = rot[j];
        P[6] = tw[src];
        P[7] = th[src];
    }
}

// ---- superblock ---------------------------------------------------------------
__device__ __forceinline__ int next_pow2(int v) { return v > 1 ? 1 << (32 - __clz(v - 1)) : 1; }

// can block `blk` take a w x h box (_Block.place, baselines.py:166-180)?  On
// success returns the shelf index to use (== n_shelves for a new shelf)
__device__ __forceinline__ int sb_probe(const int* sh_h, const int* sh_cur, int nsh, int used_h, int size, int w,
                                        int shelf_h) {
    for (int s = 0; s < nsh; s++)
        if (sh_h[s] == shelf_h && sh_cur[s] + w <= size) return s;
    if (used_h + shelf_h <= size) return nsh;
    return -1;
}

// One CTA (one warp) per halving level L: block = block0 >> L.
// state per level: used_h[nb], nsh[nb], shelves [nb][block] (h, y, cursor)
__global__ void k_superblock(const long long* __restrict__ ow, const long long* __restrict__ oh, int n,
                             long long omega, int block0, int* __restrict__ state, size_t state_stride,
                             int* __restrict__ out_xywh, size_t out_stride, int* __restrict__ level_ok) {
    FA_PDL_PROLOGUE();
    int L = blockIdx.x;
    int block = block0 >> L;
    int lane = threadIdx.x;
    int grid = (int)(omega / block);
    int nb = grid * grid;
    int* used_h = state + L * state_stride;
    int* nsh = used_h + nb;
    int* sh_h = nsh + nb;                          // [nb][block]
    int* sh_y = sh_h + (size_t)nb * block;
    int* sh_cur = sh_y + (size_t)nb * block;
    int* xywh = out_xywh + L * out_stride;
    for (int b = lane; b < nb; b += 32) {
        used_h[b] = 0;
        nsh[b] = 0;
    }
    __syncwarp();
    bool ok = true;
    for (int k = 0; k < n && ok; k++) {
        long long w64 = ow[k], h64 = oh[k];
        int w, h;
        if (w64 > block || h64 > block) {
            // uniform downscale by min(block/w, block/h) = block / max(w, h)
            long long m = w64 > h64 ? w64 : h64;
            long long ws = (w64 * block + m - 1) / m, hs = (h64 * block + m - 1) / m;
            w = (int)(ws < 1 ? 1 : ws);
            h = (int)(hs < 1 ? 1 : hs);
        } else {
            w = (int)w64;
            h = (int)h64;
        }
        int shelf_h = next_pow2(h);
        int found = -1, found_sh = -1;
        for (int base = 0; base < nb && found < 0; base += 32) {
            int blk = base + lane;
            int s = -1;
            if (blk < nb)
                s = sb_probe(sh_h + (size_t)blk * block, sh_cur + (size_t)blk * block, nsh[blk], used_h[blk], block,
                             w, shelf_h);
            unsigned m = __ballot_sync(0xffffffffu, s >= 0);
            if (m) {
                int src = __ffs(m) - 1;
                found = base + src;
                found_sh = __shfl_sync(0xffffffffu, s, src);
            }
        }
        if (found < 0) {
            ok = false;
            break;
        }
        if (lane == 0) {
            int bx = found % grid, by = found / grid;
            int* H = sh_h + (size_t)found * block;
            int* Y = sh_y + (size_t)found * block;
            int* C = sh_cur + (size_t)found * block;
            int x, y;
            if (found_sh < nsh[found]) {
                x = bx * block + C[found_sh];
                y = by * block + Y[found_sh];
                C[found_sh] += w;
            } else {
                int s = nsh[found]++;
                H[s] = shelf_h;
                Y[s] = used_h[found];
                C[s] = w;
                used_h[found] += shelf_h;
                x = bx * block;
                y = by * block + Y[s];
            }
            xywh[4 * k] = x;
            xywh[4 * k + 1] = y;
            xywh[4 * k + 2] = w;
            xywh[4 * k + 3] = h;
        }
        __syncwarp();
    }
    if (lane == 0) level_ok[L] = ok;
}

// first successful level -> placements; scale index = argmin w / target
__global__ void k_superblock_select(const long long* __restrict__ tw, const long long* __restrict__ th,
                                    const long long* __restrict__ chart_id, const unsigned char* __restrict__ rot,
                                    const int* __restrict__ perm, int n, int n_levels, const int* __restrict__ xywh,
                                    size_t out_stride, const int* __restrict__ level_ok,
                                    long long* __restrict__ placements, long long* __restrict__ out) {
    FA_PDL_PROLOGUE();
    __shared__ int s_level;
    if (threadIdx.x == 0) {
        s_level = -1;
        for (int L = 0; L < n_levels; L++)
            if (level_ok[L]) { s_level = L; break; }
        out[0] = s_level;
    }
    __syncthreads();
    int L = s_level;
    if (L < 0) return;
    const int* q = xywh + L * out_stride;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        int src = perm[j];
        long long* P = placements + 8 * (long long)j;
        P[0] = chart_id[src];
        P[1] = q[4 * j];
        P[2] = q[4 * j + 1];
        P[3] = q[4 * j + 2];
        P[4] = q[4 * j + 3];
        P[5] = rot[j];
        P[6] = tw[src];
        P[7] = th[src];
    }
    __syncthreads();
    // _min_box_scale (baselines.py:253-259): the minimum of w / target over
    // boxes, starting from 1; exact rational compare by cross-multiplication.
    // The first minimal box (placement order) wins ties, as in the reference.
    if (threadIdx.x == 0) {
        long long bn = 1, bd = 1;
        for (int j = 0; j < n; j++) {
            int src = perm[j];
            long long t = rot[j] ? th[src] : tw[src];
            long long w = q[4 * j + 2];
            if (w * bd < bn * t) { bn = w; bd = t; }
        }
        out[1] = bn;
        out[2] = bd;
    }
}

// ---- launchers --------------------------------------------------------------
void fa_launch_seq_search(const long long* ow, const long long* oh, int n, long long omega, long long n_scales,
                          long long min_dim, long long pad, int batch, int* cw, int* ch, int* cx, int* cy,
                          int* rowstart, int* gfront, long long* cand, unsigned* done, cudaStream_t s) {
    size_t dyn = gfront ? 0 : (size_t)(omega + 1) * sizeof(int);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_seq_candidates, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    for (long long hi = n_scales; hi >= 1; hi -= batch) {
        long long lo = hi - batch + 1;
        if (lo < 1) lo = 1;
        fa_launch(k_seq_candidates, (int)(hi - lo + 1), BL_THREADS, dyn, s, ow, oh, n, omega, n_scales, hi, min_dim, pad, cw,
                                                                   ch, cx, cy, rowstart, gfront, cand, done, nullptr);
        if (lo > 1) fa_launch(k_seq_batch_done, 1, 256, 0, s, cand, lo, hi, done);
    }
}

__global__ void k_widen3(const int* __restrict__ a, const int* __restrict__ b, const int* __restrict__ c, int n,
                         long long* __restrict__ oa, long long* __restrict__ ob, long long* __restrict__ oc) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        oa[i] = a[i];
        ob[i] = b[i];
        oc[i] = c[i];
    }
}

// sequential_pack / sequential_fold (baselines.py:53-107) on the caller's
// order at the stated dims: rows, x, y and the cand record [accept, used, 0]
void fa_launch_seq_single(const long long* w, const long long* h, int n, long long omega, int* cw, int* ch, int* cx,
                          int* cy, int* rowstart, int* rows, int* gfront, long long* cand, const unsigned* done_zero,
                          long long* rows_out, long long* x_out, long long* y_out, cudaStream_t s) {
    size_t dyn = gfront ? 0 : (size_t)(omega + 1) * sizeof(int);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_seq_candidates, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    fa_launch(k_seq_candidates, 1, BL_THREADS, dyn, s, w, h, n, omega, 1, 1, 1, 0, cw, ch, cx, cy, rowstart, gfront, cand,
                                               done_zero, rows);
    fa_launch(k_widen3, fa_grid(n, 256, FA_NUM_SMS), 256, 0, s, rows, cx, cy, n, rows_out, x_out, y_out);
}

void fa_launch_seq_select(const long long* tw, const long long* th, const long long* cid, const unsigned char* rot,
                          const int* perm, int n, long long n_scales, const long long* cand, const int* cw,
                          const int* ch, const int* cx, const int* cy, long long* placements, long long* out,
                          cudaStream_t s) {
    fa_launch(k_seq_select, 1, 1024, 0, s, tw, th, cid, rot, perm, n, n_scales, cand, cw, ch, cx, cy, placements, out);
}

void fa_launch_superblock(const long long* ow, const long long* oh, const long long* tw, const long long* th,
                          const long long* cid, const unsigned char* rot, const int* perm, int n, long long omega,
                          int block0, int n_levels, int* state, size_t state_stride, int* xywh, size_t out_stride,
                          int* level_ok, long long* placements, long long* out, cudaStream_t s) {
    fa_launch(k_superblock, n_levels, 32, 0, s, ow, oh, n, omega, block0, state, state_stride, xywh, out_stride, level_ok);
    fa_launch(k_superblock_select, 1, 256, 0, s, tw, th, cid, rot, perm, n, n_levels, xywh, out_stride, level_ok, placements,
                                          out);
}

FA_TRACE_TU(baselines)
