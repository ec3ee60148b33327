// fa_common.cuh — shared device helpers for the B200 atlas path.
//
// Every kernel in this library is compiled with -fmad=false: the reference
// computes in numpy float64 with one rounding per operation, so contraction
// of a*b+c into DFMA would change bits.  The only FMAs are the explicit
// __fma_rn() calls that restate OpenBLAS' dgemm chain.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fastatlas.h"

#define FA_W_EPSILON 1e-9       // geometry.py:19
#define FA_DEPTH_EPSILON 1e-6   // charts.py:26
#define FA_MAX_BOX_DIM (1 << 23)  // packing.py:25
#define FA_SCALE_GRID_BITS 24   // packing.py:29
#define FA_DIRECTION_PERIOD 3   // packing.py:32
#define FA_MAX_OVERFLOW_ITERS 8 // packing.py:34
#define FA_MAXV 16              // clipped polygon capacity (real max is 10)

#define FA_NUM_SMS 148
#define FA_HIZ 8                // hierarchical-Z tile edge (pixels)

// device status bits (fa_ctx::dstat->flags)
#define FA_VC_OFF 16  // vp_dev: 16 doubles of VP, then the frame's fa_view_consts (host-computed)
#define FA_VP_DOUBLES 64  // per uploaded camera (VP + view constants)
// triangles per culling cluster (consecutive in the setup order; 32 or 16)
#ifndef FA_CLUSTER
#define FA_CLUSTER 32
#endif
#define FA_DFLAG_POLY_OVERFLOW 1u
#define FA_DFLAG_HEIGHT_OVERFLOW 2u
#define FA_DFLAG_DEGENERATE_CHART 4u
#define FA_DFLAG_PACK_FAILURE 8u
#define FA_DFLAG_QUEUE_OVERFLOW 16u
#define FA_DFLAG_DUPLICATE_MIN_TRI 32u
#define FA_DFLAG_KEY_RANGE 64u
#define FA_DFLAG_BAD_ARGS 128u
#define FA_FX_DIGITS 6
#define FA_DFLAG_STRETCH_RANGE 256u  // a stretch partial outside [2^-80, 2^111): report the float sums

// Per-frame device counters and status (zeroed per frame).  The four append
// counters of k_raster_setup take one atomic per block step each (~4K per
// frame at C2); they sit 256 bytes apart so their atomics are served by
// different L2 slices instead of queueing on one.
struct fa_dstat {
    unsigned int flags;
    int n_vis;            // visible triangles
    int n_charts;         // chart roots (ascending)
    int n_vis_q;          // small records the visibility filter left for sampling
    int n_large;          // large-raster triangle setups
    int best;             // selected candidate (1-based), 0 = none
    int floor_fail;       // pack floor-width failure
    int n_rows_max;
    long long screen_fragments;
    long long texels_allocated;
    long long scale_num;
    long long scale_den;
    int max_h;            // max oriented height (sort key range)
    unsigned int done;    // pack batch early-exit
    int stretch_valid;    // triangles that entered the stretch sums
    int n_tiles_clip;     // tiles of clipped (generic) setups, stored downward from max_tiles - 1
    int n_vis_vertices;   // vertices touched by a visible triangle (compact UV format)
    int pad_v;
    double stretch_wsum;  // sum area * (S1^2 + S2^2) / 2   (metrics.py:103) — used only on FA_DFLAG_STRETCH_RANGE
    double stretch_area;  // sum area                       (metrics.py:104) — ditto
    unsigned long long stretch_linf_bits;  // max S1 (positive double bits)
    int n_live;           // 32-triangle clusters the setup processes (k_frame_init's cluster culling)
    int pad_l;
    // the same two sums in exact fixed point (units of 2^-80, 32-bit digits
    // in six u64 counters each, fx_add): integer adds commute, so the sums
    // are run-to-run reproducible (k_uv adds one truncated partial per block)
    unsigned long long stretch_fx[2][FA_FX_DIGITS];
    int n_vis_q2;         // larger small records the visibility filter left for warp sampling
    int pad0[9];
    int n_small3;         // stored small-triangle records (pass 2 input)
    int pad1[63];
    int n_large3;         // compact large-triangle records (stored from the back of the record array)
    int pad2[63];
    int n_clip;           // triangles routed to the generic (clipping) path
    int pad3[63];
    int n_tiles;          // large-raster tile work items
    int pad4[63];
};
static_assert(offsetof(fa_dstat, stretch_fx) % 8 == 0, "fa_dstat: aligned fixed-point limbs");
static_assert(sizeof(fa_dstat) == 1280, "fa_dstat: a 256-byte status block + four 256-byte counter slots");

// ---- float64 <-> order-preserving u64 key --------------------------------
__device__ __forceinline__ unsigned long long f64_key(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}
#define FA_KEY_POS_INF 0xfff0000000000000ull   // f64_key(+inf)
#define FA_KEY_NEG_INF 0x000fffffffffffffull   // f64_key(-inf)

// ---- projection (charts.py:273-274): OpenBLAS dgemm FMA chain -------------
struct vp_mat { double m[16]; };

__device__ __forceinline__ double4 project_point(double x, double y, double z, const double* __restrict__ m) {
    double4 o;
    double a;
    a = __dmul_rn(x, m[0]);  a = __fma_rn(y, m[1], a);  a = __fma_rn(z, m[2], a);  a = __fma_rn(1.0, m[3], a);  o.x = a;
    a = __dmul_rn(x, m[4]);  a = __fma_rn(y, m[5], a);  a = __fma_rn(z, m[6], a);  a = __fma_rn(1.0, m[7], a);  o.y = a;
    a = __dmul_rn(x, m[8]);  a = __fma_rn(y, m[9], a);  a = __fma_rn(z, m[10], a); a = __fma_rn(1.0, m[11], a); o.z = a;
    a = __dmul_rn(x, m[12]); a = __fma_rn(y, m[13], a); a = __fma_rn(z, m[14], a); a = __fma_rn(1.0, m[15], a); o.w = a;
    return o;
}

// ---- warp helpers ---------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = v > w ? v : w;
    }
    return v;
}

// warp-aggregated append: returns the slot of this lane when pred is true
__device__ __forceinline__ int warp_append(int* counter, bool pred) {
    unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return -1;
    int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane_id() == leader) base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    return pred ? base + __popc(mask & ((1u << lane_id()) - 1u)) : -1;
}

// block-wide exclusive scan of one int per thread (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ int block_exclusive_scan(int v, int* smem32, int* total) {
    int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem32[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < nw ? smem32[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) smem32[lane] = s;
    }
    __syncthreads();
    int base = wid > 0 ? smem32[wid - 1] : 0;
    int tot = smem32[nw - 1];
    __syncthreads();
    if (total) *total = tot;
    return base + x - v;
}

// same for int64
__device__ __forceinline__ long long block_exclusive_scan_ll(long long v, long long* smem32, long long* total) {
    int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem32[wid] = x;
    __syncthreads();
    if (wid == 0) {
        long long s = lane < nw ? smem32[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) smem32[lane] = s;
    }
    __syncthreads();
    long long base = wid > 0 ? smem32[wid - 1] : 0;
    long long tot = smem32[nw - 1];
    __syncthreads();
    if (total) *total = tot;
    return base + x - v;
}

// Block reductions: warp shuffles, then warp 0 reduces the per-warp partials
// and broadcasts through slot 32.  smem32 must hold 33 entries.  Two barriers;
// the broadcast slot is only rewritten after the next call's first barrier,
// which every reader of the previous value has passed.
__device__ __forceinline__ long long block_max_ll(long long v, long long* smem32) {
    int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max_ll(v);
    if (lane == 0) smem32[wid] = v;
    __syncthreads();
    if (wid == 0) {
        long long x = lane < nw ? smem32[lane] : (long long)0x8000000000000000ll;
        x = warp_max_ll(x);
        if (lane == 0) smem32[32] = x;
    }
    __syncthreads();
    return smem32[32];
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* smem32) {
    int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) smem32[wid] = v;
    __syncthreads();
    if (wid == 0) {
        long long x = lane < nw ? smem32[lane] : 0;
        x = warp_sum(x);
        if (lane == 0) smem32[32] = x;
    }
    __syncthreads();
    return smem32[32];
}

// ---- exact fixed-point accumulation (reproducible sums) ----------------
// acc += v truncated to a multiple of 2^-80.  The fixed-point value is cut
// into 32-bit digits and digit k is added to the 64-bit counter acc[k]
// (value = sum_k acc[k] * 2^(32k - 80)); counters cannot overflow below 2^32
// adds, so no carries are needed and every add is a fire-and-forget RED.
// Integer adds commute: the sum does not depend on their order.
// Returns false when v is negative, NaN or >= 2^111 (not representable).
__device__ __forceinline__ bool fx_add(unsigned long long* acc, double v) {
    if (v == 0.0) return true;
    if (!(v > 0.0) || v >= 0x1p111) return false;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const int be = (int)(bits >> 52);                                    // biased exponent (v > 0)
    if (be == 0) return true;                                            // subnormal: below 2^-80
    unsigned long long m = (bits & 0xFFFFFFFFFFFFFull) | (1ull << 52);  // v = m * 2^(be - 1075)
    int sh = be - 1075 + 80;                                             // accumulator bit of m's LSB
    if (sh < 0) {
        if (sh <= -64) return true;                                      // below 2^-80
        m >>= -sh;
        sh = 0;
    }
    const int k = sh >> 5, r = sh & 31;                                  // digit k, bit r (k <= 4)
    // m << r spans at most 85 bits: digits k, k+1, k+2
    atomicAdd(acc + k, (m << r) & 0xFFFFFFFFull);
    const unsigned long long d1 = (m >> (32 - r)) & 0xFFFFFFFFull, d2 = r ? m >> (64 - r) : 0ull;
    if (d1) atomicAdd(acc + k + 1, d1);
    if (d2 && k + 2 < FA_FX_DIGITS) atomicAdd(acc + k + 2, d2);  // (d2 == 0 for k == 4: v < 2^111)
    return true;
}

// ---- cp.async (LDGSTS): global -> shared copies that complete in the background
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// ---- bulk copies (TMA engine, cp.async.bulk): one thread moves a contiguous
// block global -> shared; completion is counted in bytes on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make mbarrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// bytes: a multiple of 16; smem and g: 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, unsigned bytes, unsigned long long* bar) {
    const unsigned b = smem_u32(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem)),
                 "l"(g), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "FA_MBAR_WAIT%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FA_MBAR_WAIT%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- programmatic dependent launch (PDL) ---------------------------------
// Frame kernels are launched with programmatic stream serialization, so a
// kernel's CTAs are scheduled while its predecessor drains instead of after
// it.  Every such kernel starts with FA_PDL_PROLOGUE(): wait until the
// predecessor grid has completed and its writes are visible (before ANY
// global read or write), then let the successor be scheduled.  Both are
// no-ops when the kernel was launched without the attribute.
__device__ __forceinline__ void fa_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void fa_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#ifdef FA_TRACE
// Debug builds only (tools/trace_frame.py): each kernel's first block start
// and last block-0-thread exit per frame, from %globaltimer, into a
// host-bound buffer (one pointer per translation unit, bound by
// fa_debug_trace_reset); a kernel is keyed by FA_TU_ID * 100000 + the line of
// its FA_PDL_PROLOGUE.
struct fa_trace_rec {
    unsigned long long name, start, end, hits;
};
static __device__ fa_trace_rec* g_fa_trace;
__device__ __forceinline__ unsigned long long fa_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifndef FA_TU_ID
#define FA_TU_ID 0
#endif
struct FaTraceGuard {
    int slot = -1;
    __device__ FaTraceGuard(unsigned long long key) {
        if (!g_fa_trace || threadIdx.x != 0) return;
        int h = (int)(((key >> 4) * 2654435761ull) & 127);
        for (int k = 0; k < 128; k++, h = (h + 1) & 127) {
            unsigned long long cur = atomicCAS(&g_fa_trace[h].name, 0ull, key);
            if (cur == 0ull || cur == key) { slot = h; break; }
        }
        if (slot >= 0) {
            atomicMin(&g_fa_trace[slot].start, fa_gtime());
            if (blockIdx.x == 0 && blockIdx.y == 0) atomicAdd(&g_fa_trace[slot].hits, 1ull);
        }
    }
    __device__ ~FaTraceGuard() {
        if (slot >= 0) atomicMax(&g_fa_trace[slot].end, fa_gtime());
    }
};
#define FA_TRACE_TU(tu) \
    void fa_trace_bind_##tu(void* p) { cudaMemcpyToSymbol(g_fa_trace, &p, sizeof(p)); }
#define FA_PDL_PROLOGUE() \
    fa_pdl_wait();        \
    fa_pdl_trigger();     \
    FaTraceGuard _fa_trace_guard((unsigned long long)FA_TU_ID * 100000ull + __LINE__)
#else
#define FA_TRACE_TU(tu)
#define FA_PDL_PROLOGUE() \
    do {                  \
        fa_pdl_wait();    \
        fa_pdl_trigger(); \
    } while (0)
#endif

bool fa_pdl_enabled();  // FASTATLAS_PDL=0 disables (fa_api.cu)
int fa_env_int(const char* name, int dflt);  // integer knob from the environment (fa_api.cu)

// Grid for a grid-stride kernel over device-counted work (the visible
// triangles): one resident wave -- every CTA fits on the GPU at once, so under
// PDL the whole grid is already resident when its predecessor finishes -- or,
// with FASTATLAS_WAVES=0, the former cap of `cap` CTAs.
template <typename... KArgs>
static inline int fa_wave_grid(void (*k)(KArgs...), int threads, size_t smem, long long max_blocks, int cap) {
    static const int waves = fa_env_int("FASTATLAS_WAVES", 1);
    if (waves <= 0) return (int)(max_blocks < cap ? max_blocks : cap);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    long long g = (long long)FA_NUM_SMS * per_sm * waves;
    if (g > max_blocks) g = max_blocks;
    return (int)(g < 1 ? 1 : g);
}

template <typename... KArgs, typename... Args>
static inline void fa_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = fa_pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Grid-stride kernels cap their grid at a multiple of the SM count; the cap
// scale (FASTATLAS_GRID_CAP, default 1) trades single-frame latency for room
// that concurrent frames' kernels can share.
float fa_grid_cap_scale();
static inline int fa_cap(int max_blocks) {
    int c = (int)(max_blocks * fa_grid_cap_scale());
    return c > 0 ? c : 1;
}

static inline int fa_grid(long long n, int block, int max_blocks) {
    max_blocks = fa_cap(max_blocks);
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

// 32-byte read-only load of a clip-space vertex (two 128-bit LDG.NC)
__device__ __forceinline__ double4 ldg4(const double4* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// Clip-space vertices for the paths that need them (clipping, and the bounds /
// UV fallbacks of triangles with a vertex outside the frustum): read from a
// stored array, or recomputed from the positions with the projection's own
// FMA chain (same bits), so the frame never writes the (V,4) clip array.
struct ClipSrc {
    const double4* clip;  // stored clip coordinates, or nullptr:
    const double* pos;    // (V,3) positions and
    const double* vp;     // the device view-projection matrix (row-major)
    __device__ __forceinline__ double4 operator()(int v) const {
        if (clip) return ldg4(clip + v);
        double m[16];
#pragma unroll
        for (int i = 0; i < 16; i++) m[i] = __ldg(vp + i);
        return project_point(__ldg(pos + 3 * (long long)v), __ldg(pos + 3 * (long long)v + 1),
                             __ldg(pos + 3 * (long long)v + 2), m);
    }
};

// ---- per-chart box dims (geometry.py:352-362 viewport_box + cli.py:379-384) --
// NDC box -> (w_px, h_px) = max(1, ceil(extent/2 * W)) -> target dims
// max(1, ceil(prescale * dim)); the packer's inputs for j < cap.  Shared by
// k_box_dims and the frame's fused order kernel.
struct fa_box_dims_args {
    const unsigned long long* keys;  // 4 order-preserving keys per chart (min x, min y, max x, max y)
    const int* survived;
    const int* roots;
    int W, H;
    double prescale;
    double* ndc;
    int* px;
    long long* target;
    long long* otw;
    long long* oth;
    long long* cid;
    int cap;
};

__device__ __forceinline__ void fa_box_dims_one(const fa_box_dims_args& a, int j, fa_dstat* st,
                                                long long* out_tw = nullptr, long long* out_th = nullptr) {
    if (!a.survived[j]) atomicOr(&st->flags, FA_DFLAG_DEGENERATE_CHART);
    double mnx = key_f64(a.keys[4 * j]), mny = key_f64(a.keys[4 * j + 1]);
    double mxx = key_f64(a.keys[4 * j + 2]), mxy = key_f64(a.keys[4 * j + 3]);
    a.ndc[4 * j] = mnx;
    a.ndc[4 * j + 1] = mny;
    a.ndc[4 * j + 2] = mxx;
    a.ndc[4 * j + 3] = mxy;
    double fw = ceil(__dmul_rn(__ddiv_rn(__dsub_rn(mxx, mnx), 2.0), (double)a.W));
    double fh = ceil(__dmul_rn(__ddiv_rn(__dsub_rn(mxy, mny), 2.0), (double)a.H));
    long long w = fw < 1.0 ? 1 : (long long)fw;
    long long h = fh < 1.0 ? 1 : (long long)fh;
    a.px[2 * j] = (int)w;
    a.px[2 * j + 1] = (int)h;
    double tw = ceil(__dmul_rn(a.prescale, (double)w));
    double th = ceil(__dmul_rn(a.prescale, (double)h));
    long long itw = tw < 1.0 ? 1 : (long long)tw, ith = th < 1.0 ? 1 : (long long)th;
    a.target[2 * j] = itw;
    a.target[2 * j + 1] = ith;
    if (out_tw) { *out_tw = itw; *out_th = ith; }
    if (j >= a.cap) {
        atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
        return;
    }
    a.otw[j] = itw;
    a.oth[j] = ith;
    a.cid[j] = a.roots[j];
}
