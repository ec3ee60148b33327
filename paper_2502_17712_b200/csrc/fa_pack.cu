// fa_pack.cu — orient/order, candidate-parallel fold + push-up packing.
//
// Reference: packing.py:109-362.
//   * orient/order (packing.py:109-130): one CTA; stable LSD radix sort
//     (8-bit digits, warp match_any ranking) on the composite key
//     (h descending, min_tri ascending).  In the frame path the boxes
//     arrive in ascending-root order, so only the height digits are sorted.
//   * pack (packing.py:295-345): one CTA per scale candidate.  Each CTA runs
//     up to 9 rounds of [scaled dims -> block max -> block prefix-sum fold
//     -> overflow m -> exact dyadic snap] (packing.py:245-268), the
//     pigeonhole check, and push_up (packing.py:170-215) against a
//     shared-memory frontline: rows in order, each row's boxes handled by
//     thread groups sized to the row population (max over the column span,
//     then write back the new top; boxes of one row never overlap when
//     m == 0, so no intra-row barrier is needed).
//   * selection (packing.py:342-345): the largest accepted candidate index.
// All scale arithmetic is exact integer arithmetic with numpy int64
// semantics; the snap uses 128-bit intermediates.
#define FA_TU_ID 5  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"

#ifndef PK_THREADS
#define PK_THREADS 512  // measured on B200: 512 > 1024 > 256 threads per candidate CTA at C2
#endif
#define SORT_THREADS 1024

#include "fa_pack.cuh"

// u128 helpers for the snap (packing.py:353-362)
struct u128 {
    unsigned long long hi, lo;
};
__device__ __forceinline__ u128 mul64(unsigned long long a, unsigned long long b) {
    u128 r;
    r.lo = a * b;
    r.hi = __umul64hi(a, b);
    return r;
}
__device__ __forceinline__ bool ge128(u128 a, u128 b) { return a.hi != b.hi ? a.hi > b.hi : a.lo >= b.lo; }
__device__ __forceinline__ u128 sub128(u128 a, u128 b) {
    u128 r;
    r.lo = a.lo - b.lo;
    r.hi = a.hi - b.hi - (a.lo < b.lo ? 1ull : 0ull);
    return r;
}
__device__ __forceinline__ u128 shl128(u128 a, int s) {
    if (s == 0) return a;
    u128 r;
    if (s >= 64) { r.hi = a.lo << (s - 64); r.lo = 0; }
    else { r.hi = (a.hi << s) | (a.lo >> (64 - s)); r.lo = a.lo << s; }
    return r;
}
// floor(n / d) for d != 0, restoring division
__device__ u128 div128(u128 n, u128 d) {
    u128 q = {0, 0}, r = {0, 0};
    for (int i = 127; i >= 0; i--) {
        r = shl128(r, 1);
        unsigned long long bit = i >= 64 ? (n.hi >> (i - 64)) & 1ull : (n.lo >> i) & 1ull;
        r.lo |= bit;
        if (ge128(r, d)) {
            r = sub128(r, d);
            if (i >= 64) q.hi |= 1ull << (i - 64); else q.lo |= 1ull << i;
        }
    }
    return q;
}

// exact floor(n / d) for 0 < d < 2^60 when the quotient is <= 2^25 (the
// snap: num <= den bounds it by 2^24): an FP32 MUFU reciprocal refined by one
// FP64 Newton step (relative error < 2^-40) puts the estimate within one of
// the quotient; the remainder checks make it exact.
__device__ __forceinline__ unsigned long long floor_div_snap(unsigned long long n, unsigned long long d) {
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)d));
    const double dd = (double)d;
    double r = (double)rf;
    r = __dmul_rn(r, __dsub_rn(2.0, __dmul_rn(dd, r)));
    unsigned long long q = (unsigned long long)__dmul_rn((double)n, r);
    long long rem = (long long)(n - q * d);  // |rem| < 3d: exact as a wrapped difference
    while (rem < 0) { q -= 1; rem += (long long)d; }
    while (rem >= (long long)d) { q += 1; rem -= (long long)d; }
    return q;
}

// (num, den) <- reduce(floor(num*omega*2^24 / (den*(omega+m))), 2^24)
__device__ __forceinline__ void snap_scale(long long& num, long long& den, long long omega, long long m) {
    long long fn;
    unsigned long long nw = (unsigned long long)num * (unsigned long long)omega;
    unsigned long long dd = (unsigned long long)den * (unsigned long long)(omega + m);
    if (num >= 0 && num < (1ll << 31) && omega < (1ll << 31) && (nw >> 40) == 0 && den > 0 &&
        den < (1ll << 31) && (omega + m) < (1ll << 32)) {
        // common case: numerator fits in 64 bits, quotient < 2^25
        const unsigned long long nn = nw << FA_SCALE_GRID_BITS;
        fn = dd < (1ull << 60) ? (long long)floor_div_snap(nn, dd) : (long long)(nn / dd);
    } else {
        u128 n = mul64((unsigned long long)num, (unsigned long long)omega);  // < 2^116 overall after shift
        n = shl128(n, FA_SCALE_GRID_BITS);
        u128 d = mul64((unsigned long long)den, (unsigned long long)(omega + m));
        u128 f = div128(n, d);
        fn = (long long)f.lo;  // < 2^24 since scale <= 1
    }
    if (fn == 0) { num = 0; den = 1; return; }
    int tz = __ffsll(fn) - 1;
    if (tz > FA_SCALE_GRID_BITS) tz = FA_SCALE_GRID_BITS;
    num = fn >> tz;
    den = (1ll << FA_SCALE_GRID_BITS) >> tz;
}

// ============================================================================
// orient + order: single CTA stable LSD radix sort
// ============================================================================
struct SortSmem {
    int hist[256];
    int base[256];
    int wcnt[32][257];
    long long red[33];
    int flag;
};

// one stable pass on digit `shift` of 64-bit keys: (ki,vi) -> (ko,vo)
__device__ void radix_pass(const unsigned long long* ki, const int* vi, unsigned long long* ko, int* vo, int n,
                           int shift, SortSmem& sm) {
    int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    for (int i = tid; i < 256; i += blockDim.x) sm.hist[i] = 0;
    for (int i = tid; i < 32 * 257; i += blockDim.x) (&sm.wcnt[0][0])[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) atomicAdd(&sm.hist[(ki[i] >> shift) & 255ull], 1);
    __syncthreads();
    if (tid < 32) {
        // exclusive scan of 256 bins by one warp (8 per lane)
        int loc[8], s = 0;
        for (int j = 0; j < 8; j++) { loc[j] = sm.hist[lane * 8 + j]; s += loc[j]; }
        int incl = s;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int run = incl - s;
        for (int j = 0; j < 8; j++) { sm.base[lane * 8 + j] = run; run += loc[j]; }
    }
    __syncthreads();
    for (int t0 = 0; t0 < n; t0 += blockDim.x) {
        int i = t0 + tid;
        bool valid = i < n;
        unsigned long long k = valid ? ki[i] : 0ull;
        int v = valid ? vi[i] : 0;
        int d = valid ? (int)((k >> shift) & 255ull) : 256;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & ((1u << lane) - 1u));
        if (rank == 0) sm.wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int off = 0;
            for (int w = 0; w < warp; w++) off += sm.wcnt[w][d];
            int pos = sm.base[d] + off + rank;
            ko[pos] = k;
            vo[pos] = v;
        }
        __syncthreads();
        if (tid < 256) {
            int s = 0;
            for (int w = 0; w < 32; w++) { s += sm.wcnt[w][tid]; sm.wcnt[w][tid] = 0; }
            sm.base[tid] += s;
        }
        if (tid < 32) sm.wcnt[tid][256] = 0;
        __syncthreads();
    }
}

// Frame mode (mt == nullptr): input order already ascending min_tri.
// With bd.keys set (frame mode) the per-chart box dims are computed first
// (fa_box_dims_one, formerly its own launch); tw/th are then the dims this
// block just wrote, so they are read without __restrict__ (no .nc loads).
__global__ void __launch_bounds__(SORT_THREADS) k_orient_sort(const long long* tw,
                                                              const long long* th,
                                                              const long long* __restrict__ mt, int n_max,
                                                              const int* __restrict__ n_dev, long long max_h,
                                                              long long* __restrict__ ow, long long* __restrict__ oh,
                                                              unsigned char* __restrict__ rot, int* __restrict__ perm,
                                                              int* __restrict__ pinv, unsigned long long* sk,
                                                              int* sv, int reject_dups, fa_dstat* __restrict__ st,
                                                              fa_box_dims_args bd) {
    FA_PDL_PROLOGUE();
    if (bd.keys) {
        const int nc = n_dev ? *n_dev : n_max;
        for (int j = threadIdx.x; j < nc; j += blockDim.x) fa_box_dims_one(bd, j, st);
        __syncthreads();
    }
    __shared__ SortSmem sm;
    int n = n_dev ? *n_dev : n_max;
    if (n > n_max) {
        if (threadIdx.x == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
        return;
    }
    int tid = threadIdx.x;
    long long hmax = 0, hmin = 0x7fffffffffffffffll, mmin = 0x7fffffffffffffffll, mmax = 0;
    bool overflow = false;
    for (int i = tid; i < n; i += blockDim.x) {
        long long w = tw[i], h = th[i];
        long long oh_ = w > h ? w : h;
        if (oh_ > max_h) overflow = true;
        hmax = oh_ > hmax ? oh_ : hmax;
        hmin = oh_ < hmin ? oh_ : hmin;
        if (mt) {
            mmin = mt[i] < mmin ? mt[i] : mmin;
            mmax = mt[i] > mmax ? mt[i] : mmax;
        }
    }
    if (tid == 0) sm.flag = 0;
    __syncthreads();
    if (overflow) sm.flag = 1;
    hmax = block_max_ll(hmax, sm.red);
    hmin = -block_max_ll(-hmin, sm.red);
    if (mt) {
        mmax = block_max_ll(mmax, sm.red);
        mmin = -block_max_ll(-mmin, sm.red);
    }
    if (sm.flag) {
        if (tid == 0) atomicOr(&st->flags, FA_DFLAG_HEIGHT_OVERFLOW);
        return;
    }
    if (n == 0) return;
    if (tid == 0) st->max_h = (int)hmax;
    int hbits = 0;
    while (hbits < 63 && ((hmax - hmin) >> hbits) != 0) hbits++;
    int mbits = 0;
    if (mt)
        while (mbits < 63 && ((unsigned long long)(mmax - mmin) >> mbits) != 0) mbits++;
    if (hbits + mbits > 64) {
        if (tid == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);  // key range unsupported
        return;
    }
    // composite key: (hmax - h) above a byte-aligned (mt - mmin) field, so the
    // first ceil(mbits/8) LSD passes leave the array ordered by min_tri alone
    int mfield = 8 * ((mbits + 7) / 8);
    if (hbits + mfield > 64) {
        if (tid == 0) atomicOr(&st->flags, FA_DFLAG_KEY_RANGE);
        return;
    }
    unsigned long long* ka = sk;
    unsigned long long* kb = sk + n_max;
    int* va = sv;
    int* vb = sv + n_max;
    for (int i = tid; i < n; i += blockDim.x) {
        long long w = tw[i], h = th[i];
        long long oh_ = w > h ? w : h;
        unsigned long long key = mfield < 64 ? ((unsigned long long)(hmax - oh_) << mfield) : 0ull;
        if (mt) key |= (unsigned long long)(mt[i] - mmin);
        ka[i] = key;
        va[i] = i;
    }
    __syncthreads();
    int mpasses = mfield / 8;
    int passes = mpasses + (hbits + 7) / 8;
    if (mt && reject_dups && mpasses == 0 && n > 1) {
        // every min_tri equal: duplicates (packing.py:319-323)
        if (tid == 0) atomicOr(&st->flags, FA_DFLAG_DUPLICATE_MIN_TRI);
        return;
    }
    for (int p = 0; p < passes; p++) {
        radix_pass(ka, va, kb, vb, n, 8 * p, sm);
        unsigned long long* tk = ka; ka = kb; kb = tk;
        int* tv = va; va = vb; vb = tv;
        if (mt && reject_dups && p == mpasses - 1) {
            // ordered by min_tri: adjacent equal ids are duplicates (packing.py:319-323)
            for (int j = tid + 1; j < n; j += blockDim.x)
                if (mt[va[j - 1]] == mt[va[j]]) sm.flag = 1;
            __syncthreads();
            if (sm.flag) {
                if (tid == 0) atomicOr(&st->flags, FA_DFLAG_DUPLICATE_MIN_TRI);
                return;
            }
        }
    }
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) {
        int i = va[j];
        long long w = tw[i], h = th[i];
        bool r = w > h;
        perm[j] = i;
        pinv[i] = j;
        ow[j] = r ? h : w;
        oh[j] = r ? w : h;
        rot[j] = r;
    }
}

// ---- the frame's order: box dims + orient + order, in shared memory -------
// The frame path of k_orient_sort (box dims at the head, charts in
// ascending-root order, so a stable radix sort on the height alone gives
// (-h, min_tri), packing.py:109-130) with every intermediate kept on chip:
// the dims stay in shared memory instead of a global write-and-read-back, the
// radix ping-pong arrays are shared memory (up to `cap` charts; beyond it the
// global scratch), and the outputs are fire-and-forget stores -- one global
// round trip (the bounds' keys) instead of about six.  Also writes the target
// dims and chart id of each packing position (ord_*), so the selection reads
// them without the perm indirection.
size_t fa_order_frame_smem(int cap) { return (size_t)cap * (4 + 4 + 8 + 8 + 4 + 4) + 64; }

__global__ void __launch_bounds__(SORT_THREADS) k_order_frame(fa_box_dims_args bd, const int* __restrict__ n_dev,
                                                              int n_max, int cap, long long max_h,
                                                              long long* __restrict__ ow, long long* __restrict__ oh,
                                                              unsigned char* __restrict__ rot, int* __restrict__ perm,
                                                              int* __restrict__ pinv, unsigned long long* sk, int* sv,
                                                              long long* __restrict__ ord_tw,
                                                              long long* __restrict__ ord_th,
                                                              long long* __restrict__ ord_cid,
                                                              fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    extern __shared__ __align__(16) unsigned char of_dyn[];
    __shared__ SortSmem sm;
    const int tid = threadIdx.x;
    const int n = *n_dev;
    if (n > n_max) {
        if (tid == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
        return;
    }
    const bool on_chip = n <= cap;
    unsigned long long* ka = reinterpret_cast<unsigned long long*>(of_dyn);
    unsigned long long* kb = ka + cap;
    int* va = reinterpret_cast<int*>(kb + cap);
    int* vb = va + cap;
    int* in_w = vb + cap;
    int* in_h = in_w + cap;
    if (!on_chip) {
        ka = sk;
        kb = sk + n_max;
        va = sv;
        vb = sv + n_max;
    }
    long long hmax = 0, nhmin = -0x7fffffffffffffffll;
    bool overflow = false;
    for (int j = tid; j < n; j += blockDim.x) {
        long long itw, ith;
        fa_box_dims_one(bd, j, st, &itw, &ith);
        const long long oh_ = itw > ith ? itw : ith;
        if (oh_ > max_h) overflow = true;
        hmax = oh_ > hmax ? oh_ : hmax;
        nhmin = -oh_ > nhmin ? -oh_ : nhmin;
        if (on_chip) {
            in_w[j] = (int)(itw < (1ll << 30) ? itw : (1ll << 30));
            in_h[j] = (int)(ith < (1ll << 30) ? ith : (1ll << 30));
        }
    }
    if (tid == 0) sm.flag = 0;
    __syncthreads();
    if (overflow) sm.flag = 1;
    {
        // hmax and -hmin in one pair of barriers
        long long a = warp_max_ll(hmax), b = warp_max_ll(nhmin);
        const int lane = lane_id(), wid = tid >> 5, nw = blockDim.x >> 5;
        __shared__ long long r2[2][32];
        if (lane == 0) { r2[0][wid] = a; r2[1][wid] = b; }
        __syncthreads();
        a = lane < nw ? r2[0][lane] : 0;
        b = lane < nw ? r2[1][lane] : -0x7fffffffffffffffll;
        hmax = warp_max_ll(a);
        nhmin = warp_max_ll(b);
    }
    if (sm.flag) {  // HeightOverflow (packing.py:127-129)
        if (tid == 0) atomicOr(&st->flags, FA_DFLAG_HEIGHT_OVERFLOW);
        return;
    }
    if (n == 0) return;
    if (tid == 0) st->max_h = (int)hmax;
    const long long hmin = -nhmin;
    int hbits = 0;
    while (hbits < 63 && ((hmax - hmin) >> hbits) != 0) hbits++;
    for (int j = tid; j < n; j += blockDim.x) {
        const long long w = on_chip ? in_w[j] : bd.otw[j], h = on_chip ? in_h[j] : bd.oth[j];
        ka[j] = (unsigned long long)(hmax - (w > h ? w : h));
        va[j] = j;
    }
    __syncthreads();
    for (int q = 0; q < (hbits + 7) / 8; q++) {
        radix_pass(ka, va, kb, vb, n, 8 * q, sm);
        unsigned long long* tk = ka; ka = kb; kb = tk;
        int* tv = va; va = vb; vb = tv;
    }
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) {
        const int i = va[j];
        const long long w = on_chip ? in_w[i] : bd.otw[i], h = on_chip ? in_h[i] : bd.oth[i];
        const bool r = w > h;
        perm[j] = i;
        pinv[i] = j;
        ow[j] = r ? h : w;
        oh[j] = r ? w : h;
        rot[j] = r;
        ord_tw[j] = w;
        ord_th[j] = h;
        ord_cid[j] = bd.roots[i];
    }
}

// ============================================================================
// packing candidates
// ============================================================================
struct PackSmem {
    long long red[33];
    long long red2[33];
    int red_i[32];
    int flag;
    int part_sum[2][32], part_max[2][32], part_m[2][32];  // narrow rounds: per-warp partials (double-buffered)
};

// block max of two values at once (one pair of barriers); red/red2 hold 33
__device__ __forceinline__ void block_max2_ll(long long& a, long long& b, long long* red, long long* red2) {
    int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    a = warp_max_ll(a);
    b = warp_max_ll(b);
    if (lane == 0) {
        red[wid] = a;
        red2[wid] = b;
    }
    __syncthreads();
    if (wid == 0) {
        long long x = lane < nw ? red[lane] : (long long)0x8000000000000000ll;
        long long y = lane < nw ? red2[lane] : (long long)0x8000000000000000ll;
        x = warp_max_ll(x);
        y = warp_max_ll(y);
        if (lane == 0) {
            red[32] = x;
            red2[32] = y;
        }
    }
    __syncthreads();
    a = red[32];
    b = red2[32];
}

// boxes per thread kept in registers by the fold rounds (n <= KREG * PK_THREADS):
// pack_candidate<4> and, for larger frames, pack_candidate<PK_KREG_WIDE>
#ifndef PK_KREG_WIDE
#define PK_KREG_WIDE 8
#endif

#ifdef FA_PACK_PROF
// debug build only: per candidate CTA [t_fold_done, t_heights, t_rowstart, t_rows_done, iterations, rows]
__device__ long long g_pack_prof[256][12];
extern "C" void fa_debug_pack_prof(long long* out) { cudaMemcpyFromSymbol(out, g_pack_prof, sizeof(g_pack_prof)); }
#define PACK_MARK(k, v) \
    if (threadIdx.x == 0 && blockIdx.x < 256) g_pack_prof[blockIdx.x][k] = (v)
#else
#define PACK_MARK(k, v)
#endif

// max of f[a, b) (>= 0: the frontline starts at 0 and only rises) and fill of
// f[a, b), 16-byte vector accesses in the aligned middle
__device__ __forceinline__ int span_max(const int* f, int a, int b) {
    int m = 0, c = a;
    for (; c < b && (reinterpret_cast<uintptr_t>(f + c) & 15); c++) m = max(m, f[c]);
    for (; c + 4 <= b; c += 4) {
        const int4 v = *reinterpret_cast<const int4*>(f + c);
        m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
    }
    for (; c < b; c++) m = max(m, f[c]);
    return m;
}
__device__ __forceinline__ void span_fill(int* f, int a, int b, int v) {
    int c = a;
    for (; c < b && (reinterpret_cast<uintptr_t>(f + c) & 15); c++) f[c] = v;
    for (; c + 4 <= b; c += 4) *reinterpret_cast<int4*>(f + c) = make_int4(v, v, v, v);
    for (; c < b; c++) f[c] = v;
}

// One candidate: returns accept; fills cand_w/h/p/y/rowstart for the CTA.
template <int PK_KREG, typename DimT>
__device__ bool pack_candidate(const DimT* __restrict__ ow, const DimT* __restrict__ oh, int n,
                               long long num, long long den, long long omega, int kbits, long long min_dim,
                               long long pad, int* cw, int* ch, long long* cp, int* cy, int* rowstart, int* front,
                               long long& out_num, long long& out_den, long long& out_used, PackSmem& sm,
                               int* sbox = nullptr, int n_sbox = 0) {
    int tid = threadIdx.x;
    bool have_fold = false;
    long long m = 0;
#ifdef FA_PACK_PROF
    long long t0 = clock64();
    PACK_MARK(0, 0);
    PACK_MARK(1, 0);
    PACK_MARK(2, 0);
    PACK_MARK(3, 0);
    PACK_MARK(4, 0);
    PACK_MARK(5, 0);
#endif
    const int K = (n + blockDim.x - 1) / blockDim.x;
    if (K <= PK_KREG) {
        // Register-resident rounds: thread tid owns boxes [tid*K, tid*K + K);
        // widths, the running fold offset and the overflow stay in registers,
        // so a round is the divisions + one block scan + one paired max.
        const int b0 = tid * K;
        long long owr[PK_KREG], ohr[PK_KREG], wr[PK_KREG];
        long long owmax = -1, negmin = 0;
        // the fast tail (heights + push-up from shared memory) needs the
        // heights too: loaded with the widths, off the critical path
        const bool fast_tail = sbox != nullptr && n <= n_sbox && omega < (1ll << 30);
#pragma unroll
        for (int k = 0; k < PK_KREG; k++) {
            owr[k] = (k < K && b0 + k < n) ? ow[b0 + k] : 0;
            ohr[k] = (fast_tail && k < K && b0 + k < n) ? oh[b0 + k] : 0;
            owmax = owr[k] > owmax ? owr[k] : owmax;
            negmin = -owr[k] > negmin ? -owr[k] : negmin;
        }
        // Narrow rounds: with scale <= 1 every width is <= wb, so when n*wb
        // < 2^31 all prefix sums and overflows fit int32: warp scans on
        // 32-bit values, REDUX max, and one barrier per block reduction
        // (every thread combines the per-warp partials itself).
        block_max2_ll(owmax, negmin, sm.red, sm.red2);
        PACK_MARK(10, clock64() - t0);
        const long long wb = (owmax > min_dim ? owmax : min_dim) + 2 * pad;
        const bool narrow = negmin <= 0 && owmax >= 0 && owmax < (1ll << 31) && wb < (1ll << 31) &&
                            (long long)n * wb < (1ll << 31);
        const int lane = lane_id(), wid = tid >> 5, nw = blockDim.x >> 5;
        int pb = 0;
        long long base = 0;
        for (int it = 0; it < FA_MAX_OVERFLOW_ITERS + 1; it++) {
            PACK_MARK(4, it + 1);
#ifdef FA_PACK_PROF
            long long ti = clock64();
#endif
            long long wmax = 0, local = 0;
            // after a snap the denominator is a power of two: the ceiling is
            // a shift (non-negative num*t < 2^62, the numpy value exactly)
            const bool pow2 = den > 0 && (den & (den - 1)) == 0 && num >= 0 && num < (1ll << 31);
            const double rdn = pow2 ? 0.0 : 1.0 / (double)den;
            const int dsh = pow2 ? __ffsll(den) - 1 : 0;
#pragma unroll
            for (int k = 0; k < PK_KREG; k++) {
                long long w = 0;
                if (k < K && b0 + k < n) {
                    if (pow2 && owr[k] >= 0 && owr[k] < (1ll << 31)) {
                        w = (num * owr[k] + (den - 1)) >> dsh;
                        w = (w < min_dim ? min_dim : w) + 2 * pad;
                    } else {
                        w = scaled_dim_rcp(owr[k], num, den, rdn, min_dim, pad);
                    }
                }
                wr[k] = w;
                wmax = w > wmax ? w : wmax;
                local += w;
            }
#ifdef FA_PACK_PROF
            if (it == 1) PACK_MARK(6, clock64() - ti);
#endif
            long long mloc = -(1ll << 62);
            if (narrow) {
                int x = (int)local;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const int wm = __reduce_max_sync(0xffffffffu, (int)wmax);
                if (lane == 31) sm.part_sum[pb][wid] = x;
                if (lane == 0) sm.part_max[pb][wid] = wm;
                __syncthreads();
                // every warp combines the partials itself: one load per lane + REDUX
                const int ps = lane < nw ? sm.part_sum[pb][lane] : 0;
                const int pm = lane < nw ? sm.part_max[pb][lane] : 0;
                const int pre = __reduce_add_sync(0xffffffffu, lane < wid ? ps : 0);
                const int bw = __reduce_max_sync(0xffffffffu, pm);
                base = (long long)(pre + x - (int)local);
                wmax = bw;
#ifdef FA_PACK_PROF
                if (it == 1) PACK_MARK(7, clock64() - ti);
#endif
                int p = (int)base, ml = -(1 << 30) - 1;
                const int om = (int)omega;
#pragma unroll
                for (int k = 0; k < PK_KREG; k++) {
                    if (k < K && b0 + k < n) {
                        const int over = (p & (om - 1)) + (int)wr[k] - om;
                        ml = over > ml ? over : ml;
                        p += (int)wr[k];
                    }
                }
                ml = __reduce_max_sync(0xffffffffu, ml);
                if (lane == 0) sm.part_m[pb][wid] = ml;
                __syncthreads();
                mloc = __reduce_max_sync(0xffffffffu, lane < nw ? sm.part_m[pb][lane] : -(1 << 30) - 1);
                pb ^= 1;
            } else {
                long long tot;
                base = block_exclusive_scan_ll(local, sm.red, &tot);
#ifdef FA_PACK_PROF
                if (it == 1) PACK_MARK(7, clock64() - ti);
#endif
                long long p = base;
#pragma unroll
                for (int k = 0; k < PK_KREG; k++) {
                    if (k < K && b0 + k < n) {
                        long long q = p & (omega - 1);
                        long long over = q + wr[k] - omega;
                        mloc = over > mloc ? over : mloc;
                        p += wr[k];
                    }
                }
                block_max2_ll(wmax, mloc, sm.red, sm.red2);
            }
#ifdef FA_PACK_PROF
            if (it == 1) PACK_MARK(8, clock64() - ti);
#endif
            if (wmax > omega) {
                m = wmax - omega;  // no fold: the widest box alone overflows
            } else {
                m = mloc > 0 ? mloc : 0;
                have_fold = true;
            }
#ifdef FA_PACK_PROF
            if (it == 0) PACK_MARK(11, clock64() - t0);
#endif
            if (m == 0) break;
            have_fold = false;
            snap_scale(num, den, omega, m);
#ifdef FA_PACK_PROF
            if (it == 1) PACK_MARK(9, clock64() - ti);
#endif
        }
        long long p = base;
        long long pr[PK_KREG];
#pragma unroll
        for (int k = 0; k < PK_KREG; k++) {
            pr[k] = p;
            if (k < K && b0 + k < n) {
                cw[b0 + k] = (int)wr[k];
                cp[b0 + k] = p;
                p += wr[k];
            }
        }
        if (fast_tail) {
            // Fast tail: the heights come from registers and the push-up
            // reads its boxes from shared memory (x, w, h and the row
            // starts), so a row costs shared-memory round trips and one
            // barrier instead of dependent global loads.  With m == 0 no box
            // straddles a row boundary, so box b starts row r exactly when
            // its fold offset is a multiple of omega.
            PACK_MARK(0, clock64() - t0);
            if (!have_fold || m != 0) return false;  // block-uniform
            int* sx = sbox;
            int* sw = sx + n_sbox;
            int* sh = sw + n_sbox;
            int* srs = sh + n_sbox;
            const double rdh = 1.0 / (double)den;
            unsigned long long area = 0;
#pragma unroll
            for (int k = 0; k < PK_KREG; k++) {
                const int b = b0 + k;
                if (k < K && b < n) {
                    const long long h = scaled_dim_rcp(ohr[k], num, den, rdh, min_dim, pad);
                    ch[b] = (int)h;
                    area += (unsigned long long)wr[k] * (unsigned long long)h;
                    const long long q = pr[k] & (omega - 1);
                    const int r = (int)(pr[k] >> kbits);
                    const bool left = (r % FA_DIRECTION_PERIOD) == 0;
                    sx[b] = left ? (int)q : (int)(omega - q - wr[k]);
                    sw[b] = (int)wr[k];
                    sh[b] = h > omega ? (int)(omega + 1) : (int)h;  // taller boxes reject anyway (saturated)
                    if (q == 0) srs[r] = b;
                    if (b == n - 1) sm.flag = r + 1;
                }
            }
            for (int c = tid; c <= omega; c += blockDim.x) front[c] = 0;
            area = (unsigned long long)block_sum_ll((long long)area, sm.red);  // its barriers publish sx..srs
            PACK_MARK(1, clock64() - t0);
            if ((long long)area > omega * omega) return false;
            const int n_rows = sm.flag;
            PACK_MARK(2, clock64() - t0);
            PACK_MARK(5, n_rows);
            int used = 0;
            for (int r = 0; r < n_rows; r++) {
                const int rb0 = srs[r];
                const int nb = ((r + 1 < n_rows) ? srs[r + 1] : n) - rb0;
                int G = 32;
                while (G > 1 && G * nb > (int)blockDim.x) G >>= 1;
                const int groups = blockDim.x / G;
                const int g = tid / G, gl = tid % G;
                for (int gbase = 0; gbase < nb; gbase += groups) {
                    const int gb = gbase + g;
                    const bool act = gb < nb;
                    const int b = rb0 + (act ? gb : 0);
                    const int x = sx[b], w = act ? sw[b] : 0, h = sh[b];
                    int rest = 0;
                    if (G == 1) rest = span_max(front, x, x + w);
                    else
                        for (int c = x + gl; c < x + w; c += G) rest = max(rest, front[c]);
                    for (int o = G >> 1; o > 0; o >>= 1) rest = max(rest, __shfl_xor_sync(0xffffffffu, rest, o, G));
                    // saturate above omega: any such top already rejects the candidate
                    const int top = min(rest + h, (int)omega + 1);
                    if (act) {
                        if (G == 1) span_fill(front, x, x + w, top);
                        else
                            for (int c = x + gl; c < x + w; c += G) front[c] = top;
                        if (gl == 0) cy[b] = rest;
                        used = max(used, top);
                    }
                }
                __syncthreads();
            }
            const long long used_b = block_max_ll((long long)used, sm.red);
            PACK_MARK(3, clock64() - t0);
            out_used = used_b;
            if (used_b > omega) return false;
            long long g2 = gcd_ll(num, den);
            if (g2 == 0) g2 = 1;
            out_num = div_by_gcd(num, g2);
            out_den = div_by_gcd(den, g2);
            return true;
        }
        __syncthreads();
    } else
    for (int it = 0; it < FA_MAX_OVERFLOW_ITERS + 1; it++) {
        PACK_MARK(4, it + 1);
        long long wmax = 0;
        for (int b = tid; b < n; b += blockDim.x) {
            long long w = scaled_dim(ow[b], num, den, min_dim, pad);
            cw[b] = (int)w;
            wmax = w > wmax ? w : wmax;
        }
        // note: widths <= omega + ... stay well inside int32 (checked by host)
        wmax = block_max_ll(wmax, sm.red);
        if (wmax > omega) {
            m = wmax - omega;
            have_fold = false;
        } else {
            long long carry = 0, mloc = -(1ll << 62);
            for (int c0 = 0; c0 < n; c0 += blockDim.x) {
                int b = c0 + tid;
                long long w = b < n ? (long long)cw[b] : 0;
                long long tot;
                long long p = carry + block_exclusive_scan_ll(w, sm.red, &tot);
                if (b < n) {
                    cp[b] = p;
                    long long q = p & (omega - 1);
                    long long over = q + w - omega;
                    mloc = over > mloc ? over : mloc;
                }
                carry += tot;
            }
            mloc = block_max_ll(mloc, sm.red);
            m = mloc > 0 ? mloc : 0;
            have_fold = true;
        }
        if (m == 0) break;
        have_fold = false;
        snap_scale(num, den, omega, m);
    }
    PACK_MARK(0, clock64() - t0);
    if (!have_fold || m != 0) return false;
    // heights + pigeonhole (packing.py:271-274), int64 wrapping sum
    unsigned long long area = 0;
    for (int b = tid; b < n; b += blockDim.x) {
        long long h = scaled_dim_rcp(oh[b], num, den, 1.0 / (double)den, min_dim, pad);
        ch[b] = (int)h;
        area += (unsigned long long)cw[b] * (unsigned long long)h;
    }
    area = (unsigned long long)block_sum_ll((long long)area, sm.red);
    PACK_MARK(1, clock64() - t0);
    if ((long long)area > omega * omega) return false;
    // row starts
    for (int b = tid; b < n; b += blockDim.x) {
        long long r = cp[b] >> kbits;
        if (b == 0 || (cp[b - 1] >> kbits) != r) rowstart[r] = b;
    }
    for (int c = tid; c <= omega; c += blockDim.x) front[c] = 0;
    if (tid == 0) sm.flag = 0;
    __syncthreads();
    int n_rows = (int)(cp[n - 1] >> kbits) + 1;
    PACK_MARK(2, clock64() - t0);
    PACK_MARK(5, n_rows);
    long long used = 0;
    for (int r = 0; r < n_rows; r++) {
        int b0 = rowstart[r];
        int b1 = (r + 1 < n_rows) ? rowstart[r + 1] : n;
        int nb = b1 - b0;
        bool left = (r % FA_DIRECTION_PERIOD) == 0;
        int G = 32;
        while (G > 1 && G * nb > (int)blockDim.x) G >>= 1;
        int groups = blockDim.x / G;
        int g = tid / G, gl = tid % G;
        // block-uniform trip count: the group shuffles below are full-warp
        for (int gbase = 0; gbase < nb; gbase += groups) {
            int gb = gbase + g;
            bool act = gb < nb;
            int b = b0 + (act ? gb : 0);
            long long q = cp[b] & (omega - 1);
            int w = act ? cw[b] : 0;
            int x = left ? (int)q : (int)(omega - q - w);
            int rest = 0;
            if (G == 1) rest = span_max(front, x, x + w);  // one thread per box: 4 columns per load
            else
                for (int c = x + gl; c < x + w; c += G) rest = max(rest, front[c]);
            for (int o = G >> 1; o > 0; o >>= 1) rest = max(rest, __shfl_xor_sync(0xffffffffu, rest, o, G));
            // saturate above omega: any such top already rejects the candidate
            long long top64 = (long long)rest + ch[b];
            int top = top64 > omega ? (int)(omega + 1) : (int)top64;
            if (act) {
                if (G == 1) span_fill(front, x, x + w, top);
                else
                    for (int c = x + gl; c < x + w; c += G) front[c] = top;
                if (gl == 0) cy[b] = rest;
                used = top > used ? top : used;
            }
        }
        // groups are warp-aligned (G divides 32), so shuffles above are full-warp;
        // the barrier orders this row's writes before the next row's reads
        __syncthreads();
    }
    used = block_max_ll(used, sm.red);
    PACK_MARK(3, clock64() - t0);
    out_used = used;
    if (used > omega) return false;
    long long g2 = gcd_ll(num, den);
    if (g2 == 0) g2 = 1;
    out_num = div_by_gcd(num, g2);
    out_den = div_by_gcd(den, g2);
    return true;
}

// cand record: [accept, num, den, used, slot]
#define CAND_REC FA_CAND_REC

__global__ void __launch_bounds__(PK_THREADS) k_pack(const long long* __restrict__ ow, const long long* __restrict__ oh,
                                                     int n_max, const int* __restrict__ n_dev, long long omega,
                                                     int kbits, long long n_scales, long long first,
                                                     long long explicit_num, long long explicit_den, long long min_dim,
                                                     long long pad, long long* __restrict__ cand,
                                                     long long* __restrict__ cand_p, int* __restrict__ cand_w,
                                                     int* __restrict__ cand_h, int* __restrict__ cand_y,
                                                     int* __restrict__ rowstart, int* __restrict__ gfront,
                                                     fa_dstat* __restrict__ st, int n_sbox) {
    FA_PDL_PROLOGUE();
    // dynamic shared memory: the frontline (omega + 1 ints, unless it lives
    // in gfront), then the push-up's box arrays (x, w, h, row starts: n_sbox
    // each) when n_sbox > 0
    extern __shared__ int dyn_front[];
    __shared__ PackSmem sm;
    int n = n_dev ? *n_dev : n_max;
    if (n > n_max) {
        if (st && threadIdx.x == 0) atomicOr(&st->flags, FA_DFLAG_QUEUE_OVERFLOW);
        return;
    }
    long long i = first - blockIdx.x;  // candidates descending within a batch
    if (i < 1) return;
    if (st && st->done) return;
    if (n <= 0) return;
    if (st && (st->flags & (FA_DFLAG_HEIGHT_OVERFLOW | FA_DFLAG_KEY_RANGE | FA_DFLAG_DUPLICATE_MIN_TRI))) return;
    long long num, den;
    if (explicit_den > 0) {
        long long g = gcd_ll(explicit_num, explicit_den);
        num = div_by_gcd(explicit_num, g);
        den = div_by_gcd(explicit_den, g);
    } else {
        long long g = gcd_ll(i, n_scales);
        num = div_by_gcd(i, g);
        den = div_by_gcd(n_scales, g);
    }
    size_t slot = blockIdx.x;
    int* front = gfront ? gfront + slot * (size_t)(omega + 1) : dyn_front;
    int* sbox = n_sbox > 0 ? dyn_front + (gfront ? 0 : ((omega + 1 + 3) & ~3ll)) : nullptr;
    long long rn = 0, rd = 1, used = 0;
    // boxes per thread in registers: 4 up to 4 * blockDim boxes (the C2
    // frames), 8 beyond (C3's ~4000 charts), else the global-memory rounds
    const int K = (n + (int)blockDim.x - 1) / (int)blockDim.x;
#ifdef FA_PACK_TWICE
    // debug: a first, discarded run warms the instruction cache; the timed
    // (second) run then shows the per-phase cost without cold-code misses
    if (K <= 4)
        pack_candidate<4>(ow, oh, n, num, den, omega, kbits, min_dim, pad, cand_w + slot * n_max,
                          cand_h + slot * n_max, cand_p + slot * n_max, cand_y + slot * n_max,
                          rowstart + slot * n_max, front, rn, rd, used, sm, sbox, n_sbox);
    __syncthreads();
#endif
    bool ok = K <= 4 ? pack_candidate<4>(ow, oh, n, num, den, omega, kbits, min_dim, pad, cand_w + slot * n_max,
                                         cand_h + slot * n_max, cand_p + slot * n_max, cand_y + slot * n_max,
                                         rowstart + slot * n_max, front, rn, rd, used, sm, sbox, n_sbox)
                     : pack_candidate<PK_KREG_WIDE>(ow, oh, n, num, den, omega, kbits, min_dim, pad,
                                                    cand_w + slot * n_max, cand_h + slot * n_max,
                                                    cand_p + slot * n_max, cand_y + slot * n_max,
                                                    rowstart + slot * n_max, front, rn, rd, used, sm, sbox, n_sbox);
    if (threadIdx.x == 0) {
        long long* rec = cand + CAND_REC * (i - 1);
        rec[0] = ok;
        rec[1] = rn;
        rec[2] = rd;
        rec[3] = used;
        rec[4] = (long long)slot;
    }
}

// after a batch: done |= any accepted in [lo, hi]
__global__ void k_batch_done(const long long* __restrict__ cand, long long lo, long long hi, fa_dstat* st) {
    FA_PDL_PROLOGUE();
    bool any = false;
    for (long long i = lo + threadIdx.x; i <= hi; i += blockDim.x) any |= cand[CAND_REC * (i - 1)] != 0;
    if (__syncthreads_or(any) && threadIdx.x == 0) st->done = 1;
}

// selection (packing.py:327-345) + placements in packing order, by one CTA;
// red: 33 long longs of shared memory.  Array types are templated so the
// frame's fused pack (k_pack_frame) can pass its shared-memory copies.
template <typename OwT, typename TwT, typename RotT>
__device__ void select_body(const OwT* ow, const TwT* tw, const TwT* th, const int* __restrict__ chart_id_i,
                            const long long* __restrict__ chart_id, const RotT* rot, const int* perm, int n,
                            long long omega, long long n_scales, long long min_dim, long long pad,
                            const long long* __restrict__ cand, const long long* __restrict__ cand_p,
                            const int* __restrict__ cand_w, const int* __restrict__ cand_h,
                            const int* __restrict__ cand_y, int n_max, long long* __restrict__ placements,
                            int4* __restrict__ plc_by_src, unsigned char* __restrict__ accept_out,
                            fa_dstat* __restrict__ st, long long* red, long long* red2,
                            const long long* __restrict__ ord_tw = nullptr, const long long* __restrict__ ord_th = nullptr,
                            const long long* __restrict__ ord_cid = nullptr) {
    const int tid = threadIdx.x;
    if (n <= 0) {
        if (tid == 0) { st->scale_num = 1; st->scale_den = 1; st->best = -1; }
        return;
    }
    // this thread's first output item's selection-independent inputs, loaded
    // before the reductions so they are in flight beside them
    int src0 = 0, rot0 = 0;
    long long cid0 = 0, tw0 = 0, th0 = 0;
    if (tid < n) {
        src0 = perm[tid];
        rot0 = rot[tid];
        if (ord_tw) {
            cid0 = ord_cid[tid];
            tw0 = ord_tw[tid];
            th0 = ord_th[tid];
        }
    }
    // floor-scale width check (packing.py:327-332) and the largest accepted
    // candidate, reduced together (one pair of barriers; every thread gets both)
    long long fmax = 0;
    const double rdn = 1.0 / (double)n_scales;
    for (int b = tid; b < n; b += blockDim.x) {
        long long f = scaled_dim_rcp((long long)ow[b], 1, n_scales, rdn, min_dim, pad);
        fmax = f > fmax ? f : fmax;
    }
    long long best = 0;
    for (long long i = tid + 1; i <= n_scales; i += blockDim.x) {
        bool acc = cand[CAND_REC * (i - 1)] != 0 && cand[CAND_REC * (i - 1) + 4] >= 0;
        if (accept_out) accept_out[i - 1] = acc;
        if (acc && i > best) best = i;
    }
    block_max2_ll(fmax, best, red, red2);
    if (fmax > omega) best = 0;
    if (best == 0) {
        if (tid == 0) { atomicOr(&st->flags, FA_DFLAG_PACK_FAILURE); st->best = 0; }
        return;
    }
    const long long* rec = cand + CAND_REC * (best - 1);
    size_t slot = (size_t)rec[4];
    const long long* p = cand_p + slot * n_max;
    const int* w = cand_w + slot * n_max;
    const int* h = cand_h + slot * n_max;
    const int* y = cand_y + slot * n_max;
    int kbits = 63 - __clzll(omega);
    long long tex = 0;
    for (int j = tid; j < n; j += blockDim.x) {
        long long q = p[j] & (omega - 1);
        int r = (int)(p[j] >> kbits);  // row index < n <= 2^31
        long long x = (r % FA_DIRECTION_PERIOD == 0) ? q : omega - q - w[j];
        const bool first = j == tid;
        int src = first ? src0 : perm[j];
        long long* P = placements + 8 * (long long)j;
        if (ord_tw) {  // packing-order copies (k_order_frame): no dependent load through perm
            P[0] = first ? cid0 : ord_cid[j];
            P[6] = first ? tw0 : ord_tw[j];
            P[7] = first ? th0 : ord_th[j];
        } else {
            P[0] = chart_id_i ? (long long)chart_id_i[src] : (chart_id ? chart_id[src] : src);
            P[6] = tw[src];
            P[7] = th[src];
        }
        P[1] = x;
        P[2] = y[j];
        P[3] = w[j];
        P[4] = h[j];
        const int rj = first ? rot0 : rot[j];
        P[5] = rj;
        if (plc_by_src) {  // k_uv reads its chart's placement directly (x, y, w, h < 2^31)
            plc_by_src[2 * src] = make_int4((int)x, y[j], w[j], h[j]);
            plc_by_src[2 * src + 1] = make_int4(rj, 0, 0, 0);
        }
        long long cw = w[j] - 2 * pad, chh = h[j] - 2 * pad;
        tex += (cw > 0 ? cw : 0) * (chh > 0 ? chh : 0);
    }
    tex = block_sum_ll(tex, red);
    if (tid == 0) {
        st->best = (int)best;
        st->scale_num = rec[1];
        st->scale_den = rec[2];
        st->texels_allocated = tex;
    }
}

__global__ void __launch_bounds__(1024) k_select(const long long* __restrict__ ow, const long long* __restrict__ tw,
                                                 const long long* __restrict__ th, const long long* __restrict__ chart_id,
                                                 const unsigned char* __restrict__ rot, const int* __restrict__ perm,
                                                 int n_max, const int* __restrict__ n_dev, long long omega,
                                                 long long n_scales, long long min_dim, long long pad,
                                                 const long long* __restrict__ cand, const long long* __restrict__ cand_p,
                                                 const int* __restrict__ cand_w, const int* __restrict__ cand_h,
                                                 const int* __restrict__ cand_y, long long* __restrict__ placements,
                                                 int4* __restrict__ plc_by_src, unsigned char* __restrict__ accept_out,
                                                 fa_dstat* __restrict__ st, const long long* __restrict__ ord_tw,
                                                 const long long* __restrict__ ord_th,
                                                 const long long* __restrict__ ord_cid) {
    FA_PDL_PROLOGUE();
    __shared__ long long red[33];
    __shared__ long long red2[33];
    int n = n_dev ? *n_dev : n_max;
    if (st->flags & (FA_DFLAG_HEIGHT_OVERFLOW | FA_DFLAG_KEY_RANGE | FA_DFLAG_DUPLICATE_MIN_TRI |
                     FA_DFLAG_QUEUE_OVERFLOW))
        return;
    select_body(ow, tw, th, (const int*)nullptr, chart_id, rot, perm, n, omega, n_scales, min_dim, pad, cand, cand_p,
                cand_w, cand_h, cand_y, n_max, placements, plc_by_src, accept_out, st, red, red2, ord_tw, ord_th,
                ord_cid);
}

// ---- standalone fold (packing.py:133-158) --------------------------------
__global__ void __launch_bounds__(1024) k_fold(const long long* __restrict__ w, int n, long long omega,
                                               long long* __restrict__ rows, long long* __restrict__ xs,
                                               long long* __restrict__ m_out) {
    FA_PDL_PROLOGUE();
    __shared__ long long red[33];
    int kbits = 63 - __clzll(omega);
    long long carry = 0, mloc = -(1ll << 62);
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        int b = c0 + threadIdx.x;
        long long wb = b < n ? w[b] : 0;
        long long tot;
        long long p = carry + block_exclusive_scan_ll(wb, red, &tot);
        if (b < n) {
            long long r = p >> kbits, q = p & (omega - 1);
            rows[b] = r;
            xs[b] = (r % FA_DIRECTION_PERIOD == 0) ? q : omega - q - wb;
            long long over = q + wb - omega;
            mloc = over > mloc ? over : mloc;
        }
        carry += tot;
    }
    mloc = block_max_ll(mloc, red);
    if (threadIdx.x == 0) *m_out = mloc > 0 ? mloc : 0;
}

// ---- standalone push_up (packing.py:170-215) -------------------------------
__global__ void __launch_bounds__(1024) k_push_up(const long long* __restrict__ rows, const long long* __restrict__ xs,
                                                  const long long* __restrict__ w, const long long* __restrict__ h,
                                                  int n, long long omega, int* __restrict__ rowstart,
                                                  long long* __restrict__ y, long long* __restrict__ used_out,
                                                  int* gfront) {
    FA_PDL_PROLOGUE();
    extern __shared__ int dyn_front[];
    __shared__ long long red[33];
    int* front = gfront ? gfront : dyn_front;
    int tid = threadIdx.x;
    for (int c = tid; c <= omega; c += blockDim.x) front[c] = 0;
    // segments of equal consecutive rows (np.split at np.diff(rows) != 0)
    __shared__ int nseg;
    if (tid == 0) nseg = 0;
    __syncthreads();
    for (int b = tid; b < n; b += blockDim.x) {
        if (b == 0 || rows[b - 1] != rows[b]) {
            // segments are numbered by order of appearance; rows are
            // nondecreasing for a genuine fold so row index works as id
            rowstart[rows[b] - rows[0]] = b;
            atomicAdd(&nseg, 1);
        }
    }
    __syncthreads();
    int nsegs = nseg;
    long long usedl = 0;
    for (int r = 0; r < nsegs; r++) {
        int b0 = rowstart[r];
        int b1 = (r + 1 < nsegs) ? rowstart[r + 1] : n;
        int nb = b1 - b0;
        int G = 32;
        while (G > 1 && G * nb > (int)blockDim.x) G >>= 1;
        int groups = blockDim.x / G;
        int g = tid / G, gl = tid % G;
        for (int gbase = 0; gbase < nb; gbase += groups) {
            int gb = gbase + g;
            bool act = gb < nb;
            int b = b0 + (act ? gb : 0);
            int x = (int)xs[b], wb = act ? (int)w[b] : 0;
            long long rest = 0;
            for (int c = x + gl; c < x + wb; c += G) rest = max(rest, (long long)front[c]);
            for (int o = G >> 1; o > 0; o >>= 1) {
                long long oth = __shfl_xor_sync(0xffffffffu, rest, o, G);
                rest = oth > rest ? oth : rest;
            }
            long long top = rest + h[b];
            if (act) {
                for (int c = x + gl; c < x + wb; c += G) front[c] = (int)top;
                if (gl == 0) y[b] = rest;
                usedl = top > usedl ? top : usedl;
            }
        }
        __syncthreads();
    }
    usedl = block_max_ll(usedl, red);
    if (tid == 0) *used_out = usedl;
}

// ---- pack_at_scale xywh output ---------------------------------------------
__global__ void k_xywh(const long long* __restrict__ cand, const long long* __restrict__ cand_p,
                       const int* __restrict__ cand_w, const int* __restrict__ cand_h, const int* __restrict__ cand_y,
                       int n, long long omega, long long* __restrict__ out) {
    FA_PDL_PROLOGUE();
    if (cand[0] == 0) return;
    int kbits = 63 - __clzll(omega);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        long long q = cand_p[j] & (omega - 1), r = cand_p[j] >> kbits;
        out[4 * j] = (r % FA_DIRECTION_PERIOD == 0) ? q : omega - q - cand_w[j];
        out[4 * j + 1] = cand_y[j];
        out[4 * j + 2] = cand_w[j];
        out[4 * j + 3] = cand_h[j];
    }
}

// ============================================================================
// host launchers
// ============================================================================
static size_t front_smem(long long omega) { return (size_t)(omega + 1) * sizeof(int); }
static const size_t kMaxFrontSmem = 200 * 1024;

// k_pack's dynamic shared memory: the frontline when it fits, then the
// push-up box arrays for up to the register path's box count (4 ints each)
struct PackSmemPlan {
    bool smem_front;
    int n_sbox;
    size_t dyn;
};
static PackSmemPlan pack_smem_plan(long long omega, int n_max) {
    PackSmemPlan pl{};
    const int cap = n_max < PK_KREG_WIDE * PK_THREADS ? n_max : PK_KREG_WIDE * PK_THREADS;
    const size_t boxes = (size_t)4 * cap * sizeof(int);
    const size_t front = ((size_t)(omega + 1 + 3) & ~(size_t)3) * sizeof(int);
    pl.smem_front = front_smem(omega) <= kMaxFrontSmem;
    if (pl.smem_front && front + boxes <= kMaxFrontSmem) {
        pl.n_sbox = cap;
        pl.dyn = front + boxes;
    } else if (pl.smem_front) {
        pl.dyn = front_smem(omega);
    } else if (boxes <= kMaxFrontSmem) {
        pl.n_sbox = cap;
        pl.dyn = boxes;
    }
    if (!fa_env_int("FASTATLAS_PACK_SMEM_TAIL", 1)) {
        pl.n_sbox = 0;
        pl.dyn = pl.smem_front ? front_smem(omega) : 0;
    }
    return pl;
}

static void ensure_smem_attr() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxFrontSmem);
    cudaFuncSetAttribute(k_push_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxFrontSmem);
    done = true;
}

void fa_launch_orient_sort(const fa_pack_bufs& b, int n_max, const int* n_dev, long long max_h, fa_dstat* st,
                           cudaStream_t s, const fa_box_dims_args* bd) {
    if (bd && b.ord_tw && fa_env_int("FASTATLAS_ORDER_ONCHIP", 1)) {
        const int cap = n_max < 4096 ? n_max : 4096;
        const size_t smem = fa_order_frame_smem(cap);
        static size_t attr = 0;
        if (smem > attr) {
            cudaFuncSetAttribute(k_order_frame, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr = smem;
        }
        fa_launch(k_order_frame, 1, SORT_THREADS, smem, s, *bd, n_dev, n_max, cap, max_h, b.ow, b.oh, b.rot, b.perm,
                  b.pinv, b.sortk, b.sortv, b.ord_tw, b.ord_th, b.ord_cid, st);
        return;
    }
    fa_box_dims_args none{};
    fa_launch(k_orient_sort, 1, SORT_THREADS, 0, s, b.tw, b.th, nullptr, n_max, n_dev, max_h, b.ow, b.oh, b.rot, b.perm,
              b.pinv, b.sortk, b.sortv, 0, st, bd ? *bd : none);
}

void fa_launch_orient_sort_mt(const long long* tw, const long long* th, const long long* mt, int n, long long max_h,
                              long long* ow, long long* oh, unsigned char* rot, int* perm, int* pinv,
                              unsigned long long* sk, int* sv, int reject_dups, fa_dstat* st, cudaStream_t s) {
    fa_box_dims_args none{};
    fa_launch(k_orient_sort, 1, SORT_THREADS, 0, s, tw, th, mt, n, nullptr, max_h, ow, oh, rot, perm, pinv, sk, sv,
              reject_dups, st, none);
}

// returns number of kernel launches
int fa_launch_pack(const fa_pack_bufs& b, int n_max, const int* n_dev, long long omega, long long n_scales,
                   long long min_dim, long long pad, int batch, fa_dstat* st, cudaStream_t s) {
    ensure_smem_attr();
    int kbits = 63 - __builtin_clzll((unsigned long long)omega);
    const PackSmemPlan pl = pack_smem_plan(omega, n_max);
    const bool smem_front = pl.smem_front;
    const size_t dyn = pl.dyn;
    int launches = 0;
    for (long long hi = n_scales; hi >= 1; hi -= batch) {
        long long lo = hi - batch + 1;
        if (lo < 1) lo = 1;
        int grid = (int)(hi - lo + 1);
        fa_launch(k_pack, grid, PK_THREADS, dyn, s, b.ow, b.oh, n_max, n_dev, omega, kbits, n_scales, hi, 0, 0, min_dim, pad,
                                             b.cand, b.cand_p, b.cand_w, b.cand_h, b.cand_y, b.rowstart,
                                             smem_front ? nullptr : b.gfront, st, pl.n_sbox);
        launches++;
        if (lo > 1) {
            fa_launch(k_batch_done, 1, 256, 0, s, b.cand, lo, hi, st);
            launches++;
        }
    }
    const bool ord = b.ord_tw && b.ord_written;
    fa_launch(k_select, 1, 1024, 0, s, b.ow, b.tw, b.th, b.chart_id, b.rot, b.perm, n_max, n_dev, omega, n_scales, min_dim,
                                pad, b.cand, b.cand_p, b.cand_w, b.cand_h, b.cand_y, b.placements, b.plc_by_src, b.accept_out, st,
                                ord ? (const long long*)b.ord_tw : nullptr, ord ? (const long long*)b.ord_th : nullptr,
                                ord ? (const long long*)b.ord_cid : nullptr);
    return launches + 1;
}

void fa_launch_pack_at_scale(const long long* ow, const long long* oh, int n, long long num, long long den,
                             long long omega, long long min_dim, long long pad, long long* cand, long long* cand_p,
                             int* cand_w, int* cand_h, int* cand_y, int* rowstart, int* gfront, cudaStream_t s) {
    ensure_smem_attr();
    int kbits = 63 - __builtin_clzll((unsigned long long)omega);
    const PackSmemPlan pl = pack_smem_plan(omega, n);
    fa_launch(k_pack, 1, PK_THREADS, pl.dyn, s, ow, oh, n, nullptr, omega, kbits, 1, 1, num, den, min_dim, pad, cand,
              cand_p, cand_w, cand_h, cand_y, rowstart, pl.smem_front ? nullptr : gfront, nullptr, pl.n_sbox);
}

void fa_launch_xywh(const long long* cand, const long long* cand_p, const int* cand_w, const int* cand_h,
                    const int* cand_y, int n, long long omega, long long* out, cudaStream_t s) {
    fa_launch(k_xywh, fa_grid(n, 256, FA_NUM_SMS), 256, 0, s, cand, cand_p, cand_w, cand_h, cand_y, n, omega, out);
}

void fa_launch_fold(const long long* w, int n, long long omega, long long* rows, long long* x, long long* m,
                    cudaStream_t s) {
    fa_launch(k_fold, 1, 1024, 0, s, w, n, omega, rows, x, m);
}

void fa_launch_push_up_impl(const long long* rows, const long long* x, const long long* w, const long long* h, int n,
                            long long omega, int* rowstart, long long* y, long long* used, int* gfront,
                            cudaStream_t s) {
    ensure_smem_attr();
    size_t dyn = gfront ? 0 : front_smem(omega);
    fa_launch(k_push_up, 1, 1024, dyn, s, rows, x, w, h, n, omega, rowstart, y, used, gfront);
}

bool fa_front_in_smem(long long omega) { return front_smem(omega) <= kMaxFrontSmem; }


// orient (packing.py:109-117): rotate boxes wider than tall
__global__ void k_orient(const long long* __restrict__ tw, const long long* __restrict__ th, int n,
                         long long* __restrict__ ow, long long* __restrict__ oh, unsigned char* __restrict__ rot) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        long long w = tw[i], h = th[i];
        bool r = w > h;
        ow[i] = r ? h : w;
        oh[i] = r ? w : h;
        rot[i] = r;
    }
}

void fa_launch_orient(const long long* tw, const long long* th, int n, long long* ow, long long* oh,
                      unsigned char* rot, cudaStream_t s) {
    fa_launch(k_orient, fa_grid(n, 256, FA_NUM_SMS * 4), 256, 0, s, tw, th, n, ow, oh, rot);
}

FA_TRACE_TU(pack)
