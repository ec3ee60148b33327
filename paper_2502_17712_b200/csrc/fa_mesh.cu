// fa_mesh.cu — binding a mesh (fa_set_mesh): index validation and the
// first-use vertex renumbering, on the GPU.
//
// The reference keeps the mesh as given (Mesh, charts.py:29-61, whose
// __post_init__ rejects indices outside [0, V), :45-48).  The context keeps
// its own copy with the vertices renumbered in order of first use by the
// triangle list: per-vertex gathers of consecutive triangles then share
// cache lines.  Triangle order -- and so every per-triangle output -- is
// unchanged; per-vertex outputs are mapped back through the permutation.
//
//   first[v]   = smallest corner slot c (= 3t + i) with tris[c] == v
//                (atomicMin; out-of-range indices raise a flag instead)
//   used v     : new id = rank of first[v] among the first-use corners
//                (ordered compaction of the corners c with first[tris[c]] == c)
//   unused v   : new id = U + rank of v among the unused vertices
//   tris'[c]   = new id of tris[c];  pos'[new] = pos[old]
//
// Each compaction is count -> one-CTA scan of the per-tile counts ->
// scatter, so the whole rebinding is O(3T + V) work in eight launches.
#define FA_TU_ID 8  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"

#define MS_THREADS 256
#define MS_ITEMS 4
#define MS_TILE (MS_THREADS * MS_ITEMS)

static int ms_tiles(long long n) {
    long long b = (n + MS_TILE - 1) / MS_TILE;
    return b > 0 ? (int)b : 1;
}

int fa_mesh_scratch_ints(long long V, long long T) { return ms_tiles(3 * T) + ms_tiles(V) + 8; }

__global__ void k_first_use(const int* __restrict__ tris, long long nc, int V, int* __restrict__ first,
                            int* __restrict__ bad) {
    FA_PDL_PROLOGUE();
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += (long long)gridDim.x * blockDim.x) {
        const int v = __ldg(tris + c);
        if (v < 0 || v >= V) atomicOr(bad, 1);
        else atomicMin(first + v, (int)c);
    }
}

// per-tile counts of first-use corners (mode 0) or of unused vertices (mode 1)
template <int MODE>
__device__ __forceinline__ bool ms_item(const int* __restrict__ tris, const int* __restrict__ first, long long i,
                                        long long n) {
    if (i >= n) return false;
    if (MODE == 0) return __ldg(first + __ldg(tris + i)) == (int)i;
    return __ldg(first + i) == 0x7fffffff;
}

template <int MODE>
__global__ void __launch_bounds__(MS_THREADS) k_ms_count(const int* __restrict__ tris, const int* __restrict__ first,
                                                         long long n, int* __restrict__ counts) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    const long long base = (long long)blockIdx.x * MS_TILE + threadIdx.x * MS_ITEMS;
    int c = 0;
#pragma unroll
    for (int i = 0; i < MS_ITEMS; i++) c += ms_item<MODE>(tris, first, base + i, n);
    c = warp_sum(c);
    if (lane_id() == 0) sm[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int i = 0; i < MS_THREADS / 32; i++) s += sm[i];
        counts[blockIdx.x] = s;
    }
}

// exclusive scan of counts[0..n) in place (one CTA); counts[n] = total
__global__ void __launch_bounds__(1024) k_ms_scan(int* __restrict__ counts, int n) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int carry = 0;
    for (int b0 = 0; b0 < n; b0 += 1024) {
        const int i = b0 + threadIdx.x;
        const int v = i < n ? counts[i] : 0;
        int tot;
        const int e = block_exclusive_scan(v, sm, &tot);
        if (i < n) counts[i] = carry + e;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[n] = carry;
}

// MODE 0: new id of each used vertex = rank of its first-use corner
// MODE 1: new id of each unused vertex = U + its rank (U = used count)
template <int MODE>
__global__ void __launch_bounds__(MS_THREADS) k_ms_scatter(const int* __restrict__ tris, const int* __restrict__ first,
                                                           long long n, const int* __restrict__ offsets,
                                                           const int* __restrict__ n_used, int* __restrict__ newidx,
                                                           int* __restrict__ perm) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    const long long base = (long long)blockIdx.x * MS_TILE + threadIdx.x * MS_ITEMS;
    bool f[MS_ITEMS];
    int c = 0;
#pragma unroll
    for (int i = 0; i < MS_ITEMS; i++) {
        f[i] = ms_item<MODE>(tris, first, base + i, n);
        c += f[i];
    }
    int tot;
    int pos = offsets[blockIdx.x] + block_exclusive_scan(c, sm, &tot) + (MODE == 1 ? *n_used : 0);
#pragma unroll
    for (int i = 0; i < MS_ITEMS; i++)
        if (f[i]) {
            const int v = MODE == 0 ? __ldg(tris + base + i) : (int)(base + i);
            newidx[v] = pos;
            perm[pos] = v;
            pos++;
        }
}

__global__ void k_ms_remap(const int* __restrict__ tris, long long nc, const int* __restrict__ newidx,
                           int* __restrict__ out) {
    FA_PDL_PROLOGUE();
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += (long long)gridDim.x * blockDim.x)
        out[c] = __ldg(newidx + __ldg(tris + c));
}

void fa_launch_mesh_remap(const int* tris, long long T, const int* newidx, int* out, cudaStream_t s) {
    fa_launch(k_ms_remap, fa_grid(3 * T, 256, FA_NUM_SMS * 8), 256, 0, s, tris, 3 * T, newidx, out);
}

// Validation only (first must hold V ints, bad one int; both device).
void fa_launch_mesh_validate(const int* tris, long long T, int V, int* first, int* bad, cudaStream_t s) {
    fa_launch_fill(first, V, 0x7fffffff, s);
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    fa_launch(k_first_use, fa_grid(3 * T, 256, FA_NUM_SMS * 8), 256, 0, s, tris, 3 * T, V, first, bad);
}

// Renumbering after fa_launch_mesh_validate (first filled).  scratch holds
// fa_mesh_scratch_ints(V, T) ints; newidx V ints; outputs tris_out (3T),
// perm (V), pos_out (3V doubles).
void fa_launch_mesh_renumber(const double* pos, const int* tris, long long T, int V, const int* first, int* scratch,
                             int* newidx, int* tris_out, int* perm, double* pos_out, cudaStream_t s) {
    const long long nc = 3 * T;
    const int nb0 = ms_tiles(nc), nb1 = ms_tiles(V);
    int* off0 = scratch;             // nb0 + 1 (total = used vertices U)
    int* off1 = scratch + nb0 + 1;   // nb1 + 1
    fa_launch(k_ms_count<0>, nb0, MS_THREADS, 0, s, tris, first, nc, off0);
    fa_launch(k_ms_scan, 1, 1024, 0, s, off0, nb0);
    fa_launch(k_ms_scatter<0>, nb0, MS_THREADS, 0, s, tris, first, nc, (const int*)off0, (const int*)nullptr, newidx,
              perm);
    fa_launch(k_ms_count<1>, nb1, MS_THREADS, 0, s, (const int*)nullptr, first, (long long)V, off1);
    fa_launch(k_ms_scan, 1, 1024, 0, s, off1, nb1);
    fa_launch(k_ms_scatter<1>, nb1, MS_THREADS, 0, s, (const int*)nullptr, first, (long long)V, (const int*)off1,
              (const int*)(off0 + nb0), newidx, perm);
    fa_launch(k_ms_remap, fa_grid(nc, 256, FA_NUM_SMS * 8), 256, 0, s, tris, nc, (const int*)newidx, tris_out);
    fa_launch_permute_pos(pos, perm, pos_out, V, s);
}

// ---------------------------------------------------------------------------
// Spatially coherent triangle order for the raster setup (per mesh, not per
// frame).  The setup walks the triangles in the order of a 30-bit Morton
// code of their centroids, 32 per warp: a warp's triangles then form a small
// surface patch, so its vertex gathers share cache lines and, above all, its
// cluster can be culled as a whole (k_raster_setup: bounding sphere outside a
// frustum plane, or normal cone facing away).  Triangle ids -- every output
// -- are unchanged: the setup reads the original id of each slot.
// ---------------------------------------------------------------------------
#define RS_THREADS 256
#define RS_ITEMS 64
#define RS_TILE (RS_THREADS * RS_ITEMS)

int fa_sort_blocks(long long n) { return (int)((n + RS_TILE - 1) / RS_TILE); }

__device__ __forceinline__ unsigned long long mesh_f64_key(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double mesh_key_f64(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// bbox[0..2] = min keys, bbox[3..5] = max keys of the vertex coordinates
__global__ void k_mesh_bbox(const double* __restrict__ pos, int V, unsigned long long* __restrict__ bbox) {
    FA_PDL_PROLOGUE();
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const unsigned long long q = mesh_f64_key(pos[3ll * v + k]);
            lo[k] = q < lo[k] ? q : lo[k];
            hi[k] = q > hi[k] ? q : hi[k];
        }
#pragma unroll
    for (int k = 0; k < 3; k++) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo[k], o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi[k], o);
            lo[k] = a < lo[k] ? a : lo[k];
            hi[k] = b > hi[k] ? b : hi[k];
        }
        if (lane_id() == 0) {
            atomicMin(bbox + k, lo[k]);
            atomicMax(bbox + 3 + k, hi[k]);
        }
    }
}

__device__ __forceinline__ unsigned morton_spread10(unsigned v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x30000ffu;
    v = (v | (v << 8)) & 0x300f00fu;
    v = (v | (v << 4)) & 0x30c30c3u;
    v = (v | (v << 2)) & 0x9249249u;
    return v;
}

// Morton code of each triangle's centroid in the mesh bbox (NaN centroids sort last)
__global__ void k_mesh_morton(const double* __restrict__ pos, const int* __restrict__ tris, int T,
                              const unsigned long long* __restrict__ bbox, unsigned* __restrict__ keys,
                              int* __restrict__ vals) {
    FA_PDL_PROLOGUE();
    double lo[3], sc[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        lo[k] = mesh_key_f64(bbox[k]);
        const double ext = mesh_key_f64(bbox[3 + k]) - lo[k];
        sc[k] = ext > 0 ? 1023.0 / ext : 0.0;
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        unsigned q[3];
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const double c = (pos[3ll * tris[3 * t] + k] + pos[3ll * tris[3 * t + 1] + k] + pos[3ll * tris[3 * t + 2] + k]) *
                             (1.0 / 3.0);
            double f = (c - lo[k]) * sc[k];
            if (!(f >= 0.0)) { ok = ok && f < 0.0; f = 0.0; }  // NaN -> not ok
            q[k] = (unsigned)fmin(f, 1023.0);
        }
        keys[t] = ok ? (morton_spread10(q[0]) | (morton_spread10(q[1]) << 1) | (morton_spread10(q[2]) << 2)) : 0xffffffffu;
        vals[t] = t;
    }
}

// LSD radix sort, 8-bit digit per pass: per-tile digit counts ...
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const unsigned* __restrict__ keys, int n, int shift,
                                                       int* __restrict__ hist, int nblocks) {
    FA_PDL_PROLOGUE();
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * RS_TILE;
    for (int k = 0; k < RS_ITEMS; k++) {
        const long long i = base + k * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];  // digit-major
}

// ... (exclusive scan of hist by k_ms_scan), then a stable scatter: items in
// order within the tile (chunk by chunk, warp by warp, lane by lane)
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const unsigned* __restrict__ ki, const int* __restrict__ vi,
                                                          unsigned* __restrict__ ko, int* __restrict__ vo, int n,
                                                          int shift, const int* __restrict__ offs, int nblocks) {
    FA_PDL_PROLOGUE();
    __shared__ int base[256];
    __shared__ int wcnt[RS_THREADS / 32][257];
    const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    base[tid] = offs[tid * nblocks + blockIdx.x];
    for (int i = tid; i < (RS_THREADS / 32) * 257; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const long long tbase = (long long)blockIdx.x * RS_TILE;
    for (int k = 0; k < RS_ITEMS; k++) {
        const long long i = tbase + k * RS_THREADS + tid;
        const bool valid = i < n;
        const unsigned key = valid ? ki[i] : 0u;
        const int val = valid ? vi[i] : 0;
        const int d = valid ? (int)((key >> shift) & 255u) : 256;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int off = 0;
            for (int w = 0; w < warp; w++) off += wcnt[w][d];
            const int pos = base[d] + off + rank;
            ko[pos] = key;
            vo[pos] = val;
        }
        __syncthreads();
        int s = 0;
        for (int w = 0; w < RS_THREADS / 32; w++) { s += wcnt[w][tid]; wcnt[w][tid] = 0; }
        base[tid] += s;
        if (tid < RS_THREADS / 32) wcnt[tid][256] = 0;
        __syncthreads();
    }
}

// sorted slot -> (original triangle id, its vertex indices)
__global__ void k_mesh_gather_tris(const int* __restrict__ tris, const int* __restrict__ order, int T,
                                   int* __restrict__ out) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += gridDim.x * blockDim.x) {
        const int t = order[i];
        out[3 * i] = tris[3 * t];
        out[3 * i + 1] = tris[3 * t + 1];
        out[3 * i + 2] = tris[3 * t + 2];
    }
}

// Scratch: 2 * T keys + 2 * T values + hist (256 * blocks + 1 ints).
size_t fa_mesh_sort_scratch_bytes(long long T) {
    return (size_t)T * 16 + ((size_t)256 * fa_sort_blocks(T) + 64) * 4 + 64;
}

// order[i] = the triangle at sorted slot i; tris_sorted = its vertex indices
void fa_launch_mesh_order(const double* pos, const int* tris, int T, int V, void* scratch, int* order,
                          int* tris_sorted, cudaStream_t s) {
    unsigned* ka = reinterpret_cast<unsigned*>(scratch);
    unsigned* kb = ka + T;
    int* va = reinterpret_cast<int*>(kb + T);
    int* vb = va + T;
    int* hist = vb + T;
    const int nb = fa_sort_blocks(T);
    unsigned long long* bbox = reinterpret_cast<unsigned long long*>(hist + 256 * nb + 2);
    bbox = reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(bbox) + 15) & ~(uintptr_t)15);
    const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    cudaMemcpyAsync(bbox, init, sizeof(init), cudaMemcpyHostToDevice, s);
    fa_launch(k_mesh_bbox, fa_grid(V, 256, FA_NUM_SMS * 4), 256, 0, s, pos, V, bbox);
    fa_launch(k_mesh_morton, fa_grid(T, 256, FA_NUM_SMS * 8), 256, 0, s, pos, tris, T,
              (const unsigned long long*)bbox, ka, va);
    for (int shift = 0; shift < 32; shift += 8) {
        fa_launch(k_rs_hist, nb, RS_THREADS, 0, s, (const unsigned*)ka, T, shift, hist, nb);
        fa_launch(k_ms_scan, 1, 1024, 0, s, hist, 256 * nb);
        fa_launch(k_rs_scatter, nb, RS_THREADS, 0, s, (const unsigned*)ka, (const int*)va, kb, vb, T, shift,
                  (const int*)hist, nb);
        unsigned* tk = ka; ka = kb; kb = tk;
        int* tv = va; va = vb; vb = tv;
    }
    cudaMemcpyAsync(order, va, (size_t)T * 4, cudaMemcpyDeviceToDevice, s);
    fa_launch(k_mesh_gather_tris, fa_grid(T, 256, FA_NUM_SMS * 8), 256, 0, s, tris, (const int*)order, T, tris_sorted);
}

// ---- per-cluster culling data: 32 consecutive sorted triangles ------------
// bounding sphere (centre of the vertex bbox, radius to the farthest vertex)
// and normal cone (axis = normalised sum of the unit normals, half angle to
// the farthest normal) of each cluster, plus the smallest triangle area.
// Rounding is absorbed by inflating the radius and the cone slightly; a
// cluster with a degenerate triangle gets amin = 0 (never back-face culled).
__global__ void k_cluster_build(const double* __restrict__ pos, const int* __restrict__ tris_sorted, int T,
                                fa_cluster* __restrict__ out) {
    FA_PDL_PROLOGUE();
    const int lane = lane_id();
    // one warp per 32 / FA_CLUSTER clusters; reductions stay within a cluster's lanes
    constexpr int CS = FA_CLUSTER;
    const int nc = (T + CS - 1) / CS;
    const int nw = (nc + 32 / CS - 1) / (32 / CS);
    for (int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nw; wi += (gridDim.x * blockDim.x) >> 5) {
        const int c = wi * (32 / CS) + lane / CS;
        const int i = c * CS + (lane % CS);
        const bool act = c < nc && i < T;
        double p[3][3];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int d = 0; d < 3; d++) p[k][d] = act ? pos[3ll * tris_sorted[3 * i + k] + d] : 0.0;
        double lo[3], hi[3];
#pragma unroll
        for (int d = 0; d < 3; d++) {
            lo[d] = act ? fmin(fmin(p[0][d], p[1][d]), p[2][d]) : INFINITY;
            hi[d] = act ? fmax(fmax(p[0][d], p[1][d]), p[2][d]) : -INFINITY;
            for (int o = CS / 2; o > 0; o >>= 1) {
                lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
                hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
            }
        }
        const double cx = 0.5 * (lo[0] + hi[0]), cy = 0.5 * (lo[1] + hi[1]), cz = 0.5 * (lo[2] + hi[2]);
        double r2 = 0.0;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const double dx = p[k][0] - cx, dy = p[k][1] - cy, dz = p[k][2] - cz;
            if (act) r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
        }
        // unit normal of (p1 - p0) x (p2 - p0)
        const double ux = p[1][0] - p[0][0], uy = p[1][1] - p[0][1], uz = p[1][2] - p[0][2];
        const double vx = p[2][0] - p[0][0], vy = p[2][1] - p[0][1], vz = p[2][2] - p[0][2];
        const double nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
        const double nl = sqrt(nx * nx + ny * ny + nz * nz);
        double area = act ? 0.5 * nl : INFINITY;
        const bool good = !act || (nl > 0 && isfinite(nl));
        double ax = good && act ? nx / nl : 0.0, ay = good && act ? ny / nl : 0.0, az = good && act ? nz / nl : 0.0;
        const double mx = ax, my = ay, mz = az;
        for (int o = CS / 2; o > 0; o >>= 1) {
            r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
            area = fmin(area, __shfl_xor_sync(0xffffffffu, area, o));
            ax += __shfl_xor_sync(0xffffffffu, ax, o);
            ay += __shfl_xor_sync(0xffffffffu, ay, o);
            az += __shfl_xor_sync(0xffffffffu, az, o);
        }
        const unsigned seg = (CS == 32 ? 0xffffffffu : ((1u << CS) - 1u)) << (lane & ~(CS - 1) & 31);
        const bool all_good = (__ballot_sync(0xffffffffu, good) & seg) == seg;
        const double al = sqrt(ax * ax + ay * ay + az * az);
        double cmin = 1.0;
        if (al > 0) {
            ax /= al; ay /= al; az /= al;
            cmin = act ? mx * ax + my * ay + mz * az : 1.0;
        }
        // (unconditional: `al` differs between the warp's clusters)
        for (int o = CS / 2; o > 0; o >>= 1) cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
        if ((lane % CS) == 0 && c < nc) {
            fa_cluster q;
            q.c[0] = cx; q.c[1] = cy; q.c[2] = cz;
            q.r = sqrt(r2) * (1.0 + 1e-12) + 1e-300;
            q.a[0] = ax; q.a[1] = ay; q.a[2] = az;
            // cone half angle, widened for the rounding of the normals
            const double ct = fmin(1.0, cmin) - 1e-9;
            q.cos_t = ct;
            q.sin_t = ct > -1.0 ? sqrt(fmax(0.0, 1.0 - ct * ct)) + 1e-9 : 1.0;
            q.amin = (all_good && al > 0 && ct > 0 && isfinite(area)) ? area * (1.0 - 1e-9) : 0.0;
            out[c] = q;
        }
    }
}

// the setup's per-slot record: vertex indices and triangle id in one int4
__global__ void k_make_slots4(const int* __restrict__ tris_sorted, const int* __restrict__ tperm, int T,
                              int4* __restrict__ out) {
    FA_PDL_PROLOGUE();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += gridDim.x * blockDim.x)
        out[i] = make_int4(tris_sorted[3 * i], tris_sorted[3 * i + 1], tris_sorted[3 * i + 2], tperm ? tperm[i] : i);
}

void fa_launch_make_slots4(const int* tris_sorted, const int* tperm, int T, int4* out, cudaStream_t s) {
    fa_launch(k_make_slots4, fa_grid(T, 256, FA_NUM_SMS * 8), 256, 0, s, tris_sorted, tperm, T, out);
}

void fa_launch_cluster_build(const double* pos, const int* tris_sorted, int T, fa_cluster* out, cudaStream_t s) {
    fa_launch(k_cluster_build, fa_grid((long long)((T + 31) / 32) * 32, 256, FA_NUM_SMS * 8), 256, 0, s, pos,
              tris_sorted, T, out);
}

FA_TRACE_TU(mesh)
