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
