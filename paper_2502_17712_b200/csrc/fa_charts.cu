// fa_charts.cu — visible-list compaction and lock-free union-find
// chartification on sm_100a.
//
// Reference: connected_charts + merge_shared_vertices (charts.py:343-406).
// The merged charts are the connected components of the visible-triangle /
// vertex incidence graph (edge adjacency is subsumed because edge neighbours
// share two vertices).  Per vertex v we keep vmin[v] = the smallest visible
// triangle touching v (which is exactly the reference's first_chart[v],
// charts.py:375-380), then union every visible triangle with vmin of its
// three vertices.  Hooking always puts the larger root under the smaller
// (atomicCAS), so each component's root is its minimum triangle index —
// the reference's canonical chart id (charts.py:335-340, 394-402).
#define FA_TU_ID 3  // trace builds (FA_TRACE): kernel key = TU id + line
#include "fa_internal.h"

#define CMP_THREADS 256
#ifndef UF_HALVE_AFTER
#define UF_HALVE_AFTER 16  // k_hook_multi: find rounds before path halving starts
#endif
// flags per thread of the visible compaction (one 32-bit load) and visible
// triangles per thread of the roots compaction: few items per thread, so the
// latency-bound gathers have many threads in flight
#ifndef CMP_ITEMS
#define CMP_ITEMS 4  // a multiple of 4
#endif
#define CMP_TILE (CMP_THREADS * CMP_ITEMS)
#ifndef ROOT_ITEMS
#define ROOT_ITEMS 2
#endif
#define ROOT_TILE (CMP_THREADS * ROOT_ITEMS)

// per-block count slots for n items (sized for the smaller tile)
int fa_compact_blocks(long long n) {
    long long b = (n + ROOT_TILE - 1) / ROOT_TILE;
    return b > 0 ? (int)b : 1;
}
static int blocks_for(long long n, int tile) {
    long long b = (n + tile - 1) / tile;
    return b > 0 ? (int)b : 1;
}

__device__ __forceinline__ int byte_sum4(unsigned int v) { return (int)((v * 0x01010101u) >> 24); }

// sum of blocks[0..b-1] computed cooperatively by the block
__device__ __forceinline__ int block_prefix_of(const int* blocks, int b, int* smem32) {
    int s = 0;
    for (int i = threadIdx.x; i < b; i += blockDim.x) s += blocks[i];
    s = warp_sum(s);
    if (lane_id() == 0) smem32[threadIdx.x >> 5] = s;
    __syncthreads();
    int tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) tot += smem32[i];
    __syncthreads();
    return tot;
}

// Bit mask of 4 items per lane, lanes in order (lane l holds items 4l..4l+3
// of the warp's 128): the 8 lanes of a group OR their nibbles into one 32-bit
// word, which the group's first lane returns (others return 0).
__device__ __forceinline__ unsigned int nibble_word(unsigned int nib) {
    unsigned int v = (nib & 15u) << (4 * (lane_id() & 7));
    v |= __shfl_xor_sync(0xffffffffu, v, 1);
    v |= __shfl_xor_sync(0xffffffffu, v, 2);
    v |= __shfl_xor_sync(0xffffffffu, v, 4);
    return v;
}

// ---- visible compaction ----------------------------------------------------
// The compactions run a wave-sized grid; CTA b handles the contiguous tiles
// [b * per, (b + 1) * per) of the fixed tile partition (vb = tile index).
__device__ __forceinline__ void tile_range(int ntiles, int& vb0, int& vb1) {
    const int per = (ntiles + (int)gridDim.x - 1) / (int)gridDim.x;
    vb0 = min(ntiles, (int)blockIdx.x * per);
    vb1 = min(ntiles, vb0 + per);
}

__global__ void __launch_bounds__(CMP_THREADS) k_count_flags(const unsigned char* __restrict__ flags, int T,
                                                             int* __restrict__ blocks, int ntiles) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int vb0, vb1;
    tile_range(ntiles, vb0, vb1);
    for (int vb = vb0; vb < vb1; vb++) {
        int base = vb * CMP_TILE + threadIdx.x * CMP_ITEMS;
        int c = 0;
        if (base + CMP_ITEMS <= T) {
#pragma unroll
            for (int q = 0; q < CMP_ITEMS / 4; q++) c += byte_sum4(reinterpret_cast<const unsigned int*>(flags + base)[q]);
        } else {
            for (int i = base; i < T; i++) c += flags[i] != 0;
        }
        c = warp_sum(c);
        if (lane_id() == 0) sm[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int i = 0; i < CMP_THREADS / 32; i++) s += sm[i];
            blocks[vb] = s;
        }
        __syncthreads();
    }
}

// With `vmin` bound it also lowers vmin[v] to the smallest visible triangle
// of each vertex (the union-find's first_chart, charts.py:330-336).
__global__ void __launch_bounds__(CMP_THREADS) k_scatter_visible(const unsigned char* __restrict__ flags, int T,
                                                                 const int* __restrict__ blocks, int nblocks,
                                                                 int* __restrict__ vis_list, int* __restrict__ label,
                                                                 const int* __restrict__ tris, int* __restrict__ vmin,
                                                                 int4* __restrict__ vis_tris,
                                                                 fa_dstat* __restrict__ st,
                                                                 unsigned int* __restrict__ vis_mask) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int vb0, vb1;
    tile_range(nblocks, vb0, vb1);
    int offset = block_prefix_of(blocks, vb0, sm);
    for (int vb = vb0; vb < vb1; vb++) {
    int base = vb * CMP_TILE + threadIdx.x * CMP_ITEMS;
    unsigned char f[CMP_ITEMS];
    if (base + CMP_ITEMS <= T) {
#pragma unroll
        for (int q = 0; q < CMP_ITEMS / 4; q++) {
            const unsigned int w = reinterpret_cast<const unsigned int*>(flags + base)[q];
#pragma unroll
            for (int i = 0; i < 4; i++) f[4 * q + i] = (w >> (8 * i)) & 0xffu;
        }
    } else {
#pragma unroll
        for (int i = 0; i < CMP_ITEMS; i++) f[i] = (base + i < T) ? flags[base + i] : 0;
    }
    int c = 0;
#pragma unroll
    for (int i = 0; i < CMP_ITEMS; i++) c += f[i] != 0;
    if (vis_mask) {
        // the visibility flags as a bit mask (the packed download format):
        // bit t of word t / 32
        static_assert(CMP_ITEMS == 4, "one nibble per thread");
        const unsigned int w = nibble_word((f[0] != 0) | ((f[1] != 0) << 1) | ((f[2] != 0) << 2) | ((f[3] != 0) << 3));
        if ((lane_id() & 7) == 0 && base < T) vis_mask[base >> 5] = w;
    }
    int total;
    int pos = offset + block_exclusive_scan(c, sm, &total);
    if (base + CMP_ITEMS <= T) {
        // CMP_ITEMS consecutive labels: 128-bit stores
        int4* l4 = reinterpret_cast<int4*>(label + base);
#pragma unroll
        for (int q = 0; q < CMP_ITEMS / 4; q++)
            l4[q] = make_int4(f[4 * q] ? base + 4 * q : -1, f[4 * q + 1] ? base + 4 * q + 1 : -1,
                              f[4 * q + 2] ? base + 4 * q + 2 : -1, f[4 * q + 3] ? base + 4 * q + 3 : -1);
    } else {
#pragma unroll
        for (int i = 0; i < CMP_ITEMS; i++)
            if (base + i < T) label[base + i] = f[i] ? base + i : -1;
    }
#pragma unroll
    for (int i = 0; i < CMP_ITEMS; i++) {
        int t = base + i;
        if (t < T && f[i]) {
            if (vis_tris) {
                // the visible triangle's vertex indices next to its id: the
                // later per-visible-triangle kernels skip one dependent load
                const int a = __ldg(tris + 3 * t), b = __ldg(tris + 3 * t + 1), c = __ldg(tris + 3 * t + 2);
                vis_tris[pos] = make_int4(a, b, c, t);
                if (vmin) {
                    atomicMin(vmin + a, t);
                    atomicMin(vmin + b, t);
                    atomicMin(vmin + c, t);
                }
            } else if (vmin) {
                // fire-and-forget REDs: a load-first check would put a round
                // trip per vertex into this thread's sequential item loop
#pragma unroll
                for (int j = 0; j < 3; j++) atomicMin(vmin + __ldg(tris + 3 * t + j), t);
            }
            vis_list[pos++] = t;
        }
    }
    if (vb == nblocks - 1 && threadIdx.x == 0) st->n_vis = offset + total;
    offset += total;
    __syncthreads();  // sm is reused by the next tile's scan
    }
}

void fa_launch_compact_visible(const unsigned char* flags, int T, int* blocks, int* vis_list, int* label,
                               fa_dstat* st, cudaStream_t s, const int* tris, int* vmin, int4* vis_tris,
                               unsigned int* vis_mask) {
    int nb = blocks_for(T, CMP_TILE);
    fa_launch(k_count_flags, fa_wave_grid(k_count_flags, CMP_THREADS, 0, nb, nb), CMP_THREADS, 0, s, flags, T, blocks,
              nb);
    fa_launch(k_scatter_visible, fa_wave_grid(k_scatter_visible, CMP_THREADS, 0, nb, nb), CMP_THREADS, 0, s, flags, T,
              blocks, nb, vis_list, label, tris, vmin,
              tris ? vis_tris : nullptr, st, vis_mask);
}

// ---- union-find ---------------------------------------------------------------
// parent[x] <= x always holds; find with pointer jumping (ECL-CC style)
// (only while hooking: every jump keeps a node inside its own set).  Loads may
// be L1-cached and stale: a stale chain still only climbs through ancestors
// (parent <= node always holds), a stale root can only make two nodes look
// unmerged (never wrongly merged), and every failed CAS returns a fresh value.
#ifndef FA_UF_VOLATILE
#define FA_UF_VOLATILE 0
#endif
__device__ __forceinline__ int uf_find(int* parent, int x) {
#if FA_UF_VOLATILE
    volatile int* p = parent;
#else
    int* p = parent;
#endif
    int cur = p[x];
    if (cur != x) {
        int next, prev = x;
        while (cur > (next = p[cur])) {
            p[prev] = next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}

// Read-only find for the flatten pass.  Pointer jumping must not run there:
// a jump computed from a stale read can overwrite a label another thread
// has already finalised with an intermediate (non-root) ancestor.
__device__ __forceinline__ int uf_find_ro(const int* parent, int x) {
    const volatile int* p = parent;
    int cur = x, next;
    while (cur > (next = p[cur])) cur = next;
    return cur;
}

#ifdef FA_UF_STATS
// debug build only: [unions, cas attempts, cas failures, find hops, max hops]
__device__ unsigned long long g_uf_stats[5];
__device__ __forceinline__ int uf_find_count(int* parent, int x) {
    volatile int* p = parent;
    int cur = p[x], hops = 0;
    if (cur != x) {
        int next, prev = x;
        while (cur > (next = p[cur])) {
            p[prev] = next;
            prev = cur;
            cur = next;
            hops++;
        }
    }
    atomicAdd(&g_uf_stats[3], (unsigned long long)hops);
    atomicMax(&g_uf_stats[4], (unsigned long long)hops);
    return cur;
}
#define UF_FIND uf_find_count
extern "C" void fa_debug_uf_stats(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_uf_stats, sizeof(g_uf_stats));
    unsigned long long z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_uf_stats, z, sizeof(z));
}
#else
#define UF_FIND uf_find
#endif

__device__ __forceinline__ void uf_union(int* parent, int a, int b) {
    int ra = UF_FIND(parent, a), rb = UF_FIND(parent, b);
#ifdef FA_UF_STATS
    atomicAdd(&g_uf_stats[0], 1ull);
#endif
    // ECL-CC hooking: a failed CAS returns the root's new parent, so the
    // loser climbs one level per round trip instead of re-running finds
    while (ra != rb) {
        if (ra < rb) { int t = ra; ra = rb; rb = t; }
        int old = atomicCAS(parent + ra, ra, rb);
#ifdef FA_UF_STATS
        atomicAdd(&g_uf_stats[1], 1ull);
        if (old != ra) atomicAdd(&g_uf_stats[2], 1ull);
#endif
        if (old == ra) break;
        ra = old;
    }
}

__global__ void k_vmin(const int* __restrict__ tris, const int* __restrict__ vis_list, int* __restrict__ vmin,
                       const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        int t = vis_list[k];
#pragma unroll
        for (int j = 0; j < 3; j++) {
            int v = __ldg(tris + 3 * t + j);
            if (*(volatile int*)(vmin + v) > t) atomicMin(vmin + v, t);
        }
    }
}

// Multi-way hooking: t joins the sets of vmin[v0..2] in one step.  First the
// ECL-CC initialisation, fused: t, if still its own root, points at the
// smallest of its vertex minima (a CAS, never a plain store, so a hook that
// already gave t a parent is never lost).  Then the four
// finds (from t's parent and from the three vertex minima) advance together,
// one parent load each per round, so the dependent chain is as long as the
// deepest path rather than the sum of three unions; every root other than
// the smallest is then hooked to it with independent CASes.  A CAS that
// loses a race (the root got a new parent) sends that node up again.
// Hooking to a node m that has meanwhile stopped being a root is still a
// valid union (parent[r] = m < r keeps the min-rooted forest).
__global__ void k_hook_multi(const int* __restrict__ tris, const int* __restrict__ vis_list,
                             const int* __restrict__ vmin, int* label, const fa_dstat* __restrict__ st,
                             const int4* __restrict__ vis_tris) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        int t, r1, r2, r3;
        if (vis_tris) {
            const int4 q = vis_tris[k];
            t = q.w;
            r1 = vmin[q.x], r2 = vmin[q.y], r3 = vmin[q.z];
        } else {
            t = vis_list[k];
            r1 = vmin[__ldg(tris + 3 * t)], r2 = vmin[__ldg(tris + 3 * t + 1)], r3 = vmin[__ldg(tris + 3 * t + 2)];
        }
        const int m0 = min(min(t, r1), min(r2, r3));
        int r0 = m0 < t ? atomicCAS(label + t, t, m0) : label[t];
        if (r0 == t) r0 = m0;
        // lock-free: every lost CAS moves a node strictly down, so this ends
        while (true) {
            // joint find: one parent load per node per round; past UF_HALVE_AFTER
            // rounds (long paths: few, large charts) each non-root is also
            // pointed at its grandparent (path halving: labels only point at
            // smaller ids, so a grandparent is always an ancestor and the racy
            // plain stores keep every path intact; roots are never written)
            int hops = 0;
            while (true) {
                int p0 = label[r0], p1 = label[r1], p2 = label[r2], p3 = label[r3];
                bool roots = (p0 == r0) & (p1 == r1) & (p2 == r2) & (p3 == r3);
                if (!roots && ++hops > UF_HALVE_AFTER) {
                    const int g0 = label[p0], g1 = label[p1], g2 = label[p2], g3 = label[p3];
                    if (g0 != p0) label[r0] = g0, p0 = g0;
                    if (g1 != p1) label[r1] = g1, p1 = g1;
                    if (g2 != p2) label[r2] = g2, p2 = g2;
                    if (g3 != p3) label[r3] = g3, p3 = g3;
                }
                r0 = p0;
                r1 = p1;
                r2 = p2;
                r3 = p3;
                if (roots) break;
            }
            int m = min(min(r0, r1), min(r2, r3));
            if (r0 == m && r1 == m && r2 == m && r3 == m) break;
            int o0 = r0 != m ? atomicCAS(label + r0, r0, m) : m;
            int o1 = r1 != m && r1 != r0 ? atomicCAS(label + r1, r1, m) : m;
            int o2 = r2 != m && r2 != r0 && r2 != r1 ? atomicCAS(label + r2, r2, m) : m;
            int o3 = r3 != m && r3 != r0 && r3 != r1 && r3 != r2 ? atomicCAS(label + r3, r3, m) : m;
            bool ok = (o0 == r0 || o0 == m) && (o1 == r1 || o1 == m) && (o2 == r2 || o2 == m) &&
                      (o3 == r3 || o3 == m);
            if (ok) break;
            // lost races: continue from the fresh parents (all still ancestors)
            if (o0 != r0 && o0 != m) r0 = o0;
            if (o1 != r1 && o1 != m) r1 = o1;
            if (o2 != r2 && o2 != m) r2 = o2;
            if (o3 != r3 && o3 != m) r3 = o3;
        }
    }
}

__global__ void k_hook_edges(const int* __restrict__ adj, const unsigned char* __restrict__ flags,
                             const int* __restrict__ vis_list, int* label, const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        int t = vis_list[k];
#pragma unroll
        for (int e = 0; e < 3; e++) {
            int nb = __ldg(adj + 3 * t + e);
            if (nb >= 0 && flags[nb]) uf_union(label, t, nb);
        }
    }
}

__global__ void k_hook_labels(const int* __restrict__ labels_in, const int* __restrict__ vis_list, int* label,
                              const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        int t = vis_list[k];
        int r = labels_in[t];
        if (r != t) uf_union(label, t, r);
    }
}

__global__ void k_compress(const int* __restrict__ vis_list, int* label, const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        int t = vis_list[k];
        label[t] = uf_find_ro(label, t);
    }
}

__global__ void k_iota(int* a, int n) {
    FA_PDL_PROLOGUE();
    int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = i;
}

__global__ void k_fill(int* a, int n, int v) {
    FA_PDL_PROLOGUE();
    int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

// canonical label = minimum VISIBLE member of each union-find root
// (charts.py:396-402).  tmp must be pre-filled with INT_MAX.
__global__ void k_canon_min(const int* __restrict__ vis_list, const int* __restrict__ label, int* tmp,
                            const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    int n = st->n_vis;
    int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        int t = vis_list[k];
        atomicMin(tmp + label[t], t);
    }
}

__global__ void k_canon_apply(const unsigned char* __restrict__ flags, int* label, const int* __restrict__ tmp, int T) {
    FA_PDL_PROLOGUE();
    int stride = gridDim.x * blockDim.x;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += stride)
        label[t] = flags[t] ? tmp[label[t]] : -1;
}

// vertex -> chart in the caller's vertex numbering (vperm: internal -> caller index)
__global__ void k_v2c(const int* __restrict__ vmin, const int* __restrict__ label, int* __restrict__ v2c, int V,
                      const int* __restrict__ vperm) {
    FA_PDL_PROLOGUE();
    int stride = gridDim.x * blockDim.x;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride) {
        int m = vmin[v];
        v2c[vperm ? vperm[v] : v] = m == 0x7fffffff ? -1 : label[m];
    }
}

__global__ void k_permute_pos(const double* __restrict__ pos, const int* __restrict__ vperm,
                              double* __restrict__ out, int V) {
    FA_PDL_PROLOGUE();
    int stride = gridDim.x * blockDim.x;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride) {
        const long long o = 3ll * vperm[v];
        out[3ll * v] = pos[o];
        out[3ll * v + 1] = pos[o + 1];
        out[3ll * v + 2] = pos[o + 2];
    }
}

void fa_launch_permute_pos(const double* pos, const int* vperm, double* out, int V, cudaStream_t s) {
    fa_launch(k_permute_pos, fa_grid(V, 256, FA_NUM_SMS * 8), 256, 0, s, pos, vperm, out, V);
}

__global__ void k_flags_from_labels(const int* __restrict__ labels, unsigned char* __restrict__ flags, int T) {
    FA_PDL_PROLOGUE();
    int stride = gridDim.x * blockDim.x;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += stride) flags[t] = labels[t] >= 0;
}

static inline int uf_grid(int T) { return fa_grid(T, 256, FA_NUM_SMS * 8); }

// ---- mesh edge adjacency (charts.py:64-77) ------------------------------------
// Open-addressing hash on the undirected edge key (min<<32 | max).  Insert
// counts the (triangle, edge) slots per key and records the first two; resolve
// links the two slots of keys used exactly twice (symmetric, so slot order
// does not matter) and leaves every other edge at -1, like the reference.
#define ADJ_EMPTY 0xffffffffffffffffull

__device__ __forceinline__ unsigned long long edge_key(const int* __restrict__ tris, int code) {
    int t = code / 3, e = code - 3 * t;
    unsigned a = (unsigned)__ldg(tris + 3 * t + e), b = (unsigned)__ldg(tris + 3 * t + (e == 2 ? 0 : e + 1));
    unsigned lo = a < b ? a : b, hi = a < b ? b : a;
    return ((unsigned long long)lo << 32) | hi;
}

__device__ __forceinline__ unsigned long long edge_hash(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

__global__ void k_adj_insert(const int* __restrict__ tris, int n_codes, unsigned long long* __restrict__ keys,
                             int* __restrict__ cnt, int* __restrict__ c0, int* __restrict__ c1,
                             unsigned long long mask) {
    FA_PDL_PROLOGUE();
    for (int code = blockIdx.x * blockDim.x + threadIdx.x; code < n_codes; code += gridDim.x * blockDim.x) {
        unsigned long long key = edge_key(tris, code);
        unsigned long long h = edge_hash(key) & mask;
        while (true) {
            unsigned long long old = atomicCAS(keys + h, ADJ_EMPTY, key);
            if (old == ADJ_EMPTY || old == key) break;
            h = (h + 1) & mask;
        }
        int k = atomicAdd(cnt + h, 1);
        if (k == 0) c0[h] = code;
        else if (k == 1) c1[h] = code;
    }
}

__global__ void k_adj_resolve(const int* __restrict__ tris, int n_codes, const unsigned long long* __restrict__ keys,
                              const int* __restrict__ cnt, const int* __restrict__ c0, const int* __restrict__ c1,
                              unsigned long long mask, int* __restrict__ adj) {
    FA_PDL_PROLOGUE();
    for (int code = blockIdx.x * blockDim.x + threadIdx.x; code < n_codes; code += gridDim.x * blockDim.x) {
        unsigned long long key = edge_key(tris, code);
        unsigned long long h = edge_hash(key) & mask;
        while (keys[h] != key) h = (h + 1) & mask;
        int other = -1;
        if (cnt[h] == 2) {
            int a = c0[h], b = c1[h];
            other = (a == code ? b : a) / 3;
        }
        adj[code] = other;
    }
}

void fa_launch_build_adjacency(const int* tris, int T, unsigned long long* keys, int* cnt, int* c0, int* c1,
                               unsigned long long table_size, int* adj, cudaStream_t s) {
    int n = 3 * T;
    cudaMemsetAsync(keys, 0xff, table_size * sizeof(unsigned long long), s);
    cudaMemsetAsync(cnt, 0, table_size * sizeof(int), s);
    int grid = fa_grid(n, 256, FA_NUM_SMS * 8);
    fa_launch(k_adj_insert, grid, 256, 0, s, tris, n, keys, cnt, c0, c1, table_size - 1);
    fa_launch(k_adj_resolve, grid, 256, 0, s, tris, n, keys, cnt, c0, c1, table_size - 1, adj);
}

int fa_launch_uf_vertex(const int* tris, const int* vis_list, int* vmin, int* label, int T, const fa_dstat* st,
                        cudaStream_t s, bool vmin_ready, const int4* vis_tris) {
    if (!vmin_ready) fa_launch(k_vmin, uf_grid(T), 256, 0, s, tris, vis_list, vmin, st);
    fa_launch(k_hook_multi, fa_wave_grid(k_hook_multi, 256, 0, ((long long)T + 255) / 256, FA_NUM_SMS * 8), 256, 0, s, tris, vis_list, vmin, label, st, vis_tris);
    return vmin_ready ? 1 : 2;
}

void fa_launch_uf_edges(const int* adjacency, const unsigned char* flags, const int* vis_list, int* label, int T,
                        const fa_dstat* st, cudaStream_t s) {
    fa_launch(k_hook_edges, uf_grid(T), 256, 0, s, adjacency, flags, vis_list, label, st);
}

void fa_launch_iota(int* label, int T, cudaStream_t s) { fa_launch(k_iota, uf_grid(T), 256, 0, s, label, T); }

// union(t, labels_in[t]) for every visible t (charts.py:372-374); run after
// fa_launch_uf_vertex, whose initialisation overwrites parent pointers
void fa_launch_uf_labels(const int* labels_in, const int* vis_list, int* label, int T, const fa_dstat* st,
                         cudaStream_t s) {
    fa_launch(k_hook_labels, uf_grid(T), 256, 0, s, labels_in, vis_list, label, st);
}

void fa_launch_uf_compress(const int* vis_list, int* label, int T, const fa_dstat* st, cudaStream_t s) {
    fa_launch(k_compress, fa_wave_grid(k_compress, 256, 0, ((long long)T + 255) / 256, FA_NUM_SMS * 8), 256, 0, s, vis_list, label, st);
}

void fa_launch_canonicalize(const int* vis_list, int* label, int* tmp, int T, const fa_dstat* st, cudaStream_t s) {
    // label holds roots for visible triangles; flags are recovered from the vis list
    fa_launch(k_fill, uf_grid(T), 256, 0, s, tmp, T, 0x7fffffff);
    fa_launch(k_canon_min, uf_grid(T), 256, 0, s, vis_list, label, tmp, st);
}

void fa_launch_canon_apply(const unsigned char* flags, int* label, const int* tmp, int T, cudaStream_t s) {
    fa_launch(k_canon_apply, uf_grid(T), 256, 0, s, flags, label, tmp, T);
}

// ---- visible vertices (the compact UV wire format) --------------------------
// A vertex is visible when a visible triangle touches it (vmin[v] != INT_MAX).
// Ordered compaction: vslot[v] = its index in the list, vlist[slot] = its id
// in the caller's numbering.  k_uv then writes one UV pair per visible vertex
// (every triangle of the vertex's chart computes the same value).
#define VTX_ITEMS 4
#define VTX_TILE (CMP_THREADS * VTX_ITEMS)
__global__ void __launch_bounds__(CMP_THREADS) k_vert_count(const int* __restrict__ vmin, int V,
                                                            int* __restrict__ blocks) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int vb0, vb1;
    tile_range((V + VTX_TILE - 1) / VTX_TILE, vb0, vb1);
    for (int vb = vb0; vb < vb1; vb++) {
        const int base = vb * VTX_TILE + threadIdx.x * VTX_ITEMS;
        int c = 0;
#pragma unroll
        for (int i = 0; i < VTX_ITEMS; i++) c += (base + i < V && vmin[base + i] != 0x7fffffff);
        c = warp_sum(c);
        if (lane_id() == 0) sm[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int i = 0; i < CMP_THREADS / 32; i++) s += sm[i];
            blocks[vb] = s;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(CMP_THREADS) k_vert_scatter(const int* __restrict__ vmin, int V,
                                                              const int* __restrict__ blocks, int nblocks,
                                                              const int* __restrict__ vperm, int* __restrict__ vslot,
                                                              int* __restrict__ vlist, float2* __restrict__ vuv,
                                                              fa_dstat* __restrict__ st,
                                                              unsigned int* __restrict__ vvis_mask) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int vb0, vb1;
    tile_range(nblocks, vb0, vb1);
    int offset = block_prefix_of(blocks, vb0, sm);
    for (int vb = vb0; vb < vb1; vb++) {
    const int base = vb * VTX_TILE + threadIdx.x * VTX_ITEMS;
    bool vis[VTX_ITEMS];
    int c = 0;
#pragma unroll
    for (int i = 0; i < VTX_ITEMS; i++) {
        vis[i] = base + i < V && vmin[base + i] != 0x7fffffff;
        c += vis[i];
    }
    if (vvis_mask) {
        // the visible vertices as a bit mask over the context's vertex order
        // (the order of vlist / vuv; the host maps it through the vertex
        // order once per mesh)
        static_assert(VTX_ITEMS == 4, "one nibble per thread");
        const unsigned int w = nibble_word(vis[0] | (vis[1] << 1) | (vis[2] << 2) | (vis[3] << 3));
        if ((lane_id() & 7) == 0 && base < V) vvis_mask[base >> 5] = w;
    }
    int total;
    int pos = offset + block_exclusive_scan(c, sm, &total);
#pragma unroll
    for (int i = 0; i < VTX_ITEMS; i++) {
        if (base + i < V) vslot[base + i] = vis[i] ? pos : -1;
        if (vis[i]) {
            vlist[pos] = vperm ? vperm[base + i] : base + i;
            // NaN until k_uv writes it: a vertex in front of the camera whose
            // visible triangles all reach behind it keeps NaN (its UV rows are
            // NaN, cli.py:433-435), never stale data
            if (vuv) vuv[pos] = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
            pos++;
        }
    }
    if (vb == nblocks - 1 && threadIdx.x == 0) st->n_vis_vertices = offset + total;
    offset += total;
    __syncthreads();  // sm is reused by the next tile's scan
    }
}

int fa_vertex_blocks(long long V) {
    long long b = (V + VTX_TILE - 1) / VTX_TILE;
    return b > 0 ? (int)b : 1;
}

void fa_launch_visible_vertices(const int* vmin, int V, const int* vperm, int* blocks, int* vslot, int* vlist,
                                fa_dstat* st, cudaStream_t s, float2* vuv, unsigned int* vvis_mask) {
    const int nb = fa_vertex_blocks(V);
    fa_launch(k_vert_count, fa_wave_grid(k_vert_count, CMP_THREADS, 0, nb, nb), CMP_THREADS, 0, s, vmin, V, blocks);
    fa_launch(k_vert_scatter, fa_wave_grid(k_vert_scatter, CMP_THREADS, 0, nb, nb), CMP_THREADS, 0, s, vmin, V, blocks,
              nb, vperm, vslot, vlist, vuv, st, vvis_mask);
}

void fa_launch_v2c(const int* vmin, const int* label, int* v2c, int V, cudaStream_t s, const int* vperm) {
    fa_launch(k_v2c, fa_wave_grid(k_v2c, 256, 0, ((long long)V + 255) / 256, FA_NUM_SMS * 8), 256, 0, s, vmin, label, v2c, V, vperm);
}

void fa_launch_flags_from_labels(const int* labels, unsigned char* flags, int T, cudaStream_t s) {
    fa_launch(k_flags_from_labels, uf_grid(T), 256, 0, s, labels, flags, T);
}

void fa_launch_fill(int* a, int n, int v, cudaStream_t s) { fa_launch(k_fill, uf_grid(n), 256, 0, s, a, n, v); }

// ---- chart roots: ordered compaction of label[t] == t over the vis list -------
__global__ void __launch_bounds__(CMP_THREADS) k_count_roots(const int* __restrict__ vis_list,
                                                             const int* __restrict__ label, int* __restrict__ blocks,
                                                             const fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int n = st->n_vis;
    int vb0, vb1;
    tile_range((n + ROOT_TILE - 1) / ROOT_TILE, vb0, vb1);
    for (int vb = vb0; vb < vb1; vb++) {
        int base = vb * ROOT_TILE + threadIdx.x * ROOT_ITEMS;
        int c = 0;
#pragma unroll
        for (int i = 0; i < ROOT_ITEMS; i++) {
            int k = base + i;
            if (k < n) {
                int t = vis_list[k];
                c += label[t] == t;
            }
        }
        c = warp_sum(c);
        if (lane_id() == 0) sm[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int i = 0; i < CMP_THREADS / 32; i++) s += sm[i];
            blocks[vb] = s;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(CMP_THREADS) k_scatter_roots(const int* __restrict__ vis_list,
                                                               const int* __restrict__ label,
                                                               const int* __restrict__ blocks, int nblocks,
                                                               int* __restrict__ roots, int* __restrict__ cidx,
                                                               unsigned long long* __restrict__ ndc_keys,
                                                               int* __restrict__ survived, fa_dstat* __restrict__ st) {
    FA_PDL_PROLOGUE();
    __shared__ int sm[32];
    int n = st->n_vis;
    int ntiles = (n + ROOT_TILE - 1) / ROOT_TILE;
    if (ntiles < 1) ntiles = 1;  // (tile 0 reports n_charts = 0)
    int vb0, vb1;
    tile_range(ntiles, vb0, vb1);
    int offset = block_prefix_of(blocks, vb0, sm);
    for (int vb = vb0; vb < vb1; vb++) {
    int base = vb * ROOT_TILE + threadIdx.x * ROOT_ITEMS;
    int tv[ROOT_ITEMS];
    int c = 0;
#pragma unroll
    for (int i = 0; i < ROOT_ITEMS; i++) {
        int k = base + i;
        tv[i] = -1;
        if (k < n) {
            int t = vis_list[k];
            if (label[t] == t) { tv[i] = t; c++; }
        }
    }
    int total;
    int pos = offset + block_exclusive_scan(c, sm, &total);
#pragma unroll
    for (int i = 0; i < ROOT_ITEMS; i++) {
        if (tv[i] >= 0) {
            roots[pos] = tv[i];
            cidx[tv[i]] = pos;
            ndc_keys[4 * pos + 0] = FA_KEY_POS_INF;
            ndc_keys[4 * pos + 1] = FA_KEY_POS_INF;
            ndc_keys[4 * pos + 2] = FA_KEY_NEG_INF;
            ndc_keys[4 * pos + 3] = FA_KEY_NEG_INF;
            survived[pos] = 0;
            pos++;
        }
    }
    if (vb == ntiles - 1 && threadIdx.x == 0) st->n_charts = offset + total;
    offset += total;
    __syncthreads();  // sm is reused by the next tile's scan
    }
}

void fa_launch_compact_roots(const int* vis_list, const int* label, int T, int* blocks, int* roots, int* cidx,
                             unsigned long long* ndc_keys, int* survived, fa_dstat* st, cudaStream_t s) {
    int nb = blocks_for(T, ROOT_TILE);
    fa_launch(k_count_roots, fa_wave_grid(k_count_roots, CMP_THREADS, 0, nb, nb), CMP_THREADS, 0, s, vis_list, label,
              blocks, st);
    fa_launch(k_scatter_roots, fa_wave_grid(k_scatter_roots, CMP_THREADS, 0, nb, nb), CMP_THREADS, 0, s, vis_list,
              label, blocks, nb, roots, cidx, ndc_keys, survived, st);
}

FA_TRACE_TU(charts)
