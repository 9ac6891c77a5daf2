// dendro.cu — dendrogram construction and the flat cut.
//
// Replaces build_dendrogram (/root/reference/pkg/src/parlink/linkage.py:160-181,
// _dendrogram_merge :103-129, _uf_find :91-100) and extract_clusters
// (:184-213, _inherit_labels :132-148).
//
// The (w, a, b) ordering of the N-1 tree edges is a device radix sort (two
// stable passes: by canonical key, then by weight).  The merge table is then
// built on the device (krt_kernel, below): the reference's sequential
// union-find fold is restated as a time-split recursion of polylog depth.
// The host fold (fold.cu, the paper's choice: PAPER.md:355) stays as the
// SLK_HOST_FOLD=1 alternative.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cooperative_groups.h>
#include <memory>
#include <thread>
#include <vector>

#include "common.cuh"

namespace slk {

namespace {

__global__ void dendro_keys_kernel(const int32_t *src, const int32_t *dst, const double *w,
                                   int64_t m, bool take_sqrt, uint64_t *keys, double *wt,
                                   int32_t *iota) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = (uint32_t)src[e], d = (uint32_t)dst[e];
        uint32_t a = s < d ? s : d, b = s < d ? d : s;
        keys[e] = ((uint64_t)a << 32) | b;
        wt[e] = take_sqrt ? __dsqrt_rn(w[e]) : w[e];  // np.sqrt is correctly rounded
        iota[e] = (int32_t)e;
    }
}

__global__ void dendro_gather_kernel(const uint64_t *keys_sorted, const int32_t *perm1,
                                     const double *wt, int64_t m, double *w1) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x)
        w1[e] = wt[perm1[e]];
}

__global__ void dendro_final_kernel(const uint64_t *keys_sorted, const int32_t *perm2, int64_t m,
                                    int32_t *a, int32_t *b) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys_sorted[perm2[e]];
        a[e] = (int32_t)(k >> 32);
        b[e] = (int32_t)(k & 0xffffffffu);
    }
}

// After the sort by w': ks = the canonical keys in w' order with every run
// of equal w' sorted by key (insertion sort, one thread per run); flag = 1 if
// a run is longer than RUN_MAX (the caller re-sorts).
constexpr int RUN_MAX = 64;
__global__ void dendro_runs_kernel(const uint64_t *keys, const int32_t *perm, const double *ws, int64_t m,
                                   uint64_t *ks, int *flag) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        if (p > 0 && ws[p] == ws[p - 1]) continue;  // not a run start
        int64_t e = p + 1;
        while (e < m && ws[e] == ws[p] && e - p <= RUN_MAX) e++;
        if (e - p > RUN_MAX) {
            atomicOr(flag, 1);
            continue;
        }
        for (int64_t i = p; i < e; i++) {
            const uint64_t v = keys[perm[i]];
            int64_t j = i - 1;
            while (j >= p && ks[j] > v) {
                ks[j + 1] = ks[j];
                j--;
            }
            ks[j + 1] = v;
        }
    }
}

__global__ void dendro_split_kernel(const uint64_t *ks, int64_t m, int32_t *a, int32_t *b) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        a[e] = (int32_t)(ks[e] >> 32);
        b[e] = (int32_t)(ks[e] & 0xffffffffu);
    }
}

template <class K, class V>
void sort_pairs(const K *kin, K *kout, const V *vin, V *vout, int64_t m, cudaStream_t s,
                int end_bit = sizeof(K) * 8) {
    if (m <= 0) return;
    size_t tmp = 0;
    SLK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)m, 0, end_bit, s));
    DevBuf<unsigned char> t(tmp, s);
    SLK_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)m, 0, end_bit, s));
}

// ---- components of the forest of the first t merges (hook + pointer jumping)
// Union-find entries that other SMs update during the same launch are read
// with ld.global.cg (L2, never a stale L1 line): the hook loops retry until
// a CAS sees the current root, so a stale cached read could spin.
__device__ __forceinline__ int32_t cc_find(int32_t *parent, int32_t x) {
    int32_t p = __ldcg(parent + x);
    while (p != x) {
        const int32_t g = __ldcg(parent + p);
        if (g != p) parent[x] = g;  // halving; a stale write still points at an ancestor
        x = p;
        p = g;
    }
    return x;
}

__global__ void cc_init_kernel(int32_t *parent, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        parent[v] = (int32_t)v;
}

// the larger root hooks under the smaller: every component ends rooted at its
// smallest vertex, whatever the interleaving
__global__ void cc_hook_kernel(const int32_t *a, const int32_t *b, int64_t t, int32_t *parent) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < t; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = a[e], v = b[e];
        while (true) {
            u = cc_find(parent, u);
            v = cc_find(parent, v);
            if (u == v) break;
            const int32_t hi = u > v ? u : v, lo = u > v ? v : u;
            if (atomicCAS(&parent[hi], hi, lo) == hi) break;
        }
    }
}

__global__ void cc_key_kernel(const int32_t *a, int64_t t, int32_t *parent, int32_t *key, int32_t *iota) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < t; e += (int64_t)gridDim.x * blockDim.x) {
        key[e] = cc_find(parent, a[e]);
        iota[e] = (int32_t)e;
    }
}

__global__ void group_gather_kernel(const int32_t *rank, int64_t t, const int32_t *a, const int32_t *b,
                                    const double *w, int32_t *ga, int32_t *gb, double *gw) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < t; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t e = rank[j];
        ga[j] = a[e];
        gb[j] = b[e];
        gw[j] = w[e];
    }
}

// ---- the flat cut on the device (linkage.py:184-213): after the first `cut`
// merges the clusters are the components of the forest of those edges; a
// component's cluster id is n + (its last merge), a point alone keeps its own
// id; labels rank the ids ascending (the roots are exactly those ids).
__global__ void cut_max_kernel(const int32_t *a, int64_t cut, int32_t *parent, int32_t *cmax) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cut; e += (int64_t)gridDim.x * blockDim.x)
        atomicMax(&cmax[cc_find(parent, a[e])], (int32_t)e);
}

__global__ void cut_rid_kernel(int64_t n, int32_t *parent, const int32_t *cmax, int32_t *rid, int32_t *flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = cc_find(parent, (int32_t)v);
        const int32_t id = cmax[r] >= 0 ? (int32_t)(n + cmax[r]) : (int32_t)v;
        rid[v] = id;
        flag[id] = 1;
    }
}

__global__ void cut_label_kernel(int64_t n, const int32_t *rid, const int32_t *pos, int32_t *lab) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        lab[v] = pos[rid[v]];
}

__global__ void fill_minus1_kernel(int32_t *v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = -1;
}

// ---- the merge table on the device: Kruskal reconstruction tree (KRT)
//
// Row i of the reference's fold (linkage.py:103-129) records the cluster ids
// of the two components that edge i joins in the forest F_{<i} of the edges
// before it: a point alone keeps its own id, a component formed by merges
// keeps n + (its largest merge).  Those ids are the KRT nodes of the
// components, so row i only needs, for both endpoints, the KRT node of
// their component in F_{<i}, and its size.
//
// Time-split recursion: a window [lo, hi) of merge ranks sees the components
// of F_{<lo} as super-vertices, labelled by their KRT node ids.  Splitting it
// at mid, the left half [lo, mid) keeps those labels; the right half needs
// the components of F_{<mid}: the connected components of the left half's
// edges over the super-vertices, each labelled n + (its largest edge), which
// is exactly the KRT node the fold would give it.  After log2(m) levels every
// window is one edge whose two labels are the row's children.  All windows of
// one level are solved together with one union-find over node ids: a label
// names a component of F_{<lo} for the windows that see it, and an edge of
// any window touching it merges it away, so no label occurs in the left
// halves of two windows of a level (nothing to separate).  The per-level
// union-find state is tagged with its level instead of being reset: a node
// whose entry carries an older level is a root with no largest edge and no
// accumulated size.  Windows of KRT_LEAF edges are folded in order by one
// warp each (labels deduplicated across the lanes, the fold itself on a
// shared-memory union-find of at most 2 * KRT_LEAF slots).  Depth:
// log2(m / KRT_LEAF) levels of three grid-wide phases, ONE cooperative launch.
constexpr int KRT_LEAF_LOG = 5, KRT_LEAF = 1 << KRT_LEAF_LOG;  // = warp size: lane j folds rank i0 + j
constexpr int KRT_THREADS = 256, KRT_WARPS = KRT_THREADS / 32;

struct KrtArgs {
    int64_t m, n;
    int levels, top;  // grid-wide levels; windows at level D hold 2^(top - D) ranks
    bool block_tail;  // the windows left after the grid levels go to krt_block_kernel
    const int32_t *a, *b;  // endpoints in merge order
    const double *w;       // merge heights in merge order
    int32_t *la, *lb;      // endpoint labels (KRT node ids) at the current level
    int32_t *size;         // [2n-1] KRT node sizes (leaves 1; a merge node once it is a label)
    // [2n-1] per-level state, tagged with the level in the high 32 bits:
    // uf = (level, parent) (an older level: a root), cmax = (level, largest
    // edge of the component), acc = (level, size of the component);
    // seen = 2 * level + 1 once the node's size went into acc
    unsigned long long *uf[2], *cmax, *acc;  // uf: one buffer per level parity
    int32_t *seen;
    int32_t *rows;   // [m][3] output: child a, child b (a < b), size; size -1 marks a cycle
    int *cycle;
    unsigned long long *stamps;  // SLK_TRACE: %globaltimer after each grid-wide phase (or null)
};

__device__ __forceinline__ void krt_stamp(const KrtArgs &k, int idx) {
    if (k.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        k.stamps[idx] = t;
    }
}

// level D is stored as D + 1, so the zero entry is "older than every level"
// and tagged maxima compare level first
__device__ __forceinline__ unsigned long long tag(int D, int32_t v) {
    return ((unsigned long long)(uint32_t)(D + 1) << 32) | (uint32_t)v;
}
__device__ __forceinline__ int tag_level(unsigned long long t) { return (int)(t >> 32) - 1; }
__device__ __forceinline__ int32_t tag_value(unsigned long long t) { return (int32_t)(uint32_t)t; }

// root of x in the level-D forest (path halving; a stale halving write still
// points at an ancestor); *rv = the root's entry, the CAS operand of a hook
__device__ __forceinline__ int32_t krt_find(unsigned long long *uf, int D, int32_t x, unsigned long long *rv) {
    unsigned long long v = __ldcg(uf + x);  // L2: see cc_find
    while (tag_level(v) == D) {
        const int32_t p = tag_value(v);
        const unsigned long long vp = __ldcg(uf + p);
        if (tag_level(vp) != D) {
            x = p;
            v = vp;
            break;
        }
        uf[x] = vp;  // x -> grandparent
        x = tag_value(vp);
        v = __ldcg(uf + x);
    }
    *rv = v;
    return x;
}

// the root with the SMALLER id hooks under the other: the labels of large
// components are recent KRT nodes (large ids), so the many small labels
// joining one of them hook under it, each CAS on its own entry
__device__ __forceinline__ void krt_union(unsigned long long *uf, int D, int32_t u, int32_t v) {
    while (true) {
        unsigned long long ru, rv;
        u = krt_find(uf, D, u, &ru);
        v = krt_find(uf, D, v, &rv);
        if (u == v) return;
        if (u < v) {
            if (atomicCAS(&uf[u], ru, tag(D, v)) == ru) return;
        } else {
            if (atomicCAS(&uf[v], rv, tag(D, u)) == rv) return;
        }
    }
}

// a left edge's share of its component: the sizes of its labels not yet
// counted at this level, added to the component root's tagged accumulator
__device__ __forceinline__ void krt_acc_add(unsigned long long *acc, int D, int32_t r, int32_t add) {
    unsigned long long v = __ldcg(acc + r);
    while (tag_level(v) != D) {  // first add of this level: replace the stale entry
        const unsigned long long old = atomicCAS(&acc[r], v, tag(D, add));
        if (old == v) return;
        v = old;
    }
    atomicAdd(&acc[r], (unsigned long long)(uint32_t)add);
}

__global__ void __launch_bounds__(KRT_THREADS) krt_kernel(KrtArgs k) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t m = k.m, n = k.n, nodes = 2 * n - 1;
    int32_t *la = k.la, *lb = k.lb, *size = k.size, *seen = k.seen;
    unsigned long long *cmax = k.cmax, *acc = k.acc;
    // every rank loop gives a warp 32 consecutive ranks
    const int64_t tid0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t i = tid0; i < m; i += nth) {
        la[i] = k.a[i];
        lb[i] = k.b[i];
    }
    const unsigned long long stale = 0ull;  // level -1
    for (int64_t v = tid0; v < nodes; v += nth) {
        k.uf[0][v] = stale;
        k.uf[1][v] = stale;
        cmax[v] = stale;
        acc[v] = stale;
        seen[v] = -1;
        if (v < n) size[v] = 1;
    }
    grid.sync();
    krt_stamp(k, 0);
    // (1) components of the left halves' edges, level 0 (later levels: in (3))
    if (k.levels > 0) {
        const int sh = k.top - 1;
        for (int64_t i = tid0; i < m; i += nth)
            if (!((i >> sh) & 1)) krt_union(k.uf[0], 0, la[i], lb[i]);
    }
    grid.sync();
    krt_stamp(k, 1);
    for (int D = 0; D < k.levels; D++) {
        const int sh = k.top - D - 1;  // rank bit of the half within the window
        const int32_t mark = 2 * D + 1;
        unsigned long long *uf = k.uf[D & 1];
        // (2) per component: its largest edge and its size (each label counted
        // once), one pair of atomics per component per warp
        for (int64_t base = tid0 - lane; base < m; base += nth) {  // warp-uniform
            const int64_t i = base + lane;
            const bool left = i < m && !((i >> sh) & 1);
            int32_t r = -1, add = 0;
            if (left) {
                unsigned long long rv;
                const int32_t x = la[i], y = lb[i];
                r = krt_find(uf, D, x, &rv);
                if (atomicExch(&seen[x], mark) != mark) add += size[x];
                if (atomicExch(&seen[y], mark) != mark) add += size[y];
            }
            const unsigned grp = __match_any_sync(0xffffffffu, r);
            const unsigned gmax = __reduce_max_sync(grp, left ? (unsigned)i : 0u);
            const unsigned gsum = __reduce_add_sync(grp, (unsigned)add);
            if (left && lane == __ffs(grp) - 1) {
                atomicMax(&cmax[r], tag(D, (int32_t)gmax));
                if (gsum) krt_acc_add(acc, D, r, (int32_t)gsum);
            }
        }
        grid.sync();
        krt_stamp(k, 2 + 2 * D);
        // (3) new KRT nodes take their sizes; the right halves move to F_{<mid};
        // then (1) of level D + 1 on the other union-find buffer (the same
        // thread owns rank i in both loops, so its labels are final)
        const bool next = D + 1 < k.levels;
        unsigned long long *uf_next = k.uf[(D + 1) & 1];
        for (int64_t i = tid0; i < m; i += nth) {
            unsigned long long rv;
            if (!((i >> sh) & 1)) {
                const int32_t r = krt_find(uf, D, la[i], &rv);
                if (tag_value(cmax[r]) == (int32_t)i) size[n + i] = tag_value(acc[r]);
            } else {
                const int32_t x = la[i], y = lb[i];
                if (seen[x] == mark) la[i] = (int32_t)(n + tag_value(cmax[krt_find(uf, D, x, &rv)]));
                if (seen[y] == mark) lb[i] = (int32_t)(n + tag_value(cmax[krt_find(uf, D, y, &rv)]));
            }
            if (next && !((i >> (sh - 1)) & 1)) krt_union(uf_next, D + 1, la[i], lb[i]);
        }
        grid.sync();
        krt_stamp(k, 3 + 2 * D);
    }
    if (k.block_tail) {
        if (k.stamps) {
            grid.sync();
            krt_stamp(k, 2 + 2 * k.levels);
        }
        return;  // uniform
    }
    // leaf windows of L <= 32 ranks, one warp each: lane j holds rank i0 + j.
    // Slots: 0..31 the x labels, 32..63 the y labels; a label's slot is its
    // first occurrence (x half first), the fold runs on lane 0 over the
    // slots' shared-memory union-find, and every lane writes its own row.
    __shared__ int32_t s_val[KRT_WARPS][64], s_par[KRT_WARPS][64], s_cid[KRT_WARPS][64], s_sz[KRT_WARPS][64];
    __shared__ int32_t s_slot[KRT_WARPS][32][2], s_res[KRT_WARPS][32][3];
    const int64_t L = (int64_t)1 << (k.top - k.levels);
    const int64_t nwin = (m + L - 1) / L;
    const int64_t nwarps = (int64_t)gridDim.x * KRT_WARPS;
    for (int64_t win = blockIdx.x * (int64_t)KRT_WARPS + wib; win < nwin; win += nwarps) {
        const int64_t i0 = win * L;
        const int cnt = (int)(m - i0 < L ? m - i0 : L);
        const bool valid = lane < cnt;
        const int64_t i = i0 + lane;
        const int32_t x = valid ? la[i] : -1 - lane, y = valid ? lb[i] : -33 - lane;  // dummies never match
        s_val[wib][lane] = x;
        s_val[wib][32 + lane] = y;
        const unsigned mx = __match_any_sync(0xffffffffu, x), my = __match_any_sync(0xffffffffu, y);
        __syncwarp();
        int sy = -1;
        for (int q = 0; q < 32 && sy < 0; q++)
            if (s_val[wib][q] == y) sy = q;
        const int sx = __ffs(mx) - 1;
        if (sy < 0) sy = 32 + __ffs(my) - 1;
        s_slot[wib][lane][0] = sx;
        s_slot[wib][lane][1] = sy;
        s_par[wib][lane] = lane;
        s_par[wib][32 + lane] = 32 + lane;
        s_cid[wib][lane] = x;
        s_cid[wib][32 + lane] = y;
        s_sz[wib][lane] = valid ? size[x] : 0;
        s_sz[wib][32 + lane] = valid ? size[y] : 0;
        __syncwarp();
        if (lane == 0) {
            int32_t *par = s_par[wib], *cid = s_cid[wib], *sz = s_sz[wib];
            for (int j = 0; j < cnt; j++) {
                int rx = s_slot[wib][j][0], ry = s_slot[wib][j][1];
                while (par[rx] != rx) rx = par[rx];
                while (par[ry] != ry) ry = par[ry];
                if (rx == ry) {
                    s_res[wib][j][2] = -1;
                    continue;
                }
                const int32_t ca = cid[rx], cb = cid[ry], tot = sz[rx] + sz[ry];
                s_res[wib][j][0] = ca < cb ? ca : cb;
                s_res[wib][j][1] = ca < cb ? cb : ca;
                s_res[wib][j][2] = tot;
                par[ry] = rx;
                cid[rx] = (int32_t)(n + i0 + j);
                sz[rx] = tot;
            }
        }
        __syncwarp();
        if (valid) {
            int32_t *row = k.rows + 3 * i;
            const int32_t tot = s_res[wib][lane][2];
            if (tot < 0) *k.cycle = 1;
            row[0] = s_res[wib][lane][0];
            row[1] = s_res[wib][lane][1];
            row[2] = tot;
        }
        __syncwarp();
    }
    if (k.stamps) {
        grid.sync();
        krt_stamp(k, 2 + 2 * k.levels);
    }
}

// ---- the lower levels of the recursion, one CTA per window of up to
// KB ranks (block-local, shared memory, block barriers instead of grid-wide
// ones).  The window's labels go into a shared-memory hash table (slot =
// table position); per level the slots' union-find, largest edge and size
// are reset and recomputed exactly as in krt_kernel, the new labels
// (n + largest edge) are inserted with their sizes, and the right halves
// move to them; windows of 32 ranks are then folded in order by lane 0 of a
// warp on the slots (labels are unique to a 32-rank window, so the warps of
// a CTA never touch the same slot).
constexpr int KB_LOG = 10, KB = 1 << KB_LOG, KB_T = 4 * KB, KB_THREADS = 256, KB_PER = KB / KB_THREADS;
constexpr size_t KB_SMEM = 5 * KB_T * sizeof(int32_t) + (KB_T / 32) * sizeof(uint32_t) + KB * 5 * sizeof(int32_t);

__device__ __forceinline__ int kb_insert(int32_t *keys, int32_t *ssz, int32_t label, int32_t sz_if_new,
                                         const int32_t *gsize) {
    uint32_t h = ((uint32_t)label * 2654435761u) >> (32 - (KB_LOG + 2));
    while (true) {
        const int32_t old = atomicCAS(&keys[h], -1, label);
        if (old == -1) {
            ssz[h] = gsize ? gsize[label] : sz_if_new;
            return (int)h;
        }
        if (old == label) return (int)h;
        h = (h + 1) & (KB_T - 1);
    }
}

// read-only walk (no path halving: concurrent halving writes in shared memory
// are benign but racecheck cannot tell; hash-slot ids link at random, so the
// trees stay shallow)
__device__ __forceinline__ int kb_find(const int32_t *uf, int x) {
    int p = uf[x];
    while (p != x) {
        x = p;
        p = uf[x];
    }
    return x;
}

__global__ void __launch_bounds__(KB_THREADS) krt_block_kernel(KrtArgs k) {
    extern __shared__ __align__(16) unsigned char kb_smem[];
    int32_t *keys = reinterpret_cast<int32_t *>(kb_smem), *uf = keys + KB_T, *cmx = uf + KB_T, *acc = cmx + KB_T,
            *ssz = acc + KB_T;
    uint32_t *sbits = reinterpret_cast<uint32_t *>(ssz + KB_T);
    int32_t(*s_slot)[2] = reinterpret_cast<int32_t(*)[2]>(sbits + KB_T / 32);
    int32_t(*s_res)[3] = reinterpret_cast<int32_t(*)[3]>(s_slot + KB);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wlog = k.top - k.levels;  // <= KB_LOG
    const int64_t m = k.m, n = k.n;
    const int64_t i0 = (int64_t)blockIdx.x << wlog;
    const int cnt = (int)(m - i0 < ((int64_t)1 << wlog) ? m - i0 : ((int64_t)1 << wlog));
    for (int e = tid; e < KB_T; e += KB_THREADS) keys[e] = -1;
    __syncthreads();
    int sx[KB_PER], sy[KB_PER];  // slots of my ranks r = j * KB_THREADS + tid
#pragma unroll
    for (int j = 0; j < KB_PER; j++) {
        const int r = j * KB_THREADS + tid;
        sx[j] = sy[j] = -1;
        if (r < cnt) {
            sx[j] = kb_insert(keys, ssz, k.la[i0 + r], 0, k.size);
            sy[j] = kb_insert(keys, ssz, k.lb[i0 + r], 0, k.size);
        }
    }
    for (int L = 0; L < wlog - KRT_LEAF_LOG; L++) {
        const int sh = wlog - L - 1;
        __syncthreads();
        for (int e = tid; e < KB_T; e += KB_THREADS) {
            uf[e] = e;
            cmx[e] = -1;
            acc[e] = 0;
        }
        for (int e = tid; e < KB_T / 32; e += KB_THREADS) sbits[e] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KB_PER; j++) {  // (1) union of the left halves' edges
            const int r = j * KB_THREADS + tid;
            if (r >= cnt || ((r >> sh) & 1)) continue;
            int u = sx[j], v = sy[j];
            while (true) {
                u = kb_find(uf, u);
                v = kb_find(uf, v);
                if (u == v) break;
                const int hi = u > v ? u : v, lo = u > v ? v : u;
                if (atomicCAS(&uf[lo], lo, hi) == lo) break;
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KB_PER; j++) {  // (2) largest edge, sizes (each slot once)
            const int r = j * KB_THREADS + tid;
            if (r >= cnt || ((r >> sh) & 1)) continue;
            const int rt = kb_find(uf, sx[j]);
            atomicMax(&cmx[rt], r);
            int add = 0;
            const uint32_t bx = 1u << (sx[j] & 31), by = 1u << (sy[j] & 31);
            if (!(atomicOr(&sbits[sx[j] >> 5], bx) & bx)) add += ssz[sx[j]];
            if (!(atomicOr(&sbits[sy[j] >> 5], by) & by)) add += ssz[sy[j]];
            if (add) atomicAdd(&acc[rt], add);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KB_PER; j++) {  // (3a) the component's new label n + (largest edge)
            const int r = j * KB_THREADS + tid;
            if (r >= cnt || ((r >> sh) & 1)) continue;
            const int rt = kb_find(uf, sx[j]);
            if (atomicAdd(&cmx[rt], 0) == r) {  // atomic read: the creator rewrites it below
                const int h = kb_insert(keys, ssz, (int32_t)(n + i0 + r), acc[rt], nullptr);
                atomicExch(&cmx[rt], -(h + 2));  // never equal to a rank
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KB_PER; j++) {  // (3b) right halves move to F_{<mid}
            const int r = j * KB_THREADS + tid;
            if (r >= cnt || !((r >> sh) & 1)) continue;
            if (sbits[sx[j] >> 5] & (1u << (sx[j] & 31))) sx[j] = -cmx[kb_find(uf, sx[j])] - 2;
            if (sbits[sy[j] >> 5] & (1u << (sy[j] & 31))) sy[j] = -cmx[kb_find(uf, sy[j])] - 2;
        }
    }
    // fold the 32-rank windows in order: slot state = union-find, cluster id, size
    __syncthreads();
    for (int e = tid; e < KB_T; e += KB_THREADS) {
        uf[e] = e;
        acc[e] = keys[e];  // cluster id
    }
#pragma unroll
    for (int j = 0; j < KB_PER; j++) {
        const int r = j * KB_THREADS + tid;
        s_slot[r][0] = sx[j];
        s_slot[r][1] = sy[j];
    }
    __syncthreads();
    if (lane == 0) {
        for (int j = 0; j < KB_PER; j++) {
            const int r0 = j * KB_THREADS + warp * 32;
            for (int r = r0; r < r0 + 32 && r < cnt; r++) {
                int rx = s_slot[r][0], ry = s_slot[r][1];
                while (uf[rx] != rx) rx = uf[rx];
                while (uf[ry] != ry) ry = uf[ry];
                if (rx == ry) {
                    s_res[r][2] = -1;
                    continue;
                }
                const int32_t ca = acc[rx], cb = acc[ry], tot = ssz[rx] + ssz[ry];
                s_res[r][0] = ca < cb ? ca : cb;
                s_res[r][1] = ca < cb ? cb : ca;
                s_res[r][2] = tot;
                uf[ry] = rx;
                acc[rx] = (int32_t)(n + i0 + r);
                ssz[rx] = tot;
            }
        }
    }
    __syncthreads();
    for (int r = tid; r < cnt; r += KB_THREADS) {
        int32_t *row = k.rows + 3 * (i0 + r);
        const int32_t tot = s_res[r][2];
        if (tot < 0) *k.cycle = 1;
        row[0] = s_res[r][0];
        row[1] = s_res[r][1];
        row[2] = tot;
    }
}

struct FoldStaging {
    PinnedBuf<int32_t> a, b, rank, labels;
    PinnedBuf<double> w;
    std::vector<int64_t> off;
};
thread_local FoldStaging staging;

constexpr int64_t FOLD_TOP = 4096;           // merges folded in order after the parallel prefix
constexpr int64_t FOLD_MIN_PARALLEL = 1 << 17;

int fold_threads() {
    if (const char *e = getenv("SLK_FOLD_THREADS")) return std::max(1, atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min(32u, std::max(1u, hc));
}

}  // namespace

namespace {

struct SortedTree {
    DevBuf<int32_t> a, b;  // canonical endpoints in merge order
    DevBuf<double> w;      // merge heights w' in merge order
};

// The n-1 tree edges sorted by (w', a, b) with w' = sqrt(w) when requested
// (linkage.py:177, 295-297): stable radix sort by the canonical key, then a
// stable one by w'.
SortedTree sort_tree(const int32_t *src, const int32_t *dst, const double *w, int64_t m, bool take_sqrt,
                     cudaStream_t s) {
    SortedTree T;
    DevBuf<uint64_t> keys(m, s), ks(m, s);
    DevBuf<double> wt(m, s);
    DevBuf<int32_t> iota(m, s), perm(m, s);
    T.a.alloc(m, s);
    T.b.alloc(m, s);
    T.w.alloc(m, s);
    const int grid = grid_for(m, 256);
    dendro_keys_kernel<<<grid, 256, 0, s>>>(src, dst, w, m, take_sqrt, keys, wt, iota);
    SLK_CHECK_LAUNCH();
    // One radix sort by w', then each run of equal w' put in (a, b) order in
    // place (tree weights rarely tie); a run longer than RUN_MAX falls back
    // to two stable sorts, by (a, b) and then by w'.
    sort_pairs(wt.get(), T.w.get(), iota.get(), perm.get(), m, s);
    DevBuf<int> flag(1, s);
    SLK_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
    dendro_runs_kernel<<<grid, 256, 0, s>>>(keys, perm, T.w, m, ks, flag);
    SLK_CHECK_LAUNCH();
    if (read_scalar<int>(flag.get(), s)) {
        DevBuf<double> w1(m, s);
        DevBuf<int32_t> perm1(m, s);
        sort_pairs(keys.get(), ks.get(), iota.get(), perm1.get(), m, s);  // by (a, b)
        dendro_gather_kernel<<<grid, 256, 0, s>>>(ks, perm1, wt, m, w1);
        SLK_CHECK_LAUNCH();
        // stable by w' → (w', a, b); iota indexes the (a, b)-sorted list
        sort_pairs(w1.get(), T.w.get(), iota.get(), perm.get(), m, s);
        dendro_final_kernel<<<grid, 256, 0, s>>>(ks, perm, m, T.a, T.b);
        SLK_CHECK_LAUNCH();
        return T;
    }
    dendro_split_kernel<<<grid, 256, 0, s>>>(ks, m, T.a, T.b);
    SLK_CHECK_LAUNCH();
    return T;
}

// The flat cut on the device (linkage.py:184-213) from the merge-ordered
// endpoints: int32 labels into lab[n].
void device_cut(const int32_t *a, const int32_t *b, int64_t n, int64_t cut, int32_t *lab, cudaStream_t s) {
    DevBuf<int32_t> parent(n, s), cmax(n, s), rid(n, s), flag(n + cut, s), pos(n + cut, s);
    cc_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(parent, n);
    fill_minus1_kernel<<<grid_for(n, 256), 256, 0, s>>>(cmax, n);
    SLK_CUDA(cudaMemsetAsync(flag.get(), 0, (n + cut) * sizeof(int32_t), s));
    if (cut > 0) {
        cc_hook_kernel<<<grid_for(cut, 256), 256, 0, s>>>(a, b, cut, parent);
        cut_max_kernel<<<grid_for(cut, 256), 256, 0, s>>>(a, cut, parent, cmax);
    }
    cut_rid_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, parent, cmax, rid, flag);
    SLK_CHECK_LAUNCH();
    size_t tmp = 0;
    SLK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.get(), pos.get(), (int)(n + cut), s));
    DevBuf<unsigned char> tb(tmp, s);
    SLK_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, flag.get(), pos.get(), (int)(n + cut), s));
    cut_label_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, rid, pos, lab);
    SLK_CHECK_LAUNCH();
}

thread_local PinnedBuf<int> cycle_flag;

}  // namespace

// Sorts the tree edges (sort_tree) and stages them on the host for the host
// fold (fold.cu, SLK_HOST_FOLD=1).  When the tree is large, the first
// t = min(n-1-FOLD_TOP, cut) merges are grouped by the component of the
// forest they form (device hook + pointer jumping, stable radix sort by
// component root, gather), so the host folds the groups in parallel.  cut < 0:
// no flat cut requested.
FoldInput dendrogram_device_sort(const int32_t *src, const int32_t *dst, const double *w, int64_t n,
                                 bool take_sqrt, int64_t cut, cudaStream_t s) {
    FoldInput in;
    in.n = n;
    in.threads = fold_threads();
    const int64_t m = n - 1;
    if (m <= 0) return in;
    SortedTree T = sort_tree(src, dst, w, m, take_sqrt, s);
    const int32_t *a = T.a.get(), *b = T.b.get();
    const double *w2 = T.w.get();
    DevBuf<int32_t> iota(m, s);
    int64_t t = std::min(m - FOLD_TOP, cut >= 0 ? cut : m);
    if (m < FOLD_MIN_PARALLEL || in.threads < 2 || t < FOLD_MIN_PARALLEL / 2) t = 0;
    int32_t *ha = staging.a.get(m), *hb = staging.b.get(m);
    double *hw = staging.w.get(m);
    if (t > 0) {
        DevBuf<int32_t> parent(n, s), key(t, s), key2(t, s), rank(t, s), ga(t, s), gb(t, s), cnt(t, s),
            uniq(t, s), nrun(1, s);
        DevBuf<double> gw(t, s);
        cc_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(parent, n);
        cc_hook_kernel<<<grid_for(t, 256), 256, 0, s>>>(a, b, t, parent);
        cc_key_kernel<<<grid_for(t, 256), 256, 0, s>>>(a, t, parent, key, iota);
        SLK_CHECK_LAUNCH();
        sort_pairs(key.get(), key2.get(), iota.get(), rank.get(), t, s);  // stable: ranks stay increasing
        group_gather_kernel<<<grid_for(t, 256), 256, 0, s>>>(rank, t, a, b, w2, ga, gb, gw);
        SLK_CHECK_LAUNCH();
        size_t tmp = 0;
        SLK_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp, key2.get(), uniq.get(), cnt.get(), nrun.get(),
                                                    (int)t, s));
        DevBuf<unsigned char> tb(tmp, s);
        SLK_CUDA(cub::DeviceRunLengthEncode::Encode(tb.get(), tmp, key2.get(), uniq.get(), cnt.get(), nrun.get(),
                                                    (int)t, s));
        const int ng = read_scalar<int32_t>(nrun.get(), s);
        std::vector<int32_t> hc(ng);
        int32_t *hr = staging.rank.get(t);
        SLK_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), ng * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(hr, rank.get(), t * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(ha, ga.get(), t * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(hb, gb.get(), t * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(hw, gw.get(), t * sizeof(double), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaStreamSynchronize(s));
        staging.off.assign(ng + 1, 0);
        for (int g = 0; g < ng; g++) staging.off[g + 1] = staging.off[g] + hc[g];
        in.rank = hr;
        in.off = staging.off.data();
        in.ngroups = ng;
    }
    SLK_CUDA(cudaMemcpyAsync(ha + t, a + t, (m - t) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaMemcpyAsync(hb + t, b + t, (m - t) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaMemcpyAsync(hw + t, w2 + t, (m - t) * sizeof(double), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaStreamSynchronize(s));
    in.a = ha;
    in.b = hb;
    in.w = hw;
    in.t = t;
    if (cut >= 0 && !getenv("SLK_HOST_CUT")) {
        // enqueued after the fold input is on the host: runs while the host
        // folds; the caller synchronises the stream before reading labels
        DevBuf<int32_t> lab(n, s);
        device_cut(a, b, n, cut, lab, s);
        int32_t *hl = staging.labels.get(n);
        SLK_CUDA(cudaMemcpyAsync(hl, lab.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        in.labels = hl;
    }
    return in;
}

// The merge table on the device (krt_kernel) and, when cut >= 0, the flat
// cut (linkage.py:103-129, 184-213), see DeviceMerges.  Enqueued only; the
// returned pinned flag is nonzero after the stream synchronises if the edges
// contain a cycle (the caller raises).
const int *dendrogram_device(const int32_t *src, const int32_t *dst, const double *w, int64_t n,
                             bool take_sqrt, int64_t cut, DeviceMerges &out, cudaStream_t s,
                             cudaStream_t cut_stream, cudaEvent_t table_done) {
    int *flag = cycle_flag.get(1);
    *flag = 0;
    const int64_t m = n - 1;
    if (m <= 0) return flag;
    if (n >= (1ll << 30)) throw_invalid("n=%lld too large for the dendrogram", (long long)n);
    // timing events only under SLK_TRACE (no per-call event churn otherwise)
    const bool trace = getenv("SLK_TRACE") != nullptr;
    std::unique_ptr<EventPair> ev_sort(trace ? new EventPair : nullptr), ev_krt(trace ? new EventPair : nullptr),
        ev_cut(trace ? new EventPair : nullptr), ev_blk(trace ? new EventPair : nullptr);
    if (trace) ev_sort->start(s);
    SortedTree T = sort_tree(src, dst, w, m, take_sqrt, s);
    out.rows.alloc(3 * m, s);
    if (cut >= 0) out.labels.alloc(n, s);
    const int64_t nodes = 2 * n - 1;
    DevBuf<int32_t> la(m, s), lb(m, s), size(nodes, s), seen(nodes, s);
    DevBuf<unsigned long long> uf0(nodes, s), uf1(nodes, s), cmax(nodes, s), acc(nodes, s);
    DevBuf<int> dcycle(1, s);
    SLK_CUDA(cudaMemsetAsync(dcycle.get(), 0, sizeof(int), s));
    int top = 0;
    while (((int64_t)1 << top) < m) top++;
    const bool block_tail = !getenv("SLK_KRT_GRID_ONLY");
    KrtArgs ka{m, n, std::max(0, top - (block_tail ? KB_LOG : KRT_LEAF_LOG)), top, block_tail, T.a.get(), T.b.get(),
               T.w.get(), la.get(), lb.get(),
               size.get(), {uf0.get(), uf1.get()}, cmax.get(), acc.get(), seen.get(), out.rows.get(), dcycle.get(),
               nullptr};
    static int coop_blocks = 0;
    if (!coop_blocks) {
        int per_sm = 0;
        SLK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, krt_kernel, KRT_THREADS, 0));
        coop_blocks = std::max(1, per_sm) * num_sms();
    }
    DevBuf<unsigned long long> stamps(trace ? 2 * ka.levels + 3 : 0, s);
    ka.stamps = trace ? stamps.get() : nullptr;
    if (trace) {
        ev_sort->stop(s);
        ev_krt->start(s);
    }
    void *kargs[] = {&ka};
    SLK_CUDA(cudaLaunchCooperativeKernel((void *)krt_kernel, dim3(coop_blocks), dim3(KRT_THREADS), kargs, 0, s));
    SLK_CHECK_LAUNCH();
    if (trace) ev_blk->start(s);
    if (block_tail) {
        static bool attr = false;
        if (!attr) {
            SLK_CUDA(cudaFuncSetAttribute(krt_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KB_SMEM));
            attr = true;
        }
        const int64_t nwin = (m + ((int64_t)1 << (top - ka.levels)) - 1) >> (top - ka.levels);
        krt_block_kernel<<<(unsigned)nwin, KB_THREADS, KB_SMEM, s>>>(ka);
        SLK_CHECK_LAUNCH();
    }
    if (trace) {
        ev_blk->stop(s);
        ev_krt->stop(s);
    }
    // the cut after the table (next to the cooperative kernel both slowed
    // down); on cut_stream when given, so the table's copies on s overlap it
    cudaStream_t cs = s;
    if (cut >= 0 && cut_stream && table_done) {
        SLK_CUDA(cudaEventRecord(table_done, s));
        SLK_CUDA(cudaStreamWaitEvent(cut_stream, table_done, 0));
        cs = cut_stream;
        T.a.stream = T.b.stream = cut_stream;  // freed after the cut has read them
    }
    if (trace) ev_cut->start(cs);
    if (cut >= 0) device_cut(T.a.get(), T.b.get(), n, cut, out.labels.get(), cs);
    if (trace) ev_cut->stop(cs);
    if (trace) {
        std::vector<unsigned long long> h(2 * ka.levels + 3);
        SLK_CUDA(cudaMemcpyAsync(h.data(), stamps.get(), h.size() * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaStreamSynchronize(s));
        const double cut_ms = ev_cut->ms();
        fprintf(stderr, "[slk] krt: sort %.3f ms; %d blocks, %d levels (leaf windows %lld): kernel %.3f ms, cut %.3f ms; "
                        "union(0) %.1f us, per level (us, max+size / relabel+next union):", ev_sort->ms(), coop_blocks,
                ka.levels, (long long)1 << (ka.top - ka.levels), ev_krt->ms(), cut_ms, (h[1] - h[0]) * 1e-3);
        for (int D = 0; D < ka.levels; D++)
            fprintf(stderr, " [%d] %.1f %.1f", D, (h[2 + 2 * D] - h[1 + 2 * D]) * 1e-3,
                    (h[3 + 2 * D] - h[2 + 2 * D]) * 1e-3);
        fprintf(stderr, " leaf %.1f; block-local tail %.3f ms\n", (h[2 + 2 * ka.levels] - h[1 + 2 * ka.levels]) * 1e-3,
                block_tail ? ev_blk->ms() : 0.0);
    }
    SLK_CUDA(cudaMemcpyAsync(flag, dcycle.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    out.w = std::move(T.w);
    return flag;
}

// linkage.py:184-213
void extract_labels(const double *merges, int64_t n, int64_t n_clusters, int64_t *labels) {
    if (n_clusters < 1 || n_clusters > n)
        throw_invalid("n_clusters must be in [1, %lld], got %lld", (long long)n, (long long)n_clusters);
    int64_t cut = (n - 1) - (n_clusters - 1), total = 2 * n - 1;
    // row i may only reference points and the clusters of earlier rows
    // (ref linkage.py:103-129 builds exactly such tables; a forward reference
    // raises IndexError there and must not index out of bounds here)
    for (int64_t i = 0; i < n - 1; i++)
        for (int c = 0; c < 2; c++) {
            const double v = merges[4 * i + c];
            if (!(v >= 0.0 && v < (double)(n + i)) || v != (double)(int64_t)v)
                throw_invalid("merge row %lld references cluster %g before it exists", (long long)i, v);
        }
    std::vector<uint8_t> consumed(n + cut, 0);
    for (int64_t i = 0; i < cut; i++) {
        consumed[(int64_t)merges[4 * i]] = 1;
        consumed[(int64_t)merges[4 * i + 1]] = 1;
    }
    std::vector<int64_t> node_label(total, -1), parent(total, -1), stack;
    int64_t nroots = 0;
    for (int64_t v = 0; v < n + cut; v++)
        if (!consumed[v]) node_label[v] = nroots++;
    if (nroots != n_clusters)
        throw_invalid("internal: found %lld label roots for %lld clusters", (long long)nroots,
                      (long long)n_clusters);
    for (int64_t i = 0; i < n - 1; i++) {
        parent[(int64_t)merges[4 * i]] = n + i;
        parent[(int64_t)merges[4 * i + 1]] = n + i;
    }
    stack.reserve(64);
    for (int64_t p = 0; p < n; p++) {
        int64_t node = p;
        stack.clear();
        while (node_label[node] < 0) {
            stack.push_back(node);
            node = parent[node];
        }
        int64_t lab = node_label[node];
        for (int64_t v : stack) node_label[v] = lab;
        labels[p] = lab;
    }
}

}  // namespace slk
