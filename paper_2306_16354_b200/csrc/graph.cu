// graph.cu — k-NN graph symmetrisation and the Boruvka spanning forest.
//
// Replaces edge_list_to_csr (/root/reference/pkg/src/parlink/core.py:264-286)
// and the solver in mst.py (weight_alteration :198-222, _hash_unit :82-91,
// _alter_weights :94-105, _min_edge_scan :108-128, _reconcile_per_color
// :131-151, _propagate_colors :154-186, solve_mst :292-344).
//
// Design: the solver's strict total order on undirected edges
// is (w_alt, a, b) with a < b.  We compute w_alt bit-exactly, then ONE stable
// device radix sort by w_alt over the (a, b)-sorted edge list gives every
// edge a 32-bit rank in that order.  Boruvka then runs on ranks: per round
// an edge-centric kernel does atomicMin(rank) into both endpoint colours
// (deterministic — ranks are unique), roots hook along their minimum edge,
// 2-cycles are broken toward the smaller id, pointers are jumped in place and
// the edge list is compacted to the edges that still cross colours.  The
// minimum spanning forest under a strict total order is unique, so the
// accepted edge set equals the reference's exactly.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace slk {

namespace {

constexpr uint32_t NONE32 = 0xffffffffu;

// ---------------------------------------------------------- sort helpers
template <class K, class V>
void sort_pairs(const K *kin, K *kout, const V *vin, V *vout, int64_t m, cudaStream_t s,
                int begin_bit = 0, int end_bit = sizeof(K) * 8) {
    if (m <= 0) return;
    size_t tmp = 0;
    SLK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)m, begin_bit,
                                             end_bit, s));
    DevBuf<unsigned char> t(tmp, s);
    SLK_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)m, begin_bit,
                                             end_bit, s));
}

template <class K>
void sort_keys(const K *kin, K *kout, int64_t m, cudaStream_t s) {
    if (m <= 0) return;
    size_t tmp = 0;
    SLK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, (int)m, 0, sizeof(K) * 8, s));
    DevBuf<unsigned char> t(tmp, s);
    SLK_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, kin, kout, (int)m, 0, sizeof(K) * 8, s));
}

template <class T>
void exclusive_sum(const T *in, T *out, int64_t m, cudaStream_t s) {
    if (m <= 0) return;
    size_t tmp = 0;
    SLK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)m, s));
    DevBuf<unsigned char> t(tmp, s);
    SLK_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, (int)m, s));
}

int bits_for(int64_t n) {
    int b = 1;
    while ((1ll << b) < n) b++;
    return b;
}

// ------------------------------------------------------------- kernels
#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void canon_keys_kernel(const int32_t *src, const int32_t *dst, int64_t m,
                                  uint64_t *keys) {
    GRID_LOOP(e, m) {
        uint32_t s = (uint32_t)src[e], d = (uint32_t)dst[e];
        uint32_t a = s < d ? s : d, b = s < d ? d : s;
        keys[e] = ((uint64_t)a << 32) | b;
    }
}

__global__ void directed_keys_kernel(const int32_t *src, const int32_t *dst, const double *w,
                                     int64_t m, uint64_t *keys, double *ws) {
    GRID_LOOP(e, m) {
        uint32_t s = (uint32_t)src[e], d = (uint32_t)dst[e];
        keys[e] = ((uint64_t)s << 32) | d;
        keys[m + e] = ((uint64_t)d << 32) | s;
        ws[e] = w[e];
        ws[m + e] = w[e];
    }
}

// run heads of a sorted key array; run minimum of the weights
__global__ void run_heads_kernel(const uint64_t *keys, int64_t m, int32_t *flag) {
    GRID_LOOP(e, m) flag[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}

__global__ void run_min_scatter_kernel(const uint64_t *keys, const double *w, const int32_t *flag,
                                       const int32_t *pos, int64_t m, int32_t *out_a,
                                       int32_t *out_b, double *out_w) {
    GRID_LOOP(e, m) {
        if (!flag[e]) continue;
        double best = w[e];
        for (int64_t f = e + 1; f < m && keys[f] == keys[e]; f++) best = fmin(best, w[f]);
        int32_t p = pos[e];
        out_a[p] = (int32_t)(keys[e] >> 32);
        out_b[p] = (int32_t)(keys[e] & 0xffffffffu);
        out_w[p] = best;
    }
}

__global__ void lower_bound_offsets_kernel(const int32_t *rows, int64_t nnz, int64_t n,
                                           int64_t *offs) {
    GRID_LOOP(v, n + 1) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((int64_t)rows[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        offs[v] = lo;
    }
}

__global__ void row_sources_kernel(const int64_t *offs, int64_t n, int32_t *src) {
    GRID_LOOP(v, n) {
        for (int64_t p = offs[v]; p < offs[v + 1]; p++) src[p] = (int32_t)v;
    }
}

__global__ void check_weights_kernel(const double *w, int64_t m, int *flags) {
    GRID_LOOP(e, m) {
        double x = w[e];
        if (!isfinite(x)) atomicOr(flags, 1);
        if (x == 0.0) atomicOr(flags, 2);
    }
}

__global__ void negate_kernel(const double *w, int64_t m, double *out, bool neg) {
    GRID_LOOP(e, m) out[e] = neg ? -w[e] : w[e];
}

// min positive gap between adjacent distinct sorted weights (mst.py:215-217)
__global__ void min_gap_kernel(const double *s, int64_t m, unsigned long long *gap_bits) {
    double g = INFINITY;
    GRID_LOOP(e, m) {
        if (e > 0 && s[e] != s[e - 1]) g = fmin(g, __dsub_rn(s[e], s[e - 1]));
    }
    for (int o = 16; o; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
    if ((threadIdx.x & 31) == 0 && g < INFINITY)
        atomicMin(gap_bits, (unsigned long long)__double_as_longlong(g));  // g > 0: bit order
}

// ref mst.py:82-91
__device__ __forceinline__ double hash_unit(uint32_t a, uint32_t b, int64_t seed) {
    uint64_t z = (uint64_t)a * 0x9E3779B97F4A7C15ULL;
    z ^= (uint64_t)b + 0xBF58476D1CE4E5B9ULL;
    z ^= (uint64_t)seed * 0x94D049BB133111EBULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return __dmul_rn((double)(z >> 11), 0x1p-53);
}

// ref mst.py:94-105: out = w + hash(a, b, seed) * eps_max (product, then sum)
__global__ void alter_kernel(const int32_t *a, const int32_t *b, const double *w, int64_t m,
                             int64_t seed, double eps_max, double *alt) {
    GRID_LOOP(e, m) {
        uint32_t s = (uint32_t)a[e], d = (uint32_t)b[e];
        uint32_t lo = s < d ? s : d, hi = s < d ? d : s;
        alt[e] = __dadd_rn(w[e], __dmul_rn(hash_unit(lo, hi, seed), eps_max));
    }
}

__global__ void iota_kernel(int32_t *v, int64_t m) {
    GRID_LOOP(e, m) v[e] = (int32_t)e;
}

template <class T>
__global__ void gather_kernel(const T *in, const int32_t *perm, int64_t m, T *out) {
    GRID_LOOP(e, m) out[e] = in[perm[e]];
}

// --- Boruvka on ranks
__global__ void fill_u32_kernel(uint32_t *v, int64_t n, uint32_t x) {
    GRID_LOOP(i, n) v[i] = x;
}

__global__ void min_edge_kernel(const int32_t *ea, const int32_t *eb, const uint32_t *erank,
                                int64_t m, const int32_t *color, uint32_t *best) {
    GRID_LOOP(e, m) {
        int32_t ca = color[ea[e]], cb = color[eb[e]];
        if (ca == cb) continue;
        uint32_t r = erank[e];
        if (best[ca] > r) atomicMin(&best[ca], r);
        if (best[cb] > r) atomicMin(&best[cb], r);
    }
}

__global__ void hook_kernel(int64_t n, const int32_t *color, const uint32_t *best,
                            const int32_t *ra, const int32_t *rb, int32_t *parent,
                            uint8_t *accepted, int *any) {
    GRID_LOOP(v, n) {
        if (color[v] != v) continue;
        uint32_t e = best[v];
        if (e == NONE32) {
            parent[v] = (int32_t)v;
            continue;
        }
        accepted[e] = 1;
        int32_t ca = color[ra[e]], cb = color[rb[e]];
        parent[v] = ca == v ? cb : ca;
        *any = 1;
    }
}

__global__ void break_cycles_kernel(int64_t n, const int32_t *color, int32_t *parent) {
    GRID_LOOP(v, n) {
        if (color[v] != v) continue;
        int32_t p = parent[v];
        if (p != v && p > v && parent[p] == v) parent[v] = (int32_t)v;
    }
}

__global__ void jump_kernel(int64_t n, const int32_t *color, int32_t *parent) {
    GRID_LOOP(v, n) {
        if (color[v] != v) continue;
        int32_t p = parent[v];
        while (true) {
            int32_t pp = parent[p];
            if (pp == p) break;
            p = pp;
        }
        parent[v] = p;
    }
}

// also clears every vertex's best edge for the next round (nothing reads
// best after the hooks)
__global__ void relabel_kernel(int64_t n, int32_t *color, const int32_t *parent, uint32_t *best) {
    GRID_LOOP(v, n) {
        color[v] = parent[color[v]];
        best[v] = NONE32;
    }
}

// edges still crossing colours after the round, in order (flag / pos from
// cross_flag_kernel and an exclusive scan)
__global__ void compact_edges_kernel(const int32_t *ea, const int32_t *eb, const uint32_t *er, const int32_t *flag,
                                     const int32_t *pos, int64_t m, int32_t *oa, int32_t *ob, uint32_t *orank) {
    GRID_LOOP(e, m) if (flag[e]) {
        const int32_t p = pos[e];
        oa[p] = ea[e];
        ob[p] = eb[e];
        orank[p] = er[e];
    }
}

// ------------------------------------------------- persistent Boruvka
// All rounds in ONE cooperative launch (grid-wide barriers between phases, no
// host round trip): per round min_edge -> hook -> break 2-cycles -> pointer
// jumping -> relabel -> compaction of the edges that still cross colours.
// Compaction appends with warp-aggregated atomics, so the order of the active
// list changes between rounds; nothing depends on it (ranks are unique and
// min_edge is an atomicMin), so the accepted set is the same unique MSF.
// counts[r] = active edges at round r (counts[0] = m, the rest zero on entry).
struct BoruvkaArgs {
    int64_t n;
    int32_t *color, *parent;
    uint32_t *best;
    const int32_t *ra, *rb;  // endpoints by rank
    uint8_t *accepted;
    int32_t *ea[2], *eb[2];
    uint32_t *er[2];
    unsigned long long *counts;  // [MAX_ROUNDS + 1]
    int *rounds;
};
constexpr int MAX_ROUNDS = 64;

__global__ void __launch_bounds__(256) boruvka_coop_kernel(BoruvkaArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t n = a.n;
    int32_t *color = a.color, *parent = a.parent;
    uint32_t *best = a.best;
    for (int r = 0; r < MAX_ROUNDS; r++) {
        const int64_t active = (int64_t)a.counts[r];
        if (active == 0) {
            if (tid == 0) *a.rounds = r;
            return;  // uniform: every thread read the same count after the last barrier
        }
        const int32_t *ea = a.ea[r & 1], *eb = a.eb[r & 1];
        const uint32_t *er = a.er[r & 1];
        for (int64_t e = tid; e < active; e += nth) {
            const int32_t ca = color[ea[e]], cb = color[eb[e]];
            if (ca == cb) continue;
            const uint32_t rk = er[e];
            if (best[ca] > rk) atomicMin(&best[ca], rk);
            if (best[cb] > rk) atomicMin(&best[cb], rk);
        }
        grid.sync();
        for (int64_t v = tid; v < n; v += nth) {  // hook every root along its minimum edge
            if (color[v] != v) continue;
            const uint32_t e = best[v];
            if (e == NONE32) {
                parent[v] = (int32_t)v;
                continue;
            }
            a.accepted[e] = 1;
            const int32_t ca = color[a.ra[e]], cb = color[a.rb[e]];
            parent[v] = ca == v ? cb : ca;
        }
        grid.sync();
        for (int64_t v = tid; v < n; v += nth) {  // a 2-cycle keeps its smaller root
            if (color[v] != v) continue;
            const int32_t p = parent[v];
            if (p != v && p > v && parent[p] == v) parent[v] = (int32_t)v;
        }
        grid.sync();
        for (int64_t v = tid; v < n; v += nth) {  // pointer jumping (in place: writes are ancestors)
            if (color[v] != v) continue;
            int32_t p = parent[v];
            while (true) {
                const int32_t pp = parent[p];
                if (pp == p) break;
                p = pp;
            }
            parent[v] = p;
        }
        grid.sync();
        for (int64_t v = tid; v < n; v += nth) {
            color[v] = parent[color[v]];
            best[v] = NONE32;
        }
        grid.sync();
        // edges that still cross colours -> the other buffer
        int32_t *oa = a.ea[(r + 1) & 1], *ob = a.eb[(r + 1) & 1];
        uint32_t *orank = a.er[(r + 1) & 1];
        for (int64_t base = tid - lane; base < active; base += nth) {
            const int64_t e = base + lane;
            bool keep = false;
            int32_t xa = 0, xb = 0;
            uint32_t xr = 0;
            if (e < active) {
                xa = ea[e];
                xb = eb[e];
                xr = er[e];
                keep = color[xa] != color[xb];
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            unsigned long long at = 0;
            if (lane == 0 && m) at = atomicAdd(&a.counts[r + 1], (unsigned long long)__popc(m));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (keep) {
                const int64_t p = (int64_t)at + __popc(m & ((1u << lane) - 1u));
                oa[p] = xa;
                ob[p] = xb;
                orank[p] = xr;
            }
        }
        grid.sync();
    }
    if (tid == 0) *a.rounds = MAX_ROUNDS;
}

__global__ void scan_total_kernel(const int32_t *pos, const int32_t *flag, int64_t m, int64_t *out) {
    *out = (int64_t)pos[m - 1] + flag[m - 1];
}

__global__ void cross_flag_kernel(const int32_t *ea, const int32_t *eb, int64_t m,
                                  const int32_t *color, int32_t *flag) {
    GRID_LOOP(e, m) flag[e] = color[ea[e]] != color[eb[e]] ? 1 : 0;
}

template <class T>
__global__ void compact_kernel(const T *in, const int32_t *flag, const int32_t *pos, int64_t m,
                               T *out) {
    GRID_LOOP(e, m) if (flag[e]) out[pos[e]] = in[e];
}

__global__ void accepted_keys_kernel(const uint8_t *accepted, const int32_t *pos, int64_t m,
                                     const int32_t *ra, const int32_t *rb, const double *rw,
                                     uint64_t *keys, double *ws) {
    GRID_LOOP(e, m) {
        if (!accepted[e]) continue;
        int32_t p = pos[e];
        keys[p] = ((uint64_t)(uint32_t)ra[e] << 32) | (uint32_t)rb[e];
        ws[p] = rw[e];
    }
}

__global__ void u8_to_i32_kernel(const uint8_t *in, int64_t m, int32_t *out) {
    GRID_LOOP(e, m) out[e] = in[e];
}

__global__ void split_keys_kernel(const uint64_t *keys, int64_t m, int32_t *a, int32_t *b) {
    GRID_LOOP(e, m) {
        a[e] = (int32_t)(keys[e] >> 32);
        b[e] = (int32_t)(keys[e] & 0xffffffffu);
    }
}

__global__ void min_member_kernel(int64_t n, const int32_t *color, int32_t *minv, int *roots) {
    GRID_LOOP(v, n) {
        // a component's vertices all hit one word: one atomic per run of
        // equal colours in the warp, from its lowest lane (smallest id)
        const int32_t c = color[v];
        const unsigned peers = __match_any_sync(__activemask(), c);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1 && minv[c] > (int32_t)v) atomicMin(&minv[c], (int32_t)v);
        if (c == v) atomicAdd(roots, 1);
    }
}

__global__ void canon_color_kernel(int64_t n, const int32_t *color, const int32_t *minv,
                                   int32_t *out) {
    GRID_LOOP(v, n) out[v] = minv[color[v]];
}

__global__ void fill_i32_kernel(int32_t *v, int64_t n, int32_t x) {
    GRID_LOOP(i, n) v[i] = x;
}

// --- CSR-level API kernels (mst.py step functions)
__device__ __forceinline__ bool key_lt(double w, int64_t a, int64_t b, double qw, int64_t qa,
                                       int64_t qb) {
    return w < qw || (w == qw && (a < qa || (a == qa && b < qb)));
}

// ref mst.py:108-128
__global__ void min_edge_scan_kernel(int64_t n, const int64_t *offs, const int32_t *cols,
                                     const double *alt, const int32_t *colors, int64_t *pos) {
    GRID_LOOP(v, n) {
        int32_t cv = colors[v];
        int64_t best = -1, ba = -1, bb = -1;
        double bw = INFINITY;
        for (int64_t p = offs[v]; p < offs[v + 1]; p++) {
            int64_t u = cols[p];
            if (colors[u] == cv) continue;
            double w = alt[p];
            int64_t a = v < u ? v : u, b = v < u ? u : v;
            if (key_lt(w, a, b, bw, ba, bb)) {
                best = p;
                bw = w;
                ba = a;
                bb = b;
            }
        }
        pos[v] = best;
    }
}

__device__ __forceinline__ unsigned long long ordered_bits(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 compares equal to +0.0 in the reference
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void reconcile_phase1(int64_t n, const int64_t *pos, const double *alt,
                                 const int32_t *colors, unsigned long long *best1) {
    GRID_LOOP(v, n) {
        if (pos[v] < 0) continue;
        atomicMin(&best1[colors[v]], ordered_bits(alt[v]));
    }
}

__global__ void reconcile_phase2(int64_t n, const int64_t *pos, const int32_t *dst,
                                 const double *alt, const int32_t *colors,
                                 const unsigned long long *best1, unsigned long long *best2) {
    GRID_LOOP(v, n) {
        if (pos[v] < 0) continue;
        int32_t c = colors[v];
        if (ordered_bits(alt[v]) != best1[c]) continue;
        uint32_t u = (uint32_t)dst[v], vv = (uint32_t)v;
        uint64_t key = ((uint64_t)(vv < u ? vv : u) << 32) | (vv < u ? u : vv);
        atomicMin(&best2[c], (unsigned long long)key);
    }
}

__global__ void reconcile_phase3(int64_t n, const int64_t *pos, const int32_t *dst,
                                 const double *alt, const double *orig, const int32_t *colors,
                                 const unsigned long long *best1, const unsigned long long *best2,
                                 int32_t *winner) {
    GRID_LOOP(v, n) {
        if (pos[v] < 0) continue;
        int32_t c = colors[v];
        if (ordered_bits(alt[v]) != best1[c]) continue;
        uint32_t u = (uint32_t)dst[v], vv = (uint32_t)v;
        uint64_t key = ((uint64_t)(vv < u ? vv : u) << 32) | (vv < u ? u : vv);
        if (key == best2[c]) atomicMin(&winner[c], (int32_t)v);
    }
}

__global__ void winner_edges_kernel(int64_t n, const int32_t *winner, const int32_t *dst,
                                    const double *orig, int32_t *flag, uint64_t *keys,
                                    double *ws) {
    GRID_LOOP(c, n) {
        int32_t v = winner[c];
        flag[c] = v != 0x7fffffff;
        if (v == 0x7fffffff) continue;
        uint32_t u = (uint32_t)dst[v], vv = (uint32_t)v;
        keys[c] = ((uint64_t)(vv < u ? vv : u) << 32) | (vv < u ? u : vv);
        ws[c] = orig[v];
    }
}

// --- label propagation (ref mst.py:154-186)
__global__ void prop_init_kernel(int64_t n, int32_t *next) {
    GRID_LOOP(c, n) next[c] = (int32_t)c;
}
__global__ void prop_edges_kernel(const int32_t *colors, const int32_t *us, const int32_t *vs,
                                  int64_t m, int32_t *next) {
    GRID_LOOP(e, m) {
        int32_t a = colors[us[e]], b = colors[vs[e]];
        if (a == b) continue;
        int32_t mn = a < b ? a : b;
        atomicMin(&next[a], mn);
        atomicMin(&next[b], mn);
    }
}
__global__ void prop_jump_kernel(int64_t n, int32_t *next) {
    GRID_LOOP(c, n) {
        int32_t p = next[c];
        while (true) {
            int32_t pp = next[p];
            if (pp >= p) break;
            p = pp;
        }
        atomicMin(&next[c], p);
    }
}
__global__ void prop_apply_kernel(int64_t n, int32_t *colors, const int32_t *next, int *changed) {
    GRID_LOOP(v, n) {
        int32_t nc = next[colors[v]];
        if (nc < colors[v]) {
            colors[v] = nc;
            *changed = 1;
        }
    }
}

// --- symmetric check
// rows strictly increasing in column: then CSR order is (src, col) order and
// there are no duplicate entries
__global__ void rows_sorted_kernel(const int32_t *src, const int32_t *cols, int64_t m, int *unsorted) {
    GRID_LOOP(e, m) if (e > 0 && src[e] == src[e - 1] && cols[e] <= cols[e - 1]) *unsorted = 1;
}

// strictly sorted rows: entry (i, j, w) needs (j, i, w); binary search of i in row j
__global__ void mirror_check_kernel(const int64_t *offs, const int32_t *src, const int32_t *cols, const double *w,
                                    int64_t m, int *diff) {
    GRID_LOOP(e, m) {
        const int32_t i = src[e], j = cols[e];
        int64_t lo = offs[j], hi = offs[j + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cols[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        if (lo >= offs[j + 1] || cols[lo] != i || !(w[lo] == w[e])) *diff = 1;
    }
}

// general rows: the reference's pairing (core.py:165-174): entries stably
// ordered by (src, col) against entries stably ordered by (col, src)
__global__ void sym_keys2_kernel(const int32_t *src, const int32_t *cols, int64_t m, uint64_t *kf, uint64_t *kr,
                                 int32_t *iota) {
    GRID_LOOP(e, m) {
        const uint32_t a = (uint32_t)src[e], b = (uint32_t)cols[e];
        kf[e] = ((uint64_t)a << 32) | b;
        kr[e] = ((uint64_t)b << 32) | a;
        iota[e] = (int32_t)e;
    }
}
__global__ void sym_compare_kernel(const uint64_t *kf, const uint64_t *kr, const int32_t *pf, const int32_t *pr,
                                   const double *w, int64_t m, int *diff) {
    GRID_LOOP(p, m) if (kf[p] != kr[p] || !(w[pf[p]] == w[pr[p]])) *diff = 1;
}

__global__ void lt_flag_kernel(const int32_t *src, const int32_t *cols, int64_t m, int32_t *flag) {
    GRID_LOOP(e, m) flag[e] = src[e] < cols[e] ? 1 : 0;
}

#undef GRID_LOOP

#define LAUNCH(kernel, n, ...)                                        \
    do {                                                              \
        kernel<<<grid_for((n), 256), 256, 0, s>>>(__VA_ARGS__);       \
        SLK_CHECK_LAUNCH();                                           \
    } while (0)

// Sort entries by (key, weight) and keep the minimum weight per key.
// Returns the number of unique keys written to (out_a, out_b, out_w).
int64_t unique_min(const uint64_t *keys_in, const double *w_in, int64_t m, int key_bits,
                   int32_t *out_a, int32_t *out_b, double *out_w, cudaStream_t s) {
    if (m == 0) return 0;
    DevBuf<uint64_t> ks(m, s);
    DevBuf<double> ws(m, s);
    sort_pairs(keys_in, ks.get(), w_in, ws.get(), m, s, 0, key_bits);
    DevBuf<int32_t> flag(m, s), pos(m, s);
    LAUNCH(run_heads_kernel, m, ks.get(), m, flag.get());
    exclusive_sum(flag.get(), pos.get(), m, s);
    int32_t last_pos = read_scalar(pos.get() + m - 1, s), last_flag = read_scalar(flag.get() + m - 1, s);
    int64_t u = (int64_t)last_pos + last_flag;
    LAUNCH(run_min_scatter_kernel, m, ks.get(), ws.get(), flag.get(), pos.get(), m, out_a, out_b, out_w);
    return u;
}

}  // namespace

#define LAUNCH(kernel, n, ...)                                        \
    do {                                                              \
        kernel<<<grid_for((n), 256), 256, 0, s>>>(__VA_ARGS__);       \
        SLK_CHECK_LAUNCH();                                           \
    } while (0)

// ---------------------------------------------------- sort-free dedups
// Undirected edges of a k-NN graph without sorting (core.py:264-286 keeps
// the minimum weight per pair; both directions of a pair carry bit-identical
// weights, knn.cu:exact_dist being symmetric in its operands): entry i -> j
// is kept as (i, j) when i < j, and as (j, i) when i > j unless row j also
// lists i (then row j keeps it).  Output order is arbitrary (msf_undirected
// orders by (w_alt, a, b) explicitly).
__global__ void knn_undirected_kernel(const int32_t *idx, const double *dist, int64_t n, int k, int32_t *oa,
                                      int32_t *ob, double *ow, unsigned long long *count) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; base < n * k;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = base + lane;
        bool keep = false;
        int32_t a = 0, b = 0;
        double w = 0.0;
        if (e < n * k) {
            const int32_t i = (int32_t)(e / k), j = idx[e];
            w = dist[e];
            if (j >= 0 && j != i) {
                if (i < j) {
                    a = i, b = j, keep = true;
                } else {
                    bool dup = false;
                    for (int t = 0; t < k; t++) dup |= idx[(int64_t)j * k + t] == i;
                    a = j, b = i, keep = !dup;
                }
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        unsigned long long at = 0;
        if (lane == 0 && m) at = atomicAdd(count, (unsigned long long)__popc(m));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (keep) {
            const int64_t p = (int64_t)at + __popc(m & ((1u << lane) - 1u));
            oa[p] = a;
            ob[p] = b;
            ow[p] = w;
        }
    }
}

// A spanning forest (canonical a < b, no duplicates) united with one
// cross-colour bridge per point (i -> bdst[i], weight bw[i]): forest edges
// join equal colours and bridges different ones, so only mutual bridge pairs
// repeat (kept from the smaller endpoint).
__global__ void union_bridges_kernel(const int32_t *bdst, const double *bw, int64_t n, int64_t ne, int32_t *oa,
                                     int32_t *ob, double *ow, unsigned long long *count) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + lane;
        bool keep = false;
        int32_t a = 0, b = 0;
        double w = 0.0;
        if (i < n) {
            const int32_t j = bdst[i];
            w = bw[i];
            if (j >= 0 && j != i) {
                keep = (int32_t)i < j || bdst[j] != (int32_t)i;
                a = min((int32_t)i, j);
                b = max((int32_t)i, j);
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        unsigned long long at = 0;
        if (lane == 0 && m) at = atomicAdd(count, (unsigned long long)__popc(m));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (keep) {
            const int64_t p = ne + (int64_t)at + __popc(m & ((1u << lane) - 1u));
            oa[p] = a;
            ob[p] = b;
            ow[p] = w;
        }
    }
}

// ------------------------------------- (w_alt, a, b) order with one sort
// w_alt = w + hash * theta (1 - 2^-20) with theta the smallest gap between
// distinct weights: for distinct w the w order IS the w_alt order (up to the
// rounding case checked below), so one stable sort by w plus an explicit
// (w_alt, a, b) sort of every run of equal w gives the solver's order.
// alter_sorted_kernel: w_alt of the w-sorted list
__global__ void alter_sorted_kernel(const int32_t *a, const int32_t *b, const double *ws, const int32_t *perm,
                                    int64_t m, int64_t seed, double eps_max, double *alt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t e = perm[p];
        const uint32_t x = (uint32_t)a[e], y = (uint32_t)b[e];
        // bit-identical to alter_kernel: hash of the canonical (min, max) pair
        alt[p] = __dadd_rn(ws[p], __dmul_rn(hash_unit(x < y ? x : y, x < y ? y : x, seed), eps_max));
    }
}

// (w_alt, a, b) order on canonical pairs (a = min, b = max of the endpoints)
__device__ __forceinline__ bool alt_less(double x, int32_t xa, int32_t xb, double y, int32_t ya, int32_t yb) {
    const int32_t xl = min(xa, xb), xh = max(xa, xb), yl = min(ya, yb), yh = max(ya, yb);
    return x < y || (x == y && (xl < yl || (xl == yl && xh < yh)));
}

// runs of equal w: insertion sort by (w_alt, a, b); flag bit 0 = a run longer
// than MAX_RUN (the caller then sorts by w_alt instead)
constexpr int MAX_RUN = 64;
__global__ void fixup_runs_kernel(const double *ws, double *alt, int32_t *perm, const int32_t *a, const int32_t *b,
                                  int64_t m, int *flag) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        if (p > 0 && ws[p] == ws[p - 1]) continue;  // not a run start
        int64_t e = p + 1;
        while (e < m && ws[e] == ws[p] && e - p <= MAX_RUN) e++;
        if (e - p == 1) continue;
        if (e - p > MAX_RUN) {
            atomicOr(flag, 1);
            continue;
        }
        for (int64_t i = p + 1; i < e; i++) {
            const double v = alt[i];
            const int32_t pi = perm[i], va = a[pi], vb = b[pi];
            int64_t j = i - 1;
            while (j >= p && alt_less(v, va, vb, alt[j], a[perm[j]], b[perm[j]])) {
                alt[j + 1] = alt[j];
                perm[j + 1] = perm[j];
                j--;
            }
            alt[j + 1] = v;
            perm[j + 1] = pi;
        }
    }
}

// flag bit 1: the list is not strictly increasing in (w_alt, a, b)
__global__ void check_order_kernel(const double *alt, const int32_t *perm, const int32_t *a, const int32_t *b,
                                   int64_t m, int *flag) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        if (p == 0) continue;
        const int32_t x = perm[p - 1], y = perm[p];
        if (!alt_less(alt[p - 1], a[x], b[x], alt[p], a[y], b[y])) atomicOr(flag, 2);
    }
}

EdgeSet dedup_undirected(int64_t n, const int32_t *src, const int32_t *dst, const double *w,
                         int64_t m, cudaStream_t s) {
    EdgeSet E;
    if (m == 0) return E;
    DevBuf<uint64_t> keys(m, s);
    LAUNCH(canon_keys_kernel, m, src, dst, m, keys.get());
    E.a.alloc(m, s);
    E.b.alloc(m, s);
    E.w.alloc(m, s);
    E.m = unique_min(keys.get(), w, m, 32 + bits_for(n), E.a.get(), E.b.get(), E.w.get(), s);
    return E;
}

EdgeSet knn_undirected(int64_t n, int k, const int32_t *idx, const double *dist, cudaStream_t s) {
    EdgeSet E;
    const int64_t m = n * k;
    if (m == 0) return E;
    E.a.alloc(m, s);
    E.b.alloc(m, s);
    E.w.alloc(m, s);
    DevBuf<unsigned long long> cnt(1, s);
    SLK_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
    LAUNCH(knn_undirected_kernel, m, idx, dist, n, k, E.a.get(), E.b.get(), E.w.get(), cnt.get());
    E.m = (int64_t)read_scalar(cnt.get(), s);
    return E;
}

EdgeSet forest_plus_bridges(int64_t n, const int32_t *fa, const int32_t *fb, const double *fw, int64_t ne,
                            const int32_t *bdst, const double *bw, cudaStream_t s) {
    EdgeSet E;
    E.a.alloc(ne + n, s);
    E.b.alloc(ne + n, s);
    E.w.alloc(ne + n, s);
    if (ne > 0) {
        SLK_CUDA(cudaMemcpyAsync(E.a.get(), fa, ne * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        SLK_CUDA(cudaMemcpyAsync(E.b.get(), fb, ne * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        SLK_CUDA(cudaMemcpyAsync(E.w.get(), fw, ne * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    DevBuf<unsigned long long> cnt(1, s);
    SLK_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
    LAUNCH(union_bridges_kernel, n, bdst, bw, n, ne, E.a.get(), E.b.get(), E.w.get(), cnt.get());
    E.m = ne + (int64_t)read_scalar(cnt.get(), s);
    return E;
}

// theta from weights already sorted ascending; m > 0.
static double theta_of_sorted(const double *sorted, int64_t m, cudaStream_t s) {
    DevBuf<unsigned long long> gap(1, s);
    unsigned long long init = (unsigned long long)0x7ff0000000000000ull;  // +inf bits
    SLK_CUDA(cudaMemcpyAsync(gap.get(), &init, sizeof(init), cudaMemcpyHostToDevice, s));
    min_gap_kernel<<<grid_for(m, 256, 2048), 256, 0, s>>>(sorted, m, gap.get());
    SLK_CHECK_LAUNCH();
    unsigned long long g = read_scalar(gap.get(), s);
    if (g != init) {
        double theta;
        memcpy(&theta, &g, sizeof theta);
        return theta;
    }
    double first = read_scalar(sorted, s);
    double a = fabs(first);
    return (a > 1.0 ? a : 1.0) * 0x1p-20;  // single distinct weight (mst.py:219)
}

// theta (mst.py:215-219) of the given weights; m > 0.
static double compute_theta(const double *w, int64_t m, cudaStream_t s) {
    DevBuf<double> sorted(m, s);
    sort_keys(w, sorted.get(), m, s);
    DevBuf<unsigned long long> gap(1, s);
    unsigned long long init = (unsigned long long)0x7ff0000000000000ull;  // +inf bits
    SLK_CUDA(cudaMemcpyAsync(gap.get(), &init, sizeof(init), cudaMemcpyHostToDevice, s));
    min_gap_kernel<<<grid_for(m, 256, 2048), 256, 0, s>>>(sorted.get(), m, gap.get());
    SLK_CHECK_LAUNCH();
    unsigned long long g = read_scalar(gap.get(), s);
    if (g != init) {
        double theta;
        memcpy(&theta, &g, sizeof theta);
        return theta;
    }
    double first = read_scalar(sorted.get(), s);
    double a = fabs(first);
    return (a > 1.0 ? a : 1.0) * 0x1p-20;  // single distinct weight (mst.py:219)
}

static void validate_weights(const double *w, int64_t m, bool check_zero, cudaStream_t s) {
    if (m == 0) return;
    DevBuf<int> flags(1, s);
    SLK_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int), s));
    LAUNCH(check_weights_kernel, m, w, m, flags.get());
    int f = read_scalar(flags.get(), s);
    if (f & 1) throw_invalid("graph contains non-finite edge weights");
    if (check_zero && (f & 2)) throw_invalid("zero-weight edges are not supported");
}

void msf_undirected(int64_t n, const int32_t *a_in, const int32_t *b_in, const double *w_in,
                    int64_t m, bool presorted, bool negate, int64_t seed, int32_t *out_src,
                    int32_t *out_dst, double *out_w, int32_t *colors_out, int64_t *n_edges,
                    int64_t *n_components, cudaStream_t s) {
    if (n <= 0) throw_invalid("empty graph: no vertices");
    EventPair ev_all, ev_rounds;
    ev_all.start(s);
    validate_weights(w_in, m, true, s);
    const int32_t *a = a_in, *b = b_in;
    const double *w = w_in;
    DevBuf<int32_t> sa, sb;
    DevBuf<double> sw;
    // --- rank order (w_alt, a, b) with ONE stable sort by w (see
    // fixup_runs_kernel), for unsorted input (the pipeline's sort-free
    // dedups).  Falls back to sorting by w_alt over the (a, b)-sorted list when
    // a run of equal weights is long or rounding breaks the order; (a, b)-
    // sorted input (CSR graphs, integer road weights with long runs of equal
    // weights) takes that path directly.
    DevBuf<int32_t> fperm;
    bool fast = false;
    if (m > 0 && !presorted && !getenv("SLK_MSF_TWO_SORTS")) {
        DevBuf<double> ww(m, s), ws(m, s), alt(m, s);
        DevBuf<int32_t> iota(m, s);
        fperm.alloc(m, s);
        LAUNCH(negate_kernel, m, w_in, m, ww.get(), negate);
        LAUNCH(iota_kernel, m, iota.get(), m);
        sort_pairs(ww.get(), ws.get(), iota.get(), fperm.get(), m, s);
        const double theta = theta_of_sorted(ws.get(), m, s);
        LAUNCH(alter_sorted_kernel, m, a_in, b_in, ws.get(), fperm.get(), m, seed, theta * (1.0 - 0x1p-20),
               alt.get());
        DevBuf<int> flag(1, s);
        SLK_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
        LAUNCH(fixup_runs_kernel, m, ws.get(), alt.get(), fperm.get(), a_in, b_in, m, flag.get());
        LAUNCH(check_order_kernel, m, alt.get(), fperm.get(), a_in, b_in, m, flag.get());
        fast = read_scalar(flag.get(), s) == 0;
        if (!fast) fperm.release();
    }
    if (!presorted && m > 0 && !fast) {
        // the (w_alt, a, b) tie-break needs the list in (a, b) order first
        DevBuf<uint64_t> keys(m, s), ks(m, s);
        DevBuf<int32_t> iota(m, s), perm(m, s);
        LAUNCH(canon_keys_kernel, m, a_in, b_in, m, keys.get());
        LAUNCH(iota_kernel, m, iota.get(), m);
        sort_pairs(keys.get(), ks.get(), iota.get(), perm.get(), m, s, 0, 32 + bits_for(n));
        sa.alloc(m, s);
        sb.alloc(m, s);
        sw.alloc(m, s);
        LAUNCH(split_keys_kernel, m, ks.get(), m, sa.get(), sb.get());
        LAUNCH(gather_kernel<double>, m, w_in, perm.get(), m, sw.get());
        a = sa.get();
        b = sb.get();
        w = sw.get();
    }
    DevBuf<int32_t> color(n, s);
    LAUNCH(iota_kernel, n, color.get(), n);
    int64_t accepted_count = 0;
    if (m > 0) {
        // --- order: w_alt (mst.py:198-222), ties by (a, b)
        DevBuf<int32_t> perm;
        if (fast) {
            perm = std::move(fperm);
        } else {
            // stable sort by w_alt over the (a, b)-sorted list
            DevBuf<double> ww(m, s), alt(m, s);
            LAUNCH(negate_kernel, m, w, m, ww.get(), negate);
            double theta = compute_theta(ww.get(), m, s);
            double eps_max = theta * (1.0 - 0x1p-20);
            LAUNCH(alter_kernel, m, a, b, ww.get(), m, seed, eps_max, alt.get());
            DevBuf<int32_t> iota(m, s);
            DevBuf<double> alt_sorted(m, s);
            perm.alloc(m, s);
            LAUNCH(iota_kernel, m, iota.get(), m);
            sort_pairs(alt.get(), alt_sorted.get(), iota.get(), perm.get(), m, s);
        }
        DevBuf<int32_t> ra(m, s), rb(m, s);
        DevBuf<double> rw(m, s);
        LAUNCH(gather_kernel<int32_t>, m, a, perm.get(), m, ra.get());
        LAUNCH(gather_kernel<int32_t>, m, b, perm.get(), m, rb.get());
        LAUNCH(gather_kernel<double>, m, w, perm.get(), m, rw.get());
        perm.release();

        // --- Boruvka rounds on ranks: one persistent cooperative launch
        DevBuf<int32_t> ea2(m, s), eb2(m, s), flag(m, s), pos(m, s);
        DevBuf<uint32_t> er(m, s), er2(m, s), best(n, s);
        DevBuf<int32_t> parent(n, s);
        DevBuf<uint8_t> accepted(m, s);
        DevBuf<unsigned long long> counts(MAX_ROUNDS + 1, s);
        DevBuf<int> nrounds(1, s);
        LAUNCH(iota_kernel, m, (int32_t *)er.get(), m);
        SLK_CUDA(cudaMemsetAsync(accepted.get(), 0, m, s));
        SLK_CUDA(cudaMemsetAsync(counts.get(), 0, (MAX_ROUNDS + 1) * sizeof(unsigned long long), s));
        {
            const unsigned long long m0 = (unsigned long long)m;
            SLK_CUDA(cudaMemcpyAsync(counts.get(), &m0, sizeof(m0), cudaMemcpyHostToDevice, s));
        }
        LAUNCH(fill_u32_kernel, n, best.get(), n, NONE32);
        ev_rounds.start(s);
        BoruvkaArgs ba{n, color.get(), parent.get(), best.get(), ra.get(), rb.get(), accepted.get(),
                       {ra.get(), ea2.get()}, {rb.get(), eb2.get()}, {er.get(), er2.get()}, counts.get(),
                       nrounds.get()};
        // the active edge lists alternate between two buffers; ra / rb stay
        // intact (hook reads endpoints by rank), so buffer 0 starts as a copy
        DevBuf<int32_t> ea0(m, s), eb0(m, s);
        SLK_CUDA(cudaMemcpyAsync(ea0.get(), ra.get(), m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        SLK_CUDA(cudaMemcpyAsync(eb0.get(), rb.get(), m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        ba.ea[0] = ea0.get();
        ba.eb[0] = eb0.get();
        static int coop_blocks = 0;
        if (!coop_blocks) {
            int per_sm = 0;
            SLK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, boruvka_coop_kernel, 256, 0));
            coop_blocks = std::max(1, per_sm) * num_sms();
        }
        void *kargs[] = {&ba};
        SLK_CUDA(cudaLaunchCooperativeKernel((void *)boruvka_coop_kernel, dim3(coop_blocks), dim3(256), kargs, 0, s));
        SLK_CHECK_LAUNCH();
        ev_rounds.stop(s);
        unsigned long long hc[MAX_ROUNDS + 1];
        int rounds = 0;
        SLK_CUDA(cudaMemcpyAsync(hc, counts.get(), sizeof(hc), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(&rounds, nrounds.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaStreamSynchronize(s));
        double mst_bytes = 0.0;
        for (int r = 0; r < rounds; r++)
            mst_bytes += 12.0 * 2.0 * (double)hc[r] + 16.0 * (double)n;  // directed entries = 2 x undirected
        profile().mst_ms += ev_rounds.ms();
        profile().mst_bytes += mst_bytes;
        profile().mst_rounds += rounds;
        // --- accepted edges, sorted by (a, b) with original weights
        LAUNCH(u8_to_i32_kernel, m, accepted.get(), m, flag.get());
        exclusive_sum(flag.get(), pos.get(), m, s);
        accepted_count = (int64_t)read_scalar(pos.get() + m - 1, s) + read_scalar(flag.get() + m - 1, s);
        if (accepted_count > n - 1) throw_internal("accepted %lld edges for %lld vertices",
                                                   (long long)accepted_count, (long long)n);
        DevBuf<uint64_t> keys(accepted_count, s), keys_sorted(accepted_count, s);
        DevBuf<double> ws(accepted_count, s);
        LAUNCH(accepted_keys_kernel, m, accepted.get(), pos.get(), m, ra.get(), rb.get(), rw.get(),
               keys.get(), ws.get());
        sort_pairs(keys.get(), keys_sorted.get(), ws.get(), out_w, accepted_count, s, 0,
                   32 + bits_for(n));
        LAUNCH(split_keys_kernel, accepted_count, keys_sorted.get(), accepted_count, out_src, out_dst);
    }
    // --- canonical colours: minimum vertex id per component
    DevBuf<int32_t> minv(n, s);
    DevBuf<int> roots(1, s);
    LAUNCH(fill_i32_kernel, n, minv.get(), n, 0x7fffffff);
    SLK_CUDA(cudaMemsetAsync(roots.get(), 0, sizeof(int), s));
    LAUNCH(min_member_kernel, n, n, color.get(), minv.get(), roots.get());
    LAUNCH(canon_color_kernel, n, n, color.get(), minv.get(), colors_out);
    int64_t ncomp = read_scalar(roots.get(), s);
    if (accepted_count != n - ncomp)
        throw_internal("internal: accepted %lld edges for %lld vertices and %lld components",
                       (long long)accepted_count, (long long)n, (long long)ncomp);
    *n_edges = accepted_count;
    *n_components = ncomp;
    ev_all.stop(s);
    profile().msf_ms += ev_all.ms();
}

// ------------------------------------------------------- C-ABI helpers
void csr_from_edges(int64_t n, const int32_t *src, const int32_t *dst, const double *w, int64_t m,
                    int64_t *offs, int32_t *cols, double *cw, int64_t *nnz, cudaStream_t s) {
    if (m == 0) {
        SLK_CUDA(cudaMemsetAsync(offs, 0, (n + 1) * sizeof(int64_t), s));
        *nnz = 0;
        return;
    }
    DevBuf<uint64_t> keys(2 * m, s);
    DevBuf<double> ws(2 * m, s);
    LAUNCH(directed_keys_kernel, m, src, dst, w, m, keys.get(), ws.get());
    DevBuf<int32_t> rows(2 * m, s);
    int64_t u = unique_min(keys.get(), ws.get(), 2 * m, 32 + bits_for(n), rows.get(), cols, cw, s);
    LAUNCH(lower_bound_offsets_kernel, n + 1, rows.get(), u, n, offs);
    *nnz = u;
}

void csr_row_sources(int64_t n, const int64_t *offs, int32_t *src, cudaStream_t s) {
    LAUNCH(row_sources_kernel, n, offs, n, src);
}

// True iff the rows are strictly increasing in column (CSR order = (src, col)
// order, no duplicate entries); src = row of every entry.
static bool rows_strictly_sorted(const int32_t *src, const int32_t *cols, int64_t m, cudaStream_t s) {
    DevBuf<int> flag(1, s);
    SLK_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
    LAUNCH(rows_sorted_kernel, m, src, cols, m, flag.get());
    return read_scalar(flag.get(), s) == 0;
}

// core.py:165-174.  Strictly sorted rows (the canonical CSR edge_list_to_csr
// builds): one binary search per entry for its mirror.  Otherwise the
// reference's pairing of the two stable orders, by two radix sorts.
bool csr_symmetric(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                   cudaStream_t s) {
    int64_t m = read_scalar(offs + n, s);
    if (m == 0) return true;
    DevBuf<int32_t> src(m, s);
    csr_row_sources(n, offs, src.get(), s);
    DevBuf<int> diff(1, s);
    SLK_CUDA(cudaMemsetAsync(diff.get(), 0, sizeof(int), s));
    if (rows_strictly_sorted(src.get(), cols, m, s)) {
        LAUNCH(mirror_check_kernel, m, offs, src.get(), cols, w, m, diff.get());
        return read_scalar(diff.get(), s) == 0;
    }
    DevBuf<uint64_t> kf(m, s), kr(m, s), k1(m, s), k2(m, s);
    DevBuf<int32_t> iota(m, s), pf(m, s), pr(m, s);
    const int bits = 32 + bits_for(n);
    LAUNCH(sym_keys2_kernel, m, src.get(), cols, m, kf.get(), kr.get(), iota.get());
    sort_pairs(kf.get(), k1.get(), iota.get(), pf.get(), m, s, 0, bits);
    sort_pairs(kr.get(), k2.get(), iota.get(), pr.get(), m, s, 0, bits);
    LAUNCH(sym_compare_kernel, m, k1.get(), k2.get(), pf.get(), pr.get(), w, m, diff.get());
    return read_scalar(diff.get(), s) == 0;
}
void csr_validate(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                  cudaStream_t s) {
    if (n <= 0) throw_invalid("empty graph: no vertices");
    int64_t m = read_scalar(offs + n, s);
    validate_weights(w, m, false, s);
    if (!csr_symmetric(n, offs, cols, w, s))
        throw_invalid("graph must be symmetric: every (i, j, w) needs its (j, i, w)");
}

double csr_weight_alteration(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                             int64_t seed, double *alt, cudaStream_t s) {
    csr_validate(n, offs, cols, w, s);
    int64_t m = read_scalar(offs + n, s);
    validate_weights(w, m, true, s);
    if (m == 0) return 0.0;
    double theta = compute_theta(w, m, s);
    DevBuf<int32_t> src(m, s);
    csr_row_sources(n, offs, src.get(), s);
    LAUNCH(alter_kernel, m, src.get(), cols, w, m, seed, theta * (1.0 - 0x1p-20), alt);
    return theta;
}

void csr_min_edge_per_vertex(int64_t n, const int64_t *offs, const int32_t *cols,
                             const double *alt, const int32_t *colors, int64_t *pos,
                             cudaStream_t s) {
    LAUNCH(min_edge_scan_kernel, n, n, offs, cols, alt, colors, pos);
}

int64_t reconcile_supervertex(int64_t n, const int64_t *pos, const int32_t *dst,
                              const double *alt, const double *orig, const int32_t *colors,
                              int32_t *out_a, int32_t *out_b, double *out_w, cudaStream_t s) {
    DevBuf<unsigned long long> best1(n, s), best2(n, s);
    DevBuf<int32_t> winner(n, s), flag(n, s), p(n, s);
    SLK_CUDA(cudaMemsetAsync(best1.get(), 0xff, n * sizeof(unsigned long long), s));
    SLK_CUDA(cudaMemsetAsync(best2.get(), 0xff, n * sizeof(unsigned long long), s));
    LAUNCH(fill_i32_kernel, n, winner.get(), n, 0x7fffffff);
    LAUNCH(reconcile_phase1, n, n, pos, alt, colors, best1.get());
    LAUNCH(reconcile_phase2, n, n, pos, dst, alt, colors, best1.get(), best2.get());
    LAUNCH(reconcile_phase3, n, n, pos, dst, alt, orig, colors, best1.get(), best2.get(), winner.get());
    DevBuf<uint64_t> keys(n, s);
    DevBuf<double> ws(n, s);
    LAUNCH(winner_edges_kernel, n, n, winner.get(), dst, orig, flag.get(), keys.get(), ws.get());
    exclusive_sum(flag.get(), p.get(), n, s);
    int64_t cnt = (int64_t)read_scalar(p.get() + n - 1, s) + read_scalar(flag.get() + n - 1, s);
    if (cnt == 0) return 0;
    DevBuf<uint64_t> k2(cnt, s);
    DevBuf<double> w2(cnt, s);
    LAUNCH(compact_kernel<uint64_t>, n, keys.get(), flag.get(), p.get(), n, k2.get());
    LAUNCH(compact_kernel<double>, n, ws.get(), flag.get(), p.get(), n, w2.get());
    return unique_min(k2.get(), w2.get(), cnt, 32 + bits_for(n), out_a, out_b, out_w, s);
}

void label_propagation(int64_t n, int32_t *colors, const int32_t *us, const int32_t *vs, int64_t m,
                       cudaStream_t s) {
    if (m == 0 || n == 0) return;
    DevBuf<int32_t> next(n, s);
    DevBuf<int> changed(1, s);
    for (int it = 0; it < 4096; it++) {
        LAUNCH(prop_init_kernel, n, n, next.get());
        LAUNCH(prop_edges_kernel, m, colors, us, vs, m, next.get());
        LAUNCH(prop_jump_kernel, n, n, next.get());
        SLK_CUDA(cudaMemsetAsync(changed.get(), 0, sizeof(int), s));
        LAUNCH(prop_apply_kernel, n, n, colors, next.get(), changed.get());
        if (!read_scalar(changed.get(), s)) return;
    }
    throw_internal("label propagation did not converge");
}

void csr_solve_mst(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                   bool maximize, int64_t seed, int32_t *out_src, int32_t *out_dst, double *out_w,
                   int32_t *colors, int64_t *n_edges, int64_t *n_components, cudaStream_t s) {
    csr_validate(n, offs, cols, w, s);
    int64_t m = read_scalar(offs + n, s);
    // undirected entries (src < col) in CSR order
    DevBuf<int32_t> src(m, s), flag(m, s), pos(m, s);
    int64_t mu = 0;
    bool presorted = true;
    DevBuf<int32_t> ua, ub;
    DevBuf<double> uw;
    if (m > 0) {
        csr_row_sources(n, offs, src.get(), s);
        validate_weights(w, m, true, s);
        LAUNCH(lt_flag_kernel, m, src.get(), cols, m, flag.get());
        exclusive_sum(flag.get(), pos.get(), m, s);
        mu = (int64_t)read_scalar(pos.get() + m - 1, s) + read_scalar(flag.get() + m - 1, s);
        ua.alloc(mu, s);
        ub.alloc(mu, s);
        uw.alloc(mu, s);
        LAUNCH(compact_kernel<int32_t>, m, src.get(), flag.get(), pos.get(), m, ua.get());
        LAUNCH(compact_kernel<int32_t>, m, cols, flag.get(), pos.get(), m, ub.get());
        LAUNCH(compact_kernel<double>, m, w, flag.get(), pos.get(), m, uw.get());
        // strictly sorted rows: the (src < col) entries are already in (a, b) order
        presorted = rows_strictly_sorted(src.get(), cols, m, s);
    }
    msf_undirected(n, ua.get(), ub.get(), uw.get(), mu, presorted, maximize, seed, out_src, out_dst,
                   out_w, colors, n_edges, n_components, s);
}

}  // namespace slk
