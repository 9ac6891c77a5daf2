// dendro.cu — dendrogram construction and the flat cut.
//
// Replaces build_dendrogram (/root/reference/pkg/src/parlink/linkage.py:160-181,
// _dendrogram_merge :103-129, _uf_find :91-100) and extract_clusters
// (:184-213, _inherit_labels :132-148).
//
// The (w, a, b) ordering of the N-1 tree edges is a device radix sort (two
// stable passes: by canonical key, then by weight).  The merge fold is the
// reference's sequential union-find (union by rank + path compression); like
// the paper it runs on the host, in native code, over the
// sorted arrays.  Its cost is O(N α(N)) and it is timed in the pipeline.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
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
__device__ __forceinline__ int32_t cc_find(int32_t *parent, int32_t x) {
    int32_t p = parent[x];
    while (p != x) {
        const int32_t g = parent[p];
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

// Sorts the n-1 tree edges by (w', a, b) with w' = sqrt(w) when requested
// (linkage.py:177, 295-297) and stages them on the host for the fold.  When
// the tree is large, the first t = min(n-1-FOLD_TOP, cut) merges are grouped
// by the component of the forest they form (device hook + pointer jumping,
// stable radix sort by component root, gather), so the host folds the groups
// in parallel (fold.cu).  cut < 0: no flat cut requested.
FoldInput dendrogram_device_sort(const int32_t *src, const int32_t *dst, const double *w, int64_t n,
                                 bool take_sqrt, int64_t cut, cudaStream_t s) {
    FoldInput in;
    in.n = n;
    in.threads = fold_threads();
    const int64_t m = n - 1;
    if (m <= 0) return in;
    DevBuf<uint64_t> keys(m, s), ks(m, s);
    DevBuf<double> wt(m, s), w1(m, s), w2(m, s);
    DevBuf<int32_t> iota(m, s), perm1(m, s), iota2(m, s), perm2(m, s), a(m, s), b(m, s);
    int grid = grid_for(m, 256);
    dendro_keys_kernel<<<grid, 256, 0, s>>>(src, dst, w, m, take_sqrt, keys, wt, iota);
    SLK_CHECK_LAUNCH();
    sort_pairs(keys.get(), ks.get(), iota.get(), perm1.get(), m, s);  // by (a, b)
    dendro_gather_kernel<<<grid, 256, 0, s>>>(ks, perm1, wt, m, w1);
    SLK_CHECK_LAUNCH();
    // stable by w' → (w', a, b); iota2 indexes the (a, b)-sorted list
    SLK_CUDA(cudaMemcpyAsync(iota2.get(), iota.get(), m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    sort_pairs(w1.get(), w2.get(), iota2.get(), perm2.get(), m, s);
    dendro_final_kernel<<<grid, 256, 0, s>>>(ks, perm2, m, a, b);
    SLK_CHECK_LAUNCH();

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
    SLK_CUDA(cudaMemcpyAsync(ha + t, a.get() + t, (m - t) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaMemcpyAsync(hb + t, b.get() + t, (m - t) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaMemcpyAsync(hw + t, w2.get() + t, (m - t) * sizeof(double), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaStreamSynchronize(s));
    in.a = ha;
    in.b = hb;
    in.w = hw;
    in.t = t;
    if (cut >= 0 && !getenv("SLK_HOST_CUT")) {
        // enqueued after the fold input is on the host: runs while the host
        // folds; the caller synchronises the stream before reading labels
        DevBuf<int32_t> parent(n, s), cmax(n, s), rid(n, s), flag(n + cut, s), pos(n + cut, s), lab(n, s);
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
        int32_t *hl = staging.labels.get(n);
        SLK_CUDA(cudaMemcpyAsync(hl, lab.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        in.labels = hl;
    }
    return in;
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
