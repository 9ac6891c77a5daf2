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

}  // namespace

// Sort the n-1 tree edges by (w', a, b) with w' = sqrt(w) when requested;
// writes host arrays (a, b, w') in merge order.
void dendrogram_device_sort(const int32_t *src, const int32_t *dst, const double *w, int64_t n,
                            bool take_sqrt, int32_t *h_a, int32_t *h_b, double *h_w,
                            cudaStream_t s) {
    int64_t m = n - 1;
    if (m <= 0) return;
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
    SLK_CUDA(cudaMemcpyAsync(h_a, a.get(), m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaMemcpyAsync(h_b, b.get(), m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaMemcpyAsync(h_w, w2.get(), m * sizeof(double), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaStreamSynchronize(s));
}

// linkage.py:184-213
void extract_labels(const double *merges, int64_t n, int64_t n_clusters, int64_t *labels) {
    if (n_clusters < 1 || n_clusters > n)
        throw_invalid("n_clusters must be in [1, %lld], got %lld", (long long)n, (long long)n_clusters);
    int64_t cut = (n - 1) - (n_clusters - 1), total = 2 * n - 1;
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
