// common.cuh — shared plumbing for libslink (status handling, scratch
// allocation, launch accounting).  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <memory>
#include <string>

#include "../../include/slink.h"

namespace slk {

// ---------------------------------------------------------------- errors
struct Error {
    int status;
    std::string msg;
};

void set_error(int status, const std::string &msg);
int fail(int status, const char *fmt, ...);

#define SLK_CUDA(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::slk::Error{SLK_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    } while (0)

#define SLK_CHECK_LAUNCH()                                                                   \
    do {                                                                                     \
        ::slk::count_launch();                                                               \
        cudaError_t _e = cudaGetLastError();                                                 \
        if (_e != cudaSuccess)                                                               \
            throw ::slk::Error{SLK_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)}; \
    } while (0)

[[noreturn]] void throw_invalid(const char *fmt, ...);
[[noreturn]] void throw_internal(const char *fmt, ...);

void count_launch();

// Run `body`, translating thrown slk::Error into a status code.
template <class F>
int guarded(F &&body) {
    try {
        body();
        return SLK_OK;
    } catch (const Error &e) {
        set_error(e.status, e.msg);
        return e.status;
    } catch (const std::exception &e) {
        set_error(SLK_ERR_INTERNAL, e.what());
        return SLK_ERR_INTERNAL;
    }
}

// ------------------------------------------------------- device scratch
// Keep freed scratch in the device's stream-ordered pool instead of returning
// it to the driver at every synchronisation (default release threshold 0).
void ensure_pool();
// Reserve `bytes` of the device pool in one piece (see slink_api.cu).
void reserve_pool(size_t bytes, cudaStream_t s);
// SLK_TRACE=1 in the environment: sub-stage timings on stderr
bool trace_on();
// SLK_TRACE: host milliseconds since the previous mark on this thread
void trace_mark(const char *what);

// Stream-ordered scratch buffer (cudaMallocAsync pool); freed on destruction.
template <class T>
struct DevBuf {
    T *ptr = nullptr;
    size_t count = 0;
    cudaStream_t stream = nullptr;
    DevBuf() = default;
    DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
    void alloc(size_t n, cudaStream_t s) {
        release();
        stream = s;
        count = n;
        if (n) {
            ensure_pool();
            SLK_CUDA(cudaMallocAsync((void **)&ptr, n * sizeof(T), s));
        }
    }
    void release() {
        if (ptr) cudaFreeAsync(ptr, stream);
        ptr = nullptr;
        count = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : ptr(o.ptr), count(o.count), stream(o.stream) {
        o.ptr = nullptr;
        o.count = 0;
    }
    DevBuf &operator=(DevBuf &&o) noexcept {
        release();
        ptr = o.ptr;
        count = o.count;
        stream = o.stream;
        o.ptr = nullptr;
        o.count = 0;
        return *this;
    }
    T *get() const { return ptr; }
    operator T *() const { return ptr; }
};

// Grow-only pinned host staging buffer (keep one per host thread: thread_local).
template <class T>
struct PinnedBuf {
    T *p = nullptr;
    size_t cap = 0;
    T *get(size_t n) {
        if (n > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            SLK_CUDA(cudaMallocHost((void **)&p, (n > 0 ? n : 1) * sizeof(T)));
            cap = n;
        }
        return p;
    }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

inline int grid_for(int64_t n, int block, int64_t cap = 148 * 32) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

template <class T>
T read_scalar(const T *d_ptr, cudaStream_t s) {
    T v;
    SLK_CUDA(cudaMemcpyAsync(&v, d_ptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaStreamSynchronize(s));
    return v;
}

// Number of SMs of the current device (cached).
int num_sms();

// ------------------------------------------------- cross-module entry points
// Scan statistics of the last neighbour search on this thread.
struct ScanStats {
    int64_t rows_refined = 0, rows_rescanned = 0, tiles_computed = 0, tiles_skipped = 0,
            rows_uncertified = 0;
};
ScanStats &scan_stats();

// Cumulative kernel profile (process-wide), read by bench.py via slk_profile.
struct Profile {
    double scan_ms = 0, scan_launches = 0, scan_flops = 0, scan_tiles = 0, refine_ms = 0,
           rescan_rows = 0, order_ms = 0, scan_flops_done = 0, scan_tiles_total = 0, tc_ms = 0,
           tc_flops_done = 0, tc_uncertified = 0;
    // graph phase (graph.cu:msf_undirected): Boruvka round loop time, its
    // algorithmic bytes (12 B per directed entry + 16 B per vertex
    // per round), rounds, and the whole forest solve incl. its sorts
    double mst_ms = 0, mst_bytes = 0, mst_rounds = 0, msf_ms = 0;
    Profile &operator+=(const Profile &o) {
        double *a = &scan_ms;
        const double *b = &o.scan_ms;
        for (size_t i = 0; i < sizeof(Profile) / sizeof(double); i++) a[i] += b[i];
        return *this;
    }
};
// per host thread (the multi-GPU driver's shard threads merge theirs into the caller's)
Profile &profile();

// CUDA-event pair on one stream.
struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
        SLK_CUDA(cudaEventCreate(&a));
        SLK_CUDA(cudaEventCreate(&b));
    }
    ~EventPair() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    void start(cudaStream_t s) { SLK_CUDA(cudaEventRecord(a, s)); }
    void stop(cudaStream_t s) { SLK_CUDA(cudaEventRecord(b, s)); }
    double ms() {
        float v = 0;
        SLK_CUDA(cudaEventSynchronize(b));
        SLK_CUDA(cudaEventElapsedTime(&v, a, b));
        return v;
    }
};

// knn.cu
// A point matrix prepared for the scans: dims-major 128-point blocks, fp64
// norms (reference order), max norm, and per-block bounding spheres.
struct SplitIndex;  // knn.cu: tight-block copy of an index for the block-centred scan
struct PointSet {
    const float *x32 = nullptr;
    const double *x64 = nullptr;
    int64_t n = 0, nb = 0, nsb = 0;
    int d = 0, dp = 0;
    float maxabs = 0.0f;  // max |x| of the float32 values (tensor-path scaling)
    DevBuf<float> centroid, radius, sb_centroid, sb_radius;
    // dims-major block layout of the exact-fp32 FFMA scan, built on first use
    mutable DevBuf<float> packed;
    DevBuf<double> norms, maxn;
    // tensor-core scan operand layout (knn.cu:tcpack_kernel), built on first use
    mutable DevBuf<float> tcpack;
    // block-centred fp16 index records (tc_bc.cu), built on first use for one scale
    mutable DevBuf<unsigned char> bcpack;
    mutable float bcpack_scale = 0.0f;
    // knn.cu:split_index: -1 not planned, 0 every block tight, 1 `split` built,
    // 2 too many wide blocks (the block-centred scan is not used)
    mutable std::shared_ptr<SplitIndex> split;
    mutable int split_state = -1;
    // virtual re-blocked index (knn.cu:split_index): position p holds row
    // rowmap[p] of x32; spheres and the block-centred records read through it
    const int32_t *rowmap = nullptr;
    // optional finest cluster labels (the k-NN graph's components): the
    // cross-colour re-blocking keeps their segments contiguous and aligned
    const int32_t *block_hint = nullptr;
};
std::shared_ptr<PointSet> make_pointset(const float *x32, const double *x64, int64_t n, int d,
                                        cudaStream_t s);
void knn_ps(const PointSet &X, int k, int64_t q0, int64_t q1, int32_t *idx, double *dist,
            cudaStream_t s);
void nn1_ps(const PointSet &Q, const PointSet &X, int mode, const uint8_t *mask,
            const int32_t *qcolor, const int32_t *xcolor, int64_t q0, int64_t q1, int32_t *idx,
            double *dist, cudaStream_t s);
void knn_rows(const float *x32, const double *x64, int64_t n, int d, int k, int64_t q0,
              int64_t q1, int32_t *idx, double *dist, cudaStream_t s);
void nn1_rows(const float *q32, const double *q64, int64_t nq, const float *x32,
              const double *x64, int64_t nx, int d, int mode, const uint8_t *mask,
              const int32_t *qcolor, const int32_t *xcolor, int64_t q0, int64_t q1, int32_t *idx,
              double *dist, cudaStream_t s);
void row_norms(const float *x32, const double *x64, int64_t n, int d, double *out, cudaStream_t s);
void pairwise_l2(const double *q, int64_t nq, const double *x, int64_t nx, int d, int squared,
                 double *out, cudaStream_t s);

// graph.cu
// Undirected, deduplicated (min weight) edge list sorted by (a, b), a < b.
struct EdgeSet {
    DevBuf<int32_t> a, b;
    DevBuf<double> w;
    int64_t m = 0;
};
// The same undirected edge sets without sorting (graph.cu), in arbitrary
// order: a k-NN graph's (rows of k ids, symmetric weights), and a spanning
// forest united with one cross-colour bridge per point.
EdgeSet knn_undirected(int64_t n, int k, const int32_t *idx, const double *dist, cudaStream_t s);
EdgeSet forest_plus_bridges(int64_t n, const int32_t *fa, const int32_t *fb, const double *fw, int64_t ne,
                            const int32_t *bdst, const double *bw, cudaStream_t s);
EdgeSet dedup_undirected(int64_t n, const int32_t *src, const int32_t *dst, const double *w,
                         int64_t m, cudaStream_t s);
// Spanning forest of an undirected edge set (alteration + Boruvka).  Outputs
// as slk_solve_mst.  When `negate` the weights are negated for ordering and
// restored on output.
// `presorted`: the input is already sorted by (a, b) (dedup_undirected output).
void msf_undirected(int64_t n, const int32_t *a, const int32_t *b, const double *w, int64_t m,
                    bool presorted, bool negate, int64_t seed, int32_t *out_src,
                    int32_t *out_dst, double *out_w, int32_t *colors, int64_t *n_edges,
                    int64_t *n_components, cudaStream_t s);
// CSR-level API helpers (graph.cu)
void csr_from_edges(int64_t n, const int32_t *src, const int32_t *dst, const double *w, int64_t m,
                    int64_t *offs, int32_t *cols, double *cw, int64_t *nnz, cudaStream_t s);
bool csr_symmetric(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                   cudaStream_t s);
double csr_weight_alteration(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                             int64_t seed, double *alt, cudaStream_t s);
void csr_min_edge_per_vertex(int64_t n, const int64_t *offs, const int32_t *cols,
                             const double *alt, const int32_t *colors, int64_t *pos,
                             cudaStream_t s);
int64_t reconcile_supervertex(int64_t n, const int64_t *pos, const int32_t *dst,
                              const double *alt, const double *orig, const int32_t *colors,
                              int32_t *out_a, int32_t *out_b, double *out_w, cudaStream_t s);
void label_propagation(int64_t n, int32_t *colors, const int32_t *us, const int32_t *vs, int64_t m,
                       cudaStream_t s);
void csr_solve_mst(int64_t n, const int64_t *offs, const int32_t *cols, const double *w,
                   bool maximize, int64_t seed, int32_t *out_src, int32_t *out_dst, double *out_w,
                   int32_t *colors, int64_t *n_edges, int64_t *n_components, cudaStream_t s);

// dendro.cu
// Host copy of the sorted spanning tree laid out for the fold
// (dendro.cu:dendrogram_device_sort).  Positions [0, t) hold the first t
// merges grouped by the component of the forest they form (group g =
// positions off[g] .. off[g+1], merge ranks rank[j] increasing within a
// group); positions [t, n-1) hold merges t .. n-2 in order.  The arrays live
// in per-thread pinned staging, valid until the next call.
struct FoldInput {
    int64_t n = 0;
    const int32_t *a = nullptr, *b = nullptr;
    const double *w = nullptr;
    int64_t t = 0;
    const int32_t *rank = nullptr;
    const int64_t *off = nullptr;
    int64_t ngroups = 0;
    int threads = 1;
    // flat cut taken on the device (dendro.cu): int32 labels in pinned host
    // memory, valid once the stream has synchronised after the fold
    const int32_t *labels = nullptr;
};
// cut: merges before the flat cut ((n-1) - (n_clusters-1)), < 0 for none
FoldInput dendrogram_device_sort(const int32_t *src, const int32_t *dst, const double *w, int64_t n,
                                 bool take_sqrt, int64_t cut, cudaStream_t s);
// labels (optional): the flat cut for n_clusters, taken during the fold
void dendrogram_fold(const FoldInput &in, double *merges, int64_t n_clusters = 0, int64_t *labels = nullptr,
                     double *extract_ms = nullptr);
void extract_labels(const double *merges, int64_t n, int64_t n_clusters, int64_t *labels);
// The merge table built on the device (dendro.cu:krt_kernel): row i of the
// reference's table is (rows[3i], rows[3i+1], w[i], rows[3i+2]) (children
// a < b, height, size), and labels[n] (int32) is the flat cut when cut >= 0.
struct DeviceMerges {
    DevBuf<int32_t> rows;  // [n-1][3]
    DevBuf<double> w;      // [n-1] merge heights (sqrt taken when requested)
    DevBuf<int32_t> labels;
};
// Enqueued on s (the cut on cut_stream after table_done when both are
// given: the caller reads labels after synchronising cut_stream); the
// returned pinned int is nonzero once s has synchronised if the edges
// contain a cycle.
const int *dendrogram_device(const int32_t *src, const int32_t *dst, const double *w, int64_t n,
                             bool take_sqrt, int64_t cut, DeviceMerges &out, cudaStream_t s,
                             cudaStream_t cut_stream = nullptr, cudaEvent_t table_done = nullptr);

}  // namespace slk
