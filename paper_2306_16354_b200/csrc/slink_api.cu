// slink_api.cu — the C ABI (include/slink.h) and the single-GPU pipeline
// driver replacing single_linkage / connect_graph
// (/root/reference/pkg/src/parlink/linkage.py:222-311).
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "host_pool.h"

namespace slk {

static thread_local std::string g_last_error;
static thread_local ScanStats g_scan_stats;
static std::atomic<int64_t> g_launches{0};

void set_error(int status, const std::string &msg) {
    (void)status;
    g_last_error = msg;
}

static std::string vformat(const char *fmt, va_list ap) {
    char buf[1024];
    vsnprintf(buf, sizeof buf, fmt, ap);
    return buf;
}

void throw_invalid(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::string m = vformat(fmt, ap);
    va_end(ap);
    throw Error{SLK_ERR_INVALID, m};
}

void throw_internal(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::string m = vformat(fmt, ap);
    va_end(ap);
    throw Error{SLK_ERR_INTERNAL, m};
}

// Grows the device pool's reservation to `bytes` in one piece (allocate,
// free, keep).  Without it the pool grows in many small mappings and a later
// call can stall for 0.1-0.5 s in cudaMallocAsync while the driver maps new
// physical memory (measured at C3 on the host-buffer path).  SLK_POOL_RESERVE_GB
// overrides the size.
void reserve_pool(size_t bytes, cudaStream_t s) {
    static size_t reserved[64] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    if (const char *e = getenv("SLK_POOL_RESERVE_GB")) bytes = (size_t)(atof(e) * (double)(1ull << 30));
    std::lock_guard<std::mutex> lock(mu);
    if (bytes <= reserved[dev]) return;
    ensure_pool();
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && bytes > free_b / 2) bytes = free_b / 2;
    void *p = nullptr;
    if (bytes && cudaMallocAsync(&p, bytes, s) == cudaSuccess) {
        cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
        reserved[dev] = bytes;
    } else {
        cudaGetLastError();  // best effort: a failed reservation is not an error
    }
}

void ensure_pool() {
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[dev] = true;
}

// SLK_TRACE=1: sub-stage timings on stderr (adds stream synchronisations)
bool trace_on() {
    static const bool on = [] {
        const char *e = getenv("SLK_TRACE");
        return e && *e && *e != '0';
    }();
    return on;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

ScanStats &scan_stats() { return g_scan_stats; }

static thread_local Profile g_profile;
Profile &profile() { return g_profile; }

int num_sms() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (!cached) cached = 148;
    }
    return cached;
}

namespace {

// The library's own stream for host-buffer entry points: one per device,
// created once and kept, so the stream-ordered pool reuses the previous
// call's scratch (a fresh stream per call made the pool map new memory:
// up to 0.5 s stalls at 1M x 64).  Calls on one device serialise on it.
struct StreamGuard {
    cudaStream_t s = nullptr;
    StreamGuard() {
        static std::mutex mu;
        static cudaStream_t streams[64] = {};
        int dev = 0;
        SLK_CUDA(cudaGetDevice(&dev));
        if (dev < 0 || dev >= 64) throw_internal("device ordinal %d out of range", dev);
        std::lock_guard<std::mutex> lock(mu);
        if (!streams[dev]) SLK_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
        s = streams[dev];
    }
};

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

}  // namespace

void trace_mark(const char *what) {
    if (!trace_on()) return;
    static thread_local double last = 0.0;
    const double t = now_ms();
    fprintf(stderr, "[slk]   %-28s +%.2f ms\n", what, last > 0.0 ? t - last : 0.0);
    last = t;
}

namespace {

std::string largest_sizes(const std::vector<int32_t> &colors) {
    std::vector<int64_t> counts(colors.size(), 0);
    for (int32_t c : colors) counts[c]++;
    std::vector<int64_t> sizes;
    for (int64_t c : counts)
        if (c > 0) sizes.push_back(c);
    std::sort(sizes.rbegin(), sizes.rend());
    if (sizes.size() > 8) sizes.resize(8);
    std::string out = "[";
    for (size_t i = 0; i < sizes.size(); i++) out += (i ? ", " : "") + std::to_string(sizes[i]);
    return out + "]";
}

}  // namespace

namespace {

// ------------------------------------------------------------ multi-GPU
// The two neighbour searches are the only sharded stages (SURVEY §8e,
// north_star): query rows are dealt to G shards in 128-aligned chunks
// round-robin (4 chunks per shard, so clusters of unequal pruning cost
// spread over the shards), the index is replicated, and each shard's rows
// come back to the main device with peer copies over NVLink; the spanning
// forests, dendrogram and cut stay on the main device.  One host thread per
// shard drives its device (the search has host synchronisation points);
// shard g uses device (main + g) % device_count, so G > device_count places
// several shards on one device (the multi-shard logic is testable on one GPU).
struct Shard {
    int dev = 0;
    cudaStream_t s = nullptr;
    DevBuf<float> x32;
    DevBuf<double> x64;
    const float *px32 = nullptr;
    const double *px64 = nullptr;
    std::shared_ptr<PointSet> P;
    DevBuf<int32_t> idx, colors;
    DevBuf<double> dist;
    Profile prof;
};

struct ShardSet {
    int main_dev = 0;
    cudaStream_t main_s = nullptr;
    std::vector<std::unique_ptr<Shard>> sh;
    std::vector<std::pair<int64_t, int64_t>> chunks;  // row ranges; chunk j -> shard j % G

    ShardSet(int G, int64_t n, cudaStream_t s) : main_s(s) {
        SLK_CUDA(cudaGetDevice(&main_dev));
        int ndev = 1;
        SLK_CUDA(cudaGetDeviceCount(&ndev));
        for (int g = 0; g < G; g++) {
            auto S = std::make_unique<Shard>();
            S->dev = (main_dev + g) % ndev;
            if (S->dev != main_dev) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(S->dev, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SLK_CUDA(e);
                (void)cudaGetLastError();
            }
            sh.push_back(std::move(S));
        }
        const int64_t nb = (n + 127) / 128;
        const int64_t nc = std::min<int64_t>(nb, 4 * (int64_t)G);
        for (int64_t j = 0; j < nc; j++) chunks.push_back({std::min(n, nb * j / nc * 128), std::min(n, nb * (j + 1) / nc * 128)});
    }
    ~ShardSet() {
        for (auto &S : sh)
            if (S->s) {
                cudaSetDevice(S->dev);
                cudaStreamSynchronize(S->s);
                S->x32.release();
                S->x64.release();
                S->idx.release();
                S->dist.release();
                S->colors.release();
                S->P.reset();
                cudaStreamDestroy(S->s);
            }
        cudaSetDevice(main_dev);
    }
    int size() const { return (int)sh.size(); }
    // fn(g, shard) on every shard concurrently (shard 0 on this thread)
    template <class F>
    void run(F fn) {
        std::vector<std::exception_ptr> err(sh.size());
        auto body = [&](int g) {
            try {
                SLK_CUDA(cudaSetDevice(sh[g]->dev));
                if (!sh[g]->s) SLK_CUDA(cudaStreamCreateWithFlags(&sh[g]->s, cudaStreamNonBlocking));
                fn(g, *sh[g]);
                SLK_CUDA(cudaStreamSynchronize(sh[g]->s));
                if (g > 0) sh[g]->prof += profile();  // worker threads hand their profile to the caller
            } catch (...) {
                err[g] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (int g = 1; g < size(); g++) th.emplace_back(body, g);
        body(0);
        for (auto &t : th) t.join();
        SLK_CUDA(cudaSetDevice(main_dev));
        for (int g = 1; g < size(); g++) {
            profile() += sh[g]->prof;
            sh[g]->prof = Profile{};
        }
        for (auto &e : err)
            if (e) std::rethrow_exception(e);
    }
    // copy rows [r0, r1) x width elements of T from shard g's buffer to dst (main device)
    template <class T>
    void gather(T *dst, const T *src, int g, int64_t r0, int64_t r1, int64_t width) {
        const size_t bytes = (size_t)(r1 - r0) * width * sizeof(T);
        if (!bytes) return;
        if (sh[g]->dev == main_dev)
            SLK_CUDA(cudaMemcpyAsync(dst + r0 * width, src + r0 * width, bytes, cudaMemcpyDeviceToDevice, main_s));
        else
            SLK_CUDA(cudaMemcpyPeerAsync(dst + r0 * width, main_dev, src + r0 * width, sh[g]->dev, bytes, main_s));
    }
};

}  // namespace

// finish_tree with the host fold (SLK_HOST_FOLD=1; fold.cu): device sort,
// parallel host fold, device cut.
static void finish_tree_host_fold(const int32_t *ts, const int32_t *td, const double *tw, int64_t n, int metric,
                        int64_t n_clusters, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                        int64_t *h_tree_dst, double *h_tree_w, double *dendro_ms, double *extract_ms_out,
                        cudaStream_t s) {
    const double t3 = now_ms();
    trace_mark("dendrogram start");
    // The caller's output arrays are usually fresh allocations: fault their
    // pages in (one write per 4 KB page, host threads) while the device sorts,
    // instead of inside the fold (measured: the dendrogram stage alternated
    // 3.4 / 6-8 ms between steps with page faults in the fold).
    const int pf_parts = (int)std::min<int64_t>(16, std::max<int64_t>(1, n / 65536));
    auto touch = [](void *base, size_t bytes, int k, int nt) {
        char *c = static_cast<char *>(base);
        const size_t pages = (bytes + 4095) / 4096, lo = pages * k / nt, hi = pages * (k + 1) / nt;
        for (size_t pg = lo; pg < hi; pg++) c[pg * 4096] = 0;
    };
    auto prefault = HostPool::get().submit(pf_parts, [=](int k) {
        if (h_merges) touch(h_merges, (size_t)(n - 1) * 4 * sizeof(double), k, pf_parts);
        if (h_labels) touch(h_labels, (size_t)n * sizeof(int64_t), k, pf_parts);
        if (h_tree_src) touch(h_tree_src, (size_t)(n - 1) * sizeof(int64_t), k, pf_parts);
        if (h_tree_dst) touch(h_tree_dst, (size_t)(n - 1) * sizeof(int64_t), k, pf_parts);
        if (h_tree_w) touch(h_tree_w, (size_t)(n - 1) * sizeof(double), k, pf_parts);
    });
    const FoldInput fin = dendrogram_device_sort(ts, td, tw, n, metric == 0, (n - 1) - (n_clusters - 1), s);
    prefault.wait();
    trace_mark("dendrogram sorted (host)");
    // the spanning tree goes to pinned staging on the copy engine while the
    // host folds
    static thread_local PinnedBuf<int32_t> st_src, st_dst;
    static thread_local PinnedBuf<double> st_w;
    const bool want_tree = h_tree_src || h_tree_dst || h_tree_w;
    if (want_tree) {
        SLK_CUDA(cudaMemcpyAsync(st_src.get(n - 1), ts, (n - 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(st_dst.get(n - 1), td, (n - 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(st_w.get(n - 1), tw, (n - 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    double extract_ms = 0.0;
    // the flat cut: on the device when dendrogram_device_sort took it (labels
    // in pinned staging after the stream syncs), else during the host fold
    dendrogram_fold(fin, h_merges, n_clusters, fin.labels ? nullptr : h_labels, &extract_ms);
    trace_mark("dendrogram folded");
    if (fin.labels) {
        const double te = now_ms();
        SLK_CUDA(cudaStreamSynchronize(s));
        const int32_t *hl = fin.labels;
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(fin.threads, n / 65536 + 1));
        pool_slices(n, nt, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; i++) h_labels[i] = hl[i];
        });
        extract_ms = now_ms() - te;
    }
    const double t5 = now_ms();
    if (want_tree) {
        SLK_CUDA(cudaStreamSynchronize(s));
        const int32_t *hs = st_src.p, *hd = st_dst.p;
        const double *hw = st_w.p;
        // widen / copy out of the pinned staging in parallel slices (the caller's
        // fresh arrays are first touched here)
        const int64_t m = n - 1;
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(fin.threads, m / 65536 + 1));
        pool_slices(m, nt, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; i++) {
                if (h_tree_src) h_tree_src[i] = hs[i];
                if (h_tree_dst) h_tree_dst[i] = hd[i];
            }
            if (h_tree_w) memcpy(h_tree_w + lo, hw + lo, (hi - lo) * sizeof(double));
        });
    }
    if (dendro_ms) *dendro_ms = t5 - t3 - extract_ms;  // the cut is taken inside the fold
    if (extract_ms_out) *extract_ms_out = extract_ms;
}

// Faults in the pages of the caller's output arrays (one write per 4 KB page,
// pool threads) while the device works: they are usually fresh allocations,
// and first touches inside the copy-out made it jitter between steps.
static HostPool::Batch prefault_outputs(int64_t n, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                                        int64_t *h_tree_dst, double *h_tree_w) {
    const int pf_parts = (int)std::min<int64_t>(16, std::max<int64_t>(1, n / 65536));
    auto touch = [](void *base, size_t bytes, int k, int nt) {
        char *c = static_cast<char *>(base);
        const size_t pages = (bytes + 4095) / 4096, lo = pages * k / nt, hi = pages * (k + 1) / nt;
        for (size_t pg = lo; pg < hi; pg++) c[pg * 4096] = 0;
    };
    return HostPool::get().submit(pf_parts, [=](int k) {
        if (h_merges) touch(h_merges, (size_t)(n - 1) * 4 * sizeof(double), k, pf_parts);
        if (h_labels) touch(h_labels, (size_t)n * sizeof(int64_t), k, pf_parts);
        if (h_tree_src) touch(h_tree_src, (size_t)(n - 1) * sizeof(int64_t), k, pf_parts);
        if (h_tree_dst) touch(h_tree_dst, (size_t)(n - 1) * sizeof(int64_t), k, pf_parts);
        if (h_tree_w) touch(h_tree_w, (size_t)(n - 1) * sizeof(double), k, pf_parts);
    });
}

static int copy_threads(int64_t count) {
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    return (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)std::min(16u, hc), count / 65536 + 1}));
}

// Enqueues the copies of a device merge table to pinned staging in chunks
// (an event after each); merges_expand then widens each chunk into the
// caller's float64 rows as soon as it lands, overlapping the next chunk's copy.
struct MergeCopies {
    static constexpr int MAX_CHUNKS = 4;
    int64_t m = 0;
    int chunks = 0;
    cudaEvent_t *ev = nullptr;
    int32_t *rows = nullptr;
    double *w = nullptr;
};

// Per host thread and device: the side stream and the events finish_tree
// reuses (created once: per-call creation showed up as rare multi-ms stalls).
struct TreeCopyRes {
    cudaStream_t side = nullptr;
    cudaEvent_t ready = nullptr, tree = nullptr, table = nullptr, chunk[MergeCopies::MAX_CHUNKS] = {};
};
static TreeCopyRes &tree_copy_res() {
    static thread_local std::vector<TreeCopyRes> res;
    int dev = 0;
    SLK_CUDA(cudaGetDevice(&dev));
    if ((int)res.size() <= dev) res.resize(dev + 1);
    TreeCopyRes &r = res[dev];
    if (!r.side) {
        SLK_CUDA(cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking));
        SLK_CUDA(cudaEventCreateWithFlags(&r.ready, cudaEventDisableTiming));
        SLK_CUDA(cudaEventCreateWithFlags(&r.tree, cudaEventDisableTiming));
        SLK_CUDA(cudaEventCreateWithFlags(&r.table, cudaEventDisableTiming));
        for (auto &e : r.chunk) SLK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return r;
}

static void merges_enqueue(const DeviceMerges &dm, int64_t m, MergeCopies &mc, cudaStream_t s) {
    static thread_local PinnedBuf<int32_t> st_rows;
    static thread_local PinnedBuf<double> st_w;
    mc.m = m;
    mc.rows = st_rows.get(3 * m);
    mc.w = st_w.get(m);
    mc.chunks = m >= (1 << 18) ? MergeCopies::MAX_CHUNKS : 1;
    mc.ev = tree_copy_res().chunk;
    for (int k = 0; k < mc.chunks; k++) {
        const int64_t lo = m * k / mc.chunks, hi = m * (k + 1) / mc.chunks;
        SLK_CUDA(cudaMemcpyAsync(mc.rows + 3 * lo, dm.rows.get() + 3 * lo, (hi - lo) * 3 * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, s));
        SLK_CUDA(cudaMemcpyAsync(mc.w + lo, dm.w.get() + lo, (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost,
                                 s));
        SLK_CUDA(cudaEventRecord(mc.ev[k], s));
    }
}

static void merges_expand(const MergeCopies &mc, double *h_merges) {
    const int32_t *hr = mc.rows;
    const double *hw = mc.w;
    for (int k = 0; k < mc.chunks; k++) {
        const int64_t lo = mc.m * k / mc.chunks, hi = mc.m * (k + 1) / mc.chunks;
        SLK_CUDA(cudaEventSynchronize(mc.ev[k]));
        if (!h_merges) continue;
        pool_slices(hi - lo, copy_threads(hi - lo), [&](int64_t a, int64_t b) {
            for (int64_t i = lo + a; i < lo + b; i++) {
                double *row = h_merges + 4 * i;
                row[0] = (double)hr[3 * i];
                row[1] = (double)hr[3 * i + 1];
                row[2] = hw[i];
                row[3] = (double)hr[3 * i + 2];
            }
        });
    }
}

// Dendrogram + cut + spanning-tree copy-out of a device spanning tree
// (linkage.py:295-311): device sort, device merge table (dendro.cu:krt_kernel)
// and device cut; the spanning tree is copied out on a side stream while the
// device builds the table, the table in chunks that the host widens as they
// land.  Returns the dendrogram and extract milliseconds.  Shared by the
// single-process driver and slk_finish_tree (the torchrun driver's rank 0).
static void finish_tree(const int32_t *ts, const int32_t *td, const double *tw, int64_t n, int metric,
                        int64_t n_clusters, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                        int64_t *h_tree_dst, double *h_tree_w, double *dendro_ms, double *extract_ms_out,
                        cudaStream_t s, bool prefaulted = false) {
    if (getenv("SLK_HOST_FOLD")) {
        finish_tree_host_fold(ts, td, tw, n, metric, n_clusters, h_merges, h_labels, h_tree_src, h_tree_dst,
                              h_tree_w, dendro_ms, extract_ms_out, s);
        return;
    }
    const double t3 = now_ms();
    trace_mark("dendrogram start");
    HostPool::Batch prefault(nullptr);
    if (!prefaulted) prefault = prefault_outputs(n, h_merges, h_labels, h_tree_src, h_tree_dst, h_tree_w);
    const int64_t m = n - 1;
    // the spanning tree: side stream, overlapping the device work below
    static thread_local PinnedBuf<int32_t> st_src, st_dst, st_lab;
    static thread_local PinnedBuf<double> st_w;
    const bool want_tree = h_tree_src || h_tree_dst || h_tree_w;
    TreeCopyRes &res = tree_copy_res();
    cudaStream_t side = res.side;
    cudaEvent_t ev_ready = res.ready, ev_tree = res.tree;
    if (want_tree) {
        SLK_CUDA(cudaEventRecord(ev_ready, s));
        SLK_CUDA(cudaStreamWaitEvent(side, ev_ready, 0));
        SLK_CUDA(cudaMemcpyAsync(st_src.get(m), ts, m * sizeof(int32_t), cudaMemcpyDeviceToHost, side));
        SLK_CUDA(cudaMemcpyAsync(st_dst.get(m), td, m * sizeof(int32_t), cudaMemcpyDeviceToHost, side));
        SLK_CUDA(cudaMemcpyAsync(st_w.get(m), tw, m * sizeof(double), cudaMemcpyDeviceToHost, side));
        SLK_CUDA(cudaEventRecord(ev_tree, side));
    }
    DeviceMerges dm;
    // the cut runs on the side stream after the table, next to the table's copies on s
    const int *cycle = dendrogram_device(ts, td, tw, n, metric == 0, (n - 1) - (n_clusters - 1), dm, s, side,
                                         res.table);
    MergeCopies mc;
    merges_enqueue(dm, m, mc, s);
    int32_t *hl = h_labels ? st_lab.get(n) : nullptr;
    if (hl) SLK_CUDA(cudaMemcpyAsync(hl, dm.labels.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, side));
    prefault.wait();
    double t_tree = 0.0;
    if (want_tree) {
        SLK_CUDA(cudaEventSynchronize(ev_tree));
        const double tt = now_ms();
        const int32_t *hs = st_src.p, *hd = st_dst.p;
        const double *hw = st_w.p;
        pool_slices(m, copy_threads(m), [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; i++) {
                if (h_tree_src) h_tree_src[i] = hs[i];
                if (h_tree_dst) h_tree_dst[i] = hd[i];
            }
            if (h_tree_w) memcpy(h_tree_w + lo, hw + lo, (hi - lo) * sizeof(double));
        });
        t_tree = now_ms() - tt;
    }
    const double t4 = now_ms();
    merges_expand(mc, h_merges);
    SLK_CUDA(cudaStreamSynchronize(s));
    SLK_CUDA(cudaStreamSynchronize(side));  // the cut and its labels
    if (*cycle) throw_invalid("edges contain a cycle: not a spanning tree");
    const double t5 = now_ms();
    if (hl)
        pool_slices(n, copy_threads(n), [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; i++) h_labels[i] = hl[i];
        });
    const double t6 = now_ms();
    trace_mark("dendrogram copied out");
    if (getenv("SLK_TRACE"))
        fprintf(stderr, "[slk] dendrogram: tree copy-out %.2f ms (overlapped), merges landed+widened %.2f ms after, "
                        "labels %.2f ms; total %.2f ms\n", t_tree, t5 - t4, t6 - t5, t6 - t3);
    if (dendro_ms) *dendro_ms = t5 - t3;
    if (extract_ms_out) *extract_ms_out = t6 - t5;
}

// Pipeline state on one device (used by slk_single_linkage); n_gpus > 1
// shards the two neighbour searches (ShardSet above).
void single_linkage_device(const float *x32, const double *x64, int64_t n, int d, int k,
                           int64_t n_clusters, int metric, int64_t seed, int64_t max_iters,
                           double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                           int64_t *h_tree_dst, double *h_tree_w, int64_t *n_iters,
                           double *timings, cudaStream_t s, int n_gpus = 1) {
    // peak scratch of the pipeline, x2 headroom: operand copies (packed,
    // tc-packed, f64), per-query-block visit bounds, k-NN lists, edge lists
    {
        const double nb = (double)((n + 127) / 128);
        const double est = 4.0 * n * d * 4 + (x64 ? 8.0 * n * d : 0.0) + 8.0 * nb * nb +
                           64.0 * n * k + 256.0 * n;
        reserve_pool((size_t)(2.0 * est), s);
    }
    double t0 = now_ms();
    // the caller's output arrays are fresh allocations: fault their pages in
    // on the host pool while the device computes (off the critical path)
    HostPool::Batch prefault = prefault_outputs(n, h_merges, h_labels, h_tree_src, h_tree_dst, h_tree_w);
    // --- k-NN graph (linkage.py:287)
    std::unique_ptr<ShardSet> shards;
    std::shared_ptr<PointSet> P;
    DevBuf<int32_t> idx(n * k, s);
    DevBuf<double> dist(n * k, s);
    if (n_gpus > 1) {
        // every shard holds the points and its own PointSet (spheres, packs)
        // for the k-NN and all connect passes
        SLK_CUDA(cudaStreamSynchronize(s));  // the caller's points are ready
        shards = std::make_unique<ShardSet>(n_gpus, n, s);
        ShardSet &SS = *shards;
        SS.run([&](int g, Shard &S) {
            if (S.dev == SS.main_dev) {
                S.px32 = x32;
                S.px64 = x64;
            } else {
                S.x32.alloc(n * (int64_t)d, S.s);
                SLK_CUDA(cudaMemcpyPeerAsync(S.x32.get(), S.dev, x32, SS.main_dev, n * (int64_t)d * sizeof(float), S.s));
                S.px32 = S.x32.get();
                if (x64) {
                    S.x64.alloc(n * (int64_t)d, S.s);
                    SLK_CUDA(cudaMemcpyPeerAsync(S.x64.get(), S.dev, x64, SS.main_dev, n * (int64_t)d * sizeof(double), S.s));
                    S.px64 = S.x64.get();
                }
            }
            S.P = make_pointset(S.px32, S.px64, n, d, S.s);
            S.idx.alloc(n * k, S.s);
            S.dist.alloc(n * k, S.s);
            for (size_t j = g; j < SS.chunks.size(); j += SS.size())
                knn_ps(*S.P, k, SS.chunks[j].first, SS.chunks[j].second, S.idx.get() + SS.chunks[j].first * k,
                       S.dist.get() + SS.chunks[j].first * k, S.s);
        });
        for (size_t j = 0; j < SS.chunks.size(); j++) {
            const int g = (int)(j % SS.size());
            SS.gather(idx.get(), (const int32_t *)SS.sh[g]->idx.get(), g, SS.chunks[j].first, SS.chunks[j].second, k);
            SS.gather(dist.get(), (const double *)SS.sh[g]->dist.get(), g, SS.chunks[j].first, SS.chunks[j].second, k);
        }
    } else {
        P = make_pointset(x32, x64, n, d, s);
        if (trace_on()) {
            SLK_CUDA(cudaStreamSynchronize(s));
            fprintf(stderr, "[slk] pointset %.1f ms\n", now_ms() - t0);
        }
        trace_mark("pointset");
        knn_ps(*P, k, 0, n, idx, dist, s);
    }
    trace_mark("knn returned");
    SLK_CUDA(cudaStreamSynchronize(s));
    trace_mark("knn synced");
    double t1 = now_ms();
    // --- symmetrise + spanning forest (linkage.py:289-290)
    EdgeSet E = knn_undirected(n, k, idx, dist, s);
    idx.release();
    dist.release();
    DevBuf<int32_t> ts(n, s), td(n, s), colors(n, s);
    DevBuf<double> tw(n, s);
    int64_t ne = 0, nc = 0;
    msf_undirected(n, E.a, E.b, E.w, E.m, false, false, seed, ts, td, tw, colors, &ne, &nc, s);
    E = EdgeSet{};
    double t2 = now_ms();
    // --- connect loop (linkage.py:222-254)
    int64_t budget = max_iters >= 0 ? max_iters : (int64_t)ceil(log2((double)std::max<int64_t>(n, 2))) + 8;
    int64_t iters = 0;
    DevBuf<int32_t> base_colors;
    if (nc > 1) {
        // the k-NN graph's components: every later colour is a union of them,
        // and the cross-colour re-blocking keeps them contiguous
        base_colors.alloc(n, s);
        SLK_CUDA(cudaMemcpyAsync(base_colors.get(), colors.get(), n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        if (P) P->block_hint = base_colors.get();
        DevBuf<int32_t> udst(2 * n, s);
        DevBuf<double> uw(2 * n, s);
        while (nc > 1) {
            if (iters >= budget) {
                std::vector<int32_t> hc(n);
                SLK_CUDA(cudaMemcpyAsync(hc.data(), colors.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
                SLK_CUDA(cudaStreamSynchronize(s));
                throw Error{SLK_ERR_CONVERGENCE,
                            "reconnection did not converge within " + std::to_string(budget) +
                                " iterations: " + std::to_string(nc) +
                                " components remain (largest sizes " + largest_sizes(hc) + ")"};
            }
            // bridges: one per point (neighbors.py:375-391), rows ne .. ne + n of udst / uw
            if (shards) {
                // every shard scans its chunks against the replicated index
                // with this iteration's colours; bridges come back by rows
                ShardSet &SS = *shards;
                SLK_CUDA(cudaStreamSynchronize(s));  // colours final on the main device
                SS.run([&](int g, Shard &S) {
                    S.colors.alloc(n, S.s);
                    if (S.dev == SS.main_dev)
                        SLK_CUDA(cudaMemcpyAsync(S.colors.get(), colors.get(), n * sizeof(int32_t), cudaMemcpyDeviceToDevice, S.s));
                    else
                        SLK_CUDA(cudaMemcpyPeerAsync(S.colors.get(), S.dev, colors.get(), SS.main_dev, n * sizeof(int32_t), S.s));
                    for (size_t j = g; j < SS.chunks.size(); j += SS.size())
                        nn1_ps(*S.P, *S.P, 2, nullptr, S.colors, S.colors, SS.chunks[j].first, SS.chunks[j].second,
                               S.idx.get() + SS.chunks[j].first, S.dist.get() + SS.chunks[j].first, S.s);
                });
                for (size_t j = 0; j < SS.chunks.size(); j++) {
                    const int g = (int)(j % SS.size());
                    SS.gather(udst.get() + ne, (const int32_t *)SS.sh[g]->idx.get(), g, SS.chunks[j].first,
                              SS.chunks[j].second, 1);
                    SS.gather(uw.get() + ne, (const double *)SS.sh[g]->dist.get(), g, SS.chunks[j].first,
                              SS.chunks[j].second, 1);
                }
            } else {
                nn1_ps(*P, *P, 2, nullptr, colors, colors, 0, n, udst.get() + ne, uw.get() + ne, s);
            }
            EdgeSet U = forest_plus_bridges(n, ts, td, tw, ne, udst.get() + ne, uw.get() + ne, s);
            msf_undirected(n, U.a, U.b, U.w, U.m, false, false, seed, ts, td, tw, colors, &ne, &nc, s);
            iters++;
        }
    }
    SLK_CUDA(cudaStreamSynchronize(s));
    double t3 = now_ms();
    double dendro_ms = 0.0, extract_ms = 0.0;
    prefault.wait();
    finish_tree(ts, td, tw, n, metric, n_clusters, h_merges, h_labels, h_tree_src, h_tree_dst, h_tree_w,
                &dendro_ms, &extract_ms, s, true);
    const double t4 = t3 + dendro_ms, t5 = t4 + extract_ms;
    if (n_iters) *n_iters = iters;
    if (timings) {
        timings[0] = t1 - t0;
        timings[1] = t2 - t1;
        timings[2] = t3 - t2;
        timings[3] = t4 - t3;
        timings[4] = t5 - t4;
    }
}

}  // namespace slk

using namespace slk;

#define STREAM(s) cudaStream_t s = (cudaStream_t)stream_

extern "C" {

int slk_version(void) { return 100; }

const char *slk_last_error(void) { return g_last_error.c_str(); }

int64_t slk_kernel_launches(void) { return g_launches.load(); }

int slk_profile(double *out, int reset) {
    out[0] = g_profile.scan_ms;
    out[1] = g_profile.scan_launches;
    out[2] = g_profile.scan_flops;
    out[3] = g_profile.scan_tiles;
    out[4] = g_profile.refine_ms;
    out[5] = g_profile.rescan_rows;
    out[6] = g_profile.order_ms;
    out[7] = g_profile.scan_flops_done;
    out[8] = g_profile.scan_tiles_total;
    out[9] = g_profile.tc_ms;
    out[10] = g_profile.tc_flops_done;
    out[11] = g_profile.tc_uncertified;
    out[12] = g_profile.mst_ms;
    out[13] = g_profile.mst_bytes;
    out[14] = g_profile.mst_rounds;
    out[15] = g_profile.msf_ms;
    if (reset) g_profile = Profile{};
    return SLK_OK;
}

int slk_last_scan_stats(int64_t *stats4) {
    stats4[0] = g_scan_stats.rows_refined;
    stats4[1] = g_scan_stats.rows_rescanned;
    stats4[2] = g_scan_stats.tiles_computed;
    stats4[3] = g_scan_stats.tiles_skipped;
    stats4[4] = g_scan_stats.rows_uncertified;
    return SLK_OK;
}

int slk_knn(const float *d_x32, const double *d_x64, int64_t n, int d, int k, int64_t q0,
            int64_t q1, int32_t *d_idx, double *d_dist, void *stream_) {
    STREAM(s);
    return guarded([&] {
        knn_rows(d_x32, d_x64, n, d, k, q0, q1, d_idx, d_dist, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

// Point-set handles: the block spheres, operand packs and split index of one
// device-resident matrix, built once and reused by every search over it
// (a rank's k-NN chunks and all its cross-colour passes).
int slk_pointset_create(const float *d_x32, const double *d_x64, int64_t n, int d, void **handle,
                        void *stream_) {
    STREAM(s);
    return guarded([&] {
        if (!handle) throw_invalid("handle pointer is NULL");
        auto *P = new std::shared_ptr<PointSet>(make_pointset(d_x32, d_x64, n, d, s));
        SLK_CUDA(cudaStreamSynchronize(s));
        *handle = P;
    });
}

int slk_pointset_destroy(void *handle) {
    return guarded([&] { delete static_cast<std::shared_ptr<PointSet> *>(handle); });
}

int slk_knn_ps(void *handle, int k, int64_t q0, int64_t q1, int32_t *d_idx, double *d_dist, void *stream_) {
    STREAM(s);
    return guarded([&] {
        if (!handle) throw_invalid("NULL point-set handle");
        const PointSet &P = **static_cast<std::shared_ptr<PointSet> *>(handle);
        if (k < 1 || k > P.n - 1) throw_invalid("k must be in [1, %lld] for %lld points, got %d",
                                                (long long)(P.n - 1), (long long)P.n, k);
        if (q0 < 0 || q1 > P.n || q0 > q1) throw_invalid("row range [%lld, %lld) outside [0, %lld)",
                                                          (long long)q0, (long long)q1, (long long)P.n);
        knn_ps(P, k, q0, q1, d_idx, d_dist, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_nn1_colour_ps(void *handle, const int32_t *d_colors, int64_t q0, int64_t q1, int32_t *d_idx,
                      double *d_dist, void *stream_) {
    STREAM(s);
    return guarded([&] {
        if (!handle) throw_invalid("NULL point-set handle");
        const PointSet &P = **static_cast<std::shared_ptr<PointSet> *>(handle);
        if (q0 < 0 || q1 > P.n || q0 > q1) throw_invalid("row range [%lld, %lld) outside [0, %lld)",
                                                          (long long)q0, (long long)q1, (long long)P.n);
        nn1_ps(P, P, 2, nullptr, d_colors, d_colors, q0, q1, d_idx, d_dist, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_finish_tree(const int32_t *d_src, const int32_t *d_dst, const double *d_w, int64_t n, int metric,
                    int64_t n_clusters, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                    int64_t *h_tree_dst, double *h_tree_w, double *h_ms, void *stream_) {
    STREAM(s);
    return guarded([&] {
        if (n < 2) throw_invalid("need at least 2 points, got %lld", (long long)n);
        if (n_clusters < 1 || n_clusters > n)
            throw_invalid("n_clusters=%lld outside [1, %lld]", (long long)n_clusters, (long long)n);
        double dm = 0.0, em = 0.0;
        finish_tree(d_src, d_dst, d_w, n, metric, n_clusters, h_merges, h_labels, h_tree_src, h_tree_dst,
                    h_tree_w, &dm, &em, s);
        SLK_CUDA(cudaStreamSynchronize(s));
        if (h_ms) {
            h_ms[0] = dm;
            h_ms[1] = em;
        }
    });
}

int slk_nn1(const float *d_q32, const double *d_q64, int64_t nq, const float *d_x32,
            const double *d_x64, int64_t nx, int d, int mode, const uint8_t *d_mask,
            const int32_t *d_qcolor, const int32_t *d_xcolor, int64_t q0, int64_t q1,
            int32_t *d_idx, double *d_dist, void *stream_) {
    STREAM(s);
    return guarded([&] {
        nn1_rows(d_q32, d_q64, nq, d_x32, d_x64, nx, d, mode, d_mask, d_qcolor, d_xcolor, q0, q1,
                 d_idx, d_dist, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_row_norms(const float *d_x32, const double *d_x64, int64_t n, int d, double *d_out,
                  void *stream_) {
    STREAM(s);
    return guarded([&] {
        row_norms(d_x32, d_x64, n, d, d_out, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_edge_list_to_csr(int64_t n, const int32_t *d_src, const int32_t *d_dst,
                         const double *d_w, int64_t m, int64_t *d_offsets, int32_t *d_cols,
                         double *d_cols_w, int64_t *nnz, void *stream_) {
    STREAM(s);
    return guarded([&] {
        csr_from_edges(n, d_src, d_dst, d_w, m, d_offsets, d_cols, d_cols_w, nnz, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_csr_is_symmetric(int64_t n, const int64_t *d_offsets, const int32_t *d_cols,
                         const double *d_w, int *is_symmetric, void *stream_) {
    STREAM(s);
    return guarded([&] { *is_symmetric = csr_symmetric(n, d_offsets, d_cols, d_w, s) ? 1 : 0; });
}

int slk_weight_alteration(int64_t n, const int64_t *d_offsets, const int32_t *d_cols,
                          const double *d_w, int64_t seed, double *d_alt, double *theta,
                          void *stream_) {
    STREAM(s);
    return guarded([&] {
        *theta = csr_weight_alteration(n, d_offsets, d_cols, d_w, seed, d_alt, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_min_edge_per_vertex(int64_t n, const int64_t *d_offsets, const int32_t *d_cols,
                            const double *d_alt, const int32_t *d_colors, int64_t *d_pos,
                            void *stream_) {
    STREAM(s);
    return guarded([&] {
        csr_min_edge_per_vertex(n, d_offsets, d_cols, d_alt, d_colors, d_pos, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_min_edge_per_supervertex(int64_t n, const int64_t *d_pos, const int32_t *d_dst,
                                 const double *d_alt, const double *d_orig,
                                 const int32_t *d_colors, int32_t *d_a, int32_t *d_b,
                                 double *d_w, int64_t *m_out, void *stream_) {
    STREAM(s);
    return guarded([&] {
        *m_out = reconcile_supervertex(n, d_pos, d_dst, d_alt, d_orig, d_colors, d_a, d_b, d_w, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_label_propagation(int64_t n, int32_t *d_colors, const int32_t *d_us, const int32_t *d_vs,
                          int64_t m, void *stream_) {
    STREAM(s);
    return guarded([&] {
        label_propagation(n, d_colors, d_us, d_vs, m, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_solve_mst(int64_t n, const int64_t *d_offsets, const int32_t *d_cols, const double *d_w,
                  int maximize, int64_t seed, int32_t *d_src, int32_t *d_dst, double *d_out_w,
                  int32_t *d_colors, int64_t *n_edges, int64_t *n_components, void *stream_) {
    STREAM(s);
    return guarded([&] {
        csr_solve_mst(n, d_offsets, d_cols, d_w, maximize != 0, seed, d_src, d_dst, d_out_w,
                      d_colors, n_edges, n_components, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_msf_edges(int64_t n, const int32_t *d_src, const int32_t *d_dst, const double *d_w,
                  int64_t m, int64_t seed, int32_t *d_out_src, int32_t *d_out_dst,
                  double *d_out_w, int32_t *d_colors, int64_t *n_edges, int64_t *n_components,
                  void *stream_) {
    STREAM(s);
    return guarded([&] {
        EdgeSet E = dedup_undirected(n, d_src, d_dst, d_w, m, s);
        msf_undirected(n, E.a, E.b, E.w, E.m, true, false, seed, d_out_src, d_out_dst, d_out_w,
                       d_colors, n_edges, n_components, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_build_dendrogram(const int32_t *d_src, const int32_t *d_dst, const double *d_w,
                         int64_t n, double *h_merges, void *stream_) {
    STREAM(s);
    return guarded([&] {
        if (n < 2) throw_invalid("dendrogram needs at least 2 points");
        if (getenv("SLK_HOST_FOLD")) {
            const FoldInput in = dendrogram_device_sort(d_src, d_dst, d_w, n, false, -1, s);
            dendrogram_fold(in, h_merges);
            return;
        }
        DeviceMerges dm;
        const int *cycle = dendrogram_device(d_src, d_dst, d_w, n, false, -1, dm, s);
        MergeCopies mc;
        merges_enqueue(dm, n - 1, mc, s);
        merges_expand(mc, h_merges);
        SLK_CUDA(cudaStreamSynchronize(s));
        if (*cycle) throw_invalid("edges contain a cycle: not a spanning tree");
    });
}

int slk_extract_clusters(const double *h_merges, int64_t n, int64_t n_clusters,
                         int64_t *h_labels) {
    return guarded([&] { extract_labels(h_merges, n, n_clusters, h_labels); });
}

int slk_pairwise_l2(const double *d_q, int64_t nq, const double *d_x, int64_t nx, int d,
                    int squared, double *d_out, void *stream_) {
    STREAM(s);
    return guarded([&] {
        pairwise_l2(d_q, nq, d_x, nx, d, squared, d_out, s);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

static void check_gpus(int n_gpus) {
    if (n_gpus < 1 || n_gpus > 64) throw_invalid("n_gpus must be in [1, 64], got %d", n_gpus);
}

int slk_single_linkage(const float *h_x32, const double *h_x64, int64_t n, int d, int k,
                       int64_t n_clusters, int metric, int64_t seed, int64_t max_connect_iters,
                       int n_gpus, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                       int64_t *h_tree_dst, double *h_tree_w, int64_t *n_connect_iters,
                       double *h_timings) {
    return guarded([&] {
        check_gpus(n_gpus);
        if (n < 2) throw_invalid("need at least 2 points, got %lld", (long long)n);
        if (n_clusters < 1) throw_invalid("n_clusters must be >= 1, got %lld", (long long)n_clusters);
        if (n_clusters > n) throw_invalid("n_clusters=%lld exceeds %lld points", (long long)n_clusters, (long long)n);
        if (k < 1) throw_invalid("k must be >= 1, got %d", k);
        if (k > n - 1) throw_invalid("k=%d exceeds N-1=%lld", k, (long long)(n - 1));
        if (n >= (1ll << 30)) throw_invalid("n=%lld exceeds the 2^30-1 point limit", (long long)n);
        StreamGuard g;
        cudaStream_t s = g.s;
        DevBuf<float> x32(n * (int64_t)d, s);
        DevBuf<double> x64;
        const double th = now_ms();
        SLK_CUDA(cudaMemcpyAsync(x32.get(), h_x32, n * (int64_t)d * sizeof(float), cudaMemcpyHostToDevice, s));
        if (h_x64) {
            x64.alloc(n * (int64_t)d, s);
            SLK_CUDA(cudaMemcpyAsync(x64.get(), h_x64, n * (int64_t)d * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        if (trace_on()) {
            SLK_CUDA(cudaStreamSynchronize(s));
            fprintf(stderr, "[slk] h2d %.1f ms\n", now_ms() - th);
        }
        single_linkage_device(x32, h_x64 ? x64.get() : nullptr, n, d, k, n_clusters, metric, seed,
                              max_connect_iters, h_merges, h_labels, h_tree_src, h_tree_dst,
                              h_tree_w, n_connect_iters, h_timings, s, n_gpus);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

int slk_single_linkage_device(const float *d_x32, const double *d_x64, int64_t n, int d, int k,
                              int64_t n_clusters, int metric, int64_t seed,
                              int64_t max_connect_iters, int n_gpus, double *h_merges,
                              int64_t *h_labels, int64_t *h_tree_src, int64_t *h_tree_dst,
                              double *h_tree_w, int64_t *n_connect_iters, double *h_timings,
                              void *stream_) {
    STREAM(s);
    return guarded([&] {
        check_gpus(n_gpus);
        if (n < 2) throw_invalid("need at least 2 points, got %lld", (long long)n);
        if (n_clusters < 1) throw_invalid("n_clusters must be >= 1, got %lld", (long long)n_clusters);
        if (n_clusters > n) throw_invalid("n_clusters=%lld exceeds %lld points", (long long)n_clusters, (long long)n);
        if (k < 1) throw_invalid("k must be >= 1, got %d", k);
        if (k > n - 1) throw_invalid("k=%d exceeds N-1=%lld", k, (long long)(n - 1));
        if (n >= (1ll << 30)) throw_invalid("n=%lld exceeds the 2^30-1 point limit", (long long)n);
        single_linkage_device(d_x32, d_x64, n, d, k, n_clusters, metric, seed, max_connect_iters,
                              h_merges, h_labels, h_tree_src, h_tree_dst, h_tree_w,
                              n_connect_iters, h_timings, s, n_gpus);
        SLK_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
