// fold.cu — host-side union-find fold of the sorted spanning tree into the
// merge table (and the flat cut), native code: the SLK_HOST_FOLD=1
// alternative to the device merge table (dendro.cu:krt_kernel), kept for
// comparison.  Replaces the reference's _dendrogram_merge / _uf_find
// (/root/reference/pkg/src/parlink/linkage.py:91-129) and, for the pipeline,
// _inherit_labels / extract_clusters (:132-148, :184-213).
//
// The fold is sequential in merge order; like the paper it
// runs on the host, split over the components of the forest of its first
// merges.  It is bound by cache misses on random vertex ids, so: one 16-byte
// node per vertex (parent, cluster id, size, rank share a cache line), and
// the nodes of the endpoints of edge i + D are prefetched while edge i is
// folded.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <memory>
#include <thread>
#include <vector>

#include "common.cuh"
#include "host_pool.h"

namespace slk {

namespace {

struct Node {
    int32_t parent;
    int32_t cid;   // current cluster id of the component (valid at roots)
    int32_t size;  // component size (valid at roots)
    int32_t rank;
};

inline int32_t find_root(Node *nd, int32_t x) {
    // path halving: same roots as the reference's full compression (_uf_find,
    // linkage.py:91-100); the merge table only depends on the roots
    while (nd[x].parent != x) {
        const int32_t g = nd[nd[x].parent].parent;
        nd[x].parent = g;
        x = g;
    }
    return x;
}

constexpr int64_t PREFETCH = 16;

// Folds merge rank i with endpoints (ea, eb) and weight ew: row i = (min(ca,
// cb), max(ca, cb), w, size); the merged component takes cluster id n + i
// (linkage.py:114-128).
inline void fold_edge(Node *nd, int32_t ea, int32_t eb, double ew, int64_t n, int64_t i, double *merges) {
    int32_t ra = find_root(nd, ea), rb = find_root(nd, eb);
    if (ra == rb) throw_invalid("edges contain a cycle: not a spanning tree");
    const int32_t ca = nd[ra].cid, cb = nd[rb].cid, merged = nd[ra].size + nd[rb].size;
    double *row = merges + 4 * i;
    row[0] = (double)(ca < cb ? ca : cb);
    row[1] = (double)(ca < cb ? cb : ca);
    row[2] = ew;
    row[3] = (double)merged;
    if (nd[ra].rank < nd[rb].rank) std::swap(ra, rb);
    nd[rb].parent = ra;
    if (nd[ra].rank == nd[rb].rank) nd[ra].rank++;
    nd[ra].cid = (int32_t)(n + i);
    nd[ra].size = merged;
}

// Folds positions [j0, j1) of the staged arrays (merge rank rank[j], or j
// itself when rank == nullptr), prefetching the endpoints' nodes ahead.
inline void fold_run(Node *nd, const FoldInput &in, const int32_t *rank, int64_t j0, int64_t j1, double *merges) {
    const int32_t *a = in.a, *b = in.b;
    for (int64_t j = j0; j < j1; j++) {
        if (j + PREFETCH < j1) {
            __builtin_prefetch(&nd[a[j + PREFETCH]]);
            __builtin_prefetch(&nd[b[j + PREFETCH]]);
        }
        if (j + PREFETCH / 2 < j1) {
            // second level: the parents of nodes prefetched half a window ago
            __builtin_prefetch(&nd[nd[a[j + PREFETCH / 2]].parent]);
            __builtin_prefetch(&nd[nd[b[j + PREFETCH / 2]].parent]);
        }
        fold_edge(nd, a[j], b[j], in.w[j], in.n, rank ? (int64_t)rank[j] : j, merges);
    }
}

// Runs body(lo, hi) over [0, n) split into `threads` contiguous slices.
template <class F>
void parallel_slices(int64_t n, int threads, F body) {
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n / 65536 + 1));
    pool_slices(n, threads, body);  // persistent host workers (host_pool.h)
}

// Flat cut from the union-find state after the first `cut` merges
// (linkage.py:184-213): a point's nearest labelled ancestor is the current
// cluster id of its component; labels rank those ids ascending.  Read-only
// finds (union by rank keeps them O(log n) deep), so the points split over
// threads.
void cut_labels(const Node *nd, int64_t n, int64_t n_clusters, int64_t *labels, int threads) {
    std::vector<std::pair<int32_t, int32_t>> roots;  // (cluster id, root vertex)
    {
        // roots found per slice in parallel, concatenated (sorted below)
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n / 65536 + 1));
        std::vector<std::vector<std::pair<int32_t, int32_t>>> part(nt);
        HostPool::get().run(nt, [&](int k) {
            const int64_t lo = n * k / nt, hi = n * (k + 1) / nt;
            for (int64_t v = lo; v < hi; v++)
                if (nd[v].parent == (int32_t)v) part[k].emplace_back(nd[v].cid, (int32_t)v);
        });
        roots.reserve(n_clusters);
        for (auto &p : part) roots.insert(roots.end(), p.begin(), p.end());
    }
    if ((int64_t)roots.size() != n_clusters)
        throw_invalid("internal: found %lld label roots for %lld clusters", (long long)roots.size(),
                      (long long)n_clusters);
    std::sort(roots.begin(), roots.end());
    // label of each root vertex (only roots are read)
    std::unique_ptr<int32_t[]> lab(new int32_t[n]);
    for (size_t r = 0; r < roots.size(); r++) lab[roots[r].second] = (int32_t)r;
    const int32_t *lp = lab.get();
    parallel_slices(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t p = lo; p < hi; p++) {
            int32_t x = (int32_t)p;
            while (nd[x].parent != x) x = nd[x].parent;
            labels[p] = lp[x];
        }
    });
}

}  // namespace

// linkage.py:103-129: fold edges in merge order; row i = (min(ca, cb),
// max(ca, cb), w, size), parent id n + i.  When `labels` is given, the flat
// cut for n_clusters (linkage.py:184-213) is taken from the union-find state
// after the first cut = (n-1) - (n_clusters-1) merges.
//
// Parallel prefix (in.t > 0): the first t merges split into the components of
// the forest they form, and row i only depends on the merges before it in its
// own component, so those components fold independently (threads take them
// largest first; vertex sets are disjoint, so the shared node array needs no
// locks).  The remaining merges t..n-2 then fold in order on top of the
// components' roots.  t <= cut, so the cut comes after the parallel part.
void dendrogram_fold(const FoldInput &in, double *merges, int64_t n_clusters, int64_t *labels, double *extract_ms) {
    const int64_t n = in.n;
    if (n >= (1ll << 30)) throw_invalid("n=%lld too large for the dendrogram fold", (long long)n);
    // uninitialised: the threads below write every node (first touch in parallel)
    std::unique_ptr<Node[]> nodes(new Node[n]);
    Node *nd = nodes.get();
    parallel_slices(n, in.threads, [&](int64_t lo, int64_t hi) {
        for (int64_t v = lo; v < hi; v++) nd[v] = Node{(int32_t)v, (int32_t)v, 1, 0};
    });
    const int64_t cut = labels ? (n - 1) - (n_clusters - 1) : -1;
    auto snapshot = [&]() {
        auto t0 = std::chrono::steady_clock::now();
        cut_labels(nd, n, n_clusters, labels, in.threads);
        if (extract_ms)
            *extract_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    int64_t start = 0;
    if (in.t > 0) {
        if (cut >= 0 && in.t > cut) throw_invalid("internal: parallel fold prefix passes the cut");
        const int64_t ng = in.ngroups;
        std::vector<int64_t> order(ng);
        for (int64_t g = 0; g < ng; g++) order[g] = g;
        std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
            const int64_t sx = in.off[x + 1] - in.off[x], sy = in.off[y + 1] - in.off[y];
            return sx != sy ? sx > sy : x < y;
        });
        std::atomic<int64_t> next{0};
        std::atomic<bool> failed{false};
        auto worker = [&]() {
            try {
                for (int64_t q; !failed.load() && (q = next.fetch_add(1)) < ng;)
                    fold_run(nd, in, in.rank, in.off[order[q]], in.off[order[q] + 1], merges);
            } catch (...) {
                failed = true;
            }
        };
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(in.threads, ng));
        HostPool::get().run(nt, [&](int) { worker(); });
        if (failed) throw_invalid("edges contain a cycle: not a spanning tree");
        start = in.t;
    }
    if (cut == start) snapshot();
    for (int64_t i = start; i < n - 1;) {
        // fold up to the cut, snapshot, then the rest
        const int64_t stop = (cut > i && cut < n - 1) ? cut : n - 1;
        fold_run(nd, in, nullptr, i, stop, merges);
        i = stop;
        if (i == cut && cut > start) snapshot();
    }
}

}  // namespace slk
