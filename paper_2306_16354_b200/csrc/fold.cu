// fold.cu — host-side union-find fold of the sorted spanning tree into the
// merge table (and the flat cut), native code.  Replaces the reference's
// _dendrogram_merge / _uf_find (/root/reference/pkg/src/parlink/linkage.py:
// 91-129) and, for the pipeline, _inherit_labels / extract_clusters
// (:132-148, :184-213).
//
// The fold is inherently sequential (row i needs the cluster ids produced by
// rows < i); like the paper it runs on the host.  It is bound by
// cache misses on random vertex ids, so: one 16-byte node per vertex (parent,
// cluster id, size, rank share a cache line), and the nodes of the endpoints
// of edge i + D are prefetched while edge i is folded.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "common.cuh"

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

}  // namespace

// linkage.py:103-129: fold edges in merge order; row i = (min(ca, cb),
// max(ca, cb), w, size), parent id n + i.  When `labels` is given, the flat
// cut for n_clusters (linkage.py:184-213) is taken from the union-find state
// after the first cut = (n-1) - (n_clusters-1) merges: a point's nearest
// labelled ancestor is the current cluster id of its component, and labels
// rank those ids ascending.
void dendrogram_fold(const int32_t *a, const int32_t *b, const double *w, int64_t n,
                     double *merges, int64_t n_clusters, int64_t *labels, double *extract_ms) {
    if (n >= (1ll << 30)) throw_invalid("n=%lld too large for the dendrogram fold", (long long)n);
    std::vector<Node> nodes(n);
    Node *nd = nodes.data();
    for (int32_t v = 0; v < (int32_t)n; v++) nd[v] = Node{v, v, 1, 0};
    const int64_t cut = labels ? (n - 1) - (n_clusters - 1) : -1;
    auto snapshot = [&]() {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<int32_t> ids;
        ids.reserve(n_clusters);
        for (int32_t v = 0; v < (int32_t)n; v++)
            if (nd[v].parent == v) ids.push_back(nd[v].cid);
        if ((int64_t)ids.size() != n_clusters)
            throw_invalid("internal: found %lld label roots for %lld clusters", (long long)ids.size(),
                          (long long)n_clusters);
        std::sort(ids.begin(), ids.end());
        // finds on a compact copy of the parent links (4 B per vertex: the
        // random walks stay in cache); a root's entry becomes -(label + 1)
        std::vector<int32_t> par(n);
        for (int32_t v = 0; v < (int32_t)n; v++)
            par[v] = nd[v].parent == v
                         ? -1 - (int32_t)(std::lower_bound(ids.begin(), ids.end(), nd[v].cid) - ids.begin())
                         : nd[v].parent;
        int32_t *pp = par.data();
        for (int32_t p = 0; p < (int32_t)n; p++) {
            int32_t x = p;
            while (pp[x] >= 0) {
                const int32_t nx = pp[x];
                if (pp[nx] >= 0) pp[x] = pp[nx];  // path halving
                x = nx;
            }
            labels[p] = -1 - pp[x];
        }
        if (extract_ms)
            *extract_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    if (cut == 0) snapshot();
    for (int64_t i = 0; i < n - 1; i++) {
        if (i + PREFETCH < n - 1) {
            __builtin_prefetch(&nd[a[i + PREFETCH]]);
            __builtin_prefetch(&nd[b[i + PREFETCH]]);
        }
        if (i + PREFETCH / 2 < n - 1) {
            // second level: the parents of nodes prefetched half a window ago
            __builtin_prefetch(&nd[nd[a[i + PREFETCH / 2]].parent]);
            __builtin_prefetch(&nd[nd[b[i + PREFETCH / 2]].parent]);
        }
        int32_t ra = find_root(nd, a[i]), rb = find_root(nd, b[i]);
        if (ra == rb) throw_invalid("edges contain a cycle: not a spanning tree");
        const int32_t ca = nd[ra].cid, cb = nd[rb].cid, merged = nd[ra].size + nd[rb].size;
        double *row = merges + 4 * i;
        row[0] = (double)(ca < cb ? ca : cb);
        row[1] = (double)(ca < cb ? cb : ca);
        row[2] = w[i];
        row[3] = (double)merged;
        if (nd[ra].rank < nd[rb].rank) std::swap(ra, rb);
        nd[rb].parent = ra;
        if (nd[ra].rank == nd[rb].rank) nd[ra].rank++;
        nd[ra].cid = (int32_t)(n + i);
        nd[ra].size = merged;
        if (i + 1 == cut) snapshot();
    }
}

}  // namespace slk
