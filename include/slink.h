/*
 * slink.h — C ABI of libslink.so, the B200 (sm_100a) single-linkage library.
 *
 * Drop-in boundary for the reference package `parlink`
 * (/root/reference/pkg/src/parlink).  Each entry point replaces one reference
 * function or numba kernel group; the citation is given beside it.  The
 * Python mirror (paper_2306_16354_b200/) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Return value: SLK_OK (0) or an error status; slk_last_error() returns the
 *    message of the calling thread's last error.  The status classes map onto
 *    the reference's exceptions (core.py:15-24): SLK_ERR_INVALID ->
 *    ValidationError, SLK_ERR_CONVERGENCE -> ConvergenceError,
 *    SLK_ERR_INTERNAL / SLK_ERR_CUDA -> LinkageError.
 *  - "d_" pointers are device pointers (cudaMalloc / torch tensors) on the
 *    current device; "h_" pointers are host pointers.  Vertex / point ids are
 *    int32 on the device (N < 2^30: merge-table node ids n + i stay below
 *    2^31); distances and weights are float64 with
 *    the reference's exact values.  The library never frees caller memory;
 *    its scratch comes from the stream-ordered pool of the current device.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls return
 *    after the stream has drained unless stated otherwise.
 */
#ifndef SLINK_H
#define SLINK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLK_OK 0
#define SLK_ERR_INTERNAL 1
#define SLK_ERR_INVALID 2
#define SLK_ERR_CONVERGENCE 3
#define SLK_ERR_CUDA 4

/* Library version (major*10000 + minor*100 + patch). */
int slk_version(void);
/* Message for the last non-zero status on this thread. */
const char *slk_last_error(void);
/* Number of CUDA kernels this library has launched in this process. */
int64_t slk_kernel_launches(void);

/* ------------------------------------------------------------ neighbours */

/*
 * Exact k nearest neighbours of query rows [q0, q1) among all n points.
 * Replaces fused_knn (neighbors.py:246-298: _row_sq_norms :80-89,
 * _knn_scan_tile :119-160, _knn_merge_rows :163-188).
 * d_x32: n x d float32 row-major (the scan operand).  d_x64: n x d float64
 * row-major, or NULL when every value of the input is exactly the float32 in
 * d_x32 (then the refine reads d_x32).  Outputs rows in [q0, q1):
 * d_idx (q1-q0) x k int32, d_dist (q1-q0) x k float64 squared distances,
 * sorted ascending by (distance, id), bit-identical to the reference.
 */
int slk_knn(const float *d_x32, const double *d_x64, int64_t n, int d, int k, int64_t q0,
            int64_t q1, int32_t *d_idx, double *d_dist, void *stream);

/*
 * Nearest admissible neighbour of query rows [q0, q1) of Q among the nx rows
 * of X.  Replaces _fused_1nn_arrays (neighbors.py:301-348: _nn1_scan_tile
 * :191-217, _nn1_merge_rows :220-226) and so fused_1nn (:351-372) and
 * cross_color_1nn (:375-391).
 *   mode 0: every candidate admissible;
 *   mode 1: d_mask (nq x nx bytes, non-zero = admissible);
 *   mode 2: colours, admissible iff d_qcolor[i] != d_xcolor[j].
 * Q may alias X (pass the same pointers).  Returns SLK_ERR_INVALID naming the
 * first query row without an admissible candidate (:343-345).
 */
int slk_nn1(const float *d_q32, const double *d_q64, int64_t nq, const float *d_x32,
            const double *d_x64, int64_t nx, int d, int mode, const uint8_t *d_mask,
            const int32_t *d_qcolor, const int32_t *d_xcolor, int64_t q0, int64_t q1,
            int32_t *d_idx, double *d_dist, void *stream);

/*
 * Dense nq x nx squared-distance tile in the reference's expanded float64
 * form.  Replaces pairwise_l2_tile / _dist_tile (neighbors.py:92-104,229-243).
 */
int slk_pairwise_l2(const double *d_q, int64_t nq, const double *d_x, int64_t nx, int d,
                    int squared, double *d_out, void *stream);

/* Float64 squared row norms in the reference's order (neighbors.py:80-89). */
int slk_row_norms(const float *d_x32, const double *d_x64, int64_t n, int d, double *d_out,
                  void *stream);

/* ----------------------------------------------------------------- graph */

/*
 * Symmetric CSR of an edge list, duplicates collapsed to their minimum weight,
 * columns ascending within each row.  Replaces edge_list_to_csr
 * (core.py:264-286).  d_cols / d_w must hold 2*m entries; *nnz receives the
 * entry count.  Inputs must satisfy 0 <= id < n and src != dst.
 */
int slk_edge_list_to_csr(int64_t n, const int32_t *d_src, const int32_t *d_dst,
                         const double *d_w, int64_t m, int64_t *d_offsets, int32_t *d_cols,
                         double *d_cols_w, int64_t *nnz, void *stream);

/* 1 if the CSR holds (j,i,w) for every (i,j,w) (core.py:165-174), else 0. */
int slk_csr_is_symmetric(int64_t n, const int64_t *d_offsets, const int32_t *d_cols,
                         const double *d_w, int *is_symmetric, void *stream);

/*
 * Seeded order-preserving weight alteration of a symmetric CSR
 * (mst.py:198-222, _hash_unit :82-91, _alter_weights :94-105).
 * SLK_ERR_INVALID on a zero weight.  *theta receives theta.
 */
int slk_weight_alteration(int64_t n, const int64_t *d_offsets, const int32_t *d_cols,
                          const double *d_w, int64_t seed, double *d_alt, double *theta,
                          void *stream);

/* Per-vertex minimum (alt, a, b) incident edge to another colour, as a CSR
 * position or -1 (mst.py:225-254 / _min_edge_scan :108-128). */
int slk_min_edge_per_vertex(int64_t n, const int64_t *d_offsets, const int32_t *d_cols,
                            const double *d_alt, const int32_t *d_colors, int64_t *d_pos,
                            void *stream);

/* Per-colour reconciliation of vertex candidates into canonical,
 * deduplicated edges sorted by (a, b) (mst.py:257-280 / _reconcile_per_color
 * :131-151).  Outputs hold n entries; *m_out receives the count. */
int slk_min_edge_per_supervertex(int64_t n, const int64_t *d_pos, const int32_t *d_dst,
                                 const double *d_alt, const double *d_orig,
                                 const int32_t *d_colors, int32_t *d_a, int32_t *d_b,
                                 double *d_w, int64_t *m_out, void *stream);

/* Minimum-colour propagation over new edges (mst.py:283-289 /
 * _propagate_colors :154-186).  d_colors is updated in place. */
int slk_label_propagation(int64_t n, int32_t *d_colors, const int32_t *d_us,
                          const int32_t *d_vs, int64_t m, void *stream);

/*
 * Minimum (or maximum) spanning forest of a symmetric CSR graph.  Replaces
 * solve_mst (mst.py:292-344).  Outputs: up to n-1 edges (a < b) sorted by
 * (a, b) with original weights, canonical colours (minimum vertex id of each
 * component), *n_edges and *n_components.  SLK_ERR_INVALID on empty,
 * non-finite, asymmetric or zero-weight input.
 */
int slk_solve_mst(int64_t n, const int64_t *d_offsets, const int32_t *d_cols, const double *d_w,
                  int maximize, int64_t seed, int32_t *d_src, int32_t *d_dst, double *d_out_w,
                  int32_t *d_colors, int64_t *n_edges, int64_t *n_components, void *stream);

/* ------------------------------------------------------- dendrogram / cut */

/*
 * Merge table (n-1) x 4 float64 of a spanning tree: rows (child_a, child_b,
 * distance, size), parent id n+i.  Replaces build_dendrogram
 * (linkage.py:160-181 / _dendrogram_merge :103-129).  Device radix sort of
 * the edges by (w, a, b), then the union-find fold.  Host output buffer.
 * SLK_ERR_INVALID on a cycle.
 */
int slk_build_dendrogram(const int32_t *d_src, const int32_t *d_dst, const double *d_w,
                         int64_t n, double *h_merges, void *stream);

/* Flat labels for n_clusters from a host merge table (linkage.py:184-213 /
 * _inherit_labels :132-148).  Host buffers. */
int slk_extract_clusters(const double *h_merges, int64_t n, int64_t n_clusters,
                         int64_t *h_labels);

/* --------------------------------------------------------------- pipeline */

/*
 * End-to-end single linkage on one GPU, host buffers in and out.  Replaces
 * single_linkage (linkage.py:257-311) including connect_graph (:222-254).
 * h_x32: n x d float32; h_x64: n x d float64 or NULL (see slk_knn).
 * metric: 0 = euclidean, 1 = sqeuclidean.  max_connect_iters < 0 selects
 * ceil(log2 n) + 8.  Outputs (host): h_merges (n-1) x 4, h_labels n,
 * optional spanning tree h_tree_src/h_tree_dst/h_tree_w (n-1, squared L2,
 * sorted (src, dst); any may be NULL), *n_connect_iters, and per-stage
 * milliseconds h_timings[5] = knn, mst, connect, dendrogram, extract
 * (may be NULL).
 */
int slk_single_linkage(const float *h_x32, const double *h_x64, int64_t n, int d, int k,
                       int64_t n_clusters, int metric, int64_t seed, int64_t max_connect_iters,
                       int n_gpus, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                       int64_t *h_tree_dst, double *h_tree_w, int64_t *n_connect_iters,
                       double *h_timings);

/* As slk_single_linkage with the points already resident on the device.
 *
 * n_gpus (both entry points): the replacement of the reference's threads=
 * knob (parallel.py:16-48).  The k-NN pass and every cross-colour pass are
 * dealt to n_gpus shards in 128-row chunks, round-robin; shard g runs on
 * device (current + g) % device_count with a replica of the points, one host
 * thread per shard, and its rows return to the current device by peer copies
 * over NVLink.  The spanning forests, dendrogram and cut run on the current
 * device.  Results do not depend on n_gpus. */
int slk_single_linkage_device(const float *d_x32, const double *d_x64, int64_t n, int d, int k,
                              int64_t n_clusters, int metric, int64_t seed,
                              int64_t max_connect_iters, int n_gpus, double *h_merges,
                              int64_t *h_labels, int64_t *h_tree_src, int64_t *h_tree_dst,
                              double *h_tree_w, int64_t *n_connect_iters, double *h_timings,
                              void *stream);

/*
 * Point-set handles (the distributed driver, parallel.py): the per-matrix
 * search state (block spheres, tensor operand packs, split index) built once
 * over device-resident points and reused by every search on them.  The
 * caller keeps d_x32 / d_x64 alive until slk_pointset_destroy.
 *   slk_knn_ps: fused_knn rows [q0, q1) (neighbors.py:246-298), outputs as slk_knn.
 *   slk_nn1_colour_ps: cross_color_1nn rows [q0, q1) (neighbors.py:375-391)
 *     with colours d_colors (n int32), outputs as slk_nn1.
 */
int slk_pointset_create(const float *d_x32, const double *d_x64, int64_t n, int d, void **handle,
                        void *stream);
int slk_pointset_destroy(void *handle);
int slk_knn_ps(void *handle, int k, int64_t q0, int64_t q1, int32_t *d_idx, double *d_dist, void *stream);
int slk_nn1_colour_ps(void *handle, const int32_t *d_colors, int64_t q0, int64_t q1, int32_t *d_idx,
                      double *d_dist, void *stream);

/*
 * The tail of single_linkage (linkage.py:295-311) on a device spanning tree
 * (n-1 edges, squared-L2 weights): device (w, a, b) sort, the union-find fold
 * and the cut, as the single-process driver runs them; the torchrun driver's
 * rank 0 calls it after its connect loop.  Outputs as slk_single_linkage;
 * h_ms[2] (may be NULL) = dendrogram and cut milliseconds.
 */
int slk_finish_tree(const int32_t *d_src, const int32_t *d_dst, const double *d_w, int64_t n, int metric,
                    int64_t n_clusters, double *h_merges, int64_t *h_labels, int64_t *h_tree_src,
                    int64_t *h_tree_dst, double *h_tree_w, double *h_ms, void *stream);

/*
 * Spanning forest of the union of two edge lists (used by the connect loop
 * and the multi-GPU driver): symmetrise + min-dedup (core.py:264-286) then
 * solve_mst (mst.py:292-344) with the given seed, without materialising the
 * CSR.  Inputs are device edge lists; outputs as slk_solve_mst.
 */
int slk_msf_edges(int64_t n, const int32_t *d_src, const int32_t *d_dst, const double *d_w,
                  int64_t m, int64_t seed, int32_t *d_out_src, int32_t *d_out_dst,
                  double *d_out_w, int32_t *d_colors, int64_t *n_edges, int64_t *n_components,
                  void *stream);

/* Scan-kernel statistics of the last slk_knn / slk_nn1 call on this thread:
 * stats[0] rows refined, [1] rows re-scanned exactly in float64, [2] index
 * tiles computed, [3] index tiles skipped by the bounds, [4] rows the
 * tensor-core pass could not certify (redone by the exact-fp32 scan).
 * stats must hold 5 values. */
int slk_last_scan_stats(int64_t *stats);

/* Process-wide kernel profile since the last reset: out[0] distance-scan
 * kernel milliseconds (CUDA events on the launching stream), [1] scan
 * launches, [2] algorithmic FLOP of those launches (2 * rows * n_index * d,
 * brute force), [3] 128x128 tiles computed, [4] refine-kernel milliseconds,
 * [5] rows re-scanned exactly, [6] visit-order (bounds + segmented sort)
 * milliseconds, [7] FLOP of the tiles actually computed (2*128*128*d each),
 * [8] tiles a brute-force scan would compute, [9] tensor-core scan kernel
 * milliseconds, [10] FLOP of the tiles it computed, [11] rows it could not
 * certify, [12] Boruvka round-loop milliseconds (spanning-forest solves),
 * [13] its algorithmic bytes (12 B per directed edge entry + 16 B per vertex
 * per round), [14] rounds, [15] milliseconds of the whole forest
 * solves (incl. weight alteration and sorts).  reset != 0 zeroes the
 * counters after reading.  out must hold 16 doubles. */
int slk_profile(double *out, int reset);

/* Diagnostic (scripts/tc_debug.py): only the tensor-core k-NN scan over all n
 * points, without refine: per row its raw candidate list d_cand (n x 32 int32,
 * unused slots -1), the K'-th approximate value d_kth (n floats, scaled
 * units), |q~|^2 d_qhat (n floats) and the power-of-two operand scale.
 * With SLK_DEBUG_BC=1 in the environment it runs the block-centred kernel
 * instead: d_cand n x 64 (two column-half lists), d_kth n x 2, d_qhat = the
 * largest visited block radius (scaled). */
int slk_debug_tc_scan(const float *d_x32, int64_t n, int d, int k, int32_t *d_cand,
                      float *d_kth, float *d_qhat, float *scale, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SLINK_H */
