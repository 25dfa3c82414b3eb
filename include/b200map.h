/*
 * b200map.h — C ABI of the B200-native Mapper-graph engine (libb200map.so).
 *
 * The reference (`nervemap`, /root/reference/pkg/src/nervemap) is pure
 * Python with no FFI; each entry point below replaces one Python function of
 * its hot path (cited file:line, relative to /root/reference/pkg/src/nervemap).
 * INTEGRATION.md shows the ctypes binding a nervemap maintainer would add.
 *
 * Conventions
 *   - Every pointer named d_* is DEVICE memory owned by the caller; h_* is
 *     host memory owned by the caller.  The library never returns memory the
 *     caller must free; internal scratch is stream-ordered (cudaMallocAsync)
 *     and freed before the call returns, but the device's default pool keeps
 *     it mapped for the next call, and scratch of 16 MB and more (bitmaps,
 *     limb planes, tile tables) stays in a per-device cache of large
 *     buffers that later calls reuse (bm_release_scratch frees both;
 *     B200MAP_POOL_RELEASE=1 disables the pool retention).
 *   - `stream` is a cudaStream_t (passed as void*); NULL = legacy stream.
 *     Calls that must size outputs synchronise that stream.
 *   - Return value: 0 on success, BM_ERR_DATA (-1) for invalid arguments
 *     (maps to nervemap.errors.DataError), BM_ERR_INTERNAL (-2) for CUDA or
 *     invariant failures (maps to InternalError), BM_ERR_NOMEM (-3) when a
 *     device allocation fails.  The message is kept per calling thread and
 *     read with bm_last_error().  No C++ exception crosses the ABI.
 *   - Calls are re-entrant across host threads (each uses its own stream and
 *     scratch), matching server.py's concurrent compute_mapper calls.
 */
#ifndef B200MAP_H
#define B200MAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_OK 0
#define BM_ERR_DATA (-1)
#define BM_ERR_INTERNAL (-2)
#define BM_ERR_NOMEM (-3)

/* Exact fp64 summation order used for an element's distances
 * (clustering.py:201-208 chooses it per element). */
#define BM_ORDER_SEQUENTIAL 0 /* scipy cdist: s=0; s+=(x-y)^2 ... ; sqrt   (clustering.py:113,217) */
#define BM_ORDER_PAIRWISE 1   /* numpy add.reduce pairwise tree; sqrt      (clustering.py:137-139) */

/* Lens kinds (filters.py:14, 133-140) */
#define BM_LENS_COLUMN 0
#define BM_LENS_L2 1
#define BM_LENS_LINF 2

/* Distance engines for bm_cluster_elements (flags) */
#define BM_ENGINE_AUTO 0  /* tensor-core candidates + exact recheck where supported */
#define BM_ENGINE_EXACT 1 /* every pair evaluated in exact fp64 order on CUDA cores   */
#define BM_ENGINE_TC 2    /* force the tcgen05 candidate engine (32 <= d <= 256:
                             full-K operand tiles live in shared memory; outside
                             that range BM_ENGINE_TC is BM_ERR_DATA and AUTO
                             uses the exact engine) */

int bm_abi_version(void);
const char* bm_last_error(void);
/* Kernel launches issued by this library since load (benchmark evidence). */
int64_t bm_launch_count(void);
/* Internal scratch is stream-ordered pool memory kept mapped between calls
 * (re-mapping GBs per call is slow); this returns it to the driver. */
int bm_release_scratch(void);
/* Number of visible CUDA devices (for the host-side GPU-count knob). */
int bm_device_count(int* out);
/* Free bytes on the current device, counting what the library's stream-ordered
 * pool retains unused (sizes the row windows of bm_big_*). */
int bm_device_free_bytes(int64_t* out);

/* ---- K1: lens (filters.py:133-140, evaluate) --------------------------------
 * out[i] = X[i,col]                         (BM_LENS_COLUMN, filters.py:135-136)
 *        = sqrt(numpy_pairwise_sum(X[i]^2))  (BM_LENS_L2,    filters.py:137-138)
 *        = max_j |X[i,j]|                    (BM_LENS_LINF,  filters.py:139-140)
 * X is n x d row-major fp64. Bit-identical to numpy 2.x on x86-64. */
int bm_lens_f64(int kind, const double* d_X, int64_t n, int64_t d, int64_t col,
                double* d_out, void* stream);

/* ---- normalize (dataset.py:165-186) ----------------------------------------
 * scheme 1 = minmax, 2 = l2 (0 = none is a caller-side no-op). d_out may not
 * alias d_X. Bit-identical to the numpy expressions in dataset.py:176-185. */
int bm_normalize_f64(int scheme, const double* d_X, int64_t n, int64_t d,
                     double* d_out, void* stream);

/* ---- O(N x M) lenses (filters.py:103-150): eccentricity and density ------
 * For every query row (d_qrows, nq; NULL = rows 0..nq-1) against the target
 * rows (d_trows, m; NULL = rows 0..m-1; the reference uses all points, or its
 * seed-1729 subsample of 50k rows when N is larger), with d = scipy cdist:
 *   BM_PLENS_ECC_MEAN  mean_j d             (eccentricity p = 1; bit-exact)
 *   BM_PLENS_ECC_RMS   sqrt(mean_j d^2)     (p = 2; bit-exact)
 *   BM_PLENS_ECC_POW   (mean_j d^p)^(1/p)   (param = p; ulp-level: CUDA pow)
 *   BM_PLENS_ECC_MAX   max_j d              (p = inf; bit-exact)
 *   BM_PLENS_DENSITY   sum_j exp(-(d^2)/param), param = 2 sigma^2 (ulp-level: exp)
 *   BM_PLENS_NN_MIN    min over targets with a different row id (bit-exact;
 *                      the default bandwidth's nearest-neighbour step)
 * Sums and means follow numpy's pairwise row reduction over the targets. */
#define BM_PLENS_ECC_MEAN 0
#define BM_PLENS_ECC_RMS 1
#define BM_PLENS_ECC_POW 2
#define BM_PLENS_ECC_MAX 3
#define BM_PLENS_DENSITY 4
#define BM_PLENS_NN_MIN 5
int bm_pairwise_lens(int kind, double param, const double* d_X, int64_t n, int64_t d,
                     const int64_t* d_qrows, int64_t nq, const int64_t* d_trows, int64_t m,
                     double* d_out, void* stream);

/* ---- K2: cover binning (cover.py:122-140, membership) -----------------------
 * f: n x m row-major fp64 filter values (m = 1 or 2).
 * h_lo/h_hi: concatenated per-axis closed-interval endpoints
 *            (axis 0 intervals first), exactly as cover._build_axis makes them.
 * h_n_axis: intervals per axis (m entries). Elements are row-major over axes
 *           (cover.py:56-61); n_el = prod(h_n_axis).
 * Pass 1 writes h_counts[n_el] (rows per element; synchronises the stream).
 * Pass 2 writes, for every element k, the ascending row ids of element k into
 * d_rows[d_offsets[k] .. d_offsets[k+1]) where d_offsets (n_el+1, device) is
 * the exclusive scan of the counts supplied by the caller. */
int bm_membership_count(const double* d_f, int64_t n, int m, const double* h_lo,
                        const double* h_hi, const int32_t* h_n_axis,
                        int64_t* h_counts, void* stream);
int bm_membership_fill(const double* d_f, int64_t n, int m, const double* h_lo,
                       const double* h_hi, const int32_t* h_n_axis,
                       const int64_t* d_offsets, int64_t* d_rows, void* stream);

/* ---- K3..K6: per-element DBSCAN (clustering.py:151-198, 238-316) ------------
 * X: n x d fp64 points. d_rows/h_offsets: memberships as produced above
 * (element k owns d_rows[h_offsets[k] .. h_offsets[k+1])).
 * h_order[k]: BM_ORDER_* for element k (clustering.py:201-208).
 * Outputs:
 *   d_labels[e]   cluster rank of membership entry e inside its element
 *                 (clusters ordered by smallest row, clustering.py:192-197),
 *                 or -1 for noise;
 *   h_n_clusters[k] number of clusters of element k (synchronises the stream).
 * engine: BM_ENGINE_*.  stats (optional, 8 int64): [0] distinct row pairs
 * inside the computed tile pairs, [1] pairs rechecked in exact fp64,
 * [2] tile pairs pruned by the centre/radius bound, [3] tile pairs total,
 * [4] bitmap bytes (largest window), [5] adjacency-stage device time (ns, CUDA
 * events on `stream`), [6] grouping/gather/quantise/prune time (ns),
 * [7] core/union-find/relabel time (ns).
 * Internally rows of an element are regrouped spatially and tile pairs that
 * provably hold no eps pair are skipped; results do not depend on either
 * (B200MAP_NO_PRUNE=1 turns both off). An element whose bitmap exceeds the
 * device budget is processed in row windows (two passes). */
int bm_cluster_elements(const double* d_X, int64_t n, int64_t d,
                        const int64_t* d_rows, const int64_t* h_offsets,
                        int64_t n_el, double eps, int32_t min_pts,
                        const uint8_t* h_order, int engine, int32_t* d_labels,
                        int32_t* h_n_clusters, int64_t* h_stats, void* stream);

/* Work estimate for scheduling elements over GPUs (clustering.py:281-315
 * runs elements as independent tasks): per element, the number of 128 x 128
 * tile pairs that survive the rigorous pruning bound (h_kept_tiles[k]) — the
 * distance work the engine will do for it. Runs the grouping, gather, tile
 * geometry and pruning of bm_cluster_elements (no distances). */
int bm_element_work(const double* d_X, int64_t n, int64_t d, const int64_t* d_rows,
                    const int64_t* h_offsets, int64_t n_el, double eps,
                    int64_t* h_kept_tiles, void* stream);

/* Full n_rows x n_rows distance matrix of X[rows] in one exact order
 * (clustering.py:96-113 pairwise_distances for BM_ORDER_SEQUENTIAL; the
 * on-the-fly rows of clustering.py:137-139 for BM_ORDER_PAIRWISE).
 * API helper for parity checks; the DBSCAN engine never materialises it. */
int bm_pairwise_distances(const double* d_X, int64_t n, int64_t d, const int64_t* d_rows,
                          int64_t n_rows, int order, double* d_out, void* stream);

/* ---- row-block protocol: one huge element over several ranks -------------
 * SURVEY §8e "huge single element" (cfg5). The element's eps-graph is a
 * triangle of T x T bit tiles (128 rows each); ranks take disjoint windows of
 * tile rows [I0, I1) (balanced by tile area) and run these per-rank steps; the
 * host does the collectives (torch.distributed / NCCL) in between:
 *   bm_big_open            gather + quantise the element's rows (once per rank)
 *   bm_big_counts          bits of a window; eps-neighbour counts of every row
 *                          they touch ADDED into d_cnt        -> all_reduce(sum)
 *   bm_big_init            core = cnt >= min_pts; par[p] = p; bmin[p] = INT_MAX
 *   bm_big_components      union-find over the window's core-core bits (in
 *                          d_par) and border minima (in d_bmin) -> par gathered
 *                          to rank 0 + bm_merge_forest; all_reduce(min) of bmin
 *   bm_big_labels          canonical labels of the element's entries (rank 0)
 * Arrays d_cnt/d_par/d_bmin hold P = 128 * T padded rows (int32); the caller
 * zeroes d_cnt before the first bm_big_counts. All calls on a handle run on the
 * stream given to bm_big_open. The same element processed by one rank with one
 * window is exactly bm_cluster_elements (which uses this path itself, on one
 * device, for an element whose bitmap exceeds the device budget).
 * Reference: clustering.py:151-198 (the dbscan of one element). */
int bm_big_open(const double* d_X, int64_t n, int64_t d, const int64_t* d_rows,
                int64_t n_rows, double eps, int32_t min_pts, int order, int engine,
                void* stream, void** handle, int64_t* h_tiles);
int bm_big_counts(void* handle, int32_t I0, int32_t I1, int32_t* d_cnt);
int bm_big_init(void* handle, const int32_t* d_cnt, int32_t* d_par, int32_t* d_bmin);
int bm_big_components(void* handle, int32_t I0, int32_t I1, int32_t* d_par, int32_t* d_bmin);
int bm_big_labels(void* handle, int32_t* d_par, const int32_t* d_bmin, int32_t* d_labels,
                  int32_t* h_n_clusters);
int bm_big_stats(void* handle, int64_t* h_stats);
/* Kept (unpruned) tile pairs before each tile row: h_row_first[I] for I in
 * [0, T], h_row_first[T] = all kept tile pairs. Ranks cut their windows at
 * equal KEPT work rather than equal triangle area. */
int bm_big_row_tiles(void* handle, int64_t* h_row_first);
int bm_big_close(void* handle);
/* d_par := union of the forests d_par and d_other (n entries each). */
int bm_merge_forest(int32_t* d_par, const int32_t* d_other, int64_t n, void* stream);

/* ---- nodes (nerve.py:84-101): stable grouping of entries into node rows ----
 * Given per-entry labels (above) and the per-element cluster counts, writes
 * the rows of node v (dense ids in (element, cluster) order) into
 * d_node_rows[d_node_offsets[v] .. d_node_offsets[v+1]) ascending, and
 * d_node_offsets (n_nodes+1). n_nodes = sum(h_n_clusters). Returns the total
 * number of clustered entries in *h_total. */
int bm_group_nodes(const int64_t* d_rows, const int64_t* h_offsets, int64_t n_el,
                   const int32_t* d_labels, const int32_t* h_n_clusters,
                   int64_t* d_node_rows, int64_t* d_node_offsets,
                   int64_t* h_total, void* stream);

/* ---- K7: nerve edges (nerve.py:103-113) --------------------------------------
 * Edges (s, t, w) with s < t, w = |rows_s ∩ rows_t| > 0, sorted
 * lexicographically. The point-centric histogram yields exactly the
 * overlapping_pairs candidates (cover.py:74-81) because a shared row implies
 * overlapping elements. n_points bounds the row ids.
 * Call with d_edges == NULL to get the count in *h_n_edges (synchronises);
 * then again with d_edges (3 * n_edges int64, row-major s,t,w). A d_edges
 * buffer of n_nodes * (n_nodes - 1) / 2 edges always suffices, so one call
 * with such a buffer both counts and writes. */
int bm_nerve_edges(const int64_t* d_node_rows, const int64_t* d_node_offsets,
                   int64_t n_nodes, int64_t n_points, int64_t* d_edges,
                   int64_t* h_n_edges, void* stream);

/* ---- canonical JSON of the node array (nerve.py:119-188) --------------------
 * Writes "[{...},...]": per node, keys sorted (composition, element,
 * filter_mean, id, rows, size, stats), floats "%.9g" with "-0" -> "0",
 * non-finite -> BM_ERR_DATA. Host memory only (no device work):
 *   h_node_rows/h_node_off  rows of node v: [off[v], off[v+1])
 *   h_elem                  2 per node: element index, or (i, j) for 2-D covers
 *                           (second value -1 for 1-D)
 *   h_stats (n_nodes x d)   column means; h_stat_order[i] = column of the i-th
 *                           key in sorted key order, h_names[h_name_off[i] ..
 *                           h_name_off[i+1]) its JSON-quoted name
 *   h_fmean (n_nodes x m)   filter means
 *   h_comp/h_comp_off       per node, the JSON text of its composition object
 * Call with out == NULL to get the length in *h_len, then with a buffer of at
 * least that many bytes: when the second call comes from the same thread with
 * the same arguments it copies the text formatted by the first instead of
 * formatting again. The cache is keyed on the pointers and sizes only, so the
 * caller must not modify the input arrays in place between the sizing call
 * and the writing call (a changed input needs a fresh sizing call). */
int bm_json_nodes(int64_t n_nodes, const int64_t* h_node_rows, const int64_t* h_node_off,
                  const int32_t* h_elem, const double* h_stats, int64_t d,
                  const int32_t* h_stat_order, const char* h_names, const int64_t* h_name_off,
                  const double* h_fmean, int32_t m, const char* h_comp,
                  const int64_t* h_comp_off, char* out, int64_t cap, int64_t* h_len);

/* ---- node payload (nerve.py:60-62, 96) --------------------------------------
 * d_stats[v*d + c] = numpy mean over node v's rows of column c (sequential
 * row sum / size, as numpy's axis-0 mean); d_fmean[v*m + a] = numpy 1-D mean
 * of the filter values (pairwise sum / size). */
int bm_node_stats(const double* d_X, int64_t d, const double* d_f, int m,
                  const int64_t* d_node_rows, const int64_t* d_node_offsets,
                  int64_t n_nodes, double* d_stats, double* d_fmean,
                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200MAP_H */
