/*
 * kdtree_b200.h -- C-ABI of the B200 kd-tree build + exact KNN library
 * (libkdtree_b200.so).  Plain pointers and sizes only; no torch types.
 *
 * Each entry point replaces one reference interface of the `kdknn` package
 * (paths relative to /root/reference/pkg/src/kdknn):
 *
 *   kd_tree_build   <- local_tree.build_local_tree(points, cfg)   local_tree.py:436-574
 *   kd_tree_import  <- (wrap an existing LocalTree; e.g. one built by the
 *                       reference or loaded from a PKDB bundle)    engine.py:267-297
 *   kd_tree_export  <- LocalTree fields node_dim/node_value/node_left/
 *                       node_right/node_count/points/depth        local_tree.py:71-108
 *   kd_knn          <- local_query.find_knn_batch(tree, queries, k, radii)
 *                                                                  local_query.py:175-216
 *   kd_tree_free    <- (Python object lifetime)
 *
 * Conventions
 *  - Coordinates: SoA (dims, n) row-major, binary32 (KD_F32) or binary64
 *    (KD_F64).  binary32 inputs are exact in binary64, so results equal the
 *    reference (which upcasts every input to binary64, core.py:55).
 *  - Queries: (nq, dims) row-major binary64, like find_knn_batch.
 *  - Distances are squared Euclidean, accumulated in ascending dimension order
 *    in binary64 without FMA (core.py:199-228): bit-identical to the reference.
 *  - Result rows are sorted by (sq_dist, point_id); ties go to the smaller id.
 *    Slots past out_counts[i] are left untouched (the reference leaves them
 *    uninitialised, local_query.py:199-200).
 *  - Return value: KD_OK (0) or a negative KD_E* code; kd_last_error() gives
 *    a thread-local message.  The library never aborts the process.
 *  - flags: KD_DEVICE_PTRS -> every array argument is a device pointer on the
 *    tree's device (e.g. torch.Tensor.data_ptr()); otherwise host pointers are
 *    staged through device memory inside the call.
 */
#ifndef KDTREE_B200_H
#define KDTREE_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define KD_API __attribute__((visibility("default")))
#else
#define KD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define KD_OK 0
#define KD_EINVAL (-1)        /* bad argument            -> ValueError   */
#define KD_ECUDA (-2)         /* CUDA runtime failure    -> RuntimeError */
#define KD_EUNSUPPORTED (-3)  /* outside device limits   -> ValueError   */
#define KD_ENOMEM (-4)        /* allocation failure      -> MemoryError  */

#define KD_F32 1
#define KD_F64 2

#define KD_DEVICE_PTRS 1u     /* all array arguments are device pointers */
#define KD_NO_SORT 2u         /* kd_knn: keep caller query order (no leaf sort) */
#define KD_THREAD_PER_QUERY 4u /* kd_knn: one thread per query, no dynamic fetch (default: persistent warps) */
#define KD_KNN_REFERENCE 16u  /* kd_knn: walk the tree exactly as local_query.py:72-172 (binary64 incremental bounds, prune at bound >= r'): results and counters bit-identical to the reference, tie quirk included */
#define KD_KNN_PACKET 8u      /* kd_knn, D <= 3: one warp per 32-query packet over tight boxes (default: per-lane traversals) */

typedef struct kd_tree kd_tree;

/* BuildConfig (local_tree.py:48-68); workers/branch_factor have no device
 * meaning and are not passed. */
typedef struct {
    int64_t bucket_size;      /* default 32   */
    int64_t local_sample_m;   /* default 1024 (device limit 1024) */
    int64_t variance_sample;  /* default 1024 (device limit 1024) */
    uint64_t seed;            /* default 0    */
} kd_build_cfg;

typedef struct {
    int64_t n_nodes;
    int64_t n;
    int64_t n_leaves;
    int64_t depth;
    int32_t dims;
    int32_t dtype;
    int32_t device;
    int32_t reserved;
    double build_ms;          /* device time of the last build (CUDA events) */
    int64_t build_levels;     /* breadth-first global-memory levels */
    int64_t build_tasks;      /* shared-memory subtree tasks */
    int64_t build_slow_nodes; /* nodes resolved by the exact slow path */
    double build_ms_levels;   /* breadth-first levels (sampling, histograms, partitions) */
    double build_ms_subtree;  /* shared-memory subtree kernel */
    double build_ms_finish;   /* preorder stitch, relocation, id gather */
} kd_tree_info;

/* Reference LocalTree layout (local_tree.py:71-108).  Export fills caller
 * buffers of the sizes reported by kd_tree_info; import reads them. */
typedef struct {
    int32_t* node_dim;        /* [n_nodes] -1 = leaf                       */
    double* node_value;       /* [n_nodes]                                 */
    int32_t* node_left;       /* [n_nodes] left child | bucket start       */
    int32_t* node_right;      /* [n_nodes] right child | bucket length     */
    int64_t* node_count;      /* [n_nodes] points under the node           */
    double* coords;           /* [dims][n] packed points, binary64         */
    uint64_t* ids;            /* [n] packed point ids                      */
    int64_t* perm;            /* [n] packed row i = input row perm[i] (export only; may be NULL) */
} kd_tree_arrays;

KD_API int kd_version(void);
KD_API const char* kd_last_error(void);
KD_API int kd_device_count(int* count);

/* build_local_tree (local_tree.py:436-574); byte-identical tree. */
KD_API int kd_tree_build(const void* coords, int dtype, int64_t n, int dims, const uint64_t* ids,
                  const kd_build_cfg* cfg, int device, unsigned flags, void* stream, kd_tree** out);

/* wrap an existing preorder LocalTree (host arrays); dtype selects the device
 * storage type of the packed coordinates (KD_F32 only if exactly representable). */
KD_API int kd_tree_import(const kd_tree_arrays* arrays, int64_t n_nodes, int64_t n, int dims, int64_t depth,
                   int dtype, int device, kd_tree** out);

KD_API int kd_tree_get_info(const kd_tree* t, kd_tree_info* info);

/* copy the tree out in the reference layout (host buffers) */
KD_API int kd_tree_export(const kd_tree* t, kd_tree_arrays* out);

/* find_knn_batch (local_query.py:175-216).  radii: NULL = +inf.
 * exclude_ids: NULL, or one id per query that must not be returned (a query
 * drawn from the dataset excludes itself: BASELINE config 2).
 * out_counters: NULL or [nq][3] (nodes visited, buckets scanned, points compared). */
KD_API int kd_knn(const kd_tree* t, const double* queries, int64_t nq, int64_t k, const double* radii,
           const uint64_t* exclude_ids, double* out_dists, uint64_t* out_ids, int64_t* out_counts,
           int64_t* out_counters, unsigned flags, void* stream);

KD_API int kd_tree_free(kd_tree* t);

/* ---- global (multi-GPU) tier, cluster.py / dist_query.py ---------------- */

/* histogram_with_equals (median.py:243-265, cluster.py:246): counts[nb+1] of
 * values by "number of boundaries <= v" and equals[nb] exact matches.
 * boundaries sorted distinct binary64, 1 <= nb <= 4096. */
KD_API int kd_histogram(const void* values, int dtype, int64_t n, const double* boundaries, int64_t nb,
                        int64_t* counts, int64_t* equals, unsigned flags, void* stream);

/* redistribute side split (cluster.py:292-294, replaces the per-side index
 * arrays of redistribute): stable two-way partition of a rank's SoA points + ids,
 * coord[dim] < value first, written as packed rows [coords (padded to 8 B) | id]
 * -- the all-to-all send buffer.  *n_low (DEVICE memory) receives the low-side
 * count.  Asynchronous on `stream`; device pointers only. */
KD_API int kd_split_rows(const void* coords, int dtype, int64_t n, int dims, const uint64_t* ids, int dim,
                         double value, void* out_rows, int64_t* n_low, unsigned flags, void* stream);

/* packed rows (kd_split_rows layout) -> SoA coords [dims][n] + ids.  Device ptrs. */
KD_API int kd_unpack_rows(const void* rows, int64_t n, int dims, int dtype, void* out_coords, uint64_t* out_ids,
                          unsigned flags, void* stream);

/* owner-side merge (dist_query.py:138-161 merge_topk / _merge_arrays): for each of
 * m owned queries, its local sorted top-k (local_c entries, this rank) and the
 * nr remote replies addressed to it (reply_slot = owned-query index; reply_c
 * entries from rank reply_rank) -> the k smallest by (sq_dist, point_id), with
 * the contributing rank.  *dup_flag (device int32) is set to 1 when one point id
 * appears twice in a query's pool (the reference's ValueError).  Device ptrs. */
KD_API int kd_merge_topk(int64_t m, int64_t k, const double* local_d, const uint64_t* local_i, const int64_t* local_c,
                         int32_t my_rank, int64_t nr, const int64_t* reply_slot, const double* reply_d,
                         const uint64_t* reply_i, const int64_t* reply_c, const int32_t* reply_rank, double* out_d,
                         uint64_t* out_i, int32_t* out_rank, int64_t* out_c, int32_t* dup_flag, unsigned flags,
                         void* stream);

/* GlobalTree.owner_of_batch + ranks_within (cluster.py:96-154): owner rank of
 * each query (ties right) and, when `within` is non-NULL, the bitmask of other
 * ranks whose region's min squared distance is strictly below radii[i]
 * (NULL = +inf).  Regions are [ranks][dims] lower/upper bounds.  Device ptrs. */
KD_API int kd_route(const int32_t* plane_dims, const double* plane_values, int32_t ranks, const double* region_lo,
                    const double* region_hi, const double* queries, int64_t nq, int dims, const double* radii,
                    int32_t* owner, uint64_t* within, unsigned flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KDTREE_B200_H */
