/*
 * h2f.h — C ABI of the B200 RS-S factorize/solve path (libh2f.so).
 *
 * The reference (h2factor, pure Python) has no FFI; its boundary is the Python
 * API in /root/reference/pkg/src/h2factor/__init__.py:11-26.  Each entry point
 * below is what a ctypes/cffi binding of that API binds:
 *
 *   h2f_matrix_create   H2Matrix as consumed by factorize()      h2core.py:97-125
 *   h2f_matvec          matvec(h2, x)                             h2core.py:285-315
 *   h2f_norm2           estimate_norm2(h2, iters, seed)           h2core.py:318-330
 *   h2f_factorize       factorize(h2, eps_lu, threads, norm_est)  factorization.py:204-271
 *   h2f_solve           solve(fac, b) / solve_multi(fac, B)       solve.py:29-60
 *   h2f_refined_solve   refined_solve(h2, fac, b, steps)          solve.py:63-77
 *   h2f_factor_*        H2Factorization / LevelRecord / ClusterFactor fields
 *                                                                 factorization.py:130-193
 *   h2f_greedy_coloring greedy_coloring + color_groups            structure.py:148-167
 *
 * Conventions: every function returns 0 on success and a nonzero H2F_E* code
 * otherwise (never throws across the ABI); h2f_last_error() gives the message.
 * Pointers are HOST pointers unless the name ends in _dev.  All matrices are
 * row-major (C order, like NumPy).  Vectors are in tree order.  Calls are
 * synchronous on return and run on the library's own CUDA stream
 * (h2f_stream()).  One process = one device context.
 */
#ifndef H2F_H
#define H2F_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    H2F_OK = 0,
    H2F_E_ARG = 1,        /* invalid argument / shape (ValueError)               */
    H2F_E_CUDA = 2,       /* CUDA runtime failure                                 */
    H2F_E_NOMEM = 3,      /* device arena exhausted                               */
    H2F_E_SINGULAR = 4,   /* FactorizationError: vanishing pivot                  */
    H2F_E_INTERNAL = 5    /* broken bookkeeping invariant (AssertionError)        */
};

typedef struct h2f_matrix_s* h2f_matrix;
typedef struct h2f_factor_s* h2f_factor;

/* Cluster tree + block partition + block values.  Node ids are the
 * reference's preorder ids (geometry.py:85-142).  Pair lists are canonical
 * (s <= t) and sorted, one list per level (structure.py:42-85). */
typedef struct {
    int64_t n;               /* number of points                                 */
    int32_t depth;           /* tree depth (leaves at this level)                */
    int32_t top_level;       /* shallowest level with admissible blocks, -1 none */
    int64_t num_nodes;
    const int64_t* parent;   /* [num_nodes]                                      */
    const int64_t* child_left, *child_right, *level, *begin, *end;
    const int64_t* rank;     /* [num_nodes] basis rank, -1 where no basis        */
    /* per-level pair lists: pairs[2*i], pairs[2*i+1]; level l owns
     * [ptr[l], ptr[l+1]) */
    const int64_t* adm_pairs;   const int64_t* adm_ptr;     /* admissible leaves   */
    const int64_t* inner_pairs; const int64_t* inner_ptr;   /* inadmissible inner  */
    const int64_t* dense_pairs; const int64_t* dense_ptr;   /* inadmissible leaves */
    /* element offsets into vals (-1 = absent):
     *   leaf_basis_off[node]  (m_c x rank_c)       transfer_off[node] (rank_c x rank_parent)
     *   coupling_off[i]  for adm pair i  (rank_s x rank_t)
     *   dense_off[i]     for dense pair i (m_s x m_t) */
    const int64_t* leaf_basis_off;
    const int64_t* transfer_off;
    const int64_t* coupling_off;
    const int64_t* dense_off;
    int64_t nvals;
} h2f_matrix_desc;

/* status of a factorization: for H2F_E_SINGULAR, cluster/level name the
 * cluster whose redundant block failed (cluster = -1: the final dense LU). */
typedef struct {
    int32_t code;
    int32_t cluster;
    int32_t level;
} h2f_status;

typedef struct {
    int64_t n;
    int32_t top_level;       /* -1 when there are no records                     */
    int32_t num_records;
    int64_t top_size;
    double eps_lu, eps_fill, norm_estimate;
    int64_t nbytes;          /* H2Factorization.nbytes() accounting              */
    /* phase seconds: norm, extract, color, augment, project, partial_lu,
     * transition, top */
    double phase_seconds[8];
} h2f_factor_info;

typedef struct {
    int32_t level;
    int32_t num_clusters;
    int32_t num_batches;
    int32_t csp, ncolors, graph_degree, max_rank;
    int64_t total_size;      /* length of the level vector                       */
    int64_t up_size;         /* length of up_index                               */
    int64_t batch_entries;   /* sum of batch lengths                             */
    double time_s;
} h2f_level_info;

typedef struct {
    int32_t cluster, level;
    int32_t size;            /* s: q is s x s                                    */
    int32_t r;               /* redundant count; lu is r x r, piv r             */
    int32_t num_edges;
    int64_t offset;          /* offset in the level vector                       */
} h2f_cluster_info;

typedef struct {
    char name[32];
    int64_t launches;
    double seconds;          /* sum of CUDA-event durations of the launches      */
    double flops;            /* algorithmic FP64 flops (SURVEY.md §8d formulas)   */
    double bytes;            /* algorithmic HBM bytes                            */
} h2f_kernel_profile;

/* ---- context ------------------------------------------------------------ */
int h2f_init(int device, double arena_gb);   /* arena_gb <= 0: automatic      */
const char* h2f_last_error(void);
int h2f_stream(void** stream_out);           /* cudaStream_t of the library    */
int h2f_device_count(int* count);
int h2f_kernel_launches(int64_t* count);     /* kernels launched so far        */
int h2f_memory_stats(int64_t* arena_bytes, int64_t* in_use, int64_t* peak);

/* ---- measurement ----------------------------------------------------------- */
int h2f_profile_enable(int on);              /* CUDA events around every launch */
int h2f_profile_reset(void);
int h2f_profile_count(int32_t* nkernels);
int h2f_profile_get(int32_t kid, h2f_kernel_profile* out);   /* syncs the stream */
/* FP64 DMMA (m8n8k4) throughput probe: all SMs, iters MMAs per warp chain */
int h2f_bench_dmma(int64_t iters, double* tflops);

/* ---- per-cluster dense kernels (test / micro-benchmark hooks) -------------
 * Host pointers, row-major.  `path` selects the implementation the
 * factorization dispatches to by size, so each can be checked on any size:
 *   svd:        0 shared-memory Jacobi (one CTA), 1 block-cyclic multi-CTA,
 *               2 pairwise multi-CTA.  R is m x n; U receives the kept
 *               rows (kept x n, sorted by sigma desc); sweeps = -1 if unknown.
 *               augment_basis's SVD step, factorization.py:79-81
 *   qr_r:       0 shared-memory TSQR, 1 blocked Householder (cooperative
 *               panels).  Y is n x wf (QR of Y^T), R is min(n,wf) x n.
 *               factorization.py:78
 *   complement: 0 one CTA, 1 blocked Householder.  BT is kt x s (columns of
 *               b_aug), Q is s x s = [complement | b_aug].  factorization.py:88-99
 * ms = device time of the kernels. */
int h2f_dense_svd(const double* R, int32_t m, int32_t n, double thresh, int32_t path, double* U, int32_t* kept,
                  int32_t* sweeps, double* ms);
int h2f_dense_qr_r(const double* Y, int32_t n, int32_t wf, int32_t path, double* R, double* ms);
int h2f_dense_complement(const double* BT, int32_t s, int32_t kt, int32_t path, double* Q, double* ms);

/* ---- H2 matrix ----------------------------------------------------------- */
int h2f_matrix_create(const h2f_matrix_desc* desc, const double* vals, h2f_matrix* out);
/* the same operator with its values given block by block (HOST pointers,
 * element counts, offsets into the value array, offsets ascending): no
 * packed host copy is needed -- the library packs pinned chunks in parallel
 * and overlaps them with the upload (what a binding of the reference's
 * dict-of-blocks H2Matrix passes) */
int h2f_matrix_create_blocks(const h2f_matrix_desc* desc, int64_t num_blocks, const double* const* block_ptrs,
                             const int64_t* block_counts, const int64_t* block_offsets, h2f_matrix* out);
int h2f_matrix_destroy(h2f_matrix m);
int h2f_matrix_nbytes(h2f_matrix m, int64_t* bytes);
int h2f_matvec(h2f_matrix m, const double* x, double* y, int64_t nrhs);
int h2f_matvec_dev(h2f_matrix m, const double* x_dev, double* y_dev, int64_t nrhs);
int h2f_norm2(h2f_matrix m, const double* v0, int32_t iters, double* est);

/* ---- device construction --------------------------------
 * build_h2 + orthogonalize_recompress (h2core.py:128-269) on the device from
 * the points (tree order), the cluster tree with its boxes and the block
 * partition; the operator never exists on the host.  Pair lists as in
 * h2f_matrix_desc.  Tolerance contract, not bit-exact. */
typedef struct {
    int64_t n;
    int32_t dim;             /* 1..3                                             */
    int32_t depth, top_level;
    int32_t p0;              /* Chebyshev degree at the leaves: p = p0 + (depth - level) / 2 */
    int64_t num_nodes;
    const int64_t* parent;
    const int64_t* child_left, *child_right, *level, *begin, *end;
    const double* points;    /* n x dim, tree order                              */
    const double* box_lo, *box_hi;  /* num_nodes x dim                           */
    const int64_t* adm_pairs;   const int64_t* adm_ptr;
    const int64_t* inner_pairs; const int64_t* inner_ptr;
    const int64_t* dense_pairs; const int64_t* dense_ptr;
    int32_t family;          /* 0 exp_covariance, 1 laplace2d, 2 helmholtz3d (kernels.py:44-86) */
    int32_t pad_;
    double corr_length, kappa, diag_value, alpha_r;
    double eps;              /* recompression tolerance; <= 0: interpolation bases only */
} h2f_build_desc;

/* rank[num_nodes] receives the final ranks (-1: no basis); seconds[2] =
 * construction, compression wall seconds */
int h2f_matrix_build(const h2f_build_desc* desc, h2f_matrix* out, int64_t* rank, double* seconds);
/* absorb_low_rank (h2core.py:342-405): a new operator for A + W W^T (W is
 * n x r row-major, tree order), bases widened to reproduce W, then
 * recompressed at eps on the device; m is not modified.  seconds[2] =
 * update, recompression. */
int h2f_matrix_absorb_low_rank(h2f_matrix m, const double* w, int32_t r, double eps, h2f_matrix* out,
                               int64_t* rank, double* seconds);
/* offsets of a matrix's blocks in its value array, in the description's
 * order (leaf/transfer per node, coupling/dense per pair), and the values
 * themselves (nvals doubles) -- the export of a device-built operator */
int h2f_matrix_layout(h2f_matrix m, int64_t* leaf_basis_off, int64_t* transfer_off, int64_t* coupling_off,
                      int64_t* dense_off, int64_t* nvals);
int h2f_matrix_values(h2f_matrix m, double* vals);

/* ---- factorization ------------------------------------------------------- */
/* norm_estimate < 0: run h2f_norm2 with start vector v0 (n values, already
 * normalised, e.g. Philox(20240901) as in h2core.py:320-322). */
int h2f_factorize(h2f_matrix m, double eps_lu, double norm_estimate, const double* v0,
                  h2f_factor* out, h2f_status* status);
int h2f_factor_destroy(h2f_factor f);

/* ---- subtree-sharded factorization ---------------------------
 * The same factorization as h2f_factorize (factorization.py:204-271: same
 * colouring, batches, kept counts, fill decisions, pivots and bits), with the
 * work split over `world` processes, one per GPU.  Cluster c is owned by the
 * rank of its ancestor at the top level (contiguous subtrees); a block (a, b)
 * lives on the owners of a and of b.  Per batch (factorization.py:433-505):
 * owners augment / eliminate their clusters; Q~ and the eliminator panels
 * [G | -W] travel to the ranks that hold a neighbour block (all-to-all);
 * every holder projects and Schur-updates its own copy; kept counts, pivot
 * status and fill-candidate norms are max-reduced so every rank's host
 * scheduler makes the same decisions.  The dense top matrix is sum-reduced
 * (each block added by one rank) and factored on every rank, and the cluster
 * factors are broadcast at the end, so the returned factor is complete and
 * replicated: h2f_solve / h2f_refined_solve work on it unchanged.
 *
 * The collectives are callbacks (the host binds them to torch.distributed:
 * NCCL over NVLink on a GPU box, gloo for tests).  Each is called with the
 * library stream drained and must return with its output written (device
 * buffers: complete with respect to the library stream, i.e. synchronised). */
typedef struct {
    int32_t rank, world;
    void* user;
    /* element-wise max over ranks of n doubles, in place, HOST memory */
    int (*allreduce_max)(void* user, double* buf, int64_t n);
    /* element-wise sum over ranks of n doubles, in place, DEVICE memory */
    int (*allreduce_sum_dev)(void* user, double* buf, int64_t n);
    /* all-to-all of DEVICE bytes: send holds send_counts[g] bytes for rank g,
     * packed in rank order; recv receives recv_counts[g] bytes from rank g,
     * in rank order (counts are known to both sides) */
    int (*alltoallv_dev)(void* user, const void* send, const int64_t* send_counts, void* recv,
                         const int64_t* recv_counts);
    /* broadcast of `bytes` DEVICE bytes from rank root, in place */
    int (*broadcast_dev)(void* user, void* buf, int64_t bytes, int32_t root);
} h2f_comm;

/* shard statistics of the last sharded factorization in this process:
 * stats[0] clusters eliminated here, [1] clusters eliminated by all ranks,
 * [2] bytes sent by the all-to-alls, [3] collective calls, [4] Schur target
 * tiles computed here, [5] batches, [6] seconds inside the collectives
 * (host wall time), [7] factor-broadcast bytes */
int h2f_factorize_sharded(h2f_matrix m, double eps_lu, double norm_estimate, const double* v0,
                          const h2f_comm* comm, h2f_factor* out, h2f_status* status);
int h2f_shard_stats(double* stats);
/* owner rank of every node under a `world`-way split into contiguous
 * subtrees of the top level (-1 above it); parent/level as in
 * h2f_matrix_desc.  Host-only, no device work. */
int h2f_shard_owners(int64_t num_nodes, const int64_t* parent, const int64_t* level, int32_t top_level,
                     int32_t world, int32_t* owner);

int h2f_solve(h2f_factor f, const double* b, double* x, int64_t nrhs);
int h2f_solve_dev(h2f_factor f, const double* b_dev, double* x_dev, int64_t nrhs);
int h2f_refined_solve(h2f_matrix m, h2f_factor f, const double* b, double* x, int32_t steps);
int h2f_refined_solve_dev(h2f_matrix m, h2f_factor f, const double* b_dev, double* x_dev,
                          int32_t steps);
/* refined_solve for an n x nrhs block (row-major, like solve_multi): block
 * substitution + block matvec per step (extension: the reference's
 * refined_solve is single-vector, solve.py:63-77) */
int h2f_refined_solve_multi(h2f_matrix m, h2f_factor f, const double* b, double* x, int64_t nrhs,
                            int32_t steps);
int h2f_refined_solve_multi_dev(h2f_matrix m, h2f_factor f, const double* b_dev, double* x_dev,
                                int64_t nrhs, int32_t steps);

/* ---- factor introspection (lazy export to host) ---------------------------- */
int h2f_factor_info_get(h2f_factor f, h2f_factor_info* info);
int h2f_factor_level_info(h2f_factor f, int32_t rec, h2f_level_info* info);
/* clusters/offsets/sizes [num_clusters]; batch_ptr [num_batches+1];
 * batch_ids [batch_entries]; up_index [up_size]  (any may be NULL) */
int h2f_factor_level_arrays(h2f_factor f, int32_t rec, int64_t* clusters, int64_t* offsets,
                            int64_t* sizes, int64_t* batch_ptr, int64_t* batch_ids,
                            int64_t* up_index);
/* fill keys of record rec (factorization.py:502-505, 573-588): the canonical
 * pairs present when the level started, init_pairs [num_init][2], and every
 * block created by the level's batches in creation order, created
 * [num_created][3] = (batch index, a, b).  Call with NULL arrays for the
 * counts. */
int h2f_factor_level_fills(h2f_factor f, int32_t rec, int64_t* num_init, int64_t* init_pairs,
                           int64_t* num_created, int64_t* created);
int h2f_factor_cluster_info(h2f_factor f, int32_t rec, int32_t cluster, h2f_cluster_info* ci);
/* q: s*s row-major; lu: r*r row-major; piv: r (0-based LAPACK swaps);
 * edge_other/kind [num_edges] (kind 0 self, 1 full, 2 skel), edge_width [num_edges] */
int h2f_factor_cluster_arrays(h2f_factor f, int32_t rec, int32_t cluster, double* q,
                              double* lu, int32_t* piv, int64_t* edge_other,
                              int32_t* edge_kind, int64_t* edge_width);
/* edge matrix e: r x edge_width[e] row-major */
int h2f_factor_cluster_edge(h2f_factor f, int32_t rec, int32_t cluster, int32_t e, double* mat);
int h2f_factor_top(h2f_factor f, double* top_lu, int32_t* top_piv);

/* ---- factor import (serialization) -------------------------
 * Rebuilds a device factor from the arrays h2f_factor_level_arrays /
 * h2f_factor_cluster_arrays / h2f_factor_cluster_edge / h2f_factor_top
 * export (the reference has no factor format, factorization.py:130-193):
 * begin, then every record and every cluster of it, the top, end.  mw is the
 * cluster's r x (sum of edge widths) eliminator block, edges in order.  The
 * imported factor solves exactly like the exported one. */
int h2f_factor_import_begin(int64_t n, int32_t top_level, int32_t num_records, int64_t top_size, double eps_lu,
                            double eps_fill, double norm_estimate, h2f_factor* out);
int h2f_factor_import_record(h2f_factor f, int32_t rec, int32_t level, int32_t num_clusters,
                             const int64_t* clusters, const int64_t* offsets, const int64_t* sizes,
                             int32_t num_batches, const int64_t* batch_ptr, const int64_t* batch_ids,
                             int64_t up_size, const int64_t* up_index, int32_t csp, int32_t ncolors,
                             int32_t graph_degree, int32_t max_rank, double time_s);
int h2f_factor_import_cluster(h2f_factor f, int32_t rec, int32_t cluster, int32_t s, int32_t r, const double* q,
                              const double* lu, const int32_t* piv, int32_t num_edges, const int64_t* edge_other,
                              const int32_t* edge_kind, const int64_t* edge_width, const double* mw);
int h2f_factor_import_top(h2f_factor f, const double* top_lu, const int32_t* top_piv);
int h2f_factor_import_end(h2f_factor f);

/* ---- scheduling primitives (exposed for parity tests) ---------------------- */
/* greedy colouring in ascending id order of the graph given by canonical
 * pairs over `clusters`; colors_out[i] = colour of clusters[i]. */
int h2f_greedy_coloring(int64_t num_clusters, const int64_t* clusters, int64_t num_pairs,
                        const int64_t* pairs, int32_t* colors_out, int32_t* num_colors,
                        int32_t* max_degree);

/* ---- structure replay (parity diagnostics) ----------------------------------
 * Replaces this library's threshold decisions by those of another run (the
 * CPU oracle) for every later h2f_factorize until cleared:
 *   kept_rows    [nkept][3]     (level, cluster, kept)   factorization.py:80
 *   created_rows [ncreated][4]  (level, creating cluster, a, b) for every
 *                               fill block the run created  factorization.py:502-505
 * With identical decisions the batches, ranks and fill pattern coincide, so
 * the solutions differ only by floating-point rounding. */
int h2f_debug_replay_set(const int64_t* kept_rows, int64_t nkept, const int64_t* created_rows,
                         int64_t ncreated);
int h2f_debug_replay_clear(void);
/* stats[8]: kept counts taken from the table, of which differing from this
 * run's own count; fill decisions differing from this run's own norm test,
 * then those by |log10(own norm / tolerance)| in [0, .01), [.01, .1), [.1, .5),
 * [.5, 1), [1, inf) */
int h2f_debug_replay_stats(int64_t* stats);

#ifdef __cplusplus
}
#endif
#endif /* H2F_H */
