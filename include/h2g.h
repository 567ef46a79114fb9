/*
 * h2g — B200-native (sm_100a) H² factorize / solve, C ABI.
 *
 * Drop-in boundary for the hot path of the reference h2lu library
 * (arXiv 1703.06155, Ma & Jiao). The reference is header-only C++ on Eigen and
 * exposes no C ABI; each entry point below names the reference interface it
 * replaces (paths relative to /root/reference/proj). Plain pointers and sizes
 * only; complex data is interleaved complex128 (re, im), column-major — the
 * memory layout of Eigen::MatrixXcd / VectorXcd. Vectors are in TREE order,
 * like the reference library (solve.hpp:104-110; the CLI permutes at I/O,
 * tools/h2lu_cli.cpp:47-57).
 *
 * Every call returns H2G_OK (0) or an error code; details land in the
 * optional h2g_error* (and in h2g_last_error for the calling thread). The
 * codes mirror the reference exception types (include/h2lu/types.hpp:18-47).
 * There is no CPU fallback: without a CUDA device every compute call fails
 * with H2G_ERR_CUDA.
 */
#ifndef H2G_H
#define H2G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum h2g_status {
  H2G_OK = 0,
  H2G_ERR_INVALID_INPUT = 1,   /* InvalidInputError */
  H2G_ERR_SIZE_GUARD = 2,      /* SizeGuardError */
  H2G_ERR_NON_FINITE = 3,      /* NonFiniteError */
  H2G_ERR_SINGULAR_PIVOT = 4,  /* SingularPivotError{pivot_index, pivot_magnitude, cluster, level} */
  H2G_ERR_UNDEFINED_METRIC = 5,/* UndefinedMetricError */
  H2G_ERR_CUDA = 8,            /* no device / CUDA runtime failure / out of memory */
  H2G_ERR_INTERNAL = 9
};

typedef struct h2g_error {
  int32_t code;
  int32_t cluster;          /* heap id of the failing cluster; -1 = root block / none */
  int32_t level;            /* tree level; -1 = none */
  int32_t pad_;
  int64_t pivot_index;
  double pivot_magnitude;
  char msg[256];
} h2g_error;

/* Within-level elimination order. REFERENCE reproduces the reference's
 * ascending-heap-id order (factorization.hpp:618) exactly, executed as
 * dependency wavefronts; COLORED runs a greedy distance-1 colouring, one
 * colour per batch (a different, equally valid elimination order). */
enum h2g_schedule {
  H2G_SCHEDULE_REFERENCE = 0,
  H2G_SCHEDULE_COLORED = 1,
  H2G_SCHEDULE_SERIAL = 2,
  H2G_SCHEDULE_INTERIOR_FIRST = 3,
  H2G_SCHEDULE_SUBTREE = 4
};
/* SERIAL: the reference order one cluster per batch (the hooks' debug mode).
 * INTERIOR_FIRST: the north_star's 8-way subtree split as an order (SURVEY
 * §8e option 2): per level with >= 8 clusters, the clusters whose dense
 * neighbours all lie in their own level-3 subtree first, then the boundary
 * clusters (each group ascending id); coarser levels in reference order.
 * SUBTREE: the same split with the interior clusters grouped subtree by
 * subtree (subtree 0's interior wavefronts, then subtree 1's, ..., then the
 * boundary clusters): every interior batch belongs to one subtree, which is
 * what the multi-GPU partition (h2g_factorize_dist) hands to the ranks. */

/* Solve modes: solve.hpp:105 solve, :43 forward, :65 backward, :113
 * apply_inverse (alias of solve), plus the explicit-inverse application
 * (precomputed triangular inverses, applied as ZGEMMs). */
enum h2g_solve_mode {
  H2G_SOLVE = 0,
  H2G_FORWARD = 1,
  H2G_BACKWARD = 2,
  H2G_APPLY_INVERSE = 3,
  H2G_APPLY_INVERSE_EXPLICIT = 4
};

/* Kernel of the H² construction (kernel.hpp:13-61; the diagonal is widened to
 * complex for the BASELINE volume integral equation). Off-diagonal entries are
 * scale * f(r), f = 1/(4 pi r) (LAPLACE) or exp(-i k r)/(4 pi r) (HELMHOLTZ);
 * ZERO is the reference's zero custom kernel. */
enum h2g_kernel_kind { H2G_KERNEL_LAPLACE = 0, H2G_KERNEL_HELMHOLTZ = 1, H2G_KERNEL_ZERO = 2 };

typedef struct h2g_kernel_spec {
  int32_t kind;
  int32_t pad_;
  double wavenumber_re, wavenumber_im;
  double scale_re, scale_im;
  double diag_re, diag_im;
} h2g_kernel_spec;

/* Host description of an H2Matrix (h2_matrix.hpp:29-39) with its cluster
 * tree (cluster_tree.hpp:31-69, heap order, uniform depth) and block
 * partition (block_tree.hpp:21-97, pair lists sorted by (row, col)).
 * num_clusters = 2^(depth+1) - 1. */
typedef struct h2g_matrix_desc {
  int64_t n;
  int32_t depth;
  int32_t pad_;
  double eta;
  double eps_h2;
  const int64_t* cluster_begin;   /* [num_clusters] tree-order ranges */
  const int64_t* cluster_end;
  const int64_t* adm_offsets;     /* [depth+2]: admissible pairs of level l at [adm_offsets[l], adm_offsets[l+1]) */
  const int32_t* adm_pairs;       /* 2 * num_adm, (row, col) heap ids */
  const int64_t* split_offsets;   /* [depth+2] */
  const int32_t* split_pairs;
  int64_t num_leaf_pairs;
  const int32_t* leaf_pairs;      /* inadmissible leaf pairs (dense blocks) */
  /* numerical data, offsets in complex elements */
  const int64_t* basis_rows;      /* [num_clusters]: leaf size, or rank(c1)+rank(c2) */
  const int64_t* basis_rank;      /* [num_clusters]: columns */
  const int64_t* basis_offset;
  const double* basis_data;
  const int64_t* coupling_offset; /* [num_adm], level-major admissible order; rank_t x rank_s */
  const double* coupling_data;
  const int64_t* dense_offset;    /* [num_leaf_pairs]; |t| x |s| */
  const double* dense_data;
  /* optional (needed only by h2g_matrix_save / h2g_chain_save, which write
   * the tree like serialize.hpp:121-132): points n x 3 in TREE order, the
   * tree permutation (tree index -> original index) and the leaf size */
  const double* points_tree;
  const int64_t* perm;
  int64_t leafsize;
} h2g_matrix_desc;

typedef struct h2g_context h2g_context;
typedef struct h2g_matrix h2g_matrix;
typedef struct h2g_chain h2g_chain;

/* ---- runtime -------------------------------------------------------- */
int h2g_device_count(void);
int h2g_context_create(int device, h2g_context** out, h2g_error* err);
int h2g_context_destroy(h2g_context* ctx);
int h2g_last_error(h2g_error* err);
const char* h2g_version(void);

/* ---- input ------------------------------------------------------------ */
/* Replaces passing `const H2Matrix&` into factorize (factorization.hpp:600):
 * uploads a host H2Matrix; the device copy is immutable (factorize never
 * modifies its input, test_factorization.cpp:241-254). */
int h2g_matrix_upload(h2g_context* ctx, const h2g_matrix_desc* desc, h2g_matrix** out, h2g_error* err);
/* build_cluster_tree + build_block_tree (cluster_tree.hpp:71, block_tree.hpp:114)
 * on the host and build_h2 (h2_matrix.hpp:300) on the device. points: n x 3
 * row-major doubles in original order. */
int h2g_matrix_build(h2g_context* ctx, const double* points, int64_t n, int64_t leafsize, double eta,
                     const h2g_kernel_spec* kernel, double eps_h2, h2g_matrix** out, h2g_error* err);
int h2g_matrix_destroy(h2g_matrix* m);
/* sizes[8]: n, depth, num_clusters, num_adm, num_leaf_pairs, basis_elems, coupling_elems, dense_elems */
int h2g_matrix_sizes(const h2g_matrix* m, int64_t* sizes);
/* Download into caller arrays sized from h2g_matrix_sizes (same layout as the
 * desc; pair arrays optional). perm: tree index -> original index. */
int h2g_matrix_download(const h2g_matrix* m, int64_t* cluster_begin, int64_t* cluster_end, int64_t* perm,
                        int64_t* adm_offsets, int32_t* adm_pairs, int64_t* split_offsets, int32_t* split_pairs,
                        int32_t* leaf_pairs, int64_t* basis_rows, int64_t* basis_rank, int64_t* basis_offset,
                        double* basis_data, int64_t* coupling_offset, double* coupling_data, int64_t* dense_offset,
                        double* dense_data);
/* y = A x through the compressed operator (h2_matrix.hpp:80-137), host buffers, nrhs columns. */
int h2g_matvec(h2g_context* ctx, const h2g_matrix* m, const double* x, double* y, int32_t nrhs, h2g_error* err);

/* ---- H2LU v1 container (serialize.hpp:27-343) ----------------------------
 * The reference's on-disk format, byte compatible: little-endian, header
 * "H2LU" / version 1 / kind (1 matrix, 2 chain, 3 vector), column-major
 * complex128 matrices. Loads validate like the reference loaders and fail
 * with H2G_ERR_INVALID_INPUT (SerializationError) on malformed files. */
/* save_h2 (:186-196); the matrix must know its points (h2g_matrix_build, or
 * points_tree / perm / leafsize in the upload desc) */
int h2g_matrix_save(const h2g_matrix* m, const char* path, h2g_error* err);
/* load_h2 (:198-243): the block partition is recomputed from the stored
 * tree, the data uploaded to the device */
int h2g_matrix_load(h2g_context* ctx, const char* path, h2g_matrix** out, h2g_error* err);
/* save_chain (:245-284): the chain of a factorization of `source` (whose
 * tree the file carries) downloaded into the reference's record layout */
int h2g_chain_save(const h2g_chain* c, const h2g_matrix* source, const char* path, h2g_error* err);
/* load_chain (:286-343) into a device chain that h2g_solve can apply (the
 * records' elimination order is kept; triangular inverses formed on load) */
int h2g_chain_load(h2g_context* ctx, const char* path, h2g_chain** out, h2g_error* err);
/* The tree permutation (tree index -> original index) of the chain's matrix
 * (the CLI applies it to vectors on the way in and out, h2lu_cli.cpp:47-57) */
int h2g_chain_perm_tree(const h2g_chain* c, int64_t* perm);
/* save_vector / load_vector (:345-353), host only. load: call with
 * data == NULL to get the length in *n, then again with a buffer of 2 n doubles */
int h2g_vector_save(const char* path, const double* data, int64_t n, h2g_error* err);
int h2g_vector_load(const char* path, double* data, int64_t* n, h2g_error* err);

/* y[q] = sum_j Z(rows[q], j) x[j] with Z generated directly from the kernel
 * (the reference's assemble_block, kernel.hpp:64-102): the north_star's dense
 * sampled-row residual computed on the device. points: n x 3
 * row-major in TREE order; rows: tree indices; x: n x nrhs, y: nrows x nrhs,
 * column-major interleaved complex128, host buffers. */
int h2g_kernel_rows_matvec(h2g_context* ctx, const double* points_tree, int64_t n, const h2g_kernel_spec* kernel,
                           const int64_t* rows, int64_t nrows, const double* x, double* y, int32_t nrhs, h2g_error* err);

/* ---- hot path --------------------------------------------------------- */
/* factorize(A, eps_fill_in, stop_level_override) (factorization.hpp:600-653).
 * stop_level < 0 means "default" (l0). */
int h2g_factorize(h2g_context* ctx, const h2g_matrix* m, double eps_fill_in, int32_t stop_level, int32_t schedule,
                  h2g_chain** out, h2g_error* err);
int h2g_chain_destroy(h2g_chain* c);

/* ---- multi-GPU subtree partition (north_star, SURVEY §8e option 2) --------
 * One process per GPU, every rank holding the same matrix. Per level with
 * >= 8 clusters the 8 level-3 subtrees are dealt to the ranks (subtree s to
 * rank s * nranks / 8, nranks in {1, 2, 4, 8}); under the SUBTREE order the
 * eliminations of a subtree's interior clusters (all dense neighbours inside
 * the subtree) touch only blocks of that subtree, so every rank runs the
 * interior batches of its own subtrees and skips the others'. At the level's
 * interior / boundary border the ranks exchange what their interior phase
 * produced - final ranks, factor records, the updated dense blocks and the
 * fill-in blocks of their subtrees - through `exchange`, an all-gather with
 * per-rank sizes over NCCL (NVLink); the boundary clusters, the merge and the
 * coarse levels (< 8 clusters) then run replicated on every rank, so each
 * rank ends with the complete chain. The result is bitwise the single-GPU
 * factorization in the SUBTREE order.
 * exchange(user, buf, offsets, nranks): buf is a DEVICE buffer of
 * offsets[nranks] bytes; on entry this rank's part [offsets[rank],
 * offsets[rank + 1]) is filled, on return every part must hold the owning
 * rank's bytes on every rank (ncclBroadcast per part inside one group, or
 * torch.distributed.broadcast; all work complete on return). Nonzero return
 * = failure. */
typedef int (*h2g_exchange_fn)(void* user, void* device_buf, const int64_t* offsets, int32_t nranks);
typedef struct h2g_dist {
  int32_t rank, nranks;
  h2g_exchange_fn exchange;
  void* user;
} h2g_dist;
int h2g_factorize_dist(h2g_context* ctx, const h2g_matrix* m, double eps_fill_in, int32_t stop_level, const h2g_dist* dist, h2g_chain** out,
                       h2g_error* err);
/* Host-only view of the partition of one factorized level (no device needed):
 * counts[4] = clusters, batches, dense blocks, fill blocks of the level;
 * batch_of[nl] = batch of every cluster under the SUBTREE order;
 * part_batch[9]: batches [part_batch[s], part_batch[s+1]) are subtree s's
 * interior, batches from part_batch[8] on the boundary; dense_part[ndense] /
 * fill_part[nfill] = the subtree whose interior phase writes the block, -1 =
 * none (only the boundary phase does), -2 = two subtrees (never happens; the
 * CPU tests assert it); dense_rc[2 ndense] / fill_rc[2 nfill] = (row, column)
 * cluster (level-local ids) of every block. Output arrays may be null. */
int h2g_partition_plan(const h2g_matrix_desc* d, int32_t stop_level, int32_t level, int64_t* counts, int32_t* batch_of, int32_t* part_batch,
                       int32_t* dense_part, int32_t* fill_part, int32_t* dense_rc, int32_t* fill_rc, h2g_error* err);
/* Bytes this rank sent / all ranks exchanged and the seconds spent inside
 * `exchange` during the factorization that produced c (0 for h2g_factorize). */
int h2g_chain_dist_stats(const h2g_chain* c, double* out3);

/* solve / forward_substitute / backward_substitute / apply_inverse
 * (solve.hpp:43-113) with host buffers: b, x are n x nrhs column-major
 * complex128 (x may alias b: solve_in_place). */
int h2g_solve(h2g_chain* c, const double* b, double* x, int64_t n, int32_t nrhs, int32_t mode, h2g_error* err);
/* Same on device memory (x_dev holds b on entry), on the chain's stream. */
int h2g_solve_device(h2g_chain* c, double* x_dev, int64_t n, int32_t nrhs, int32_t mode, h2g_error* err);

/* ---- chain inspection (FactorChain fields, factorization.hpp:22-98) ---- */
/* info[6]: n, stop_level, root_size, num_levels, storage_bytes, schedule */
int h2g_chain_info(const h2g_chain* c, int64_t* info);
/* out[9]: level, nrecs, rank_sum_before, rank_sum_after, eliminated, ledger_blocks, chain_bytes, perm_len, active_after */
int h2g_chain_level(const h2g_chain* c, int32_t level_index, int64_t* out);
/* 10 per record, in the level's record order: cluster, level, pos, bsize,
 * eliminated, rank_before, rank_after, fill_targets, n_lbar, n_ubar */
int h2g_chain_records(const h2g_chain* c, int32_t level_index, int64_t* out);
int h2g_chain_perm(const h2g_chain* c, int32_t level_index, int64_t* src);
/* Qtilde (bsize^2), L11 and U11 (eliminated^2) of one record (record order). */
int h2g_chain_record_mats(const h2g_chain* c, int32_t level_index, int32_t record, double* qtilde, double* l11, double* u11);
/* Lbar / Ubar blocks of one record: positions and column-major data
 * concatenated in record order; sizes from h2g_chain_record_blocks_sizes. */
int h2g_chain_record_blocks_sizes(const h2g_chain* c, int32_t level_index, int32_t record, int64_t* sizes4);
int h2g_chain_record_blocks(const h2g_chain* c, int32_t level_index, int32_t record, int64_t* lbar_pos, int64_t* lbar_rows,
                            double* lbar_data, int64_t* ubar_pos, int64_t* ubar_cols, double* ubar_data);
int h2g_chain_root(const h2g_chain* c, double* root_l, double* root_u);
/* FNV-1a over the chain contents (determinism checks). */
uint64_t h2g_chain_hash(const h2g_chain* c);
/* Device time (ms, CUDA events on the chain's stream) of the last factorize
 * and the last solve, and the number of kernels each launched. */
int h2g_chain_timing(const h2g_chain* c, double* factor_ms, double* solve_ms, int64_t* factor_launches, int64_t* solve_launches);
/* Host symbolic plan of the factorization (CSR neighbour lists, fill
 * targets, Schur target lists, merge maps; it replaces the reference's
 * whole-map scans, factorization.hpp:268-293): its build time for this chain
 * (outside the device factor time of h2g_chain_timing) and whether it was
 * built (1) or reused from the matrix / context plan cache (0). */
/* k_schur per level (4 doubles each: level, executed flops, executed bytes,
 * event ms - the ms only after a profiled run); out may be null (count). */
int h2g_chain_schur_levels(const h2g_chain* c, int32_t* nlevels, double* out);
int h2g_chain_plan(const h2g_chain* c, double* plan_ms, int32_t* built);
/* Drop the context's structure-keyed plan cache (a later factorize of a new
 * matrix handle then builds its plan from scratch: a cold-structure run). */
int h2g_context_clear_plans(h2g_context* ctx);

/* ---- FactorizeHooks debug mode (factorization.hpp:588-593) -------------
 * factorize with callbacks after every cluster's basis update (step 0),
 * projection (step 2) and elimination (step 3) and after every level merge,
 * in the reference order: the run uses the SERIAL schedule and synchronises
 * at every step; inside a callback the h2g_state_* calls inspect the device
 * state (FactorState, :115-251). */
typedef struct h2g_state h2g_state;
typedef struct h2g_factorize_hooks {
  void* user;
  void (*after_basis_update)(void* user, const h2g_state* st, int32_t cluster);
  void (*after_projection)(void* user, const h2g_state* st, int32_t cluster);
  void (*after_elimination)(void* user, const h2g_state* st, int32_t cluster);
  void (*after_merge)(void* user, const h2g_state* st);
} h2g_factorize_hooks;
int h2g_factorize_hooked(h2g_context* ctx, const h2g_matrix* m, double eps_fill_in, int32_t stop_level, const h2g_factorize_hooks* hooks,
                         h2g_chain** out, h2g_error* err);
/* info[3]: level, active length, n */
int h2g_state_info(const h2g_state* st, int64_t* info);
/* out[5] for a cluster of the current level (heap id): pos, bsize, rank
 * (kfin once its basis was updated, else the level-entry rank), rotated
 * (projected) flag, eliminated count (0 until eliminated) */
int h2g_state_cluster(const h2g_state* st, int32_t cluster, int64_t* out);
/* Qtilde (bsize x bsize) of a cluster whose basis was updated */
int h2g_state_qtilde(const h2g_state* st, int32_t cluster, double* out);
/* FactorState::shadow() (:240-245): the dense n x n matrix the state
 * represents (painted on the host from the device blocks; SizeGuardError
 * above n = 4096) */
int h2g_state_shadow(const h2g_state* st, double* out);
/* inside after_merge: the permutation src of the level just merged */
int h2g_state_perm(const h2g_state* st, int64_t* src, int64_t* len);

/* Per-kernel-class device timing of factorize (CUDA events around every
 * launch on the context stream; off by default). Classes: 0 complement,
 * 1 step-0 projection/Gram GEMMs, 2 column norms, 3 eig pass 1, 4 head,
 * 5 panels, 6 Schur scatter, 7 level merge, 8 root LU, 9 other, 10 eigenvectors,
 * 11 retained-basis construction. */
int h2g_set_profiling(h2g_context* ctx, int32_t on);
/* out[4] for class cls: ms, launches, algorithmic flops, algorithmic bytes */
int h2g_chain_kernel_stats(const h2g_chain* c, int32_t cls, double* out);

/* Algorithmic work of the factorization (SURVEY §8d F_factor, from the shapes
 * executed) and of one nrhs=1 solve (bytes of chain + vector traffic):
 * out[4]: factor_flops, schur_flops, solve_bytes, schur_bytes */
int h2g_chain_work(const h2g_chain* c, double* out);

/* The Schur products k_schur actually executed: rows / columns of a dense
 * target whose cluster was eliminated in an earlier batch are exact zeros
 * (cleanup, factorization.hpp:431-439) and are skipped.
 * out[2]: flops, bytes (targets read + written once, panels once per target) */
int h2g_chain_schur_executed(const h2g_chain* c, double* out);

/* Seeded complex-normal vector: mt19937_64(seed) + std::normal_distribution,
 * cxd(g(rng), g(rng)) (tools/h2lu_cli.cpp:181-191), ORIGINAL order. */
void h2g_random_rhs(int64_t n, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif /* H2G_H */
