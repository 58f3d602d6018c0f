/*
 * libgraphblast_sm100a -- C ABI of the B200-native GraphBLAST backend.
 *
 * The reference (/root/reference/pkg/src/graphalg) is a Python package whose
 * operator layer is kernels.py.  Its "plugin boundary" is the set of module
 * functions listed in __init__.py:70-85.  This header is what those functions
 * bind to (via ctypes): each entry point below names the
 * reference function it replaces (file:line relative to pkg/src/graphalg/).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless its name ends in `_host`.
 *     Buffers are owned by the caller (PyTorch tensors on the Python side);
 *     the library only borrows them for the duration of the call, plus a
 *     grow-only scratch pool owned by the context.
 *   - Index arrays: offsets are int64, column/row/vector indices int32
 *     (vertex counts < 2^31).  Values are int64 or float64 (`dtype`).
 *   - A matrix orientation with `values == NULL` is "iso": every stored entry
 *     equals `iso_i64` / `iso_f64` (structure-only storage).
 *   - Calls are asynchronous on the context's stream except where they return
 *     a host scalar (documented per function).
 *   - Return codes: GB_OK or a negative gb_status; gb_last_error() has text.
 */
#ifndef GRAPHBLAST_H
#define GRAPHBLAST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gb_status;
enum {
  GB_OK = 0,
  GB_ERR_SHAPE = -1,       /* errors.py ShapeError       */
  GB_ERR_FORMAT = -2,      /* errors.py FormatError      */
  GB_ERR_INDEX = -3,       /* IndexError                 */
  GB_ERR_VALUE = -4,       /* ValueError                 */
  GB_ERR_UNSUPPORTED = -5, /* NotImplementedError        */
  GB_ERR_CUDA = -6,
  GB_ERR_OOM = -7,
  GB_ERR_ARG = -8
};

/* value dtypes */
enum { GB_I64 = 0, GB_F64 = 1 };

/* operator ids (algebra.py:146-158) */
enum {
  GB_OP_PLUS = 0,      /* builtin Plus: saturating when pairwise         */
  GB_OP_PLUS_WRAP = 1, /* a user op on np.add without the saturating fn  */
  GB_OP_MINUS = 2,
  GB_OP_TIMES = 3,
  GB_OP_MIN = 4,
  GB_OP_MAX = 5,
  GB_OP_LOR = 6,
  GB_OP_LAND = 7,
  GB_OP_LESS = 8,
  GB_OP_NE = 9,
  GB_OP_SECOND = 10,
  GB_OP_FIRST = 11
};

/* direction policy (containers.py:32-35) and chosen direction */
enum { GB_DIR_AUTO = 0, GB_DIR_PUSH = 1, GB_DIR_PULL = 2 };
/* pull partitioning (containers.py:43-46) */
enum { GB_PART_NONZERO = 0, GB_PART_ROW = 1 };

typedef struct gb_ctx gb_ctx;

/* One orientation of a sparse matrix: `n` rows of A (CSR) or of A^T (CSC). */
typedef struct gb_csr {
  int64_t nrows;
  int64_t ncols;
  int64_t nnz;
  const int64_t* offsets; /* [nrows+1] */
  const int32_t* indices; /* [nnz]     */
  const void* values;     /* [nnz] of dtype, or NULL when iso */
  int32_t dtype;
  int32_t pad_;
  int64_t iso_i64;
  double iso_f64;
  /* Identity of the arrays' CONTENTS, assigned by the owner (the Python
   * package stamps every orientation with a fresh id).  Per-matrix device
   * caches (BFS column samples, the instantiated BFS graph) are reused only
   * for an equal non-zero gen -- never on equal pointers alone, which the
   * caching allocator recycles.  0 = never cached. */
  uint64_t gen;
} gb_csr;

/* ----------------------------------------------------------------------------
 * context
 * --------------------------------------------------------------------------*/
gb_status gb_ctx_create(int device, gb_ctx** out);
gb_status gb_ctx_destroy(gb_ctx* ctx);
gb_status gb_ctx_set_stream(gb_ctx* ctx, void* cuda_stream);
/* Synchronize the stream; reports a device-detected error (GB_ERR_INDEX). */
gb_status gb_ctx_sync(gb_ctx* ctx);
const char* gb_last_error(gb_ctx* ctx);
int32_t gb_abi_version(void);
/* bytes currently held by the context's scratch pool */
int64_t gb_scratch_bytes(gb_ctx* ctx);
/* release the scratch pool (e.g. after a large graph build) */
gb_status gb_ctx_trim(gb_ctx* ctx);
/* number of kernels this context has launched (all entry points) */
int64_t gb_launch_count(gb_ctx* ctx);
/* Event timing of the fused drivers' main kernels: when on, each main kernel
 * launch records (kind, arg, ms); gb_prof_read returns and clears them. */
gb_status gb_ctx_set_profiling(gb_ctx* ctx, int32_t on);
int32_t gb_prof_read(gb_ctx* ctx, int32_t max, int32_t* kind_host, int64_t* arg_host,
                     float* ms_host);

/* ----------------------------------------------------------------------------
 * element-wise utilities of the operator layer (gb_util.cu); dtype codes
 * GB_I64 = 0, GB_F64 = 1 and GB_I32 = 2 (index vectors).  Asynchronous unless
 * they return a host count.
 * --------------------------------------------------------------------------*/
enum { GB_I32 = 2 };
/* out[i] = i */
gb_status gb_iota(gb_ctx* ctx, int32_t code, int64_t n, void* out);
/* numpy astype between int32 / int64 / float64 (float -> int truncates) */
gb_status gb_cast(gb_ctx* ctx, int64_t n, int32_t in_code, const void* in, int32_t out_code,
                  void* out);
/* keep entries i with flags[i] != 0, in order: out_idx (idx[i], or i when idx
 * is NULL; NULL = not wanted) and out_vals (vals of dtype; NULL = not wanted);
 * *count_host = kept.  Synchronizes. */
gb_status gb_select_flags(gb_ctx* ctx, int64_t k, const int32_t* flags, const int32_t* idx,
                          const void* vals, int32_t dtype, int32_t* out_idx, void* out_vals,
                          int64_t* count_host);
/* out[i] = src[tgt[i]] with int32 targets (dtype GB_I64 / GB_F64 / GB_I32) */
gb_status gb_gather_i32(gb_ctx* ctx, int32_t dtype, int64_t k, const int32_t* tgt,
                        const void* src, void* out);
/* preprocess of weighted edges (io.py:220-249 before the dedup): drop
 * src == dst, append the mirror when `mirror`; int64 outputs sized 2m;
 * *count_host = edges written.  Synchronizes. */
gb_status gb_edges_clean(gb_ctx* ctx, int64_t m, const int32_t* src, const int32_t* dst,
                         const double* w, int32_t mirror, int64_t* out_src, int64_t* out_dst,
                         double* out_w, int64_t* count_host);
/* vals[p] = alpha / (row length) for every entry of row r (algorithms.py:122-129) */
gb_status gb_scale_rows(gb_ctx* ctx, int64_t n, const int64_t* offsets, double alpha,
                        double* vals);
/* algorithms.py:206-218: vertices ranked by a stable ascending sort of their
 * row length; the entries (rank[i], rank[j], a_ij) with rank[i] > rank[j]
 * (outputs sized nnz; *count_host = kept).  Synchronizes. */
gb_status gb_lower_by_rank(gb_ctx* ctx, const gb_csr* a, int64_t* out_rows, int64_t* out_cols,
                           void* out_vals, int64_t* count_host);

/* ----------------------------------------------------------------------------
 * matrix construction   (containers.py:307-364, io.py:220-315)
 * --------------------------------------------------------------------------*/

/* SparseMatrix.from_tuples (containers.py:307-345): stable sort by (row, col),
 * fold duplicates with `dedup_op`, emit CSR.  Outputs are sized nnz_in; the
 * kept count is written to *nnz_out_host (synchronizes).  Returns
 * GB_ERR_INDEX when a coordinate is out of range. */
gb_status gb_build_csr(gb_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz_in,
                       const int64_t* rows, const int64_t* cols, const void* vals,
                       int32_t dtype, int32_t dedup_op, int64_t* out_offsets,
                       int32_t* out_indices, void* out_vals, int64_t* nnz_out_host);

/* SparseMatrix._build_csc (containers.py:357-364): the other orientation,
 * stable in row order.  `vals`/`out_vals` may be NULL (iso). */
gb_status gb_transpose_csr(gb_ctx* ctx, const gb_csr* a, int64_t* out_offsets,
                           int32_t* out_indices, void* out_vals);

/* Traversal layout (no reference counterpart; an internal layout of the
 * matrix the reference stores as plain CSR/CSC, containers.py:276-364).
 * gb_degree_order: order[r] = the vertex with the r-th largest row length
 * (ties by ascending id), rank = its inverse.  Synchronizes. */
gb_status gb_degree_order(gb_ctx* ctx, int64_t n, const int64_t* offsets, int32_t* order,
                          int32_t* rank);

/* The relabelled TRANSPOSE of a square orientation: out = P A^T P^T with
 * new id rank[i] for vertex i, every output row sorted ascending; values
 * (if any) carried along.  For a symmetric matrix this is P A P^T.
 * Outputs: offsets[n+1], indices[nnz], vals[nnz].  Synchronizes. */
gb_status gb_csr_relabel_t(gb_ctx* ctx, const gb_csr* a, const int32_t* order,
                           const int32_t* rank, int64_t* out_offsets, int32_t* out_indices,
                           void* out_vals);

/* 1 when the two orientations hold identical arrays (A == A^T);
 * algorithms.py:41-45 _require_symmetric.  Synchronizes. */
gb_status gb_csr_equal(gb_ctx* ctx, const gb_csr* a, const gb_csr* b, int32_t* equal_host);

/* 1 when every stored value equals the first one (iso detection). Sync. */
gb_status gb_values_iso(gb_ctx* ctx, int64_t n, const void* vals, int32_t dtype,
                        int32_t* iso_host);

/* min / max of a value array (sssp weight check, algorithms.py:92). Sync. */
gb_status gb_values_minmax(gb_ctx* ctx, int64_t n, const void* vals, int32_t dtype,
                           double* min_host, double* max_host);

/* generate_rmat (io.py:275-295): edge e, level l uses SplitMix64 draw
 * e*scale+l; thresholds are the caller's double sums a, a+b, a+b+c. */
gb_status gb_rmat_generate(gb_ctx* ctx, int32_t scale, int64_t nedges, uint64_t seed,
                           double a, double t_ab, double t_abc, int32_t* src, int32_t* dst);

/* preprocess + edges_to_matrix (io.py:220-249, 298-315) for pattern edges:
 * drop self loops, optionally mirror, sort by (src,dst), dedup -> CSR.
 * out_indices must hold 2*nedges (mirrored) entries. Synchronizes. */
gb_status gb_edges_to_csr(gb_ctx* ctx, int64_t n, int64_t nedges, const int32_t* src,
                          const int32_t* dst, int32_t make_undirected, int64_t* out_offsets,
                          int32_t* out_indices, int64_t* nnz_out_host);

/* assign_weights (io.py:252-272): one integer weight in [low, high] per
 * unordered pair, drawn from SplitMix64(seed) in order of the pair's first
 * appearance in the (src, dst) list; both directions get the same value.
 * Writes float64 weights in list order. Synchronizes. */
gb_status gb_assign_weights(gb_ctx* ctx, int64_t n, int64_t nedges, const int32_t* src,
                            const int32_t* dst, uint64_t seed, int64_t low, int64_t high,
                            double* out_weights);

/* row id of every stored entry of a CSR (extract_tuples, containers.py:404-407) */
gb_status gb_csr_row_ids(gb_ctx* ctx, int64_t nrows, int64_t nnz, const int64_t* offsets,
                         int32_t* out_rows);

/* ----------------------------------------------------------------------------
 * vectors and masks   (containers.py:175-252, kernels.py:67-84)
 * --------------------------------------------------------------------------*/

/* Vector.nvals_for on dense storage: count of values != zero. Synchronizes. */
gb_status gb_count_ne(gb_ctx* ctx, int64_t n, const void* vals, int32_t dtype,
                      const void* zero_host, int64_t* count_host);

/* to_sparse (containers.py:242-252): keep entries != zero (dense input of n
 * values when k < 0; sparse input of k entries with indices idx otherwise).  Writes the kept count
 * to *count_host (synchronizes). */
gb_status gb_compact(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx, const void* vals,
                     int32_t dtype, const void* zero_host, int32_t* out_idx, void* out_vals,
                     int64_t* count_host);

/* to_dense (containers.py:230-240): fill `zero`, scatter k entries. */
gb_status gb_scatter_dense(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx,
                           const void* vals, int32_t dtype, const void* zero_host,
                           void* out_vals);

/* _effective_mask (kernels.py:67-84) as a bitmap of ceil(n/32) words: a stored
 * entry allows its position iff its value != 0; complement flips.  k < 0: a
 * dense mask of n values; otherwise k sparse entries (idx, vals). */
gb_status gb_mask_bitmap(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx,
                         const void* vals, int32_t dtype, int32_t complement, uint32_t* out);

/* number of set bits in the first n bits of a bitmap. Synchronizes. */
gb_status gb_bitmap_count(gb_ctx* ctx, int64_t n, const uint32_t* bitmap, int64_t* count_host);

/* bitmap of rows with at least one stored entry */
gb_status gb_nonempty_rows(gb_ctx* ctx, int64_t n, const int64_t* offsets, uint32_t* out);

/* ----------------------------------------------------------------------------
 * matrix-vector   (kernels.py:108-322)
 * --------------------------------------------------------------------------*/

/* decide_direction (kernels.py:108-126): pure host function, exported so the
 * rule has exactly one implementation shared by every fused driver. */
int32_t gb_decide_direction(int64_t nnz, int64_t nrows, int64_t nnz_u, double switch_ratio,
                            int32_t policy, int64_t* estimate_out);

/* Edge-balanced work plan of one orientation (the nonzero split,
 * kernels.py:133-150): the non-empty rows (nz_rows[R], their offsets
 * nz_off[R+1]) and, for every 512-entry tile, the plan row holding its first
 * entry (tile_first[nnz/512 + 2]).  Built once per matrix orientation by the
 * caller (gb_row_plan_build) and passed to the pull kernels; NULL = build it
 * per call. */
typedef struct gb_row_plan {
  int64_t nrows_nz;
  const int32_t* nz_rows;
  const int64_t* nz_off;
  const int32_t* tile_first;
} gb_row_plan;

/* fill caller buffers nz_rows[nrows], nz_off[nrows+1], tile_first[nnz/512+2];
 * *nrows_nz_host = R. Synchronizes. */
gb_status gb_row_plan_build(gb_ctx* ctx, const gb_csr* a, int32_t* nz_rows, int64_t* nz_off,
                            int32_t* tile_first, int64_t* nrows_nz_host);

/* Pull SpMV (kernels.py:153-229): for every row i of `a` allowed by `mask`
 * (NULL = all), out[i] = fold over stored (i,j) with u[j] != identity of
 * mult(a_ij, u[j]); rows without contributions get the identity.  `u` and
 * `out` are dense of dtype T = a->dtype.  counters (may be NULL) accumulates
 * {entries read, multiplies, adds} exactly as the reference counts them. */
gb_status gb_mxv_pull(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                      const gb_row_plan* plan, const void* u, const uint32_t* mask,
                      int32_t early_exit, int32_t partition, void* out, int64_t* counters);

/* Row bins of an orientation (gb_mv_binned.cu), built once per matrix:
 * short rows (1..16 entries), medium rows (17..512) and the 512-entry tiles
 * of the long rows, cut at absolute multiples of 512.  The row split of
 * kernels.py:133-150 (Partition.ROW_SPLIT) made row-granular so the mask is
 * tested per row before any entry is read. */
typedef struct gb_bin_plan {
  int64_t n_short, n_mid, n_long_tiles;
  const int32_t* short_rows;  /* [n_short] */
  const int32_t* mid_rows;    /* [n_mid] */
  const int32_t* tile_row;    /* [n_long_tiles] */
  const int64_t* tile_beg;    /* [n_long_tiles] first entry */
  const int64_t* tile_end;    /* [n_long_tiles] one past the last entry */
} gb_bin_plan;

/* counts_host[3] = {n_short, n_mid, n_long_tiles}.  Synchronizes. */
gb_status gb_bin_plan_counts(gb_ctx* ctx, const gb_csr* a, int64_t* counts_host);

/* fill the caller's arrays of `plan` (sizes from gb_bin_plan_counts).  Sync. */
gb_status gb_bin_plan_fill(gb_ctx* ctx, const gb_csr* a, gb_bin_plan* plan);

/* Pull SpMV over the row bins (same contract as gb_mxv_pull without early
 * exit; commutative folds).  Rows are mask-tested before their entries are
 * read.  Asynchronous. */
gb_status gb_mxv_pull_binned(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                             const gb_bin_plan* plan, const void* u, const uint32_t* mask,
                             void* out, int64_t* counters);

/* The binned pull over COLUMN STRIPES of a matrix (stripes[k]: the same rows,
 * the entries with columns in stripe k -- gb_csr_column_block -- and
 * plans[k] its row bins): the stripes are multiplied one after the other and
 * folded into `out`, so each stripe's slice of u stays L2-resident while it
 * is gathered.  Same contract and counters as gb_mxv_pull_binned.
 * Asynchronous. */
gb_status gb_mxv_pull_striped(gb_ctx* ctx, int32_t add_op, int32_t mult_op, int32_t nstripes,
                              const gb_csr* stripes, const gb_bin_plan* plans, const void* u,
                              const uint32_t* mask, void* out, int64_t* counters);

/* gb_mxv_pull on the degree-ordered layout of the same matrix (same results,
 * kernels.py:153-229; commutative folds without early exit).  `a` is the
 * relabelled orientation P A P^T (gb_csr_relabel_t), `plan` its row plan with
 * nz_rows mapped back to ORIGINAL row ids (gb_row_plan_remap), order[r] the
 * original id of new id r, reach = 1 + the largest column id of `a`.  u, mask
 * and out use the original ids.  Asynchronous. */
gb_status gb_mxv_pull_ordered(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                              const gb_row_plan* plan, const int32_t* order, int64_t reach,
                              const void* u, const uint32_t* mask, void* out, int64_t* counters);

/* out[i] = map[ids[i]] for i < count (row plans of a relabelled matrix in the
 * original ids).  Asynchronous. */
gb_status gb_row_plan_remap(gb_ctx* ctx, int64_t count, const int32_t* ids, const int32_t* map,
                            int32_t* out);

/* largest entry of idx[count] (-1 when empty).  Synchronizes. */
gb_status gb_index_max(gb_ctx* ctx, int64_t count, const int32_t* idx, int64_t* max_host);

/* Push SpMSpV (kernels.py:242-280): expand the columns named by the sparse u
 * (k entries), multiply, fold per output row, drop identity results, apply
 * the mask.  `a` is the column orientation (rows of `a` = the columns walked).
 * Output is sorted by index; count written to *count_host (synchronizes). */
gb_status gb_mxv_push(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                      int64_t out_size, int64_t k, const int32_t* u_idx, const void* u_vals,
                      const uint32_t* mask, int32_t* out_idx, void* out_vals,
                      int64_t* count_host, int64_t* counters);

/* ----------------------------------------------------------------------------
 * masked matrix-matrix   (kernels.py:329-391)
 * --------------------------------------------------------------------------*/

/* mxm_masked: for every stored mask entry (i, j) whose value is non-zero,
 * C(i,j) = fold over k in A(i,:) & B(:,j) of mult(A(i,k), B(k,j)).  `b` is the
 * orientation whose row j is column j of B.  Entries with no match are kept
 * (value = identity) only when the identity is non-zero.  Output is CSR in
 * mask order (out_offsets: m->nrows+1; indices/values sized m->nnz).
 * *nnz_host receives the kept count (synchronizes). */
gb_status gb_mxm_masked(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                        const gb_csr* b, const gb_csr* m, int64_t* out_offsets,
                        int32_t* out_indices, void* out_vals, int64_t* nnz_host,
                        int64_t* counters);

/* 1 when some row i stores column i (triangle_count check, algorithms.py:229-231). */
gb_status gb_has_diagonal(gb_ctx* ctx, const gb_csr* a, int32_t* found_host);

/* ----------------------------------------------------------------------------
 * element-wise, assign, gather, apply, reduce   (kernels.py:422-665)
 * --------------------------------------------------------------------------*/

/* out[i] = mask[i] ? op(a[i], b[i] or *b_scalar_host) : *zero_host (swap: op(b, a)). */
gb_status gb_ewise_dense(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t n, const void* a,
                         const void* b, const void* b_scalar_host, int32_t swap,
                         const uint32_t* mask, const void* zero_host, void* out);

/* ewise_add sparse+sparse (kernels.py:454-466): union of two sorted index
 * sets; shared indices fold op(a, b), single entries fold alone (logical ops
 * give 0/1).  Output sized ka+kb; *count_host = union size (synchronizes). */
gb_status gb_union_sparse(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t ka, const int32_t* ia,
                          const void* va, int64_t kb, const int32_t* ib, const void* vb,
                          int32_t* out_idx, void* out_vals, int64_t* count_host);

/* ewise_mult sparse*sparse: op(a, b) on shared indices, then the mask. */
gb_status gb_intersect_sparse(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t ka,
                              const int32_t* ia, const void* va, int64_t kb, const int32_t* ib,
                              const void* vb, const uint32_t* mask, int32_t* out_idx,
                              void* out_vals, int64_t* count_host);

/* ewise_mult sparse*dense: out[i] = op(vals[i], dense[idx[i]]) (swap: op(dense, vals)). */
gb_status gb_gather_pair(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t k, const int32_t* idx,
                         const void* vals, const void* dense, int32_t swap, void* out);

/* _mask_sparse_result (kernels.py:414-419): keep sparse entries the mask allows. */
gb_status gb_filter_mask(gb_ctx* ctx, int32_t dtype, int64_t k, const int32_t* idx,
                         const void* vals, const uint32_t* mask, int32_t* out_idx, void* out_vals,
                         int64_t* count_host);

/* assign (kernels.py:519-535): w[i] = value where the mask allows (NULL = all). */
gb_status gb_assign_scalar(gb_ctx* ctx, int32_t dtype, int64_t n, void* w,
                           const void* value_host, const uint32_t* mask);

/* 1 when some t[i] is outside [0, n). Synchronizes. */
gb_status gb_check_bounds(gb_ctx* ctx, int64_t k, const int64_t* t, int64_t n, int32_t* bad_host);

/* assign_scatter (kernels.py:538-583): w[tgt[i]] = min over colliding i of
 * vals[i] (overwrite), targets filtered by the mask; GB_ERR_INDEX when a
 * target is out of range. */
gb_status gb_scatter_min(gb_ctx* ctx, int32_t dtype, int64_t n, void* w, int64_t k,
                         const int64_t* tgt, const void* vals, const uint32_t* mask);

/* extract_gather (kernels.py:586-619), dense source: out[i] = src[tgt[i]]. */
gb_status gb_gather(gb_ctx* ctx, int32_t dtype, int64_t k, const int64_t* tgt, int64_t usize,
                    const void* src, void* out);

/* extract_gather with a sparse source: present[i] = tgt[i] is stored in u. */
gb_status gb_gather_sparse(gb_ctx* ctx, int32_t dtype, int64_t k, const int64_t* tgt,
                           int64_t usize, int64_t uk, const int32_t* uidx, const void* uval,
                           int32_t* present, void* out);

/* apply (kernels.py:622-639) for affine maps: out = in * scale + shift. */
gb_status gb_apply_affine(gb_ctx* ctx, int32_t dtype, int64_t n, const void* in,
                          const void* scale_host, const void* shift_host, void* out);

/* reduce / reduce_scalar_matrix (kernels.py:642-647, 663-665): fold values
 * (skipping those equal to *zero_host when given) into *out_host; the number
 * of folded values goes to *count_host.  Synchronizes. */
gb_status gb_reduce(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t n, const void* vals,
                    const void* zero_host, void* out_host, int64_t* count_host);

/* reduce_rows (kernels.py:650-660): per-row fold, identity for empty rows. */
gb_status gb_reduce_rows(gb_ctx* ctx, int32_t op, const gb_csr* a, void* out);

/* ----------------------------------------------------------------------------
 * fused algorithms   (algorithms.py)
 * --------------------------------------------------------------------------*/

/* ---- 1D-partitioned BFS (multi-GPU; one rank's steps, see distributed.py).
 * Rank p owns vertices [lo, hi); lo is a multiple of 1024.  Buffers levels
 * (int64[n]), vbm/vprev/fbm/xbm (uint32[ceil(n/32)]) and F (int32[n]) are
 * global-sized and replicated; only xbm is exchanged (all-reduce SUM: the
 * ranks' owned words are disjoint). */
gb_status gb_bfs_dist_init(gb_ctx* ctx, int64_t n, int64_t source, int64_t* levels,
                           uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int32_t* F);
/* push over the rank's column block (all n rows of A, columns in [lo,hi)) */
gb_status gb_bfs_dist_push(gb_ctx* ctx, const gb_csr* colblock, int64_t K, const int32_t* F,
                           uint32_t* vbm);
/* xbm = owned words of vbm & ~vprev, zero elsewhere (after a push) */
gb_status gb_bfs_dist_collect(gb_ctx* ctx, int64_t n, int64_t lo, int64_t hi,
                              const uint32_t* vbm, const uint32_t* vprev, uint32_t* xbm);
/* pull over the rank's row block (rows lo..hi-1 of A^T); owned new bits -> xbm */
gb_status gb_bfs_dist_pull(gb_ctx* ctx, const gb_csr* rowblock, int64_t lo, int64_t hi,
                           const uint32_t* nonempty_block, int64_t n, int64_t depth,
                           uint32_t* vbm, uint32_t* vprev, const uint32_t* fbm, uint32_t* xbm,
                           int64_t* levels);
/* apply the exchanged new-frontier bitmap xbm: stamp `depth`, rebuild F and
 * fbm; *K_host = global frontier size (synchronizes), or K_host = NULL when
 * the caller knows it from the exchange (asynchronous) */
gb_status gb_bfs_dist_apply(gb_ctx* ctx, int64_t n, int64_t depth, const uint32_t* xbm,
                            uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int64_t* levels,
                            int32_t* F, int64_t* K_host);

/* Frontier exchange of the 1D-partitioned BFS (distributed.FrontierExchange).
 * owned: list this rank's new vertices (owned words of xbm) into ids and
 *   their count into *count_dev (device int64).  Asynchronous.
 * pack_words: out[i] = owned word i of xbm, zero padded to wmax words.
 * unpack_words: xbm[wb[p] + i] = gathered[p*wmax + i] for the P slices
 *   (wb: device int64[P+1] word bounds).
 * set_ids: xbm = the bits of every gathered id (rank p: gathered[p*kmax ..
 *   + counts[p]), counts a device int64[P]). */
gb_status gb_bfs_dist_owned(gb_ctx* ctx, int64_t lo, int64_t hi, const uint32_t* xbm,
                            int32_t* ids, int64_t* count_dev);
gb_status gb_bfs_dist_pack_words(gb_ctx* ctx, int64_t lo, int64_t hi, int64_t wmax,
                                 const uint32_t* xbm, uint32_t* out);
gb_status gb_bfs_dist_unpack_words(gb_ctx* ctx, int32_t P, int64_t wmax, const int64_t* wb,
                                   const uint32_t* gathered, uint32_t* xbm);
gb_status gb_bfs_dist_set_ids(gb_ctx* ctx, int64_t n, int32_t P, int64_t kmax,
                              const int64_t* counts, const int32_t* gathered, uint32_t* xbm);
/* clear the levels of the K vertices in F (loop cap reached, algorithms.py:69) */
gb_status gb_bfs_dist_unstamp(gb_ctx* ctx, int64_t K, const int32_t* F, int64_t* levels);
/* Device-resident partitioned levels (distributed.bfs_partitioned_device):
 * the host never reads K.  `state` is an int64[16] device block (frontier
 * size, depth, iteration, mode, done, the loop cap), `log` the raw decision
 * log int64[1 + 3*max_iters] (count, then (dir, K, estimate) per iteration,
 * like gb_bfs_ordered_async).  Per level: gb_bfs_dist_dev_level (the
 * reference rule on the device -- kernels.py:108-126 -- then the push over
 * the column block or the pull over the row block, whichever the state's mode
 * says, each returning at once otherwise), the dense word exchange
 * (gb_bfs_dist_pack_words / allgather / gb_bfs_dist_unpack_words), then
 * gb_bfs_dist_dev_apply (stamp, new K, loop exit and cap).  Levels enqueued
 * after `done` are no-ops.  prefix_cut (rows sorted by column, e.g. the
 * degree-ordered layout): the push skips each list's entries below the dense
 * visited prefix, as the single-GPU push does.  Replaces the per-level host loop of
 * algorithms.py:48-77 on a 1D partition. */
gb_status gb_bfs_dist_dev_init(gb_ctx* ctx, int64_t* state, int64_t* log, int64_t n, int64_t nnz,
                               int64_t source, int64_t max_iters, double ratio, int32_t policy,
                               int64_t* levels, uint32_t* vbm, uint32_t* vprev, uint32_t* fbm,
                               int32_t* F);
gb_status gb_bfs_dist_dev_level(gb_ctx* ctx, int64_t* state, int64_t* log,
                                const gb_csr* rowblock, const gb_csr* colblock, int64_t lo,
                                int64_t hi, const uint32_t* nonempty_block, int64_t n,
                                uint32_t* vbm, uint32_t* vprev, const uint32_t* fbm,
                                uint32_t* xbm, int64_t* levels, const int32_t* F,
                                int32_t prefix_cut);
gb_status gb_bfs_dist_dev_apply(gb_ctx* ctx, int64_t* state, int64_t n, const uint32_t* xbm,
                                uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int64_t* levels,
                                int32_t* F);
/* entries of every row of `a` whose column lies in [lo, hi): CSR with the
 * same row count (out_offsets: nrows+1); pass out_indices = NULL to size. */
gb_status gb_csr_column_block(gb_ctx* ctx, const gb_csr* a, int64_t lo, int64_t hi,
                              int64_t* out_offsets, int32_t* out_indices, int64_t* nnz_host);

/* ---- 1D-partitioned connected components (one rank's FastSV steps).
 * int32 label vectors parent/mn/gp/gpp/pp/hook/prop are global-sized and
 * replicated; `prop` is exchanged with an all-reduce MIN after
 * gb_cc_dist_propose.  rowblock / colblock as for the partitioned BFS. */
gb_status gb_cc_dist_init(gb_ctx* ctx, int64_t n, int32_t* parent, int32_t* mn, int32_t* gp,
                          int32_t* gpp);
gb_status gb_cc_dist_hook(gb_ctx* ctx, int32_t pull, const gb_csr* rowblock,
                          const gb_csr* colblock, int64_t lo, int64_t hi, int64_t n,
                          const int32_t* gp, const int32_t* parent, int32_t* pp, int32_t* hook);
gb_status gb_cc_dist_propose(gb_ctx* ctx, int64_t n, int64_t lo, int64_t hi, const int32_t* hook,
                             int32_t* mn, const int32_t* pp, int32_t* prop);
gb_status gb_cc_dist_shortcut(gb_ctx* ctx, int64_t n, const int32_t* pp, const int32_t* prop,
                              int32_t* parent, int32_t* gp, int32_t* gpp, int32_t sparsify,
                              int64_t* changed_host, int64_t* live_host);
/* int32 -> int64 widening of a label vector (the API returns int64 labels) */
gb_status gb_widen_i32(gb_ctx* ctx, int64_t n, const int32_t* in, int64_t* out);

/* Per-iteration host callback of the fused drivers (the sssp on_iteration hook). */
typedef void (*gb_iter_cb)(int64_t iteration, void* user);

/* Engine of the SSSP / PageRank / CC iteration loops: 0 = one CUDA-graph
 * launch per call (WHILE conditional node, device-side direction decisions
 * and exit tests; the default), 1 = the host-driven loop (one synchronisation
 * per iteration; also used under per-kernel profiling and for an SSSP
 * on_iteration callback).  Returns the previous engine. */
int32_t gb_loop_engine(int32_t engine);

/* sssp (algorithms.py:80-119): dist (float64[n]) receives the distances
 * (+inf unreached).  Weights must be positive (checked by the caller);
 * min_weight is a lower bound on them (their minimum, which the caller's
 * check computes; 0 is always valid) -- the pull skips rows no candidate can
 * improve. */
gb_status gb_sssp(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull, int64_t source,
                  int64_t max_iters, double switch_ratio, int32_t policy, double min_weight,
                  double* dist,
                  int32_t* log_dir_host, int64_t* log_nvals_host, int64_t* log_est_host,
                  int64_t* iters_host, gb_iter_cb cb, void* user);

/* pagerank (algorithms.py:132-162): `pull` is the in-edge orientation (CSC of
 * A), out_offsets the CSR offsets of A (out-degrees).  err_host[i] = L2 step
 * of iteration i. */
gb_status gb_pagerank(gb_ctx* ctx, const gb_csr* pull, const int64_t* out_offsets, double alpha,
                      double eps, int64_t max_iters, double switch_ratio, int32_t policy,
                      double* ranks, int32_t* log_dir_host, int64_t* log_nvals_host,
                      int64_t* log_est_host, double* err_host, int64_t* iters_host);

/* connected_components (algorithms.py:165-203): parent (int64[n]) receives
 * the minimum vertex id of each component.  rows = CSR, cols = CSC. */
gb_status gb_cc(gb_ctx* ctx, const gb_csr* rows, const gb_csr* cols, int64_t max_iters,
                double switch_ratio, int32_t policy, int32_t sparsify, int64_t* parent,
                int32_t* log_dir_host, int64_t* log_nvals_host, int64_t* log_est_host,
                int64_t* iters_host);

/* triangle_count (algorithms.py:221-240) of a symmetric pattern matrix. Sync. */
gb_status gb_tc(gb_ctx* ctx, const gb_csr* a, int64_t* count_host);

/* bfs (algorithms.py:48-77) fused: levels (int64[n], written entirely) get the
 * 1-based level, 0 = unreached.  `push` is the orientation walked by push
 * (rows = out-edges), `pull` the orientation walked by pull (rows = in-edges)
 * with `pull_nonempty` its nonempty-row bitmap.  One decision per iteration
 * is written to log_dir/log_nvals/log_est (host arrays of max_iters entries);
 * *iters_host receives the number of decisions. */
gb_status gb_bfs(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                 const uint32_t* pull_nonempty, int64_t source, int64_t max_iters,
                 double switch_ratio, int32_t policy, int64_t* levels,
                 int32_t* log_dir_host, int64_t* log_nvals_host, int64_t* log_est_host,
                 int64_t* iters_host);

/* Engine of the fused bfs (no reference counterpart; a test / A-B knob):
 * 0 = one CUDA graph with conditional nodes for the whole level loop
 * (default), 1 = host-driven loop.  Negative values only query.  Returns the
 * previous setting; process-wide. */
int32_t gb_bfs_engine(int32_t engine);

/* Result certificates (the CLI's --verify; independent of the kernels that
 * computed the result).  gb_sssp_certify: errors_host[3] = {dist[source] != 0,
 * stored edges (u, v, w) with dist[u] + w < dist[v], reached v != source
 * without a tight in-edge}; `in_edges` = rows of A^T with A's weights.
 * gb_cc_certify: errors_host[2] = {vertices with label > v or label[label] !=
 * label, stored edges joining different labels}.  Both synchronize. */
gb_status gb_sssp_certify(gb_ctx* ctx, const gb_csr* in_edges, int64_t source, const double* dist,
                          int64_t* errors_host);
gb_status gb_cc_certify(gb_ctx* ctx, const gb_csr* a, const int64_t* labels,
                        int64_t* errors_host);

/* BFS parents (extension; the reference returns levels only,
 * algorithms.py:66-77): parent[v] = the smallest u with (u, v) stored in A and
 * level[u] = level[v] - 1; parent[source] = source; -1 when unreached.
 * `in_edges` = rows of A^T (the CSR itself for a symmetric matrix), `levels`
 * a bfs result (1-based, 0 = unreached).  Asynchronous. */
gb_status gb_bfs_parents(gb_ctx* ctx, const gb_csr* in_edges, const int64_t* levels,
                         int64_t source, int64_t* parents);

/* Work counters of a BFS run as the reference tallies them over its vxm
 * calls (kernels.py:153-191, 242-280), recomputed from the final levels and
 * the direction log (dirs_host[iters], GB_DIR_*): totals_host[3] = {entries
 * read, multiplies, adds}.  out_edges = rows of A (push), in_edges = rows of
 * A^T (pull); pattern matrices with <= 64 iterations, <= 4 of them pull
 * (else GB_ERR_UNSUPPORTED).  Synchronizes. */
gb_status gb_bfs_counters(gb_ctx* ctx, const gb_csr* out_edges, const gb_csr* in_edges,
                          const int64_t* levels, int64_t iters, const int32_t* dirs_host,
                          int32_t early_exit, int64_t* totals_host);

/* Graph500-style validation of a BFS tree: errors_host[4] counts violations of
 * {source is its own parent at level 1; every reached v != source has a
 * reached parent one level up with (parent, v) stored; unreached vertices
 * have parent -1; every stored (u, v) with u reached has v reached and
 * level[v] <= level[u] + 1 (for a symmetric matrix: both ends reached or
 * neither, at most one level apart)}.  Synchronizes. */
gb_status gb_bfs_validate(gb_ctx* ctx, const gb_csr* a, const gb_csr* in_edges, int64_t source,
                          const int64_t* levels, const int64_t* parents, int64_t* errors_host);

/* bfs (algorithms.py:48-77) over the degree-ordered relabelling of the
 * matrix (gb_csr_relabel_t): `push`/`pull`/`pull_nonempty` are the relabelled
 * orientations, rank[i] the new id of vertex i.  `source` and `levels` use
 * the ORIGINAL ids, so results equal gb_bfs on the original matrix; the
 * direction log is identical (frontier sizes do not depend on labels).  The
 * push keeps the visited bits of the low-id prefix in shared memory. */
gb_status gb_bfs_ordered(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                         const uint32_t* pull_nonempty, const int32_t* rank, int64_t source,
                         int64_t max_iters, double switch_ratio, int32_t policy,
                         int64_t* levels, int32_t* log_dir_host, int64_t* log_nvals_host,
                         int64_t* log_est_host, int64_t* iters_host);

/* Asynchronous gb_bfs_ordered (same algorithm and results): enqueues the run
 * on the context stream and returns without synchronising when the device
 * loop can run it (otherwise it runs synchronously).  log_dev: device buffer
 * of 1 + 3*max_iters int64 receiving [iters, (dir, frontier, estimate) x
 * iters]; log_host: pinned host buffer of 1 + 3*21 int64 that receives the
 * first 1 + 3*min(iters, 21) entries in stream order -- synchronise the
 * stream before reading it, and read entries past 21 decisions from log_dev.
 * launch_info[6] = launches of the fixed part, of one push level, of one
 * pull level (0 on the synchronous path), the levels per device-loop pass u,
 * of one push level whose frontier is a single vertex (it skips the degree
 * scan) and of one tiny push level (2..4096 entries: one expansion kernel
 * that appends its discoveries, no scan or bitmap finalize); pass fixed +
 * per-level launches + (u - iters % u) % u (no-op steps of the last pass) to
 * gb_count_launches once the log is read.  Replaces
 * the synchronous return of algorithms.py:48-77 + the direction_log appends
 * of kernels.py:303-304, resolved lazily by the host. */
gb_status gb_bfs_ordered_async(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                               const uint32_t* pull_nonempty, const int32_t* rank, int64_t source,
                               int64_t max_iters, double switch_ratio, int32_t policy,
                               int64_t* levels, int64_t* log_dev, int64_t* log_host,
                               int64_t* launch_info);

/* Largest graph (vertices) a default-layout BFS runs as ONE cooperative
 * kernel (gb_bfs_coop.cu) instead of the device-graph loop; n >= 0 sets it
 * (0 = never), n < 0 only reads.  Returns the previous value. */
int64_t gb_bfs_coop_max_n(int64_t n);

/* Completion events on a context's stream (host-side waits for asynchronous
 * calls): create, record on ctx's stream, wait, destroy. */
gb_status gb_event_create(void** ev);
gb_status gb_event_record(gb_ctx* ctx, void* ev);
gb_status gb_event_sync(void* ev);
gb_status gb_event_destroy(void* ev);

/* Adds n to the context's launch counter (asynchronous entries). */
void gb_count_launches(gb_ctx* ctx, int64_t n);

/* ----------------------------------------------------------------------------
 * measurement support (bench.py)
 * --------------------------------------------------------------------------*/

/* Random-probe ceiling: uniformly random 4-byte ld.global.ca probes of a
 * `words`-word bitmap (>= min_probes of them) at full occupancy; writes
 * probes per second.  Synchronizes. */
gb_status gb_probe_rate(gb_ctx* ctx, int64_t words, int64_t min_probes, double* probes_per_s_host);

/* Gather ceiling of a pull SpMV on `a`: gathers/s of a kernel that only
 * streams a's column indices and gathers x[col] (f64, n entries) for every
 * stored entry.  Measurement support for bench.py.  Synchronizes. */
gb_status gb_gather_replay_rate(gb_ctx* ctx, const gb_csr* a, const double* x,
                                double* gathers_per_s_host);

#ifdef __cplusplus
}
#endif
#endif /* GRAPHBLAST_H */
