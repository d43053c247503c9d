/*
 * isvd.h -- C ABI of the B200-native implicit randomized SVD (arXiv 2111.06312).
 *
 * Citations: P:n = line n of the paper's text; "Alg. 1" = iSVD
 * (P:834-863), "Alg. 2" = orthonormalisation, "Eq. 3" = the NE
 * design matrix, "Eq. 6" = the NC design matrix,
 * "SymbolicPF" = the product contract shape()/dot()/T().
 * Readings of unclear passages (O1..O22) are listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every call returns isvd_status.  Nothing throws or aborts across the ABI.
 *    Arguments and shapes are validated before any work is enqueued; on a
 *    non-OK status no output buffer is marked valid and isvd_last_error(ctx)
 *    holds a one-line description.
 *  - Dense matrices are fp32, ROW-MAJOR, with an explicit leading dimension
 *    (elements, >= number of columns).  Leading dimensions that are multiples
 *    of 4 and 16-byte aligned base pointers take the vectorised (float4) paths;
 *    other values are rejected with ISVD_ERR_INVALID_ARG.
 *  - Device pointers are CUDA device pointers on the ctx's device.  Work is
 *    enqueued on the ctx stream; isvd_matmul / isvd_matmul_T / isvd_sample_omega
 *    return without synchronising.  isvd_svd synchronises once at its end
 *    (it reads back the singular values and the device status flags).
 *  - Distributed layout (world > 1, 1-D row partition of the graph): every
 *    n-long dimension is row-partitioned, rank p owning rows
 *    [row_begin, row_begin + n_local) with row_begin = p * ceil(n / world)
 *    (isvd_partition computes it); the short NC dimension c = d (L + 1) is
 *    replicated on every rank.
 *  - Threading: one host thread per ctx at a time.  Graphs and ops are
 *    immutable after creation.
 *  - Determinism: for a fixed (seed, world) the results are bitwise
 *    reproducible: no floating-point atomics anywhere, every reduction runs in
 *    a fixed order.
 */
#ifndef ISVD_H_
#define ISVD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISVD_ABI_VERSION 2

typedef enum {
  ISVD_OK = 0,
  ISVD_ERR_INVALID_ARG = 1, /* null pointer, bad flag, bad leading dimension / alignment   */
  ISVD_ERR_SHAPE = 2,       /* operand dims do not match the op (SymbolicPF shape)   */
  ISVD_ERR_RANK = 3,        /* k < 1 or k > min(r, c)  (SVD_k defined for k <= rank) */
  ISVD_ERR_INDEX = 4,       /* col_idx outside [0, n) or row_ptr not monotone               */
  ISVD_ERR_NONFINITE = 5,   /* NaN / Inf met in an input or produced by the solver          */
  ISVD_ERR_OOM = 6,         /* device allocation failed                                     */
  ISVD_ERR_CUDA = 7,        /* a CUDA runtime call failed (text in isvd_last_error)         */
  ISVD_ERR_NCCL = 8,        /* an NCCL call failed                                          */
  ISVD_ERR_NOT_PD = 9,      /* Cholesky of Q^T Q broke down even after the shifted retry    */
  ISVD_ERR_BUSY = 10,       /* object still referenced (graph with live ops)                */
  ISVD_ERR_UNSUPPORTED = 11 /* valid request this build does not implement                  */
} isvd_status;

typedef struct isvd_ctx_s* isvd_ctx;
typedef struct isvd_graph_s* isvd_graph;
typedef struct isvd_op_s* isvd_op;
typedef struct isvd_sim_group_s* isvd_sim_group;

/* Device memory supplier (north_star: "PyTorch is used only for device memory, streams and
 * process groups").  alloc(bytes, stream, user) returns a 16-byte aligned device pointer on the
 * ctx's device, usable on `stream` (a cudaStream_t as void*), or NULL on failure
 * (-> ISVD_ERR_OOM); free(ptr, stream, user) gives it back.  The library calls free only after
 * the work that used the block has completed on the host-visible timeline (it synchronises its
 * stream first), so a stream-ordered caching allocator may reuse the block at once.  With an
 * allocator the library keeps no cache of its own. */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* ptr, void* stream, void* user);
  void* user;
} isvd_allocator;

/* ------------------------------------------------------------------ context */

/* Create a context on CUDA device `device`, enqueuing on `stream`
 * (a cudaStream_t passed as void*; NULL = the legacy default stream).
 * alloc == NULL: device workspace comes from cudaMalloc, cached by the context (buffers of
 *             destroyed graphs / operators are reused by later objects of the same sizes, trimmed
 *             when an allocation fails, released by isvd_ctx_destroy; ISVD_NO_POOL=1 disables
 *             the cache).  alloc != NULL: every device buffer comes from the caller's allocator
 *             (copied struct; the Python binding wires PyTorch's caching allocator).
 * nccl_unique_id == NULL: single GPU (world must be 1).  Large graphs are then
 *             relabelled internally by degree (hub rows contiguous and kept
 *             L2-persisting; every caller-ordered input and output is mapped at
 *             this boundary, and cudaLimitPersistingL2CacheSize is raised once).
 * nccl_unique_id != NULL: distributed mode over `world` >= 1 ranks; it points to
 *             the 128-byte ncclUniqueId that rank 0 created (isvd_nccl_unique_id)
 *             and every rank received out of band; the call is collective.  The
 *             row-partitioned schedule (all-gather of every SpMM gather source,
 *             fp64 all-reduce of Gram / column sums / X^T Z) runs even for world 1. */
isvd_status isvd_ctx_create(int device, void* stream, const isvd_allocator* alloc, const void* nccl_unique_id,
                            int rank, int world, isvd_ctx* out);
isvd_status isvd_ctx_destroy(isvd_ctx ctx);
/* Fill the 128-byte buffer `id_out` with a fresh ncclUniqueId (rank 0 only). */
isvd_status isvd_nccl_unique_id(void* id_out, size_t id_bytes);
const char* isvd_status_string(isvd_status s);
const char* isvd_last_error(isvd_ctx ctx); /* never NULL; "" when no error */
int isvd_abi_version(void);

/* Simulated ranks (a TEST backend of the distributed layout, SURVEY 8(c) "simulation mode"):
 * `world` (1..16) logical ranks on ONE device, one context per rank, each driven by its own
 * host thread.  The contexts run the same row-partitioned schedule as the NCCL path (padded
 * all-gathers of every SpMM gather source, fp64 all-reduces, the sign-rule candidate gather);
 * the collectives move data with one cudaMemcpyAsync per peer slice (all-gather) or one
 * rank-ordered sum kernel (all-reduce), ordered across the ranks' streams by events and host
 * barriers only (no kernel waits on another rank).  Every collective call (graph/op creation
 * do none; isvd_matmul, isvd_matmul_T, isvd_svd and isvd_least_norm do) must be made by all
 * ranks of the group, in the same order.  The solver is not captured as a CUDA graph in this
 * mode.  isvd_sim_group_destroy returns ISVD_ERR_BUSY while contexts of the group live. */
isvd_status isvd_sim_group_create(int world, isvd_sim_group* out);
isvd_status isvd_sim_group_destroy(isvd_sim_group group);
isvd_status isvd_ctx_create_sim(int device, void* stream, const isvd_allocator* alloc, isvd_sim_group group,
                                int rank, isvd_ctx* out);

/* Row partition used by the distributed layout: rows [*row_begin, *row_begin + *n_local). */
isvd_status isvd_partition(int64_t n, int world, int rank, int64_t* row_begin, int64_t* n_local);

/* -------------------------------------------------------------------- graph */

enum {
  ISVD_PTR_DEVICE = 1u,        /* row_ptr / col_idx (or X) are device pointers (else host)       */
  ISVD_GRAPH_SYMMETRIC = 2u,   /* caller asserts A = A^T (required by this build, see below)     */
  ISVD_GRAPH_VALIDATE = 4u,    /* check monotone row_ptr and 0 <= col_idx < n (one pass, O(nnz))  */
  ISVD_BORROW = 8u             /* op keeps the caller's device X instead of copying it            */
};

/* Graph A given as this rank's rows in CSR: row_ptr int64[n_local + 1] (row_ptr[0] may be
 * nonzero: it is subtracted), col_idx int32[nnz] holding GLOBAL node ids, and
 * values: NULL (unweighted, A_ij = 1 for every stored (i, j); reading O12) or fp32[nnz] edge
 * weights A_ij ("A_ij is set to their edge weight"; finite, >= 0; same host/device
 * kind as col_idx).  Rows must hold no self-loop and no duplicate (reading O16; A + I adds the
 * diagonal itself).  The graph copies every array into device memory it owns (the caller may
 * free its inputs on return) and computes, once, in fp64 from the degrees d_i = sum_j A_ij
 * (integer for unweighted graphs):
 *   inv_deg_i = 1 / d_i      (T = D^-1 A; d_i = 0 -> 0, reading O3)
 *   s_i = (d_i + 1)^-1/2     (A_hat = (D+I)^-1/2 (A+I) (D+I)^-1/2)
 * stored in fp32.  Transposes are never built: this build requires
 * ISVD_GRAPH_SYMMETRIC (all configs are undirected), so T^T = A D^-1 and
 * A_hat^T = A_hat are the same CSR with the scale moved; without the flag
 * the call returns ISVD_ERR_UNSUPPORTED.  ISVD_GRAPH_VALIDATE also checks every weight.
 * Row partition: (row_begin, n_local) must equal isvd_partition(n_global, world, rank). */
isvd_status isvd_graph_create(isvd_ctx ctx, int64_t n_global, int64_t row_begin, int64_t n_local,
                              const int64_t* row_ptr, const int32_t* col_idx, const float* values, uint32_t flags,
                              isvd_graph* out);
/* ISVD_ERR_BUSY while ops reference it.  Device memory of destroyed graphs / operators goes
 * back to the context's cache (reused by later graphs / operators of the same sizes, trimmed
 * when an allocation fails) and is released by isvd_ctx_destroy; ISVD_NO_POOL=1 frees it
 * immediately instead. */
isvd_status isvd_graph_destroy(isvd_graph g);
isvd_status isvd_graph_info(isvd_graph g, int64_t* n_global, int64_t* n_local, int64_t* nnz_local,
                            int64_t* max_degree);

/* ---------------------------------------------------------------- operators */

typedef enum {
  ISVD_OP_POWER_SUM = 1,           /* NE, Eq. 3: M = sum_c w_c T^c - lambda_ones 1 1^T          */
  ISVD_OP_STACKED_PROPAGATION = 2  /* NC, Eq. 6: M = [X | A_hat X | ... | A_hat^L X]            */
} isvd_op_kind;

/* NE basis (Section 2.1: "replace T by A_hat, recovering a basis where L = R"). */
typedef enum {
  ISVD_BASIS_DEFAULT = 0,  /* = ISVD_BASIS_T_ROW                                                 */
  ISVD_BASIS_T_ROW = 1,    /* T = D^-1 A (Eq. 3 as printed)                           */
  ISVD_BASIS_AHAT_SYM = 2  /* A_hat = (D+I)^-1/2 (A+I) (D+I)^-1/2: M is symmetric  */
} isvd_basis;

typedef struct {
  isvd_op_kind kind;
  int32_t num_terms;      /* NE: C >= 1 (number of powers of T); NC: L >= 0 (blocks after X) */
  const double* weights;  /* NE: host array w_1..w_C (copied).  Configs: 1/C (footnote P:137);
                             Fig. 1 uses (C-q+1)/(C(C+1)/2) (reading O1).  NC: NULL. */
  double lambda_ones;     /* NE: coefficient of the rank-1 term -lambda 1 1^T (Eq. 3, P:145;
                             configs: 1/n).  Applied matrix-free in fp64.           */
  double lambda_adj;      /* NE: coefficient of +lambda A (Eq. 3's -lambda (1 1^T - A), P:145;
                             the configs use 0).  Applied as one extra SpMM of Q per product,
                             added in the last Horner step's epilogue.       */
  const float* X;         /* NC: this rank's rows of X, n_local x d, row-major, leading dim ldx */
  int64_t d, ldx;         /* NC: feature width d (>= 1) and leading dimension (multiple of 4) */
  uint32_t x_flags;       /* NC: ISVD_PTR_DEVICE and/or ISVD_BORROW                           */
  /* NC label re-use: M_LR = [M | B Y | B^2 Y | ... | B^P Y] with
   * B = A_hat - (D + I)^-1 (A_hat without its diagonal: no label leaks to its own row).
   * Y: this rank's rows of Y_train (n_local x y, one-hot on labelled rows, zero elsewhere),
   * copied (host or device per y_flags & ISVD_PTR_DEVICE); ldy % 4 == 0.  P = 0: none.      */
  const float* Y;
  int64_t y, ldy;
  int32_t lr_powers;
  uint32_t y_flags;
  int32_t basis;          /* NE: isvd_basis (0 = T).  NC: 0 or ISVD_BASIS_AHAT_SYM (its basis is
                             A_hat)                                                      */
  int32_t pad0;
  /* Implicit row gather (semi-supervised option (ii): "SVD of submatrix of M without
   * explicitly computing M nor the submatrix"): the op is M_S = M[S, :] for the n_rows sorted,
   * distinct GLOBAL row ids in `rows` (host array, the same full list on every rank; copied).
   * Shape (|S|, c).  The r-side (isvd_matmul output, isvd_matmul_T input, U) then has this
   * rank's subset rows -- those of S inside its row block, in S order.  Products are
   * M_S G = (M G)[S] and M_S^T H = M^T (H scattered to the rows S, zero elsewhere).
   * n_rows = 0: the whole M. */
  const int64_t* rows;
  int64_t n_rows;
} isvd_op_desc;

/* Define an implicit matrix over graph g.  No O(nnz) work; copies w (and X
 * unless borrowed).  The op holds a reference on g. */
isvd_status isvd_op_define(isvd_graph g, const isvd_op_desc* desc, isvd_op* out);
/* Global shape (r, c) of M (SymbolicPF.shape): NE (n, n); NC (n, d (L+1) + y P); with a row
 * subset S, r = |S|. */
isvd_status isvd_op_shape(isvd_op op, int64_t* rows, int64_t* cols);
isvd_status isvd_op_destroy(isvd_op op);

/* out = M . Q   (SymbolicPF.dot; Alg. 1 lines 5/7).
 *   Q   : device, rows = this rank's share of c (NE: n_local; NC: all c, replicated), w columns.
 *   out : device, this rank's r-side rows (n_local, or its subset rows) x w.  Must not alias Q.
 * Accumulation: fp32 products summed in fp64 per row (blocks of 8 neighbours in
 * fp32, then fp64); the rank-1 term is applied in fp64 before the single
 * rounding to fp32 (reading O15).  Asynchronous on the ctx stream. */
isvd_status isvd_matmul(isvd_op op, const float* Q, int64_t w, int64_t ldq, float* out, int64_t ldo);
/* out = M^T . Q (SymbolicPF.T().dot; Alg. 1 lines 6/9).
 *   Q   : device, this rank's r-side rows x w.   out : device, NE: n_local x w; NC: c x w (replicated). */
isvd_status isvd_matmul_T(isvd_op op, const float* Q, int64_t w, int64_t ldq, float* out, int64_t ldo);

/* -------------------------------------------------------------------- solver */

enum {
  ISVD_SVD_OMEGA_PROVIDED = 1u, /* start from params.omega instead of the built-in generator   */
  ISVD_SVD_HOST_OUTPUT = 2u,    /* U and V are host pointers (copied back inside the call)      */
  ISVD_SVD_NO_GRAPH = 4u,       /* do not capture/replay the solver as a CUDA graph             */
  ISVD_SVD_FORCE_CHOL_FAIL = 8u,/* fault injection: treat every first Cholesky as broken down   */
  ISVD_SVD_PROFILE = 16u        /* bracket every SpMM step with CUDA events (report.ms_spmm)     */
};

typedef struct {
  int32_t k;            /* target rank, 1 <= k <= min(r, c)                                      */
  int32_t oversampling; /* p; l = min(k + p, r, c).  p < 0 -> l = min(2k, r, c) (Alg. 1) */
  int32_t power_iters;  /* q = Alg. 1's `iterations`: 2q + 2 products in total          */
  uint64_t seed;        /* Omega stream key (reading O11)                                       */
  uint32_t flags;       /* ISVD_SVD_*                                                           */
  const float* omega;   /* device c_local x l (ld = round_up(l, 4)) iff ISVD_SVD_OMEGA_PROVIDED */
} isvd_svd_params;

typedef struct {
  int32_t l;              /* working width                                                  */
  int32_t ld;             /* leading dimension used for n x l iterates (round_up(l, 4))      */
  int32_t chol_fallbacks; /* Cholesky breakdowns repaired by the shifted retry (reading O10) */
  int32_t jacobi_sweeps;  /* sweeps of the one-sided Jacobi SVD of the l x l factor          */
  int32_t world;
  int32_t kernel_launches;/* kernels enqueued by this call (all ours)                        */
  double ms_total;        /* CUDA-event time of the whole call on the ctx stream            */
  int32_t spmm_steps;     /* fused SpMM steps (K1 launches, fixup included) in this call     */
  int32_t pad0;
  double ms_spmm;         /* ISVD_SVD_PROFILE: summed CUDA-event time of those steps, else 0 */
  double spmm_alg_bytes;  /* algorithmic bytes of those steps (CSR + scales + gather source
                             read once + epilogue operand + output)           */
  /* ISVD_SVD_PROFILE: CUDA-event time by phase (the solver's stream, so the phases sum to about
   * ms_total); 0 otherwise.  products = every M Q / M^T Q (SpMM chains, NC dense terms, their
   * all-gathers); orth = the CholeskyQR passes (Grams, Cholesky, applies, their all-reduces);
   * small = Omega, the final SVD of R^T, U / V and the sign rule; comm = the collectives alone
   * (a subset of the other three). */
  double ms_products, ms_orth, ms_small, ms_comm;
  int32_t gram_probe_fallbacks; /* first-pass tensor-core Gram probes that fell back to the exact fp64
                                   Gram (ill-conditioned M Omega)                   */
  int32_t gram_probe_skipped;   /* 1: this call skipped the probe and took the exact first Gram
                                   directly, because an earlier call on this op fell back       */
  /* ISVD_SVD_PROFILE, distributed with the local / remote split: summed duration of the
   * all-gathers of SpMM gather sources on the collectives stream, and the part of it that ran
   * concurrently with the local SpMM pass issued meanwhile (CUDA-event intervals); 0 otherwise. */
  double ms_allgather, ms_allgather_hidden;
} isvd_svd_report;

/* Rank-k randomized SVD of M (Alg. 1) with CholeskyQR2
 * orthonormalisation (Alg. 2 right, applied twice) and the final
 * SVD of B = (M^T Q)^T computed as CQR2(M^T Q) = Q_W R followed
 * by a one-sided Jacobi SVD of R^T (B = R^T Q_W^T).
 *   U : r-side rows x k (ldu): this rank's rows (n_local, or its subset rows), left singular vectors.
 *   S : HOST double[k], non-increasing (reading O9).
 *   V : NE: n_local x k (this rank's rows); NC: c x k replicated (ldv).
 *   Sign rule (reading O9): each (U_j, V_j) is flipped so that the largest-
 *   magnitude entry of column U_j (lowest global row on ties) is positive.
 *   rep: nullable.
 * Device pointers unless ISVD_SVD_HOST_OUTPUT.  Synchronises the ctx stream once. */
isvd_status isvd_svd(isvd_op op, const isvd_svd_params* params, float* U, int64_t ldu, double* S, float* V,
                     int64_t ldv, isvd_svd_report* rep);

/* Write the Omega the solver starts from (Alg. 1 line 4; stream of
 * reading O11: Philox4x32-10 + Box-Muller keyed by the global (row, column))
 * into device `omega` (this rank's c-rows x l, ld = round_up(l, 4)). */
isvd_status isvd_sample_omega(isvd_op op, const isvd_svd_params* params, float* omega, int64_t ldo);

/* ---------------------------------------------------------- after the SVD
 * Embeddings (Eq. 5): L = U S^1/2 (and R = V S^1/2 by a second call).
 *   M: rows x k fp32 device, ld % 4 == 0; out may equal M (in place); S: host, k values >= 0.
 *   Errors: ISVD_ERR_INVALID_ARG (null / bad ld), ISVD_ERR_NONFINITE (S < 0 or not finite). */
isvd_status isvd_embeddings(isvd_ctx ctx, int64_t rows, int64_t k, const float* M, int64_t ldm, const double* S,
                            float* out, int64_t ldo);

/* Least-norm parameters (Eq. 7): W = V S^+ (U[rows]^T Y[rows]), multiplied right to
 * left.  U^T Y is exact fp64 (FP64 tensor cores) over this rank's rows, all-reduced over
 * the ranks in distributed mode; S^+ reciprocates S_i > max(r, c) eps_fp64 max(S) (reading O24);
 * W = V (S^+ U^T Y) on the device.
 *   U: r_local x k, Y: r_local x ny (labels, e.g. one-hot), V: v_rows x k (NE: this rank's rows,
 *   NC: all c rows), W: v_rows x ny -- fp32 device, every ld % 4 == 0, 16-byte aligned.
 *   rows: NULL (every row) or device int32[n_rows] of local row ids, the labelled rows
 *   (semi-supervised option (i)).  S: host double[k].  (r, c): the shape of M.
 *   Synchronises the ctx stream.  Errors: ISVD_ERR_INVALID_ARG, ISVD_ERR_NONFINITE. */
isvd_status isvd_least_norm(isvd_ctx ctx, int64_t r_local, int64_t k, const float* U, int64_t ldu, const double* S,
                            int64_t r, int64_t c, int64_t v_rows, const float* V, int64_t ldv, int64_t ny,
                            const float* Y, int64_t ldy, const int32_t* rows, int64_t n_rows, float* W,
                            int64_t ldw);

/* Gaussian spectral kernel (Eq. 9; discretisation P:1057-1065): out_i =
 * sum_{x in Omega} S_i^x softmax_x(-(x - mu)^2 exp(s_bar)), Omega = {0.5, 0.505, ..., 2.0}
 * (301 points), s_bar = log(1 / (2 s^2)); then f(i, j) = U_i^T diag(out) V_j.  Host arrays of k
 * doubles (a k-vector epilogue; fp64 on the host side of the library).  S_i >= 0.
 * Errors: ISVD_ERR_INVALID_ARG, ISVD_ERR_NONFINITE. */
isvd_status isvd_spectral_kernel(const double* S, int64_t k, double mu, double s_bar, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ISVD_H_ */
