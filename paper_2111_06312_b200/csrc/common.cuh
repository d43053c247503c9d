// Shared device/host helpers of the isvd CUDA library (sm_100a only).
// Not shared with oracle/ (the oracle is independent test infrastructure).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define ISVD_DEVICE __device__ __forceinline__

// Checked build (ISVD_BOUNDS_CHECK=1 python -m paper_2111_06312_b200._build --force): device-side
// bounds asserts on every gathered / mapped row index (compute-sanitizer is closed on this pool).
#if defined(ISVD_BOUNDS_CHECK) && defined(__CUDACC__)
#include <cassert>
#define ISVD_ASSERT(c) assert(c)
#else
#define ISVD_ASSERT(c) ((void)0)
#endif

namespace isvd {

// Device-side status word shared by every kernel of one solver call.
// Kernels set bits; the host reads the word once at the end of isvd_svd.
struct DevStatus {
  int chol_breakdown;   // Cholesky pivot <= tol met (count of factorizations that needed the shift)
  int chol_failed;      // still broken after the shifted retry
  int nonfinite;        // NaN/Inf produced
  int jacobi_sweeps;    // sweeps used by the last Jacobi SVD
  int need_extra_pass;  // set by a Cholesky that used the shift: run the third CQR pass
  int need_exact_gram;  // set by a probe-mode Cholesky: recompute the Gram exactly (fp64) and refactor
  int probes_failed;    // count of those (reported)
  int pad;
};

#if defined(__CUDACC__)
ISVD_DEVICE float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
ISVD_DEVICE void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
ISVD_DEVICE float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
// paired fp32 FMA (sm_100 FFMA2: same FLOP rate as FFMA, half the issue slots; a scalar first
// operand compiles to the .F32 broadcast form): d = a * b + c, elementwise, round-to-nearest
ISVD_DEVICE float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
// flat index t -> (row, column) of a width-w grid-stride loop: a 32-bit division whenever t fits
// (a 64-bit division is a ~70-instruction subroutine call per element)
ISVD_DEVICE int64_t row_of(int64_t t, int64_t w) {
  return (uint64_t)t <= 0xFFFFFFFFull ? (int64_t)((uint32_t)t / (uint32_t)w) : t / w;
}
#endif

// Kernels enqueued by this host thread (each launcher adds the number it launched);
// isvd_svd reports the difference over one call.
extern thread_local int64_t g_launches;

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Row maps.  A graph may be relabelled internally (degree-descending, so hub rows are
// contiguous and L2-persistable); `new2old[i]` is the caller's row of internal row i.
// Kernels that read a caller-ordered operand take an `in_map`, kernels that write a
// caller-ordered result take an `out_map` (nullptr = identity).

// ---------------------------------------------------------------- launchers
// All launchers enqueue on `st` and return cudaGetLastError().

// Omega (Alg. 1 line 4): `rows` rows of the c x l matrix, ld >= l; row i is global
// row (row_map ? row_map[i] : row0 + i).  Padding columns [l, ld) are written as 0.
cudaError_t launch_omega(uint64_t seed, int64_t row0, int64_t rows, int l, int64_t ld, float* out,
                         const int32_t* row_map, cudaStream_t st);

// Column sums (fp64) of a rows x w fp32 matrix: out[j] = sum_i Q[i, j], j < wpad (wpad = round_up(w,4)).
// Deterministic two-stage reduction; `ws` needs colsum_ws_doubles(rows, wpad) doubles.
int64_t colsum_ws_doubles(int64_t rows, int64_t wpad);
cudaError_t launch_colsum(const float* Q, int64_t rows, int64_t wpad, int64_t ldq, double* ws, double* out,
                          cudaStream_t st);

// out[i, :] = coef * (vec ? vec[i] : 1) * in[in_map ? in_map[i] : i, :]  for i < rows, columns < wpad.
cudaError_t launch_scale_rows(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows,
                              int64_t wpad, const float* vec, float coef, const int* gate, cudaStream_t st,
                              const int32_t* in_map = nullptr);
// out[out_map[i], :] = in[i, :] for i < rows, columns < wpad (other rows of out untouched).
cudaError_t launch_scatter_rows(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int64_t wpad,
                               const int32_t* out_map, cudaStream_t st);
// out[i] = inv[idx[i]] (i < m) with inv the inverse of the permutation perm of [0, n) (inv_ws: n ints).
cudaError_t launch_compose_inverse(const int32_t* perm, int64_t n, const int32_t* idx, int64_t m, int32_t* inv_ws,
                                   int32_t* out, cudaStream_t st);
// out[i, j] = in[i, j] * colvec[j]  (i < rows, j < wpad, wpad % 4 == 0; out may equal in)
cudaError_t launch_scale_cols(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int64_t wpad,
                              const float* colvec, cudaStream_t st);

// ------------------------------------------------------------------- SpMM
// Fused CSR SpMM step (K1):  for each local row i (global id row_offset + i)
//   acc_i = self_coef * Y[row_offset + i] + sum_{j in N(i)} A_ij Y[j]     (fp32 blocks of 8, fp64 across)
//   out_i = post_coef * post_vec[i] * acc_i
//         + term_coef * term_vec[i] * T[i]
//         - rank1_coef * colsum                                          (all in fp64, one rounding)
// written to out row (out_map ? out_map[i] : i).
// Rows are processed as segments of <= kSegEdges edges; long rows are split and
// their fp32 partial sums combined in a fixed order by a fixup pass.
struct SpmmPlan {
  int64_t n_local = 0;
  int64_t n_seg = 0;          // number of segments
  int64_t n_split_rows = 0;   // rows split into >1 segment
  int64_t n_slots = 0;        // partial slots (= segments of split rows)
  // device arrays
  int32_t* seg_row = nullptr;     // [n_seg] local row of the segment
  int64_t* seg_beg = nullptr;     // [n_seg] first edge
  int32_t* seg_len = nullptr;     // [n_seg] number of edges
  int32_t* seg_slot = nullptr;    // [n_seg] partial slot or -1 (whole row)
  int32_t* split_row = nullptr;   // [n_split_rows] local row id
  int32_t* split_slot0 = nullptr; // [n_split_rows] first slot
  int32_t* split_nslot = nullptr; // [n_split_rows] number of slots
};
constexpr int kSegEdges = 512;
constexpr int kIdxPad = 16;  // readable zero entries after col_idx[nnz - 1] (index prefetch)

struct SpmmArgs {
  const int32_t* col_idx;
  const float* val;        // edge weights A_ij (nullable: unweighted, every A_ij = 1)
  int64_t row_offset;
  const float* Y; int64_t ldy;
  float self_coef;
  const float* post_vec; float post_coef;
  const float* T; int64_t ldt; const float* term_vec; float term_coef;
  const double* colsum; double rank1_coef;
  float* out; int64_t ldo;
  const int32_t* out_map;  // nullable
  int64_t wpad;            // columns processed (multiple of 4)
  const float* pre; int64_t ldpre;  // nullable: fp32 partial row sums added to acc first (split passes)
  int64_t n_src;                    // rows readable in Y (bounds-checked builds assert every gather)
};
int64_t spmm_ws_floats(const SpmmPlan& plan, int64_t wpad);
// Graph relabelling on the device: new row t = old row order[t], neighbour ids renamed by new_of_old
// (edge weights, if any, move with their edges; the order inside a row is kept).
cudaError_t launch_relabel_csr(const int64_t* rp_old, const int32_t* ci_old, const float* val_old,
                               const int32_t* order, const int32_t* new_of_old, const int64_t* rp_new,
                               int32_t* ci_new, float* val_new, int64_t n, cudaStream_t st);
// Device-side graph build (graph_build.cu): degree order (stable, decreasing degree) with its
// maps and the relabelled row_ptr; fp64-derived scale vectors; SpMM segment plan (count + scan,
// then fill once the host has read the totals).  temp: graph_build_temp_bytes(n) bytes.
size_t graph_build_temp_bytes(int64_t n);
cudaError_t launch_degree_order(const int64_t* rp, int64_t n, uint32_t* keys2, int32_t* idx, int32_t* order,
                                int32_t* new_of_old, int64_t* deg_tmp, int64_t* rp_new, void* temp, size_t temp_bytes,
                                cudaStream_t st);
// val: null (unweighted: d_i = edge count) or fp32 edge weights (d_i = sum_j A_ij in fp64).
cudaError_t launch_scales(const int64_t* rp, const float* val, int64_t n, float* inv, float* s, float* s2, float* rs,
                          cudaStream_t st);
cudaError_t launch_plan_count(const int64_t* rp, int64_t n, int64_t* nseg, int32_t* nsplit, int32_t* nslot,
                              int64_t* seg_off, int32_t* split_off, int32_t* slot_off, void* temp, size_t temp_bytes,
                              cudaStream_t st);
cudaError_t launch_plan_fill(const int64_t* rp, int64_t n, const int64_t* seg_off, const int32_t* split_off,
                             const int32_t* slot_off, const SpmmPlan& p, cudaStream_t st);
// Distributed local / remote CSR split (SURVEY 8(e) overlap item 1): per row, the edges whose
// column is in [lo, hi) (this rank's own rows) and the others, each as a CSR in the same order as
// the input.  Count pass (cnt_loc[i], int64, n + 1 entries) then fill pass (warp per row, stable).
cudaError_t launch_split_count(const int64_t* rp, const int32_t* ci, int64_t n, int64_t lo, int64_t hi,
                               int64_t* cnt_loc, int64_t* cnt_rem, cudaStream_t st);
cudaError_t launch_split_fill(const int64_t* rp, const int32_t* ci, const float* val, int64_t n, int64_t lo, int64_t hi,
                              const int64_t* rp_loc, const int64_t* rp_rem, int32_t* ci_loc, float* val_loc,
                              int32_t* ci_rem, float* val_rem, cudaStream_t st);
// Dense adjacency (SURVEY 8(f) f3 comparison): out (n x ld fp32, zero-filled here) gets A_ij at (i, j).
cudaError_t launch_dense_adjacency(const int64_t* rp, const int32_t* ci, const float* val, int64_t n, int64_t ld,
                                   float* out, cudaStream_t st);
// Unweighted dense adjacency as bytes (entries are small integer counts; n x ldo, zero padded columns).
cudaError_t launch_dense_to_u8(const float* in, int64_t n, int64_t ldi, uint8_t* out, int64_t ldo, cudaStream_t st);
// Exact A Y on the INT8 tensor cores (dense_i8.cu): A = n x n bytes (lda = round_up(n, 16)), Y n x w fp32.
// ws: dense_i8_ws_bytes bytes (fp64 integer partials + column maxima), Qws: *q_bytes bytes.  Outputs the
// partial layout and the column-maximum bits for launch_spmm_dense64_epilogue.
int64_t dense_i8_ws_bytes(int64_t n, int64_t w, int num_sms, int64_t* q_bytes);
cudaError_t launch_dense_i8(const uint8_t* A, int64_t lda, int64_t n, const float* Y, int64_t ldy, int64_t w,
                            uint8_t* Qws, void* ws, int num_sms, cudaStream_t st, int64_t* parts, int64_t* ws_rows,
                            int64_t* ws_ld, const unsigned** cmax_out, const double** part_out);
// acc[row, col] = 2^(E_col - 22) * sum_p ws[p][row][col] (E_col from the column-maximum bits), then
// the SpMM epilogue of `a`.
cudaError_t launch_spmm_dense64_epilogue(const double* ws, int64_t parts, int64_t ws_rows, int64_t ws_ld,
                                         const unsigned* cmax, const SpmmArgs& a, int64_t n_local, int num_sms,
                                         cudaStream_t st);
// Epilogue of the dense-A product (f3): acc = sum over `parts` fp32 partial tiles ws32[p][row][col]
// (ws_lda rows, ws_ld columns per part; summed in fp64 in part order), then the SpMM epilogue of `a`
// (self term, scales, Horner term, rank-1 correction, out_map) for rows < n_local.
cudaError_t launch_spmm_dense_epilogue(const float* ws32, int64_t parts, int64_t ws_lda, int64_t ws_ld,
                                       const SpmmArgs& a, int64_t n_local, int num_sms, cudaStream_t st);
cudaError_t launch_exclusive_scan64(const int64_t* in, int64_t* out, int64_t n1, void* temp, size_t temp_bytes,
                                    cudaStream_t st);
// `persist_bytes` > 0: the first persist_bytes of Y (the hub rows of a degree-relabelled
// graph) are marked L2-persisting for this launch (cudaAccessPolicyWindow on `st`).
// col_block > 0: process the columns in blocks of that width (one launch each).
cudaError_t launch_spmm(const SpmmPlan& plan, const SpmmArgs& a, float* ws_partial, int num_sms,
                        cudaStream_t st, size_t persist_bytes = 0, int64_t col_block = 0);

// ------------------------------------------------------------------- dense
// C[out_map ? out_map[i] : i, j] = alpha * row_scale(i) * sum_k A[i, k] B[k, j],  i < M, j < N (N multiple of 4).
// B is K x N row-major (ldb).  upper_tri_b: B[k, j] = 0 for k > j (skips those k).
cudaError_t launch_gemm_tn(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                           int64_t M, int64_t N, int64_t K, const float* row_scale, float alpha,
                           bool upper_tri_b, const int* gate, cudaStream_t st, const int32_t* out_map = nullptr);

// Tensor-core (tcgen05, 3xTF32) tall GEMM: C[map(i), j] = alpha row_scale(i) sum_k A[i, k] B[k, j],
// i < rows, j < N; A rows x K (lda % 4 == 0), B K x N (ldb), C ldc.  ws_bt: tc_gemm_ws_floats floats.
bool tc_gemm_supported(int64_t rows, int64_t N, int64_t K, int64_t lda, int64_t ldc);
int64_t tc_gemm_ws_floats(int64_t N, int64_t K);
cudaError_t launch_tc_gemm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                           int64_t rows, int64_t N, int64_t K, const float* row_scale, float alpha, const int* gate,
                           cudaStream_t st, const int32_t* out_map, float* ws_bt, int num_sms);

// G = A^T diag(row_scale) B over `rows` rows, A: rows x Ka, B: rows x Kb -> fp64 Ka x ldg.
// symmetric: A == B, only the upper triangle of tiles is computed and mirrored.
// If out32 != null the result is also written as fp32 (ld32).
// f32_stage: fp32 sums over <= 1024-row chunks (register-tiled SIMT), fixed-order fp64 across
// chunks; else exact fp64 (fp64 tensor cores, or DFMA with ISVD_DMMA=0).
int64_t atb_ws_doubles(int64_t rows, int64_t Ka, int64_t Kb, int num_sms);
cudaError_t launch_atb(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t rows, int64_t Ka,
                       int64_t Kb, const float* row_scale, bool symmetric, double* ws, double* G, int64_t ldg,
                       float* out32, int64_t ld32, int num_sms, const int* gate, cudaStream_t st,
                       bool f32_stage = false);
// fp64 fixed-order sum of `chunks` fp32 partial tiles ws32[c][Ka_pad = ws_lda][ws_ld] -> G / out32.
cudaError_t launch_atb_f32_reduce(const float* ws32, int64_t ws_lda, int64_t ws_ld, int64_t chunks, int64_t Ka,
                                  int64_t Kb, bool symmetric, double* G, int64_t ldg, float* out32, int64_t ld32,
                                  int num_sms, const int* gate, cudaStream_t st);
// Tensor-core (tcgen05, 3xTF32) partials of C = (diag(row_scale) A)^T B (A: rows x Ka, B: rows x Kb,
// row-major, ld % 4 == 0): one fp32 tile per row part into ws32 (tc_atb_ws_floats floats),
// ws32[part][ws_lda][ws_ld]; reduce with launch_atb_f32_reduce over `parts`.  symmetric: A == B,
// only the tiles holding some i <= j are computed (the reduce mirrors).
bool tc_atb_supported(int64_t rows, int64_t Ka, int64_t Kb, int64_t lda, int64_t ldb);
int64_t tc_atb_ws_floats(int64_t rows, int64_t Ka, int64_t Kb, bool symmetric, int num_sms);
// diag0 (symmetric only): if non-null, the launch may leave a trailing diagonal block [*diag0, Ka)^2
// (when the last 128-row tile holds <= 64 valid rows) for the caller to compute; *diag0 = -1 if not.
cudaError_t launch_tc_atb(const float* A, int64_t lda, int64_t Ka, const float* row_scale, const float* B,
                          int64_t ldb, int64_t Kb, int64_t rows, bool symmetric, float* ws32, int64_t* ws_lda,
                          int64_t* ws_ld, int64_t* parts, int num_sms, const int* gate, cudaStream_t st,
                          int64_t* diag0 = nullptr);
// out = *flag ? I : Rinv  (l x l, ld x ld fp32; the deferred CholeskyQR2 factor)
cudaError_t launch_select_rfold(const float* Rinv, float* out, int l, int64_t ld, const int* flag, cudaStream_t st);
// out32[i, j] = (float) G[i, j]
cudaError_t launch_f64_to_f32(const double* G, int64_t ldg, float* out, int64_t ldo, int64_t rows,
                              int64_t cols, cudaStream_t st);

// -------------------------------------------------------------- small fp64
// `gate` (nullable, device int): when non-null and *gate == 0 the kernel does nothing
// (used for the conditional third CholeskyQR pass without a host sync).
//
// Cholesky G = R^T R (upper R) of the l x l fp64 SPD matrix G (ldg; upper triangle
// read) and the inverse of R.  Outputs: Rinv32 (ld x ld fp32, upper, zero elsewhere
// incl. padding), R64 (l x l fp64, upper, zeros below) if non-null.
// Breakdown (pivot <= 1e-14 * max diag, or non-finite) -> shift the diagonal by
// 1e-10 * trace (x100 per retry, 3 retries); status->chol_breakdown++ and
// status->need_extra_pass = 1.  force_fail treats the first attempt as broken.
// `ws` needs l*l doubles when l > 512 (global-memory path).
constexpr int kCholSmemMax = 160;
// probe_tol > 0 (blocked path, l <= 512 only): probe mode -- no shift; a breakdown or a pivot spread
// min r_kk^2 < probe_tol max r_kk^2 sets *probe_flag (the Gram was too inexact for this conditioning).
cudaError_t launch_chol_inv(const double* G, int64_t ldg, int l, int64_t ld, float* Rinv32, double* R64,
                            double* ws, DevStatus* status, bool force_fail, const int* gate, cudaStream_t st,
                            double probe_tol = 0.0, int* probe_flag = nullptr);
// out = Rnew * Racc (upper l x l fp64, ld = l); when gated off: out = Racc.
cudaError_t launch_trmm(const double* Rnew, const double* Racc, double* out, int l, const int* gate,
                        cudaStream_t st);
// One-sided Jacobi SVD of A = R^T (R upper l x l fp64, ld = l).  Writes sigma_k
// (k values, descending), Ub (l x ldk fp32: the first k left singular vectors of
// R^T) and Vb (l x ldk fp32: the matching right singular vectors).
int64_t jacobi_ws_doubles(int l);
cudaError_t launch_jacobi_svd(const double* R, int l, int k, int64_t ldk, double* sigma_k, float* Ub, float* Vb,
                              double* ws, DevStatus* status, int num_sms, cudaStream_t st);
// Sign rule: per column c < k of U (rows x ldu), the entry of largest |.| (lowest row on
// ties) -> cand[c] = {|u|, row + row_offset, sign} (3 doubles; row -1 if rows == 0).
int64_t absmax_ws_doubles(int64_t rows, int k);
cudaError_t launch_col_absmax(const float* U, int64_t ldu, int64_t rows, int k, int64_t row_offset,
                              double* ws, double* cand, cudaStream_t st);
// Select over `world` candidate sets (cand: world x k x 3) and flip the columns of
// U (rows x k) and V (vrows x k) whose selected entry is negative.
cudaError_t launch_sign_flip(const double* cand, int world, int k, float* sgn_ws, float* U, int64_t ldu,
                             int64_t rows, float* V, int64_t ldv, int64_t vrows, cudaStream_t st, DevStatus* status = nullptr);
// status->nonfinite |= any(!isfinite(A[:rows, :cols])).
cudaError_t launch_check_finite(const float* A, int64_t lda, int64_t rows, int64_t cols, DevStatus* status,
                                cudaStream_t st);

// Simulated ranks (capi.cpp SimGroup, a test backend): out[i] = sum over q < world of p.p[q][i],
// summed in rank order (bitwise identical on every logical rank).
constexpr int kMaxSimRanks = 16;
struct RankPtrs {
  const double* p[kMaxSimRanks];
};
cudaError_t launch_sum_ranks(const RankPtrs& p, int world, int64_t count, double* out, cudaStream_t st);

}  // namespace isvd
