// Small l x l fp64 kernels of the solver (l = 42 ... 400).
//
//  K6/K7 chol_inv   R = chol(G) (upper, G = R^T R) and R^-1 in place:
//                   Alg. 2 right, P:886-887 ("L <- Choleskydecomposition(Q^T Q);
//                   Q (L^-1)^T", with L = R^T).  One CTA; the matrix lives in shared
//                   memory for l <= kCholSmemMax and in an L2-resident global buffer
//                   above that.  Breakdown (reading O10) shifts the diagonal and
//                   raises a device flag that gates the third CholeskyQR pass.
//  trmm             R_acc <- R_new R_acc for the final CQR2 of W = M^T Q.
//  K9  jacobi       one-sided (Hestenes) Jacobi SVD of R^T (B = (M^T Q)^T = R^T Q_W^T,
//                   replacing tf.linalg.svd(B)), round-robin parallel ordering,
//                   one warp per column pair, cooperative grid barrier per round.
//  K17 sort/sign    descending order (reading O9) and the sign rule.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace isvd {
namespace {

ISVD_DEVICE double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ Cholesky + inverse
// Returns 1 (block-uniform) on breakdown.
__device__ int chol_upper_inplace(double* A, int l, double tol, double* s_scal, int* s_flag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int k = 0; k < l; ++k) {
    if (tid == 0) {
      double piv = A[(int64_t)k * l + k];
      int bad = !(piv > tol) || !isfinite(piv);
      *s_flag = bad;
      double r = bad ? 1.0 : sqrt(piv);
      A[(int64_t)k * l + k] = r;
      s_scal[0] = 1.0 / r;
    }
    __syncthreads();
    if (*s_flag) return 1;
    const double inv = s_scal[0];
    for (int j = k + 1 + tid; j < l; j += nt) A[(int64_t)k * l + j] *= inv;
    __syncthreads();
    const double* rk = A + (int64_t)k * l;
    for (int i = k + 1 + warp; i < l; i += nw) {
      const double rki = rk[i];
      double* ai = A + (int64_t)i * l;
      for (int j = i + lane; j < l; j += 32) ai[j] -= rki * rk[j];
    }
    __syncthreads();
  }
  return 0;
}

// In-place inverse of the upper triangular A (LAPACK trti2 order, column by column).
__device__ void trinv_upper_inplace(double* A, int l, double* tmp) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  for (int j = 0; j < l; ++j) {
    // tmp[i] = sum_{k=i}^{j-1} Xinv[i][k] * U[k][j]   (top-left block already inverted)
    for (int i = warp; i < j; i += nw) {
      const double* xi = A + (int64_t)i * l;
      double s = 0.0;
      for (int k = i + lane; k < j; k += 32) s += xi[k] * A[(int64_t)k * l + j];
      s = warp_sum(s);
      if (lane == 0) tmp[i] = s;
    }
    const double ajj = 1.0 / A[(int64_t)j * l + j];
    __syncthreads();
    for (int i = tid; i < j; i += blockDim.x) A[(int64_t)i * l + j] = -ajj * tmp[i];
    if (tid == 0) A[(int64_t)j * l + j] = ajj;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) chol_inv_kernel(const double* __restrict__ G, int64_t ldg, int l, int64_t ld,
                                                        float* __restrict__ Rinv32, double* __restrict__ R64,
                                                        double* __restrict__ ws, DevStatus* status, int force_fail,
                                                        const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  extern __shared__ double smem[];
  __shared__ double s_scal[4];
  __shared__ int s_flag;
  __shared__ double s_tmp[1024];  // l <= 1024 (isvd_svd rejects wider working widths)
  double* A = (l <= kCholSmemMax) ? smem : ws;
  const int tid = threadIdx.x, nt = blockDim.x;
  // trace and max diagonal (thread 0)
  if (tid == 0) {
    double tr = 0.0, mx = 0.0;
    for (int i = 0; i < l; ++i) {
      double d = G[(int64_t)i * ldg + i];
      tr += d;
      mx = d > mx ? d : mx;
    }
    s_scal[1] = tr;
    s_scal[2] = mx;
  }
  __syncthreads();
  const double trace = s_scal[1];
  const double tol = 1e-14 * s_scal[2];
  double shift = 0.0;
  int attempt = 0;
  int failed = 1;
  for (attempt = 0; attempt < 4; ++attempt) {
    for (int64_t t = tid; t < (int64_t)l * l; t += nt) {
      int i = (int)(t / l), j = (int)(t - (int64_t)i * l);
      double v = (j >= i) ? G[(int64_t)i * ldg + j] : 0.0;
      if (i == j) v += shift;
      A[t] = v;
    }
    __syncthreads();
    int bad = chol_upper_inplace(A, l, tol, s_scal, &s_flag);
    if (force_fail && attempt == 0) bad = 1;
    if (!bad) { failed = 0; break; }
    // shifted CholeskyQR (reading O10): s = 11 (m l + l (l+1)) u ||G||, bounded here by
    // a trace-relative shift that grows by 100x per retry.
    shift = (attempt == 0) ? 1e-10 * trace : shift * 100.0;
    __syncthreads();
  }
  if (tid == 0) {
    if (attempt > 0) {
      atomicAdd(&status->chol_breakdown, 1);
      status->need_extra_pass = 1;
    }
    if (failed) status->chol_failed = 1;
  }
  if (R64) {
    for (int64_t t = tid; t < (int64_t)l * l; t += nt) {
      int i = (int)(t / l), j = (int)(t - (int64_t)i * l);
      R64[t] = (j >= i) ? A[t] : 0.0;
    }
  }
  __syncthreads();
  trinv_upper_inplace(A, l, s_tmp);
  for (int64_t t = tid; t < ld * ld; t += nt) {
    int64_t i = t / ld, j = t - i * ld;
    float v = 0.f;
    if (i < l && j < l && j >= i) v = (float)A[i * l + j];
    Rinv32[t] = v;
  }
}

// out = Rnew * Racc (upper x upper), or out = Racc when gated off.
__global__ void trmm_kernel(const double* __restrict__ Rnew, const double* __restrict__ Racc, double* __restrict__ out,
                            int l, const int* gate) {
  const bool mult = !(gate && *((volatile const int*)gate) == 0);
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < l; j += blockDim.x) {
    double s = 0.0;
    if (mult) {
      if (j >= i)
        for (int k = i; k <= j; ++k) s += Rnew[(int64_t)i * l + k] * Racc[(int64_t)k * l + j];
    } else {
      s = Racc[(int64_t)i * l + j];
    }
    out[(int64_t)i * l + j] = s;
  }
}

// ------------------------------------------------------------ Jacobi SVD
ISVD_DEVICE int rr_index(int pos, int round, int m) {
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (m - 1);
}

// A: l x l, column j of R^T (= row j of R); J: accumulated rotations (column j = v_j).
// kMode 0: one CTA (columns in its shared memory when they fit, else global memory);
// kMode 1: cooperative grid, columns in (L2-resident) global memory, grid barrier per round;
// kMode 2: thread-block cluster, column c in the shared memory of CTA c % CS (slot c / CS),
//          read and rotated through DSMEM, one cluster barrier per round.
// Column norms are carried across rotations (Rutishauser: ||a_i'||^2 = ||a_i||^2 - t g,
// ||a_j'||^2 = ||a_j||^2 + t g) and recomputed exactly at every sweep, so a pair costs one
// dot-product reduction instead of three.
template <int kMode>
__global__ void __launch_bounds__(1024) jacobi_kernel(const double* __restrict__ R, int l, double* Ag, double* Jg,
                                                      int* counters, DevStatus* status, int max_sweeps,
                                                      double* __restrict__ Aout, double* __restrict__ Jout,
                                                      double* nrm_g) {
  extern __shared__ double smem[];
  __shared__ double nrm_s[kMode == 0 ? 1024 : 1];
  double* nrm = kMode == 0 ? nrm_s : nrm_g;
  int CS = 1, crank = 0;
  if constexpr (kMode == 2) {
    CS = (int)cg::this_cluster().num_blocks();
    crank = (int)cg::this_cluster().block_rank();
  }
  const int cols_per = (l + CS - 1) / CS;
  const bool in_smem = (kMode == 0 && 2 * l * l * (int)sizeof(double) <= 200 * 1024) || kMode == 2;
  double* A = in_smem ? smem : Ag;
  double* J = in_smem ? smem + (int64_t)(kMode == 2 ? cols_per : l) * l : Jg;
  auto colA = [&](int c) -> double* {
    if constexpr (kMode == 2) return cg::this_cluster().map_shared_rank(A, c % CS) + (int64_t)(c / CS) * l;
    return A + (int64_t)c * l;
  };
  auto colJ = [&](int c) -> double* {
    if constexpr (kMode == 2) return cg::this_cluster().map_shared_rank(J, c % CS) + (int64_t)(c / CS) * l;
    return J + (int64_t)c * l;
  };
  auto jsync = [&]() {
    if constexpr (kMode == 0) __syncthreads();
    else if constexpr (kMode == 1) cg::this_grid().sync();
    else cg::this_cluster().sync();
  };
  const int64_t gtid = (kMode == 1 ? (int64_t)blockIdx.x : (int64_t)crank) * blockDim.x + threadIdx.x;
  const int64_t gthreads = (kMode == 1 ? (int64_t)gridDim.x : (int64_t)CS) * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
  if constexpr (kMode == 2) {  // own columns c = q*CS + crank
    for (int64_t t = threadIdx.x; t < (int64_t)cols_per * l; t += blockDim.x) {
      const int q = (int)(t / l), r = (int)(t - (int64_t)q * l);
      const int c = q * CS + crank;
      A[t] = c < l ? R[(int64_t)c * l + r] : 0.0;
      J[t] = (c < l && r == c) ? 1.0 : 0.0;
    }
  } else {
    for (int64_t t = gtid; t < (int64_t)l * l; t += gthreads) {
      A[t] = R[t];
      int64_t j = t / l, i = t - j * l;
      J[t] = (i == j) ? 1.0 : 0.0;
    }
  }
  if (gtid == 0) { counters[0] = 0; counters[1] = 0; }
  jsync();
  const int m = (l & 1) ? l + 1 : l;
  const double tol = (double)l * 1.1102230246251565e-16;
  int sweep = 0;
  for (sweep = 0; sweep < max_sweeps; ++sweep) {
    int* cnt = counters + (sweep & 1);
    for (int64_t c = gwarp; c < l; c += nwarps) {
      const double* ac = colA((int)c);
      double q = 0.0;
      for (int r = lane; r < l; r += 32) q += ac[r] * ac[r];
      q = warp_sum(q);
      if (lane == 0) nrm[c] = q;
    }
    jsync();
    for (int round = 0; round < m - 1; ++round) {
      for (int64_t p = gwarp; p < m / 2; p += nwarps) {
        int i = rr_index((int)p, round, m), j = rr_index(m - 1 - (int)p, round, m);
        if (i >= l || j >= l) continue;
        if (i > j) { int t = i; i = j; j = t; }
        double* ai = colA(i);
        double* aj = colA(j);
        double ga = 0.0;
        for (int r = lane; r < l; r += 32) ga += ai[r] * aj[r];
        ga = warp_sum(ga);
        const double al = nrm[i], be = nrm[j];
        if (al > 0.0 && be > 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          double zeta = (be - al) / (2.0 * ga);
          double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < l; r += 32) {
            double x = ai[r], y = aj[r];
            ai[r] = c * x - s * y;
            aj[r] = s * x + c * y;
          }
          double* ji = colJ(i);
          double* jj = colJ(j);
          for (int r = lane; r < l; r += 32) {
            double x = ji[r], y = jj[r];
            ji[r] = c * x - s * y;
            jj[r] = s * x + c * y;
          }
          if (lane == 0) {
            atomicAdd(cnt, 1);
            nrm[i] = al - t * ga;
            nrm[j] = be + t * ga;
          }
        }
        __syncwarp();
      }
      jsync();
    }
    int rotations = *((volatile int*)cnt);
    jsync();
    if (gtid == 0) counters[(sweep + 1) & 1] = 0;
    jsync();
    if (rotations == 0) { ++sweep; break; }
  }
  if (gtid == 0) status->jacobi_sweeps = sweep;
  if constexpr (kMode == 2) {
    for (int64_t t = threadIdx.x; t < (int64_t)cols_per * l; t += blockDim.x) {
      const int q = (int)(t / l), r = (int)(t - (int64_t)q * l);
      const int c = q * CS + crank;
      if (c < l) {
        Aout[(int64_t)c * l + r] = A[t];
        Jout[(int64_t)c * l + r] = J[t];
      }
    }
    jsync();  // keep shared memory alive until every remote access is done
  } else if (in_smem) {
    for (int64_t t = threadIdx.x; t < (int64_t)l * l; t += blockDim.x) {
      Aout[t] = A[t];
      Jout[t] = J[t];
    }
  }
}

// Block one-sided Jacobi (cooperative grid of P CTAs): the l columns are cut into 2P blocks of
// b columns; in each outer round CTA p takes the block pair the round-robin tournament gives it,
// loads those 2b columns of A and J into shared memory, runs one inner sweep over all
// (2b choose 2) column pairs there (2b - 1 inner rounds of b disjoint pairs, a warp per pair,
// norms carried as in jacobi_kernel), and writes the columns back; one grid barrier per outer
// round.  Every column pair meets in every outer sweep, so the outer sweep is a (reordered)
// full Jacobi sweep: 2P - 1 grid barriers per sweep instead of l - 1.
constexpr int kJbThreads = 256;

__global__ void __launch_bounds__(kJbThreads) jacobi_block_kernel(const double* __restrict__ R, int l, int b,
                                                                  double* A, double* J, int* counters,
                                                                  DevStatus* status, int max_sweeps) {
  extern __shared__ double smem[];
  cg::grid_group grid = cg::this_grid();
  const int P = gridDim.x, nb = 2 * P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = kJbThreads / 32;
  double* sA = smem;                           // 2b columns of A (l each)
  double* sJ = smem + (int64_t)2 * b * l;      // 2b columns of J
  double* snrm = smem + (int64_t)4 * b * l;    // 2b squared norms
  int* scol = reinterpret_cast<int*>(snrm + 2 * b);  // global column of local slot (or -1)
  for (int64_t t = blockIdx.x * (int64_t)kJbThreads + tid; t < (int64_t)l * l; t += (int64_t)P * kJbThreads) {
    A[t] = R[t];
    const int64_t j = t / l, i = t - j * l;
    J[t] = (i == j) ? 1.0 : 0.0;
  }
  if (blockIdx.x == 0 && tid == 0) { counters[0] = 0; counters[1] = 0; }
  grid.sync();
  const double tol = (double)l * 1.1102230246251565e-16;
  const int m2 = 2 * b;  // local columns (even)
  int sweep = 0;
  for (sweep = 0; sweep < max_sweeps; ++sweep) {
    int* cnt = counters + (sweep & 1);
    for (int round = 0; round < nb - 1; ++round) {
      const int bi = rr_index(blockIdx.x, round, nb), bj = rr_index(nb - 1 - blockIdx.x, round, nb);
      // load the two blocks (slot q < b: block bi, else bj)
      for (int q = tid; q < m2; q += kJbThreads) {
        const int c = (q < b ? bi : bj) * b + (q % b);
        scol[q] = c < l ? c : -1;
      }
      __syncthreads();
      // a warp per column (columns are contiguous): no index division, 16-byte L2 loads (.cg: the
      // columns were written by other CTAs since the last grid barrier), several in flight per lane
      // (round 2: the element loop with a 64-bit division per element made this copy the longest
      // phase of an outer round)
      for (int q = warp; q < m2; q += nw) {
        const int c = scol[q];
        double* la = sA + (int64_t)q * l;
        double* lj = sJ + (int64_t)q * l;
        if (c < 0) {
          for (int r = lane; r < l; r += 32) la[r] = lj[r] = 0.0;
        } else if ((l & 1) == 0) {
          const double2* ga = reinterpret_cast<const double2*>(A + (int64_t)c * l);
          const double2* gj = reinterpret_cast<const double2*>(J + (int64_t)c * l);
#pragma unroll 4
          for (int r = lane; r < l / 2; r += 32) {
            const double2 x = __ldcg(ga + r), y = __ldcg(gj + r);
            reinterpret_cast<double2*>(la)[r] = x;
            reinterpret_cast<double2*>(lj)[r] = y;
          }
        } else {
          for (int r = lane; r < l; r += 32) {
            la[r] = __ldcg(A + (int64_t)c * l + r);
            lj[r] = __ldcg(J + (int64_t)c * l + r);
          }
        }
      }
      __syncthreads();
      for (int q = warp; q < m2; q += nw) {
        const double* a = sA + (int64_t)q * l;
        double v = 0.0;
        for (int r = lane; r < l; r += 32) v += a[r] * a[r];
        v = warp_sum(v);
        if (lane == 0) snrm[q] = v;
      }
      __syncthreads();
      // inner sweep: m2 - 1 rounds of m2 / 2 disjoint pairs
      for (int ir = 0; ir < m2 - 1; ++ir) {
        for (int pp = warp; pp < m2 / 2; pp += nw) {
          int i = rr_index(pp, ir, m2), j = rr_index(m2 - 1 - pp, ir, m2);
          if (scol[i] < 0 || scol[j] < 0) continue;
          if (scol[i] > scol[j]) { const int t = i; i = j; j = t; }  // orient as in the global order
          double* ai = sA + (int64_t)i * l;
          double* aj = sA + (int64_t)j * l;
          double g0 = 0.0, g1 = 0.0;  // two chains: the dot is latency-bound
          int r = lane;
#pragma unroll 4
          for (; r + 32 < l; r += 64) {
            g0 += ai[r] * aj[r];
            g1 += ai[r + 32] * aj[r + 32];
          }
          if (r < l) g0 += ai[r] * aj[r];
          const double ga = warp_sum(g0 + g1);
          const double al = snrm[i], be = snrm[j];
          if (al > 0.0 && be > 0.0 && fabs(ga) > tol * sqrt(al * be)) {
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
#pragma unroll 4
            for (int r2 = lane; r2 < l; r2 += 32) {
              const double x = ai[r2], y = aj[r2];
              ai[r2] = c * x - s * y;
              aj[r2] = s * x + c * y;
            }
            double* ji = sJ + (int64_t)i * l;
            double* jj = sJ + (int64_t)j * l;
#pragma unroll 4
            for (int r2 = lane; r2 < l; r2 += 32) {
              const double x = ji[r2], y = jj[r2];
              ji[r2] = c * x - s * y;
              jj[r2] = s * x + c * y;
            }
            if (lane == 0) {
              atomicAdd(cnt, 1);
              snrm[i] = al - t * ga;
              snrm[j] = be + t * ga;
            }
          }
          __syncwarp();
        }
        __syncthreads();
      }
      for (int q = warp; q < m2; q += nw) {
        const int c = scol[q];
        if (c < 0) continue;
        const double* la = sA + (int64_t)q * l;
        const double* lj = sJ + (int64_t)q * l;
        if ((l & 1) == 0) {
          double2* ga = reinterpret_cast<double2*>(A + (int64_t)c * l);
          double2* gj = reinterpret_cast<double2*>(J + (int64_t)c * l);
#pragma unroll 4
          for (int r = lane; r < l / 2; r += 32) {
            __stcg(ga + r, reinterpret_cast<const double2*>(la)[r]);
            __stcg(gj + r, reinterpret_cast<const double2*>(lj)[r]);
          }
        } else {
          for (int r = lane; r < l; r += 32) {
            __stcg(A + (int64_t)c * l + r, la[r]);
            __stcg(J + (int64_t)c * l + r, lj[r]);
          }
        }
      }
      grid.sync();
    }
    const int rotations = *((volatile int*)cnt);
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) counters[(sweep + 1) & 1] = 0;
    grid.sync();
    if (rotations == 0) { ++sweep; break; }
  }
  if (blockIdx.x == 0 && tid == 0) status->jacobi_sweeps = sweep;
}

// sigma_j = ||A_j||; descending order; Ub = A_perm / sigma, Vb = J_perm (first k columns).
__global__ void __launch_bounds__(1024) jacobi_finish_kernel(const double* __restrict__ A, const double* __restrict__ J,
                                                             int l, int k, int64_t ldk, double* sig_ws,
                                                             double* __restrict__ sigma_k, float* __restrict__ Ub,
                                                             float* __restrict__ Vb, DevStatus* status) {
  __shared__ int perm[1024];  // l <= 1024 (isvd_svd rejects wider)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < l; j += nw) {
    const double* aj = A + (int64_t)j * l;
    double s = 0.0;
    for (int r = lane; r < l; r += 32) s += aj[r] * aj[r];
    s = warp_sum(s);
    if (lane == 0) {
      // a non-finite norm is flagged below and ranked last as -1 so the ranking stays a total order
      // (NaN compares false both ways) and perm[] is a permutation -- no out-of-range gathers
      if (!isfinite(s)) atomicOr(&status->nonfinite, 1);
      sig_ws[j] = isfinite(s) ? sqrt(s) : -1.0;
    }
  }
  __syncthreads();
  for (int j = tid; j < l; j += blockDim.x) {
    double sj = sig_ws[j];
    int rank = 0;
    for (int i = 0; i < l; ++i) {
      double si = sig_ws[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    if (rank < k) perm[rank] = j;
  }
  __syncthreads();
  for (int t = tid; t < k; t += blockDim.x) sigma_k[t] = sig_ws[perm[t]];
  for (int64_t e = tid; e < (int64_t)l * ldk; e += blockDim.x) {
    int64_t r = e / ldk;
    int t = (int)(e - r * ldk);
    float u = 0.f, v = 0.f;
    if (t < k) {
      int j = perm[t];
      double s = sig_ws[j];
      u = s > 0.0 ? (float)(A[(int64_t)j * l + r] / s) : 0.f;
      v = (float)J[(int64_t)j * l + r];
    }
    Ub[e] = u;
    Vb[e] = v;
  }
}

// Rfold = flag ? I : Rinv (l x l in an ld x ld fp32 buffer; padding zero): the factor a deferred
// CholeskyQR2 leaves for its consumers (capi.cpp cqr2_deferred).
__global__ void select_rfold_kernel(const float* __restrict__ Rinv, float* __restrict__ out, int l, int64_t ld,
                                    const int* flag) {
  const bool ident = *((volatile const int*)flag) != 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ld * ld; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld, j = e - (e / ld) * ld;
    float v = 0.f;
    if (i < l && j < l) v = ident ? (i == j ? 1.f : 0.f) : Rinv[e];
    out[e] = v;
  }
}

// ------------------------------------------------------------ sign rule
constexpr int64_t kAbsmaxRows = 4096;

__global__ void col_absmax_partial_kernel(const float* __restrict__ U, int64_t ldu, int64_t rows, int k,
                                          double* __restrict__ part) {
  // blockDim (32, 8)
  const int64_t r0 = blockIdx.x * kAbsmaxRows;
  int64_t r1 = r0 + kAbsmaxRows;
  if (r1 > rows) r1 = rows;
  __shared__ float bv[8][32];
  __shared__ int64_t br[8][32];
  for (int c0 = 0; c0 < k; c0 += 32) {
    int c = c0 + threadIdx.x;
    float best = -1.f;
    int64_t brow = -1;
    if (c < k)
      for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
        float v = fabsf(U[r * ldu + c]);
        if (v > best) { best = v; brow = r; }  // rows visited in increasing order: ties keep the lowest
      }
    bv[threadIdx.y][threadIdx.x] = best;
    br[threadIdx.y][threadIdx.x] = brow;
    __syncthreads();
    if (threadIdx.y == 0 && c < k) {
      float b = -1.f;
      int64_t rb = -1;
      for (int y = 0; y < 8; ++y) {
        float v = bv[y][threadIdx.x];
        int64_t r = br[y][threadIdx.x];
        if (r >= 0 && (v > b || (v == b && r < rb))) { b = v; rb = r; }
      }
      double* o = part + ((int64_t)blockIdx.x * k + c) * 3;
      o[0] = b;
      o[1] = (double)rb;
      o[2] = rb >= 0 ? (U[rb * ldu + c] < 0.f ? -1.0 : 1.0) : 1.0;
    }
    __syncthreads();
  }
}

__global__ void col_absmax_final_kernel(const double* __restrict__ part, int nblocks, int k, int64_t row_offset,
                                        double* __restrict__ cand) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    double b = -1.0, rb = -1.0, sg = 1.0;
    for (int blk = 0; blk < nblocks; ++blk) {
      const double* o = part + ((int64_t)blk * k + c) * 3;
      if (o[1] >= 0.0 && (o[0] > b || (o[0] == b && o[1] < rb))) { b = o[0]; rb = o[1]; sg = o[2]; }
    }
    cand[c * 3 + 0] = b;
    cand[c * 3 + 1] = rb >= 0.0 ? rb + (double)row_offset : -1.0;
    cand[c * 3 + 2] = sg;
  }
}

__global__ void sign_select_kernel(const double* __restrict__ cand, int world, int k, float* __restrict__ sgn) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    double b = -1.0, rb = -1.0, sg = 1.0;
    for (int w = 0; w < world; ++w) {
      const double* o = cand + ((int64_t)w * k + c) * 3;
      if (o[1] >= 0.0 && (o[0] > b || (o[0] == b && o[1] < rb))) { b = o[0]; rb = o[1]; sg = o[2]; }
    }
    sgn[c] = (float)sg;
  }
}

// U[:, c] *= sgn[c]; with `status`, also flags a non-finite entry (the output check of isvd_svd,
// fused here so U is read once).  k % 4 == 0 and ldu % 4 == 0: float4 path.
__global__ void flip_kernel(const float* __restrict__ sgn, int k, float* U, int64_t ldu, int64_t rows,
                            DevStatus* status) {
  int bad = 0;
  if ((k & 3) == 0 && (ldu & 3) == 0) {
    const int k4 = k >> 2;
    const int64_t tot = rows * k4;
    // four independent 16-byte loads in flight per thread
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t0 < tot; t0 += 4 * S) {
      float4* p[4];
      float4 v[4];
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = t0 + u * S;
        p[u] = nullptr;
        if (t < tot) {
          const int64_t i = row_of(t, k4);
          c[u] = (int)(t - i * k4) * 4;
          p[u] = reinterpret_cast<float4*>(U + i * ldu + c[u]);
          v[u] = *p[u];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!p[u]) continue;
        float4 w = v[u];
        w.x *= sgn[c[u]]; w.y *= sgn[c[u] + 1]; w.z *= sgn[c[u] + 2]; w.w *= sgn[c[u] + 3];
        bad |= !isfinite(w.x) | !isfinite(w.y) | !isfinite(w.z) | !isfinite(w.w);
        *p[u] = w;
      }
    }
  } else {
    const int64_t tot = rows * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = row_of(t, k);
      const int c = (int)(t - i * k);
      const float v = U[i * ldu + c] * sgn[c];
      bad |= !isfinite(v);
      U[i * ldu + c] = v;
    }
  }
  if (status && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status->nonfinite, 1);
}

int grid_for(int64_t work, int threads, int cap) {
  int64_t b = (work + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// ------------------------------------------------- cluster Cholesky + inverse (l > kCholSmemMax)
// The l x l matrix is spread over a thread-block cluster (8 CTAs, 16 above l = 400) in
// shared memory, block-cyclic by panels of kPanel rows.  Right-looking blocked Cholesky:
// the owner of panel B factors its kPanel rows locally, the cluster syncs once, every CTA
// copies the panel through DSMEM and applies the rank-kPanel update to its own rows.
// The inverse of R is the blocked Gauss-Jordan back-substitution, in place, with the
// same panel broadcast.  One cluster barrier per panel instead of one grid-wide barrier
// per row.
constexpr int kPanel = 8;

struct ClusterLayout {
  int CS, c, nblk, rows_max;
  ISVD_DEVICE int owner(int i) const { return (i / kPanel) % CS; }
  ISVD_DEVICE int local_row(int i) const { return ((i / kPanel) / CS) * kPanel + (i % kPanel); }
  ISVD_DEVICE int global_row(int r) const { return ((r / kPanel) * CS + c) * kPanel + (r % kPanel); }
};

// probe_tol > 0 (probe mode, for a Gram with fp32-class error): a breakdown, or a pivot spread
// min_k r_kk^2 < probe_tol * max_k r_kk^2 (kappa(Y)^2 too large for that Gram), sets *probe_flag
// instead of shifting; the caller then recomputes the Gram exactly and refactors (gated on the flag).
__global__ void __launch_bounds__(512) chol_inv_cluster_kernel(const double* __restrict__ G, int64_t ldg, int l,
                                                               int64_t ld, float* __restrict__ Rinv32,
                                                               double* __restrict__ R64, DevStatus* status,
                                                               int force_fail, const int* gate, double probe_tol,
                                                               int* probe_flag) {
  if (gate && *((volatile const int*)gate) == 0) return;  // same value for every CTA of the cluster
  cg::cluster_group cl = cg::this_cluster();
  ClusterLayout L;
  L.CS = (int)cl.num_blocks();
  L.c = (int)cl.block_rank();
  L.nblk = (l + kPanel - 1) / kPanel;
  L.rows_max = ((L.nblk + L.CS - 1) / L.CS) * kPanel;
  extern __shared__ double sm[];
  double* A = sm;                                  // rows_max x l (own rows)
  double* P = sm + (size_t)L.rows_max * l;         // kPanel x l (panel copy)
  double* colk = P + (size_t)kPanel * l;           // rows_max x kPanel
  __shared__ double s_misc[4];
  __shared__ double s_pinv[kPanel], s_pblk[kPanel * kPanel];  // in-panel: 1 / r_kk, the diagonal block
  __shared__ double s_pmin, s_pmax;  // pivots factored by this CTA (probe mode)
  __shared__ int s_bad, s_remote_bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int my_rows = ((L.nblk - L.c + L.CS - 1) / L.CS) * kPanel;
  if (tid == 0) {
    s_pmin = INFINITY;
    s_pmax = 0.0;
  }

  if (tid == 0) {
    double tr = 0.0, mx = 0.0;
    for (int i = 0; i < l; ++i) {
      double d = G[(int64_t)i * ldg + i];
      tr += d;
      mx = d > mx ? d : mx;
    }
    s_misc[1] = tr;
    s_misc[2] = mx;
  }
  __syncthreads();
  const double trace = s_misc[1], tol = 1e-14 * s_misc[2];
  double shift = 0.0;
  int attempt, failed = 1;
  for (attempt = 0; attempt < 4; ++attempt) {
    cl.sync();  // nobody still reads our rows from a previous attempt
    for (int t = tid; t < my_rows * l; t += nt) {
      int r = t / l, j = t - r * l;
      int gi = L.global_row(r);
      double v = 0.0;
      if (gi < l && j >= gi) v = G[(int64_t)gi * ldg + j] + (j == gi ? shift : 0.0);
      A[t] = v;
    }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    int bad = 0;
    for (int B = 0; B < L.nblk; ++B) {
      const int own = B % L.CS, k0 = B * kPanel, kend = min(k0 + kPanel, l);
      const int lb = (B / L.CS) * kPanel;
      if (L.c == own) {
        // In-panel factorisation without a CTA barrier per column (round 2; the column-by-column
        // form took 3 barriers and a serial pivot per column, 400 of them at l = 400): thread 0
        // factors the nb x nb diagonal block in registers, then every other column of the panel
        // is an independent nb-step forward substitution, one thread per column.  The operations
        // on each entry and their order are those of the column-by-column form.
        const int nbo = kend - k0;
        if (tid == 0) {
          double D[kPanel][kPanel];
#pragma unroll
          for (int a = 0; a < kPanel; ++a)
#pragma unroll
            for (int b = 0; b < kPanel; ++b)
              D[a][b] = (a < nbo && b < nbo && b >= a) ? A[(size_t)(lb + a) * l + k0 + b] : 0.0;
#pragma unroll
          for (int a = 0; a < kPanel; ++a) {
            if (a < nbo) {
              const double piv = D[a][a];
              const int b_ = !(piv > tol) || !isfinite(piv);
              if (b_) s_bad = 1;
              s_pmin = fmin(s_pmin, piv);
              s_pmax = fmax(s_pmax, piv);
              const double rr = b_ ? 1.0 : sqrt(piv);
              const double inv = 1.0 / rr;
              D[a][a] = rr;
              s_pinv[a] = inv;
#pragma unroll
              for (int b = a + 1; b < kPanel; ++b) D[a][b] *= inv;
#pragma unroll
              for (int a2 = a + 1; a2 < kPanel; ++a2)
#pragma unroll
                for (int b = a2; b < kPanel; ++b) D[a2][b] -= D[a][a2] * D[a][b];
            }
          }
#pragma unroll
          for (int a = 0; a < kPanel; ++a)
#pragma unroll
            for (int b = 0; b < kPanel; ++b) {
              if (a < nbo && b < nbo && b >= a) A[(size_t)(lb + a) * l + k0 + b] = D[a][b];
              s_pblk[a * kPanel + b] = D[a][b];
            }
        }
        __syncthreads();
        for (int j = kend + tid; j < l; j += nt) {
          double v[kPanel];
#pragma unroll
          for (int a = 0; a < kPanel; ++a) v[a] = a < nbo ? A[(size_t)(lb + a) * l + j] : 0.0;
#pragma unroll
          for (int a = 0; a < kPanel; ++a) {
            if (a < nbo) {
              v[a] *= s_pinv[a];
#pragma unroll
              for (int a2 = a + 1; a2 < kPanel; ++a2) v[a2] -= s_pblk[a * kPanel + a2] * v[a];
            }
          }
#pragma unroll
          for (int a = 0; a < kPanel; ++a)
            if (a < nbo) A[(size_t)(lb + a) * l + j] = v[a];
        }
        __syncthreads();
      }
      cl.sync();  // panel B final
      const double* rem = cl.map_shared_rank(A, own) + (size_t)lb * l;
      if (tid == 0) s_remote_bad = *cl.map_shared_rank(&s_bad, own);
      const int nb = kend - k0;
      {  // warp w copies panel row w % kPanel (two warps per row at 512 threads)
        const int w = tid >> 5, q = w % kPanel, part = w / kPanel, parts = (nt >> 5) / kPanel;
        if (q < nb && part < parts)
          for (int j = k0 + part * 32 + (tid & 31); j < l; j += 32 * parts) P[(size_t)q * l + j] = rem[(size_t)q * l + j];
      }
      __syncthreads();
      if (s_remote_bad) { bad = 1; break; }
      // rank-nb update of own rows i >= kend, columns j >= i
      // (a warp per row, lanes over its columns j >= i: no index division per entry)
      for (int r = tid >> 5; r < my_rows; r += nt >> 5) {
        const int gi = L.global_row(r);
        if (gi < kend || gi >= l) continue;
        double pg[kPanel];
#pragma unroll
        for (int q = 0; q < kPanel; ++q) pg[q] = q < nb ? P[(size_t)q * l + gi] : 0.0;
        for (int j = gi + (tid & 31); j < l; j += 32) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < kPanel; ++q)
            if (q < nb) s += pg[q] * P[(size_t)q * l + j];
          A[(size_t)r * l + j] -= s;
        }
      }
      __syncthreads();
    }
    if (force_fail && attempt == 0) bad = 1;
    if (probe_tol > 0.0) {  // probe mode: never shift; flag breakdown or a too-wide pivot spread
      cl.sync();
      if (L.c == 0 && tid == 0) {
        double pmin = INFINITY, pmax = 0.0;
        for (int q = 0; q < L.CS; ++q) {
          pmin = fmin(pmin, *cl.map_shared_rank(&s_pmin, q));
          pmax = fmax(pmax, *cl.map_shared_rank(&s_pmax, q));
        }
        if (bad || !(pmin >= probe_tol * pmax)) {
          *probe_flag = 1;
          atomicAdd(&status->probes_failed, 1);
        }
      }
      failed = 0;
      break;
    }
    if (!bad) { failed = 0; break; }
    shift = (attempt == 0) ? 1e-10 * trace : shift * 100.0;
  }
  if (L.c == 0 && tid == 0 && probe_tol <= 0.0) {
    if (attempt > 0) {
      atomicAdd(&status->chol_breakdown, 1);
      status->need_extra_pass = 1;
    }
    if (failed) status->chol_failed = 1;
  }
  if (R64) {
    for (int t = tid; t < my_rows * l; t += nt) {
      int r = t / l, j = t - r * l;
      int gi = L.global_row(r);
      if (gi < l) R64[(int64_t)gi * l + j] = A[t];
    }
  }
  // ---- blocked Gauss-Jordan inverse, in place, panels from the bottom
  for (int B = L.nblk - 1; B >= 0; --B) {
    const int own = B % L.CS, k0 = B * kPanel, kend = min(k0 + kPanel, l);
    const int lb = (B / L.CS) * kPanel;
    const int nb = kend - k0;
    // rows of a panel are final once its owner factored them; only the switch from the
    // Cholesky (whose last panel is still being read) to the inverse needs a barrier
    if (B == L.nblk - 1) cl.sync();
    if (L.c == own) {
      // the panel's own Gauss-Jordan steps, as above: thread 0 transforms the nb x nb diagonal block
      // in registers (keeping the original block for the others), then one thread per remaining
      // column runs the nb-step back substitution
      __syncthreads();
      if (tid == 0) {
        double D[kPanel][kPanel];
#pragma unroll
        for (int a = 0; a < kPanel; ++a)
#pragma unroll
          for (int b = 0; b < kPanel; ++b) {
            D[a][b] = (a < nb && b < nb && b >= a) ? A[(size_t)(lb + a) * l + k0 + b] : 0.0;
            s_pblk[a * kPanel + b] = D[a][b];
          }
#pragma unroll
        for (int a = kPanel - 1; a >= 0; --a) {
          if (a < nb) {
            const double inv = 1.0 / D[a][a];
            s_pinv[a] = inv;
#pragma unroll
            for (int b = a + 1; b < kPanel; ++b) D[a][b] *= inv;
            D[a][a] = inv;
#pragma unroll
            for (int q = 0; q < a; ++q) {
              const double rik = D[q][a];
#pragma unroll
              for (int b = a; b < kPanel; ++b) D[q][b] = (b == a) ? -rik * inv : D[q][b] - rik * D[a][b];
            }
          }
        }
#pragma unroll
        for (int a = 0; a < kPanel; ++a)
#pragma unroll
          for (int b = 0; b < kPanel; ++b)
            if (a < nb && b < nb && b >= a) A[(size_t)(lb + a) * l + k0 + b] = D[a][b];
      }
      __syncthreads();
      for (int j = kend + tid; j < l; j += nt) {
        double v[kPanel];
#pragma unroll
        for (int a = 0; a < kPanel; ++a) v[a] = a < nb ? A[(size_t)(lb + a) * l + j] : 0.0;
#pragma unroll
        for (int a = kPanel - 1; a >= 0; --a) {
          if (a < nb) {
            v[a] *= s_pinv[a];
#pragma unroll
            for (int q = 0; q < a; ++q) v[q] -= s_pblk[q * kPanel + a] * v[a];
          }
        }
#pragma unroll
        for (int a = 0; a < kPanel; ++a)
          if (a < nb) A[(size_t)(lb + a) * l + j] = v[a];
      }
      __syncthreads();
    }
    cl.sync();  // panel rows of X final
    const double* rem = cl.map_shared_rank(A, own) + (size_t)lb * l;
    {
      const int w = tid >> 5, q = w % kPanel, part = w / kPanel, parts = (nt >> 5) / kPanel;
      if (q < nb && part < parts)
        for (int j = k0 + part * 32 + (tid & 31); j < l; j += 32 * parts) P[(size_t)q * l + j] = rem[(size_t)q * l + j];
    }
    // save R[i][k0..kend) of own rows i < k0
    for (int t = tid; t < my_rows * kPanel; t += nt) {
      int r = t / kPanel, q = t - r * kPanel;
      int gi = L.global_row(r);
      colk[t] = (gi < k0 && q < nb) ? A[(size_t)r * l + k0 + q] : 0.0;
    }
    __syncthreads();
    for (int r = tid >> 5; r < my_rows; r += nt >> 5) {
      const int gi = L.global_row(r);
      if (gi >= k0) continue;
      double ck[kPanel];
#pragma unroll
      for (int q = 0; q < kPanel; ++q) ck[q] = colk[(size_t)r * kPanel + q];
      for (int j = k0 + (tid & 31); j < l; j += 32) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kPanel; ++q)
          if (q < nb && k0 + q <= j) s += ck[q] * P[(size_t)q * l + j];
        double* a = A + (size_t)r * l + j;
        *a = (j >= kend ? *a : 0.0) - s;
      }
    }
    __syncthreads();
  }
  // ---- R^-1 -> fp32, upper, zero padded (ld x ld)
  for (int t = tid; t < my_rows * ld; t += nt) {
    int r = (int)(t / ld);
    int64_t j = t - (int64_t)r * ld;
    int gi = L.global_row(r);
    if (gi >= l) continue;
    Rinv32[(int64_t)gi * ld + j] = (j < l && j >= gi) ? (float)A[(size_t)r * l + j] : 0.f;
  }
  if (L.c == 0)
    for (int64_t t = tid; t < (ld - l) * ld; t += nt) Rinv32[(int64_t)l * ld + t] = 0.f;
  cl.sync();  // keep every CTA's shared memory alive until all remote reads are done
}

}  // namespace

cudaError_t launch_chol_inv(const double* G, int64_t ldg, int l, int64_t ld, float* Rinv32, double* R64, double* ws,
                            DevStatus* status, bool force_fail, const int* gate, cudaStream_t st, double probe_tol,
                            int* probe_flag) {
  // Blocked (panel) algorithm: one CTA for l <= kCholSmemMax (whole matrix in its shared
  // memory), a cluster of 8 / 16 CTAs sharing it through DSMEM above that.
  if (l <= 512 && !getenv("ISVD_CHOL_UNBLOCKED")) {
    int CS = l <= kCholSmemMax ? 1 : (l <= 400 ? 8 : 16);
    if (const char* e = getenv("ISVD_CHOL_CLUSTER"))  // tuning override: 8 or 16 (l > kCholSmemMax)
      if (l > kCholSmemMax && (atoi(e) == 8 || atoi(e) == 16)) CS = atoi(e);
    const int nblk = (l + kPanel - 1) / kPanel;
    const int rows_max = ((nblk + CS - 1) / CS) * kPanel;
    size_t smem = sizeof(double) * ((size_t)rows_max * l + (size_t)kPanel * l + (size_t)rows_max * kPanel);
    static bool cattr = false;
    if (!cattr) {
      cudaFuncSetAttribute(chol_inv_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      cudaFuncSetAttribute(chol_inv_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cattr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ++g_launches;
    return cudaLaunchKernelEx(&cfg, chol_inv_cluster_kernel, G, ldg, l, ld, Rinv32, R64, status,
                              force_fail ? 1 : 0, gate, probe_tol, probe_flag);
  }
  size_t smem = (l <= kCholSmemMax) ? sizeof(double) * (size_t)l * l : 0;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * kCholSmemMax * kCholSmemMax));
    attr_set = true;
  }
  ++g_launches; chol_inv_kernel<<<1, 1024, smem, st>>>(G, ldg, l, ld, Rinv32, R64, ws, status, force_fail ? 1 : 0, gate);
  return cudaGetLastError();
}

cudaError_t launch_trmm(const double* Rnew, const double* Racc, double* out, int l, const int* gate, cudaStream_t st) {
  ++g_launches; trmm_kernel<<<l, 128, 0, st>>>(Rnew, Racc, out, l, gate);
  return cudaGetLastError();
}

int64_t jacobi_ws_doubles(int l) { return 4LL * l * l + 2LL * l + 64; }

cudaError_t launch_jacobi_svd(const double* R, int l, int k, int64_t ldk, double* sigma_k, float* Ub, float* Vb,
                              double* ws, DevStatus* status, int num_sms, cudaStream_t st) {
  double* A = ws;
  double* J = ws + (int64_t)l * l;
  double* Aout = ws + 2LL * l * l;  // smem path copies results here
  double* Jout = ws + 3LL * l * l;
  double* sig = ws + 4LL * l * l;
  double* nrm = ws + 4LL * l * l + l;  // column norms of the cooperative variant
  int* counters = reinterpret_cast<int*>(ws + 4LL * l * l + 2LL * l);
  const int max_sweeps = 60;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(jacobi_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(jacobi_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(jacobi_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_set = true;
  }
  bool done = false;
  if (l <= 112) {
    size_t smem = 2 * (size_t)l * l * sizeof(double);
    ++g_launches;
    jacobi_kernel<0><<<1, 1024, smem, st>>>(R, l, A, J, counters, status, max_sweeps, Aout, Jout, nrm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    done = true;
  } else if (l <= 448 && getenv("ISVD_JACOBI_CLUSTER")) {
    // measured slower than the cooperative-grid variant at l = 160 / 256 / 400 (DSMEM
    // column reads per pair); kept behind a switch for experiments
    // cluster: the smallest cluster (8, else 16 CTAs) whose shared memory holds A and J
    for (int CS : {8, 16}) {
      const int cols_per = (l + CS - 1) / CS;
      const size_t smem = 2 * (size_t)cols_per * l * sizeof(double);
      if (smem > 200 * 1024) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CS);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CS;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      ++g_launches;
      cudaError_t e = cudaLaunchKernelEx(&cfg, jacobi_kernel<2>, R, l, A, J, counters, status, max_sweeps, Aout,
                                         Jout, nrm);
      if (e == cudaSuccess) {
        done = true;
        break;
      }
      --g_launches;
      (void)cudaGetLastError();
    }
  }
  if (!done && !getenv("ISVD_JACOBI_PAIRWISE")) {
    // block Jacobi: blocks of b columns, 2P blocks, P CTAs.  b = 8 gives each of the 8 warps one
    // pair per inner round; b = 4 when 16 columns of A and J do not fit 200 KB of shared memory
    for (int b : {8, 4}) {
      const int P = (int)ceil_div(l, 2 * b);
      const size_t smem = (size_t)(4 * b * l + 2 * b) * sizeof(double) + 2 * b * sizeof(int);
      if (smem > 200 * 1024 || P > num_sms) continue;
      static bool battr = false;
      if (!battr) {
        cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        battr = true;
      }
      void* args[] = {(void*)&R, (void*)&l, (void*)&b, (void*)&A, (void*)&J, (void*)&counters, (void*)&status,
                      (void*)&max_sweeps};
      ++g_launches;
      cudaError_t e = cudaLaunchCooperativeKernel((const void*)jacobi_block_kernel, dim3(P), dim3(kJbThreads), args,
                                                  smem, st);
      if (e != cudaSuccess) {
        --g_launches;
        (void)cudaGetLastError();
        continue;
      }
      Aout = A;
      Jout = J;
      done = true;
      break;
    }
  }
  if (!done) {
    int m = (l & 1) ? l + 1 : l;
    int warps_needed = m / 2;
    int threads = 256;
    int blocks = (warps_needed * 32 + threads - 1) / threads;
    if (blocks > num_sms) blocks = num_sms;
    void* args[] = {(void*)&R, (void*)&l, (void*)&A, (void*)&J, (void*)&counters, (void*)&status,
                    (void*)&max_sweeps, (void*)&A, (void*)&J, (void*)&nrm};
    ++g_launches;
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)jacobi_kernel<1>, dim3(blocks), dim3(threads), args,
                                                0, st);
    if (e != cudaSuccess) return e;
    Aout = A;
    Jout = J;
  }
  ++g_launches; jacobi_finish_kernel<<<1, 1024, 0, st>>>(Aout, Jout, l, k, ldk, sig, sigma_k, Ub, Vb, status);
  return cudaGetLastError();
}

cudaError_t launch_select_rfold(const float* Rinv, float* out, int l, int64_t ld, const int* flag, cudaStream_t st) {
  ++g_launches; select_rfold_kernel<<<grid_for(ld * ld, 256, 148), 256, 0, st>>>(Rinv, out, l, ld, flag);
  return cudaGetLastError();
}

int64_t absmax_ws_doubles(int64_t rows, int k) { return (ceil_div(rows, kAbsmaxRows) + 1) * k * 3; }

cudaError_t launch_col_absmax(const float* U, int64_t ldu, int64_t rows, int k, int64_t row_offset, double* ws,
                              double* cand, cudaStream_t st) {
  int64_t nb = ceil_div(rows, kAbsmaxRows);
  if (nb < 1) {
    // no local rows: candidates with row -1
    ++g_launches; col_absmax_final_kernel<<<1, 256, 0, st>>>(ws, 0, k, row_offset, cand);
    return cudaGetLastError();
  }
  ++g_launches; col_absmax_partial_kernel<<<(unsigned)nb, dim3(32, 8), 0, st>>>(U, ldu, rows, k, ws);
  ++g_launches; col_absmax_final_kernel<<<grid_for(k, 256, 16), 256, 0, st>>>(ws, (int)nb, k, row_offset, cand);
  return cudaGetLastError();
}

cudaError_t launch_sign_flip(const double* cand, int world, int k, float* sgn_ws, float* U, int64_t ldu, int64_t rows,
                             float* V, int64_t ldv, int64_t vrows, cudaStream_t st, DevStatus* status) {
  ++g_launches; sign_select_kernel<<<grid_for(k, 256, 16), 256, 0, st>>>(cand, world, k, sgn_ws);
  if (rows > 0) {
    ++g_launches; flip_kernel<<<grid_for(rows * k, 256, 148 * 8), 256, 0, st>>>(sgn_ws, k, U, ldu, rows, status);
  }
  if (vrows > 0) {
    ++g_launches; flip_kernel<<<grid_for(vrows * k, 256, 148 * 8), 256, 0, st>>>(sgn_ws, k, V, ldv, vrows, nullptr);
  }
  return cudaGetLastError();
}

}  // namespace isvd
