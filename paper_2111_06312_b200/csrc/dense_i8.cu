// Exact dense-adjacency product on the INT8 tensor cores (the dense-T NE comparison).
//
// For an unweighted graph A is binary, so A Y needs no rounding in the products at all: every
// product A_ij Y_j is Y_j or 0.  The rounding of the 3xTF32 variant (gram_tc.cu) comes from the
// tensor core's truncating fp32 accumulation over K = n (config 3: n = 4267, 625 neighbours per row,
// and a result that cancels against the rank-1 term of Eq. 3), which misses this suite's per-column
// bar at config 3.  Here the accumulation is exact instead:
//   * each column c of the gather source Y is put on a fixed-point grid: with m_c = max_j |Y_jc| =
//     f 2^E (f in [0.5, 1)), q_jc = rint(Y_jc 2^(22 - E)) is an integer with |q| <= 2^22, i.e. Y_jc to
//     within 2^-23 of the column's largest entry (an fp32 Y carries 2^-24 relative to its own value);
//   * q = 65536 s2 + 256 u1 + u0 with u0, u1 in [0, 255] (unsigned bytes) and s2 in [-64, 64]
//     (a signed byte): three int8 slices, written K-major (slice s, column c, row j) by quant_kernel;
//   * tcgen05.mma.kind::i8 forms D_s = A Q_s with A as unsigned bytes (0 / 1) and int32 accumulation,
//     exact while K * 255 < 2^31 (K <= 8.4M); three TMEM accumulators, one per slice;
//   * the drain combines D_2 65536 + D_1 256 + D_0 (an integer < 2^39) in fp64, exactly; split-K
//     partials are summed in fp64 (still exact integers) and scaled by 2^(E - 22) (exact) in the
//     SpMM epilogue (spmm.cu), which then applies 1/d, the Horner term and the rank-1 correction in
//     fp64 exactly as the CSR kernel does.
// So A Y is computed exactly for the fixed-point Y; the only rounding is the 23-bit quantisation
// of Y and the epilogue's usual fp64 -> fp32 store.
//
// Operand staging: A (n x n bytes, K-major: A = A^T, row i = the neighbours of i) and the slices
// (3 Wr x n bytes, K-major) are loaded by TMA with SWIZZLE_64B, 64 K-bytes per stage: the UMMA
// K-major SWIZZLE_64B canonical layout (8-row atoms of 512 B), the same byte geometry as the tf32
// operands of gemm_tc.cu; an MMA (K = 32 bytes) advances 32 B inside the swizzled row.
#include <algorithm>

#include "common.cuh"
#include "umma.cuh"

namespace isvd {
namespace {

constexpr int kIM = 128;       // output rows per tile (UMMA M)
constexpr int kIK = 64;        // K bytes per pipeline stage (one SWIZZLE_64B row)
constexpr int kIStages = 5;
constexpr int kIThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2..5 drain (TMEM lane quadrants)
constexpr uint32_t kSw64 = 4;

// kind::i8 instruction descriptor: S32 accumulate, A unsigned bytes, B unsigned / signed, M x N
__host__ __device__ constexpr uint32_t i8_idesc(int M, int N, bool b_signed) {
  return (2u << 4) | (0u << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

ISVD_DEVICE void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// column maxima of |Y| as float bits (non-negative floats order like their bit patterns)
__global__ void colmax_kernel(const float* __restrict__ Y, int64_t ldy, int64_t n, int w, unsigned* __restrict__ cmax) {
  const int64_t r0 = (int64_t)blockIdx.x * 128;
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    float m = 0.f;
    for (int64_t r = r0; r < r0 + 128 && r < n; ++r) m = fmaxf(m, fabsf(Y[r * ldy + c]));
    atomicMax(cmax + c, __float_as_uint(m));
  }
}

// exponent E of the column maximum (m = f 2^E, f in [0.5, 1)); -1000 for an all-zero column
ISVD_DEVICE int col_exp(unsigned bits) {
  const float m = __uint_as_float(bits);
  if (!(m > 0.f)) return -1000;
  int e;
  frexpf(m, &e);
  return e;
}

// Q_s[c][j] (s = 0, 1, 2; c < Wr; j < n, row length kp bytes): the three byte slices of the
// fixed-point Y, K-major.  Block: 128 rows j x 32 columns c, transposed through shared memory.
__global__ void __launch_bounds__(256) quant_kernel(const float* __restrict__ Y, int64_t ldy, int64_t n, int w, int Wr,
                                                    const unsigned* __restrict__ cmax, uint8_t* __restrict__ Q,
                                                    int64_t kp) {
  __shared__ __align__(16) uint8_t t[3][32][128 + 16];
  const int64_t j0 = (int64_t)blockIdx.x * 128;
  const int c0 = blockIdx.y * 32;
  for (int e = threadIdx.x; e < 128 * 32; e += 256) {
    const int jj = e >> 5, cc = e & 31;
    const int64_t j = j0 + jj;
    const int c = c0 + cc;
    int q = 0;
    if (j < n && c < w) {
      const int E = col_exp(cmax[c]);
      const float y = Y[j * ldy + c];
      if (E > -1000 && isfinite(y) && isfinite(__uint_as_float(cmax[c]))) q = __float2int_rn(ldexpf(y, 22 - E));
    }
    t[0][cc][jj] = (uint8_t)(q & 0xFF);
    t[1][cc][jj] = (uint8_t)((q >> 8) & 0xFF);
    t[2][cc][jj] = (uint8_t)(int8_t)(q >> 16);
  }
  __syncthreads();
  const int64_t nbytes = kp - j0 < 128 ? kp - j0 : 128;  // this block's bytes of each slice row
  for (int e = threadIdx.x; e < 3 * 32 * 8; e += 256) {
    const int s = e / 256, rem = e % 256, cc = rem >> 3, v = rem & 7;
    const int c = c0 + cc;
    if (c >= Wr || 16 * v >= nbytes) continue;
    *reinterpret_cast<uint4*>(Q + ((int64_t)s * Wr + c) * kp + j0 + 16 * v) =
        *reinterpret_cast<const uint4*>(&t[s][cc][16 * v]);
  }
}

template <int N>
struct ICfg {
  static constexpr int A_B = kIM * kIK;   // 8 KB
  static constexpr int B_B = N * kIK;     // one slice box
  static constexpr int STAGE_B = A_B + 3 * B_B;
  static constexpr size_t smem_bytes() { return (size_t)kIStages * STAGE_B + 1024; }
};

// grid (m tiles x n tiles, parts): tile (m0, n0) over K range [k_begin, k_end) of this part; writes
// fp64 integer partials ws[part][row][col] (row < m_tiles 128, col < ntn N).
template <int N>
__global__ void __launch_bounds__(kIThreads, 1)
    dense_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmQ, int64_t n, int Wr,
                    int ntn, int64_t k_per_part, double* __restrict__ ws, int64_t ws_rows, int64_t ws_ld) {
  using C = ICfg<N>;
  static_assert(N % 16 == 0 && N >= 16 && N <= 160, "3 N TMEM columns");
  constexpr uint32_t kCols = 3 * N <= 128 ? 128 : (3 * N <= 256 ? 256 : 512);
  extern __shared__ uint8_t smraw[];
  uint8_t* const base = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kIStages], empty[kIStages], done;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x;
  const int m0 = (tile / ntn) * kIM, n0 = (tile % ntn) * N;
  const int64_t kb = (int64_t)blockIdx.y * k_per_part;
  const int64_t ke = kb + k_per_part < n ? kb + k_per_part : n;
  const int nst = ke > kb ? (int)((ke - kb + kIK - 1) / kIK) : 0;

  if (tid == 0) {
    for (int i = 0; i < kIStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {
      for (int st = 0; st < nst; ++st) {
        const int s = st % kIStages;
        if (st >= kIStages) mbar_wait(&empty[s], (uint32_t)((st / kIStages - 1) & 1));
        uint8_t* const p = base + s * C::STAGE_B;
        const int k0 = (int)(kb + (int64_t)st * kIK);
        mbar_expect_tx(&full[s], (uint32_t)C::STAGE_B);
        tma_2d(p, &tmA, k0, m0, &full[s]);
#pragma unroll
        for (int q = 0; q < 3; ++q) tma_2d(p + C::A_B + q * C::B_B, &tmQ, k0, q * Wr + n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idu = i8_idesc(kIM, N, false), ids = i8_idesc(kIM, N, true);
      for (int st = 0; st < nst; ++st) {
        const int s = st % kIStages;
        mbar_wait(&full[s], (uint32_t)((st / kIStages) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a = smem_u32(base + s * C::STAGE_B), b = a + C::A_B;
#pragma unroll
        for (int kk = 0; kk < kIK / 32; ++kk) {
          const uint32_t ko = (uint32_t)kk * 32;
          const uint64_t da = umma_desc(a + ko, 16, 512, kSw64);
#pragma unroll
          for (int q = 0; q < 3; ++q)
            mma_i8(tmem + (uint32_t)(q * N), da, umma_desc(b + q * C::B_B + ko, 16, 512, kSw64), q == 2 ? ids : idu,
                   (st == 0 && kk == 0) ? 0u : 1u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(&done);
    }
  } else {
    // drain: warp w reads TMEM lanes 32 (w % 4) .. +31 = tile rows; combine the slices exactly
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32;
    const int64_t row = m0 + lane_base + lane;
    double* const out = ws + ((int64_t)blockIdx.y * ws_rows + row) * ws_ld + n0;
    if (nst > 0) {
      mbar_wait(&done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
#pragma unroll 1
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[3][8];
      if (nst > 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                       : "=r"(r[q][0]), "=r"(r[q][1]), "=r"(r[q][2]), "=r"(r[q][3]), "=r"(r[q][4]), "=r"(r[q][5]),
                         "=r"(r[q][6]), "=r"(r[q][7])
                       : "r"(tmem + (lane_base << 16) + (uint32_t)(q * N + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int u = 0; u < 8; ++u) r[q][u] = 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const double v0 = 65536.0 * (double)(int)r[2][u] + 256.0 * (double)(int)r[1][u] + (double)(int)r[0][u];
        const double v1 =
            65536.0 * (double)(int)r[2][u + 1] + 256.0 * (double)(int)r[1][u + 1] + (double)(int)r[0][u + 1];
        *reinterpret_cast<double2*>(out + c0 + u) = make_double2(v0, v1);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

struct ITiling {
  int N, ntn, mt, parts;
  int64_t Wr, kp, k_per_part;
};

ITiling i_tiling(int64_t n, int64_t w, int num_sms) {
  ITiling t{};
  t.ntn = (int)ceil_div(w, 160);
  t.N = (int)round_up(ceil_div(w, t.ntn), 16);
  t.Wr = (int64_t)t.ntn * t.N;
  t.kp = round_up(std::max<int64_t>(n, 1), 16);
  t.mt = (int)ceil_div(std::max<int64_t>(n, 1), kIM);
  const int tiles = t.mt * t.ntn;
  int parts = std::max(1, num_sms / tiles);
  t.k_per_part = round_up(ceil_div(std::max<int64_t>(n, 1), parts), kIK);
  t.parts = (int)ceil_div(std::max<int64_t>(n, 1), t.k_per_part);
  return t;
}

template <int N>
cudaError_t launch_i8_n(const ITiling& t, const uint8_t* A, int64_t lda, const uint8_t* Q, int64_t n, double* ws,
                        cudaStream_t st) {
  CUtensorMap tmA, tmQ;
  if (!make_map_u8(&tmA, A, n, n, lda, kIK, kIM, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map_u8(&tmQ, Q, 3 * t.Wr, n, t.kp, kIK, N, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  const size_t smem = ICfg<N>::smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dense_i8_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  ++g_launches;
  dense_i8_kernel<N><<<dim3((unsigned)(t.mt * t.ntn), (unsigned)t.parts), kIThreads, smem, st>>>(
      tmA, tmQ, n, (int)t.Wr, t.ntn, t.k_per_part, ws, (int64_t)t.mt * kIM, t.Wr);
  return cudaGetLastError();
}

}  // namespace

int64_t dense_i8_ws_bytes(int64_t n, int64_t w, int num_sms, int64_t* q_bytes) {
  const ITiling t = i_tiling(n, w, num_sms);
  *q_bytes = 3 * t.Wr * t.kp;
  return (int64_t)t.parts * t.mt * kIM * t.Wr * (int64_t)sizeof(double) + 4 * round_up(std::max<int64_t>(w, 1), 4);
}

cudaError_t launch_dense_i8(const uint8_t* A, int64_t lda, int64_t n, const float* Y, int64_t ldy, int64_t w,
                            uint8_t* Qws, void* ws, int num_sms, cudaStream_t st, int64_t* parts, int64_t* ws_rows,
                            int64_t* ws_ld, const unsigned** cmax_out, const double** part_out) {
  const ITiling t = i_tiling(n, w, num_sms);
  double* const parts_ws = static_cast<double*>(ws);
  unsigned* const cmax = reinterpret_cast<unsigned*>(parts_ws + (int64_t)t.parts * t.mt * kIM * t.Wr);
  *parts = t.parts;
  *ws_rows = (int64_t)t.mt * kIM;
  *ws_ld = t.Wr;
  *cmax_out = cmax;
  *part_out = parts_ws;
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(unsigned) * (size_t)w, st);
  if (e != cudaSuccess) return e;
  ++g_launches;
  colmax_kernel<<<(unsigned)ceil_div(n, 128), 256, 0, st>>>(Y, ldy, n, (int)w, cmax);
  ++g_launches;
  quant_kernel<<<dim3((unsigned)ceil_div(n, 128), (unsigned)ceil_div(t.Wr, 32)), 256, 0, st>>>(Y, ldy, n, (int)w,
                                                                                              (int)t.Wr, cmax, Qws, t.kp);
  switch (t.N) {
    case 16: return launch_i8_n<16>(t, A, lda, Qws, n, parts_ws, st);
    case 32: return launch_i8_n<32>(t, A, lda, Qws, n, parts_ws, st);
    case 48: return launch_i8_n<48>(t, A, lda, Qws, n, parts_ws, st);
    case 64: return launch_i8_n<64>(t, A, lda, Qws, n, parts_ws, st);
    case 80: return launch_i8_n<80>(t, A, lda, Qws, n, parts_ws, st);
    case 96: return launch_i8_n<96>(t, A, lda, Qws, n, parts_ws, st);
    case 112: return launch_i8_n<112>(t, A, lda, Qws, n, parts_ws, st);
    case 128: return launch_i8_n<128>(t, A, lda, Qws, n, parts_ws, st);
    case 144: return launch_i8_n<144>(t, A, lda, Qws, n, parts_ws, st);
    default: return launch_i8_n<160>(t, A, lda, Qws, n, parts_ws, st);
  }
}

}  // namespace isvd
