// Tensor-core tall GEMM  C[map(i), j] = alpha s_i sum_k A[i, k] B[k, j]  on tcgen05, 3xTF32, for
//   * the NC blocks X G_j of M G (Eq. 6; A = X, K = d),
//   * the CholeskyQR update Y R^-1 (Alg. 2 right; A = Y, K = l),
//   * the final U = Q U_hat (Alg. 1 step 9; A = Q, K = l).
// A is tall (rows x K fp32, row-major, i.e. K-major for UMMA), B is small (K x N).
//
// 3xTF32 as in gram_tc.cu: a*b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi, where the tensor core itself
// truncates an fp32 operand to TF32 (measured: profiles/umma_mn_probe.cu variant 3) -- so the
// raw fp32 tile of A loaded by TMA *is* A_hi, and only A_lo = A - A_hi is computed in shared
// memory (same swizzled positions).  B is split once per launch into Bt_hi / Bt_lo (N x K,
// K contiguous) by split_bt_kernel (forming Bt_lo per tile instead measured slower: the
// per-step conversion is on the critical path, the extra L2 traffic is not).  A TMEM accumulator
// covers kGChunk K steps (48 truncating MMAs) and is drained into fp32 register sums while the
// next chunk's MMAs run (two accumulators alternate).
//
// Persistent CTAs (one per SM, 256 threads) loop over 128 x N tiles (consecutive CTAs share A
// rows across N tiles, so A is read ~once from DRAM).  Per K step:
//   * TMA (thread 0) loads A[128 x 16] and Bt_hi / Bt_lo[N x 16] boxes with SWIZZLE_64B into a
//     4-stage ring -- exactly the UMMA K-major SWIZZLE_64B canonical layout (8-row atoms of
//     512 B), so no transposition;
//   * all threads write A_lo (two float4 each);
//   * thread 0 issues 2 k-steps x 3 tcgen05.mma.kind::tf32 (M = 128, N <= 256, K = 8) and
//     commits; after the previous step's MMAs completed it refills that step's stage;
//   * every kGChunk steps, warp w drains TMEM lanes 32 (w % 4) .. +31, column half w / 4
//     (tcgen05.ld.32x32b; TMEM reads run at ~64 B/clk, so draining every step would cost more
//     than the MMAs) into register sums and, after the tile's last chunk, writes its rows of C
//     (alpha, row scale, row map) transposed through shared memory as full 128-byte segments.
#include <algorithm>

#include "common.cuh"
#include "umma.cuh"

namespace isvd {
namespace {

constexpr int kGM = 128;      // rows per tile (UMMA M)
constexpr int kGK = 16;       // K per pipeline step: one 64-byte SWIZZLE_64B row
constexpr int kGChunk = 8;    // K steps per TMEM accumulation (48 truncating MMAs; TMEM-read budget)
constexpr int kGThreads = 256;  // 8 warps: 4 TMEM lane quadrants x 2 column halves
constexpr uint32_t kSw64 = 4;  // UMMA descriptor layout type SWIZZLE_64B

template <int N>
struct GCfg {
  static constexpr int A_B = kGM * kGK * 4;            // bytes of one A box (8 KB)
  static constexpr int B_B = N * kGK * 4;              // bytes of one Bt box
  static constexpr int STAGE_B = 2 * A_B + 2 * B_B;    // A (TMA) | A lo | Bt hi (TMA) | Bt lo (TMA)
  static constexpr int TMA_B = A_B + 2 * B_B;          // bytes landed by TMA per stage
  static constexpr int EPI_B = 8 * 32 * 32 * 4;        // per-warp 32 x 32 fp32 epilogue transpose buffers
  static constexpr int STAGES = 4;                     // ring depth
  static constexpr size_t smem_bytes() { return (size_t)STAGES * STAGE_B + EPI_B + 1024; }
};

// Bt_hi / Bt_lo [n][k] (Npad x Kpad, zero padded) from B (K x N, row-major, ldb): the K-major
// split of the small operand, loaded by TMA for every 128-row tile.
__global__ void split_bt_kernel(const float* __restrict__ B, int64_t ldb, int K, int N, int Kpad, int Npad,
                                float* __restrict__ hi, float* __restrict__ lo, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  const int64_t tot = (int64_t)Npad * Kpad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(e / Kpad), k = (int)(e - (int64_t)n * Kpad);
    const float v = (n < N && k < K) ? B[(int64_t)k * ldb + n] : 0.f;
    const float h = tf32_hi(v);
    hi[e] = h;
    lo[e] = v - h;
  }
}

template <int N>
__global__ void __launch_bounds__(kGThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
                   const __grid_constant__ CUtensorMap tmBlo, int64_t rows, int K, int ntn, int ntiles,
                   float* __restrict__ C, int64_t ldc, int64_t ncols, const float* __restrict__ rs, float alpha,
                   const int32_t* __restrict__ out_map, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  using G = GCfg<N>;
  static_assert(N % 16 == 0 && N >= 32 && N <= 256, "UMMA N");
  constexpr int HALF = N / 2;  // columns drained per thread
  static_assert(HALF % 4 == 0, "drain granularity");
  constexpr uint32_t kCols = 2 * N <= 256 ? 256 : 512;

  extern __shared__ uint8_t smraw[];
  uint8_t* const base = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  constexpr int S = G::STAGES;
  float* const epi = reinterpret_cast<float*>(base + S * G::STAGE_B);
  __shared__ __align__(8) uint64_t full[S];   // stage landed (TMA tx bytes)
  __shared__ __align__(8) uint64_t empty[S];  // stage's MMAs (and the lo buffer's) done
  __shared__ __align__(8) uint64_t cdone[2];         // chunk accumulator b complete
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int ksteps = (K + kGK - 1) / kGK;
  const int cpt = (ksteps + kGChunk - 1) / kGChunk;  // chunks per tile
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nsteps = my_tiles * ksteps;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&cdone[0], 1);
    mbar_init(&cdone[1], 1);
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
  const uint32_t idesc = umma_idesc(kGM, N);

  // step g -> (local tile i, k step kk); tile t = blockIdx.x + i gridDim.x -> (m0, n0)
  auto fill = [&](int g) {  // thread 0
    const int s = g % S;
    uint8_t* st = base + s * G::STAGE_B;
    const int i = g / ksteps, kk = g - i * ksteps;
    const int t = (int)blockIdx.x + i * (int)gridDim.x;
    const int m0 = (t / ntn) * kGM, n0 = (t - (t / ntn) * ntn) * N;
    mbar_expect_tx(&full[s], (uint32_t)G::TMA_B);
    tma_2d(st, &tmA, kk * kGK, m0, &full[s]);
    tma_2d(st + 2 * G::A_B, &tmBhi, kk * kGK, n0, &full[s]);
    tma_2d(st + 2 * G::A_B + G::B_B, &tmBlo, kk * kGK, n0, &full[s]);
  };
  // thread 0 keeps the ring full without blocking the MMA issue: step j may be loaded once the
  // MMAs of step j - S (same stage) are done
  int next_fill = 0;
  auto top_up = [&](int upto, bool block) {
    while (next_fill < nsteps && next_fill <= upto) {
      if (next_fill >= S) {
        const int j = next_fill - S;
        uint64_t* e = &empty[j % S];
        const uint32_t par = (uint32_t)((j / S) & 1);
        if (block) mbar_wait(e, par);
        else if (!mbar_test(e, par)) break;
      }
      fill(next_fill++);
    }
  };
  if (tid == 0) top_up(S - 1, true);

  float acc[HALF];
#pragma unroll
  for (int q = 0; q < HALF; ++q) acc[q] = 0.f;
  const uint32_t lane_base = (uint32_t)(warp & 3) * 32;
  const uint32_t col_h = (uint32_t)(warp >> 2) * HALF;

  // add chunk c (global id) of local tile i into acc; after the tile's last chunk write C
  auto drain = [&](int c, int i, bool last) {
    mbar_wait(&cdone[c & 1], (uint32_t)((c >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem + (lane_base << 16) + (uint32_t)(c & 1) * N + col_h;
#pragma unroll
    for (int q0 = 0; q0 < HALF; q0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int q = 0; q < 16; q += 4)
        if (q0 + q < HALF)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(r[q]), "=r"(r[q + 1]), "=r"(r[q + 2]), "=r"(r[q + 3])
                       : "r"(tb + (uint32_t)(q0 + q)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q0 + q < HALF) acc[q0 + q] += __uint_as_float(r[q]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (last) {
      // C rows of this warp (32 rows x HALF columns), transposed through a 32 x 32 smem buffer in
      // pieces of 32 columns so each store instruction writes 4 full 128-byte row segments
      const int t = (int)blockIdx.x + i * (int)gridDim.x;
      const int64_t m0 = (int64_t)(t / ntn) * kGM, n0 = (int64_t)(t - (t / ntn) * ntn) * N;
      const int64_t row = m0 + lane_base + lane;
      const float sc = row < rows ? alpha * (rs ? __ldg(rs + row) : 1.f) : 0.f;
      const int64_t orow = row < rows ? (out_map ? (int64_t)__ldg(out_map + row) : row) : -1;
      float4* const eb = reinterpret_cast<float4*>(epi + warp * 32 * 32);  // [32 rows][8 float4], XOR-swizzled
      const int64_t cbase = n0 + col_h;
#pragma unroll
      for (int p0 = 0; p0 < HALF; p0 += 32) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (p0 + 4 * j < HALF)
            eb[lane * 8 + (j ^ (lane & 7))] = make_float4(sc * acc[p0 + 4 * j], sc * acc[p0 + 4 * j + 1],
                                                          sc * acc[p0 + 4 * j + 2], sc * acc[p0 + 4 * j + 3]);
        __syncwarp();
        const int c4 = lane & 7;
        const int64_t col = cbase + p0 + 4 * c4;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = it * 4 + (lane >> 3);
          const int64_t orr = __shfl_sync(0xffffffffu, orow, r);
          if (orr >= 0 && p0 + 4 * c4 < HALF && col < ncols)
            *reinterpret_cast<float4*>(C + orr * ldc + col) = eb[r * 8 + (c4 ^ (r & 7))];
        }
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < HALF; ++q) acc[q] = 0.f;
    }
  };

  int pend_c = -1, pend_i = 0;  // chunk whose drain is due
  bool pend_last = false;
  for (int g = 0; g < nsteps; ++g) {
    const int s = g % S;
    uint8_t* const st = base + s * G::STAGE_B;
    const int i = g / ksteps, kk = g - i * ksteps;
    const int c = i * cpt + kk / kGChunk;  // global chunk id -> accumulator c & 1
    if (tid == 0) top_up(g, true);         // step g itself must be in flight
    mbar_wait(&full[s], (uint32_t)((g / S) & 1));
    // A_lo = A - tf32(A), position for position (the swizzle is irrelevant elementwise); the raw
    // TMA tile itself is the hi operand
    static_assert(GCfg<N>::A_B == 2 * kGThreads * 16, "two float4 of A per thread");
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 v = reinterpret_cast<const float4*>(st)[tid + h * kGThreads];
      reinterpret_cast<float4*>(st + G::A_B)[tid + h * kGThreads] =
          make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const bool chunk_end = (kk % kGChunk) == kGChunk - 1 || kk == ksteps - 1;
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + (uint32_t)(c & 1) * N;
      const uint32_t ah = smem_u32(st), al = ah + G::A_B;
      const uint32_t bh = ah + 2 * G::A_B, bl = bh + G::B_B;
#pragma unroll
      for (int ks = 0; ks < kGK / 8; ++ks) {
        const uint32_t ko = (uint32_t)ks * 32;  // 8 TF32 values along the swizzled 64-byte row
        const uint64_t dah = umma_desc(ah + ko, 16, 512, kSw64), dal = umma_desc(al + ko, 16, 512, kSw64);
        const uint64_t dbh = umma_desc(bh + ko, 16, 512, kSw64), dbl = umma_desc(bl + ko, 16, 512, kSw64);
        mma_tf32(d, dah, dbh, idesc, ((kk % kGChunk) == 0 && ks == 0) ? 0u : 1u);
        mma_tf32(d, dah, dbl, idesc, 1u);
        mma_tf32(d, dal, dbh, idesc, 1u);
      }
      umma_commit(&empty[s]);
      if (chunk_end) umma_commit(&cdone[c & 1]);
      // step g-1's MMAs are done shortly after step g's start: refill its stage with step g-1+S
      top_up(g - 1 + S, true);
    }
    // the chunk that ended at step g-1 is drained while step g's MMAs run (other accumulator);
    // its accumulator is next written by chunk c + 1, issued after the next __syncthreads
    if (pend_c >= 0) {
      drain(pend_c, pend_i, pend_last);
      pend_c = -1;
    }
    if (chunk_end) {
      pend_c = c;
      pend_i = i;
      pend_last = kk == ksteps - 1;
    }
  }
  if (pend_c >= 0) drain(pend_c, pend_i, pend_last);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

constexpr int kGNs[] = {128, 160, 208, 256};  // instantiated tile widths

int gemm_tile_n(int64_t N) {
  const int64_t tb = ceil_div(N, 256);
  const int64_t need = round_up(ceil_div(N, tb), 16);
  for (int n : kGNs)
    if (n >= need) return n;
  return 256;
}

template <int NT>
cudaError_t tc_gemm_launch(const float* A, int64_t lda, float* C, int64_t ldc, int64_t rows, int64_t N, int64_t K,
                           const float* rs, float alpha, const int* gate, cudaStream_t st, const int32_t* out_map,
                           float* bt, int num_sms) {
  const int64_t ntn = ceil_div(N, NT), Npad = ntn * NT, Kpad = round_up(K, kGK);
  CUtensorMap tmA, tmBhi, tmBlo;
  if (!make_map(&tmA, A, rows, K, lda, kGK, kGM, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map(&tmBhi, bt, Npad, Kpad, Kpad, kGK, NT, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map(&tmBlo, bt + Npad * Kpad, Npad, Kpad, Kpad, kGK, NT, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  const size_t smem = GCfg<NT>::smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_gemm_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t ntiles = ceil_div(rows, kGM) * ntn;
  const int grid = (int)std::min<int64_t>(ntiles, num_sms);
  ++g_launches;
  tc_gemm_kernel<NT><<<grid, kGThreads, smem, st>>>(tmA, tmBhi, tmBlo, rows, (int)K, (int)ntn, (int)ntiles, C, ldc, N,
                                                    rs, alpha, out_map, gate);
  return cudaGetLastError();
}

}  // namespace

bool tc_gemm_supported(int64_t rows, int64_t N, int64_t K, int64_t lda, int64_t ldc) {
  return rows >= 65536 && N >= 16 && N <= 1024 && N % 4 == 0 && K >= 1 && K <= 4096 && lda % 4 == 0 &&
         ldc % 4 == 0;
}

int64_t tc_gemm_ws_floats(int64_t N, int64_t K) {
  const int nt = gemm_tile_n(N);
  return 2 * ceil_div(N, nt) * nt * round_up(K, kGK);
}

cudaError_t launch_tc_gemm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                           int64_t rows, int64_t N, int64_t K, const float* row_scale, float alpha, const int* gate,
                           cudaStream_t st, const int32_t* out_map, float* ws_bt, int num_sms) {
  if (rows <= 0 || N <= 0) return cudaSuccess;
  const int nt = gemm_tile_n(N);
  const int64_t Npad = ceil_div(N, nt) * nt, Kpad = round_up(K, kGK);
  ++g_launches;
  split_bt_kernel<<<(unsigned)std::min<int64_t>(ceil_div(Npad * Kpad, 256), 4LL * num_sms), 256, 0, st>>>(
      B, ldb, (int)K, (int)N, (int)Kpad, (int)Npad, ws_bt, ws_bt + Npad * Kpad, gate);
  switch (nt) {
    case 128: return tc_gemm_launch<128>(A, lda, C, ldc, rows, N, K, row_scale, alpha, gate, st, out_map, ws_bt, num_sms);
    case 160: return tc_gemm_launch<160>(A, lda, C, ldc, rows, N, K, row_scale, alpha, gate, st, out_map, ws_bt, num_sms);
    case 208: return tc_gemm_launch<208>(A, lda, C, ldc, rows, N, K, row_scale, alpha, gate, st, out_map, ws_bt, num_sms);
    default: return tc_gemm_launch<256>(A, lda, C, ldc, rows, N, K, row_scale, alpha, gate, st, out_map, ws_bt, num_sms);
  }
}

}  // namespace isvd
