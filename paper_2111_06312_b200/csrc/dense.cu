// Tall-skinny dense kernels of the solver (FP32 SIMT; fp64 where a reduction
// over the n-long dimension is taken).
//
//  K2  gemm_tn   C = alpha * diag(row_scale) * A * B   (A: M x K tall, B: K x N small)
//                X.G_j of the NC operator (DenseMatrixPF.dot), the
//                CholeskyQR apply Q (L^-1)^T = Q R^-1 (Alg. 2 right, upper
//                triangular B skips the zero half) and U = Q U_B (Alg. 1).
//  K5/K16 atb    G = A^T diag(s) B in fp64 (Gram Q^T Q of Alg. 2; X^T Z_j of
//                the NC transpose).  Split-K over rows, fp32 tiles promoted to fp64
//                once when staged in shared memory, fp64 FMA, deterministic
//                fixed-order reduction of the per-CTA partials (no atomics).
//  K15 colsum    1^T Q in fp64 for the rank-1 term of Eq. 3.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace isvd {
namespace {

// ------------------------------------------------------------------ GEMM
// Thread (tx, ty) owns rows {g*4*TY + ty*4 + 0..3} and columns {g*4*TX + tx*4 + 0..3}: every
// shared-memory float4 read of a quarter-warp covers 128 contiguous bytes (no bank conflicts).
// A is stored transposed with 4 floats of padding per k-row so the transposing stores do
// not conflict either.  __launch_bounds__(., 2): <= 128 registers, two CTAs per SM.
// Thread -> (tx, ty) of a register-tiled kernel whose thread reads B float4 tx*4 (and A
// float4 ty*4) of each smem row.  A quarter-warp's 8 float4 reads must hit 8 distinct 16-byte
// bank groups: with TX a multiple of 8 the plain tid % TX mapping does that; with TX = 10 no
// cyclic window of 8 consecutive tx can (tx and tx + 8 share banks), so the first 8 TY threads
// take tx = 0..7 (one ty per quarter-warp) and the last 2 TY take tx = 8, 9 (four ty per
// quarter-warp: 2 distinct B and 4 distinct A float4s).
template <int TX>
ISVD_DEVICE void thread_xy(int tid, int* tx, int* ty) {
  if constexpr (TX % 8 == 0 || TX < 8) {
    *tx = tid % TX;
    *ty = tid / TX;
  } else {
    // TX = 8a + b: groups of 8 threads take tx = 8j + 0..7 (one ty per quarter-warp), the last
    // b TY threads take tx = 8a .. 8a + b - 1 (TX = 10: a = 1, b = 2; TX = 25: a = 3, b = 1)
    constexpr int A8 = TX / 8, B8 = TX % 8;
    const int ty_n = blockDim.x / TX;
    if (tid < 8 * A8 * ty_n) {
      const int g = tid >> 3;
      *tx = 8 * (g / ty_n) + (tid & 7);
      *ty = g % ty_n;
    } else {
      const int t = tid - 8 * A8 * ty_n;
      *tx = 8 * A8 + t % B8;
      *ty = t / B8;
    }
  }
}

template <int BM, int BN, int BK, int TM, int TN, int MINB = 2>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
    gemm_tn_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                   float* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                   const float* __restrict__ row_scale, float alpha, int upper_tri_b, const int* gate,
                   const int32_t* __restrict__ out_map) {
  if (gate && *((volatile const int*)gate) == 0) return;
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int TX = BN / TN;  // threads along N
  constexpr int TY = BM / TM;  // threads along M
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  int tx, ty;
  thread_xy<TX>(tid, &tx, &ty);
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  int64_t kend = K;
  if (upper_tri_b) kend = (n0 + BN < K) ? (n0 + BN) : K;

  // loader mapping: A tile BM x BK as float4 along K; B tile BK x BN as float4 along N
  constexpr int A_F4 = BM * BK / 4;
  constexpr int B_F4 = BK * BN / 4;
  float4 ra[(A_F4 + NT - 1) / NT];
  float4 rb[(B_F4 + NT - 1) / NT];

  auto load_tiles = [&](int64_t k0) {
#pragma unroll
    for (int t = 0; t < (A_F4 + NT - 1) / NT; ++t) {
      int f = tid + t * NT;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < A_F4) {
        int r = f / (BK / 4), kk = (f % (BK / 4)) * 4;
        int64_t gm = m0 + r, gk = k0 + kk;
        if (gm < M) {
          const float* p = A + gm * lda + gk;
          if (gk + 3 < kend) {
            v = *reinterpret_cast<const float4*>(p);
          } else {
            if (gk < kend) v.x = p[0];
            if (gk + 1 < kend) v.y = p[1];
            if (gk + 2 < kend) v.z = p[2];
          }
        }
      }
      ra[t] = v;
    }
#pragma unroll
    for (int t = 0; t < (B_F4 + NT - 1) / NT; ++t) {
      int f = tid + t * NT;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < B_F4) {
        int kk = f / (BN / 4), c = (f % (BN / 4)) * 4;
        int64_t gk = k0 + kk, gn = n0 + c;
        if (gk < kend && gn < N) v = *reinterpret_cast<const float4*>(B + gk * ldb + gn);
      }
      rb[t] = v;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int t = 0; t < (A_F4 + NT - 1) / NT; ++t) {
      int f = tid + t * NT;
      if (f < A_F4) {
        int r = f / (BK / 4), kk = (f % (BK / 4)) * 4;
        As[buf][kk][r] = ra[t].x;
        As[buf][kk + 1][r] = ra[t].y;
        As[buf][kk + 2][r] = ra[t].z;
        As[buf][kk + 3][r] = ra[t].w;
      }
    }
#pragma unroll
    for (int t = 0; t < (B_F4 + NT - 1) / NT; ++t) {
      int f = tid + t * NT;
      if (f < B_F4) {
        int kk = f / (BN / 4), c = (f % (BN / 4)) * 4;
        *reinterpret_cast<float4*>(&Bs[buf][kk][c]) = rb[t];
      }
    }
  };

  float2 acc[TM][TN / 2];  // column pairs (FFMA2)
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);

  int64_t ntiles = (kend + BK - 1) / BK;
  if (ntiles > 0) {
    load_tiles(0);
    store_tiles(0);
    __syncthreads();
  }
  for (int64_t t = 0; t < ntiles; ++t) {
    int buf = (int)(t & 1);
    if (t + 1 < ntiles) load_tiles((t + 1) * BK);
    // fragments of step kk + 1 are read from shared memory while step kk's FMAs issue
    float a[2][TM], b[2][TN];
    auto frag = [&](int kk, int s) {
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        float4 v = *reinterpret_cast<const float4*>(&As[buf][kk][(i / 4) * 4 * TY + ty * 4]);
        a[s][i] = v.x; a[s][i + 1] = v.y; a[s][i + 2] = v.z; a[s][i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        float4 v = *reinterpret_cast<const float4*>(&Bs[buf][kk][(j / 4) * 4 * TX + tx * 4]);
        b[s][j] = v.x; b[s][j + 1] = v.y; b[s][j + 2] = v.z; b[s][j + 3] = v.w;
      }
    };
    frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      if (kk + 1 < BK) frag(kk + 1, (kk + 1) & 1);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN / 2; ++j)
          acc[i][j] = ffma2(make_float2(a[kk & 1][i], a[kk & 1][i]),
                            make_float2(b[kk & 1][2 * j], b[kk & 1][2 * j + 1]), acc[i][j]);
    }
    if (t + 1 < ntiles) {
      store_tiles(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t gm = m0 + (i / 4) * 4 * TY + ty * 4 + (i & 3);
    if (gm >= M) continue;
    float s = alpha;
    if (row_scale) s *= row_scale[gm];
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      int64_t gn = n0 + (j / 4) * 4 * TX + tx * 4;
      if (gn < N)
        *reinterpret_cast<float4*>(C + (out_map ? (int64_t)out_map[gm] : gm) * ldc + gn) =
            make_float4(s * acc[i][j / 2].x, s * acc[i][j / 2].y, s * acc[i][j / 2 + 1].x, s * acc[i][j / 2 + 1].y);
    }
  }
}

// ------------------------------------------------------------------ GEMM, K-resident (round 2)
// C = alpha * diag(row_scale) * A * B for a short contraction (K <= 128: X G_j of the NC operator,
// K = d) with the whole B panel (K x N, N <= 416) resident in shared memory for the life of a
// persistent CTA, and 64-row A tiles streamed through a two-slot ring by bulk copies
// (cp.async.bulk, one per row, completing on an mbarrier).  The K loop of a tile has no CTA
// barrier at all (gemm_tn_kernel: one per 8 k-steps, its first stall reason in ncu), B is read from
// L2 once per CTA instead of once per 128 x 80 tile, and the next tile's rows land while this one
// computes.  Warp w owns columns {16 w + 4 t .. +3} and {NP/2 + 16 w + 4 t .. +3} (t = lane & 3) of
// all 64 rows; lane row group r = lane >> 2 owns rows {r + 8 i}: a B fragment read touches 64
// contiguous bytes per warp (broadcast over r), an A fragment read (float2 along k, row pitch K
// floats, K = 4 mod 32 for K = 100) 8 distinct bank pairs (broadcast over t).
constexpr int kResBM = 64;

ISVD_DEVICE uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
ISVD_DEVICE void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
ISVD_DEVICE void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
ISVD_DEVICE void mbar_wait(const uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1u << 28)) __trap();  // a copy that never lands fails the launch instead of hanging
  }
}
ISVD_DEVICE void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// One 64 x 32 warp tile over the whole K (K % 4 == 0).  Fragments of the next k-step are read from
// shared memory while this step's FMAs issue.  kHalf: only the lower 16 columns (acc[.][0..1]).
// KT / NPT: compile-time K and panel pitch (0: run-time), so every shared-memory address of the loop
// is base + immediate (the run-time form spends one IMAD -- an FMA-pipe cycle -- per fragment load,
// 16 % of the pipe at K = 100).
// MODE: 0 both column halves, 1 the lower 16 columns only (acc[.][0..1]), 2 the upper only
// (acc[.][2..3]).  APT: compile-time A row pitch in floats (0: K).  ZERO: clear acc first.
template <int MODE, int KT, int NPT, int APT = 0, bool ZERO = true>
ISVD_DEVICE void kres_tile_m(const float* __restrict__ a_base, const float* __restrict__ b0p,
                             const float* __restrict__ b1p, int Krt, int NPrt, float2 acc[8][4], int APrt = 0) {
  const int K = KT ? KT : Krt, NP = NPT ? NPT : NPrt;
  const int AP = APT ? APT : (APrt ? APrt : K);
  if constexpr (ZERO) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  }
  auto lda2 = [&](float2 a[8], int k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float2*>(a_base + (size_t)(8 * i) * AP + k);
  };
  auto ldb = [&](float4& bl, float4& bh, int k) {
    if constexpr (MODE != 2) bl = *reinterpret_cast<const float4*>(b0p + (size_t)k * NP);
    if constexpr (MODE != 1) bh = *reinterpret_cast<const float4*>(b1p + (size_t)k * NP);
  };
  auto fma_step = [&](const float2 a[8], bool hi, float4 bl, float4 bh) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float av = hi ? a[i].y : a[i].x;
      const float2 a2 = make_float2(av, av);
      if constexpr (MODE != 2) {
        acc[i][0] = ffma2(a2, make_float2(bl.x, bl.y), acc[i][0]);
        acc[i][1] = ffma2(a2, make_float2(bl.z, bl.w), acc[i][1]);
      }
      if constexpr (MODE != 1) {
        acc[i][2] = ffma2(a2, make_float2(bh.x, bh.y), acc[i][2]);
        acc[i][3] = ffma2(a2, make_float2(bh.z, bh.w), acc[i][3]);
      }
    }
  };
  float2 a0[8], a1[8];
  float4 bl0 = make_float4(0.f, 0.f, 0.f, 0.f), bh0 = bl0, bl1 = bl0, bh1 = bl0;
  lda2(a0, 0);
  ldb(bl0, bh0, 0);
  auto block4 = [&](int k, int kn) {
    ldb(bl1, bh1, k + 1);
    fma_step(a0, false, bl0, bh0);
    lda2(a1, k + 2);
    ldb(bl0, bh0, k + 2);
    fma_step(a0, true, bl1, bh1);
    ldb(bl1, bh1, k + 3);
    fma_step(a1, false, bl0, bh0);
    lda2(a0, kn);
    ldb(bl0, bh0, kn);
    fma_step(a1, true, bl1, bh1);
  };
  if constexpr (KT != 0) {
#pragma unroll
    for (int k = 0; k < KT; k += 4) block4(k, k + 4 < KT ? k + 4 : k);  // the last prefetch re-reads valid data
  } else {
#pragma unroll 1
    for (int k = 0; k < K; k += 4) block4(k, k + 4 < K ? k + 4 : k);
  }
}
template <bool kHalf, int KT, int NPT>
ISVD_DEVICE void kres_tile(const float* __restrict__ a_base, const float* __restrict__ b0p,
                           const float* __restrict__ b1p, int Krt, int NPrt, float2 acc[8][4]) {
  kres_tile_m<kHalf ? 1 : 0, KT, NPT>(a_base, b0p, b1p, Krt, NPrt, acc);
}

ISVD_DEVICE void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// blockDim = 32 (compute warps + 1): warps 0 .. ncw-1 compute, warp ncw feeds the A ring.  No CTA
// barrier after the start: a compute warp waits only for its tile's rows (full[slot]) and releases
// the slot (empty[slot]) as soon as its k-loop has read them, before its stores, so the warps of
// one SM sub-partition drift apart and one warp's epilogue overlaps the others' FMAs.  (With a
// __syncthreads per tile, 18 % of the warp samples sat at the barrier: ncu, profiles/r02h_*.)
// (14 warps put 4 on an SM sub-partition: at most 128 registers per thread.)
template <int KT, int NPT>
__global__ void __launch_bounds__(448, 1)
    gemm_kres_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                     float* __restrict__ C, int64_t ldc, int64_t M, int N, int Krt, const float* __restrict__ row_scale,
                     float alpha, const int* gate, const int32_t* __restrict__ out_map) {
  if (gate && *((volatile const int*)gate) == 0) return;
  extern __shared__ __align__(128) uint8_t kres_sm[];
  const int ncw = (int)(blockDim.x >> 5) - 1;
  const int K = KT ? KT : Krt;
  const int NP = NPT ? NPT : 32 * ncw;  // 32 columns per compute warp
  float* const Bs = reinterpret_cast<float*>(kres_sm);                       // [K][NP]
  float* const As = Bs + (size_t)K * NP;                                      // [2][64][K]
  uint64_t* const bars = reinterpret_cast<uint64_t*>(As + 2 * kResBM * K);   // full[2], empty[2], bfull
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, t = lane & 3;
  const int64_t ntile = (M + kResBM - 1) / kResBM;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], (uint32_t)ncw);
    mbar_init(&bars[3], (uint32_t)ncw);
    mbar_init(&bars[4], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t t0 = blockIdx.x, dt = gridDim.x;
  if (warp == ncw) {
    // ---------------------------------------------------------------- producer warp
    if (lane == 0) mbar_expect_tx(&bars[4], (uint32_t)(K * N * 4));
    __syncwarp();
    for (int k = lane; k < K; k += 32) bulk_g2s(Bs + (size_t)k * NP, B + (int64_t)k * ldb, (uint32_t)(N * 4), &bars[4]);
    int it = 0;
    for (int64_t tl = t0; tl < ntile; tl += dt, ++it) {
      const int slot = it & 1;
      if (it >= 2) mbar_wait(&bars[2 + slot], (uint32_t)(((it >> 1) - 1) & 1));  // every compute warp released it
      const int64_t m0 = tl * kResBM;
      const int rows = (int)((M - m0) < kResBM ? (M - m0) : kResBM);
      if (lane == 0) mbar_expect_tx(&bars[slot], (uint32_t)(rows * K * 4));
      __syncwarp();
      for (int e = lane; e < rows; e += 32)  // lane e copies rows e and e + 32
        bulk_g2s(As + ((size_t)slot * kResBM + e) * K, A + (m0 + e) * lda, (uint32_t)(K * 4), &bars[slot]);
    }
    return;
  }
  // ------------------------------------------------------------------ compute warps
  const int c0 = 16 * warp + 4 * t, c1 = NP / 2 + c0;
  const float* const b0p = Bs + c0;
  const float* const b1p = Bs + c1;
  mbar_wait(&bars[4], 0);
  int it = 0;
  for (int64_t tl = t0; tl < ntile; tl += dt, ++it) {
    const int slot = it & 1;
    mbar_wait(&bars[slot], (uint32_t)((it >> 1) & 1));
    const float* const a_base = As + ((size_t)slot * kResBM + r) * K;
    float2 acc[8][4];
    if (NP / 2 + 16 * warp < N) kres_tile<false, KT, NPT>(a_base, b0p, b1p, K, NP, acc);
    else kres_tile<true, KT, NPT>(a_base, b0p, b1p, K, NP, acc);  // the last warp's upper columns are padding
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[2 + slot]);  // this warp has read the slot
    const int64_t m0 = tl * kResBM;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t gm = m0 + r + 8 * i;
      if (gm >= M) continue;
      float sc = alpha;
      if (row_scale) sc *= row_scale[gm];
      float* const crow = C + (out_map ? (int64_t)out_map[gm] : gm) * ldc;
      if (c0 < N)
        *reinterpret_cast<float4*>(crow + c0) =
            make_float4(sc * acc[i][0].x, sc * acc[i][0].y, sc * acc[i][1].x, sc * acc[i][1].y);
      if (c1 < N)
        *reinterpret_cast<float4*>(crow + c1) =
            make_float4(sc * acc[i][2].x, sc * acc[i][2].y, sc * acc[i][3].x, sc * acc[i][3].y);
    }
  }
}

// ------------------------------------------------------------------ GEMM, K-chunked (round 2)
// The same warp tiling and producer / consumer ring for a long contraction (Y R^-1 of the
// CholeskyQR apply, K = l = 400): the C tile (64 x N) stays in registers while K-chunks of KC
// k-steps of B (KC x N per stage, as many stages as fit beside the A tile: 3 at KC = 20, N = 400) stream through shared memory; the 64 x K row tile of A is copied once per tile
// (B is re-read from L2 for every row tile: 2.5 TB/s over the GPU, inside what L2 delivers).
// upper_tri_b: chunk c only touches columns >= KC c, so a warp skips a 16-column group whose
// columns all lie left of the chunk (warp-uniform), and the producer copies only the columns from
// the first live group on.  A rows are padded to K + 4 floats in shared memory (the 8 row groups of
// an A fragment read hit 8 distinct bank pairs).  Measured on the way: A and B per chunk in two
// stages of 40 k-steps left the compute warps waiting for data 29 % of the time (11.1 ms; ncu), five
// stages of 20 k-steps with per-chunk 80-byte A row copies ran 15.9 ms (1,680 small bulk copies per
// tile): hence whole A rows once per tile.
// Chunk order of a row tile.  With a triangular B the late chunks carry little work (few live column
// groups) and finish before the next copy lands (ncu: 16 % of the warp samples waited on full[]), so
// early and late chunks alternate (0, n-1, 1, n-2, ...): every pair of consecutive chunks then has
// about the same work, which the ring's prefetch distance covers.
ISVD_DEVICE int chunk_order(int i, int nch, int tri) {
  if (!tri) return i;
  return (i & 1) ? nch - 1 - (i >> 1) : (i >> 1);
}

template <int KC, int APT, int NPT>
__global__ void __launch_bounds__(448, 1)
    gemm_kchunk_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                       float* __restrict__ C, int64_t ldc, int64_t M, int N, int K, const float* __restrict__ row_scale,
                       float alpha, int upper_tri_b, int S, const int* gate, const int32_t* __restrict__ out_map) {
  if (gate && *((volatile const int*)gate) == 0) return;
  extern __shared__ __align__(128) uint8_t kres_sm[];
  const int ncw = (int)(blockDim.x >> 5) - 1;
  const int NP = NPT ? NPT : 32 * ncw;
  const int AP = APT ? APT : K + 4;
  float* const Bs = reinterpret_cast<float*>(kres_sm);                        // [S][KC][NP]
  float* const As = Bs + (size_t)S * KC * NP;                                  // [64][AP]: the whole row tile
  uint64_t* const full = reinterpret_cast<uint64_t*>(As + (size_t)kResBM * AP);
  uint64_t* const empty = full + S;
  uint64_t* const a_full = empty + S;
  uint64_t* const a_empty = a_full + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, t = lane & 3;
  const int64_t ntile = (M + kResBM - 1) / kResBM;
  const int nch = K / KC;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], (uint32_t)ncw);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, (uint32_t)ncw);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t t0 = blockIdx.x, dt = gridDim.x;
  int st = 0;
  uint32_t ph = 0;  // ring slot and the parity of its current use
  if (warp == ncw) {
    // ---------------------------------------------------------------- producer warp
    bool first_lap = true;
    uint32_t it = 0;
    for (int64_t tl = t0; tl < ntile; tl += dt, ++it) {
      const int64_t m0 = tl * kResBM;
      const int rows = (int)((M - m0) < kResBM ? (M - m0) : kResBM);
      if (it > 0) mbar_wait(a_empty, (it - 1) & 1u);  // every compute warp is done with the previous tile's rows
      if (lane == 0) mbar_expect_tx(a_full, (uint32_t)(rows * K * 4));
      __syncwarp();
      for (int e = lane; e < rows; e += 32) bulk_g2s(As + (size_t)e * AP, A + (m0 + e) * lda, (uint32_t)(K * 4), a_full);
      for (int i = 0; i < nch; ++i) {
        if (!first_lap) mbar_wait(&empty[st], ph ^ 1u);  // every compute warp released the previous use
        const int c = chunk_order(i, nch, upper_tri_b);
        const int k0 = c * KC;
        const int cb = upper_tri_b ? (k0 / 16) * 16 : 0;  // first live column
        if (lane == 0) mbar_expect_tx(&full[st], (uint32_t)(KC * (N - cb) * 4));
        __syncwarp();
        for (int k = lane; k < KC; k += 32)
          bulk_g2s(Bs + ((size_t)st * KC + k) * NP + cb, B + (int64_t)(k0 + k) * ldb + cb, (uint32_t)((N - cb) * 4),
                   &full[st]);
        if (++st == S) {
          st = 0;
          ph ^= 1u;
          first_lap = false;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------ compute warps
  // warp w owns the 16-column groups w and G - 1 - w: with a triangular B group g is live for the
  // first ~(16 g + 16) / KC chunks, so pairing a short-lived group with a long-lived one gives every
  // warp the same work per tile and keeps it busy to the late chunks
  const int hi_g = NP / 16 - 1 - warp;
  const int c0 = 16 * warp + 4 * t, c1 = 16 * hi_g + 4 * t;
  const bool hi_cols = 16 * hi_g < N;  // the last group of a padded panel is padding
  uint32_t it = 0;
  for (int64_t tl = t0; tl < ntile; tl += dt, ++it) {
    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
    mbar_wait(a_full, it & 1u);
    for (int i = 0; i < nch; ++i) {
      mbar_wait(&full[st], ph);
      const int c = chunk_order(i, nch, upper_tri_b);
      const int k0 = c * KC;
      const bool lo_on = !upper_tri_b || 16 * warp + 16 > k0;
      const bool hi_on = hi_cols && (!upper_tri_b || 16 * hi_g + 16 > k0);
      const float* const a_base = As + (size_t)r * AP + k0;
      const float* const b0p = Bs + (size_t)st * KC * NP + c0;
      const float* const b1p = Bs + (size_t)st * KC * NP + c1;
      if (lo_on && hi_on) kres_tile_m<0, KC, NPT, APT, false>(a_base, b0p, b1p, KC, NP, acc, AP);
      else if (hi_on) kres_tile_m<2, KC, NPT, APT, false>(a_base, b0p, b1p, KC, NP, acc, AP);
      else if (lo_on) kres_tile_m<1, KC, NPT, APT, false>(a_base, b0p, b1p, KC, NP, acc, AP);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[st]);
        if (i == nch - 1) mbar_arrive(a_empty);
      }
      if (++st == S) {
        st = 0;
        ph ^= 1u;
      }
    }
    const int64_t m0 = tl * kResBM;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t gm = m0 + r + 8 * i;
      if (gm >= M) continue;
      float sc = alpha;
      if (row_scale) sc *= row_scale[gm];
      float* const crow = C + (out_map ? (int64_t)out_map[gm] : gm) * ldc;
      if (c0 < N)
        *reinterpret_cast<float4*>(crow + c0) =
            make_float4(sc * acc[i][0].x, sc * acc[i][0].y, sc * acc[i][1].x, sc * acc[i][1].y);
      if (c1 < N)
        *reinterpret_cast<float4*>(crow + c1) =
            make_float4(sc * acc[i][2].x, sc * acc[i][2].y, sc * acc[i][3].x, sc * acc[i][3].y);
    }
  }
}

// whether the K-chunked kernel takes the product (KC = 20 or 16); ring depth *stages (as many as fit,
// at most 8) and *smem, its dynamic shared memory
int gemm_kchunk_kc(int64_t N, int64_t K, size_t* smem, int* stages) {
  if (K < 160 || K % 4 || N % 4 || N <= 128 || N > 416) return 0;
  const int kc = K % 20 == 0 ? 20 : (K % 16 == 0 ? 16 : 0);
  if (!kc) return 0;
  // the A pitch K + 4 must keep the 8 row groups of a fragment read on distinct bank pairs
  const int64_t ap = K + 4;
  bool used[16] = {};
  for (int rr = 0; rr < 8; ++rr) {
    const int b = (int)((rr * ap) % 32) / 2;
    if ((rr * ap) % 2 || used[b]) return 0;
    used[b] = true;
  }
  const int64_t NP = round_up(N, 32);
  const size_t a_bytes = (size_t)kResBM * ap * 4, stage = (size_t)kc * NP * 4;
  if (a_bytes + 2 * stage + 512 > 227 * 1024) return 0;
  int S = (int)((227 * 1024 - 512 - a_bytes) / (stage + 16));
  if (S > 8) S = 8;
  *stages = S;
  *smem = a_bytes + (size_t)S * (stage + 16) + 64;
  return kc;
}

// whether the K-resident kernel takes the product; *smem its dynamic shared memory
bool gemm_kres_fits(int64_t N, int64_t K, size_t* smem) {
  if (K < 16 || K > 128 || K % 4 || N % 4 || N <= 128 || N > 416) return false;
  const int64_t NP = round_up(N, 32);
  *smem = (size_t)(K * NP + 2 * kResBM * K) * 4 + 64;
  return *smem <= 227 * 1024;
}

// ------------------------------------------------------------------ A^T B (fp64)
constexpr int ATB_T = 64;   // output tile edge
constexpr int ATB_R = 16;   // rows per smem stage

constexpr int ATB_THREADS = 64;  // 8 x 8 threads, each an 8 x 8 register tile of the 64 x 64 output tile

// Exact fp64 A^T B by DFMA (ISVD_DMMA=0; the default is atb_dmma_kernel): operands promoted to
// fp64 once when staged, fp64 FMA (exact products of the fp32 inputs, fp64 sums), for Grams
// whose input may be ill-conditioned.
using S = double;
__global__ void __launch_bounds__(ATB_THREADS)
    atb_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb, int64_t rows,
               int64_t Ka, int64_t Kb, const float* __restrict__ row_scale, int symmetric, int tiles_a,
               int tiles_b, int64_t rows_per_chunk, double* __restrict__ ws, int64_t ws_ld, const int* gate,
               int /*unused*/) {
  if (gate && *((volatile const int*)gate) == 0) return;
  __shared__ __align__(16) S As[2][ATB_R][ATB_T];
  __shared__ __align__(16) S Bs[2][ATB_R][ATB_T];
  // output tile (ti, tj); symmetric: upper-triangular tiles only, enumerated row by row
  int ti = 0, tj = 0;
  {
    int t = blockIdx.x;
    if (symmetric) {
      while (t >= tiles_a - ti) { t -= tiles_a - ti; ++ti; }
      tj = ti + t;
    } else {
      ti = t / tiles_b;
      tj = t - ti * tiles_b;
    }
  }
  const int64_t a0 = (int64_t)ti * ATB_T, b0 = (int64_t)tj * ATB_T;
  const int64_t chunk = blockIdx.y;
  const int64_t r_begin = chunk * rows_per_chunk;
  int64_t r_end = r_begin + rows_per_chunk;
  if (r_end > rows) r_end = rows;
  const int tid = threadIdx.x;
  const int tx = tid & 7, ty = tid >> 3;
  // staging map: 16 rows x 64 cols = 256 float4 per operand, 4 per thread
  float4 pa[4], pb[4];
  auto load = [&](int64_t r0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int f = tid + u * ATB_THREADS;
      int rr = f >> 4, cc = (f & 15) * 4;
      int64_t gr = r0 + rr;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      if (gr < r_end) {
        if (a0 + cc < Ka) va = __ldg(reinterpret_cast<const float4*>(A + gr * lda + a0 + cc));
        if (b0 + cc < Kb) vb = __ldg(reinterpret_cast<const float4*>(B + gr * ldb + b0 + cc));
        if (row_scale) {
          float s = __ldg(row_scale + gr);
          vb.x *= s; vb.y *= s; vb.z *= s; vb.w *= s;
        }
      }
      pa[u] = va;
      pb[u] = vb;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int f = tid + u * ATB_THREADS;
      int rr = f >> 4, cc = (f & 15) * 4;
      double2* da = reinterpret_cast<double2*>(&As[buf][rr][cc]);
      double2* db = reinterpret_cast<double2*>(&Bs[buf][rr][cc]);
      da[0] = make_double2(pa[u].x, pa[u].y); da[1] = make_double2(pa[u].z, pa[u].w);
      db[0] = make_double2(pb[u].x, pb[u].y); db[1] = make_double2(pb[u].z, pb[u].w);
    }
  };
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  const int64_t nst = (r_end - r_begin + ATB_R - 1) / ATB_R;
  if (nst > 0) {
    load(r_begin);
    store(0);
  }
  __syncthreads();
  for (int64_t st = 0; st < nst; ++st) {
    const int buf = (int)(st & 1);
    if (st + 1 < nst) load(r_begin + (st + 1) * ATB_R);
#pragma unroll 4
    for (int r = 0; r < ATB_R; ++r) {
      double a[8], b[8];
      // 4 x LDS.128 per operand; 8 lanes of a phase read 128 contiguous bytes (no conflicts)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 va = *reinterpret_cast<const double2*>(&As[buf][r][q * 16 + ty * 2]);
        double2 vb = *reinterpret_cast<const double2*>(&Bs[buf][r][q * 16 + tx * 2]);
        a[2 * q] = va.x; a[2 * q + 1] = va.y;
        b[2 * q] = vb.x; b[2 * q + 1] = vb.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (st + 1 < nst) store(buf ^ 1);
    __syncthreads();
  }
  // partial tile -> ws[chunk][a][b]  (ws_ld = padded Kb).  Register element (i, j) of thread
  // (tx, ty) is tile row rowmap(ty, i), column rowmap(tx, j).
  auto tmap = [](int t, int q) { return (q >> 1) * 16 + t * 2 + (q & 1); };
  double* W = ws + chunk * (int64_t)((Ka + ATB_T - 1) / ATB_T * ATB_T) * ws_ld;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double v = acc[i][j];
      W[(a0 + tmap(ty, i)) * ws_ld + b0 + tmap(tx, j)] = v;
    }
}

// Exact fp64 A^T diag(s) B on the FP64 tensor cores (mma.sync m8n8k4 f64): the product of two
// fp32 values is exact in fp64 and the sums are fp64, as in atb_kernel<double>, whose FMA form is
// bound by shared-memory reads (8x8 fp64 fragments: 128 B per 64 DFMA).  Same tiles, chunks and
// workspace layout as atb_kernel (64 x 64 output tile per CTA, upper tiles when symmetric, one
// fp64 partial tile per row chunk, reduced by atb_reduce_kernel).  4 warps, each a 32 x 32 quarter
// as 4 x 4 MMA tiles of 8 x 8; operands staged as fp32 (row stride 72: the fragment loads of a
// warp hit 32 distinct banks) and widened to fp64 in registers.
constexpr int ATBD_THREADS = 128;
constexpr int ATBD_LD = ATB_T + 8;

ISVD_DEVICE void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(ATBD_THREADS)
    atb_dmma_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                    int64_t rows, int64_t Ka, int64_t Kb, const float* __restrict__ row_scale, int symmetric,
                    int tiles_a, int tiles_b, int64_t rows_per_chunk, double* __restrict__ ws, int64_t ws_ld,
                    const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  __shared__ __align__(16) float As[2][ATB_R][ATBD_LD];
  __shared__ __align__(16) float Bs[2][ATB_R][ATBD_LD];
  int ti = 0, tj = 0;
  {
    int t = blockIdx.x;
    if (symmetric) {
      while (t >= tiles_a - ti) { t -= tiles_a - ti; ++ti; }
      tj = ti + t;
    } else {
      ti = t / tiles_b;
      tj = t - ti * tiles_b;
    }
  }
  const int64_t a0 = (int64_t)ti * ATB_T, b0 = (int64_t)tj * ATB_T;
  const int64_t chunk = blockIdx.y;
  const int64_t r_begin = chunk * rows_per_chunk;
  const int64_t r_end = r_begin + rows_per_chunk < rows ? r_begin + rows_per_chunk : rows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;
  // staging: 16 rows x 64 columns = 256 float4 per operand, 2 per thread
  float4 pa[2], pb[2];
  auto load = [&](int64_t r0) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int f = tid + u * ATBD_THREADS;
      const int rr = f >> 4, cc = (f & 15) * 4;
      const int64_t gr = r0 + rr;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      if (gr < r_end) {
        if (a0 + cc < Ka) va = __ldg(reinterpret_cast<const float4*>(A + gr * lda + a0 + cc));
        if (b0 + cc < Kb) vb = __ldg(reinterpret_cast<const float4*>(B + gr * ldb + b0 + cc));
        if (row_scale) {
          const float sc = __ldg(row_scale + gr);
          vb.x *= sc; vb.y *= sc; vb.z *= sc; vb.w *= sc;
        }
      }
      pa[u] = va;
      pb[u] = vb;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int f = tid + u * ATBD_THREADS;
      const int rr = f >> 4, cc = (f & 15) * 4;
      *reinterpret_cast<float4*>(&As[buf][rr][cc]) = pa[u];
      *reinterpret_cast<float4*>(&Bs[buf][rr][cc]) = pb[u];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int g = lane >> 2, q = lane & 3;
  const int64_t nst = (r_end - r_begin + ATB_R - 1) / ATB_R;
  if (nst > 0) {
    load(r_begin);
    store(0);
  }
  __syncthreads();
  for (int64_t st = 0; st < nst; ++st) {
    const int buf = (int)(st & 1);
    if (st + 1 < nst) load(r_begin + (st + 1) * ATB_R);
#pragma unroll
    for (int k0 = 0; k0 < ATB_R; k0 += 4) {
      // A fragment (8 x 4, row): A[m = g][k = q] = Y[k0 + q][col + g]; B (4 x 8, col): B[k = q][n = g]
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        fa[i] = (double)As[buf][k0 + q][wm * 32 + i * 8 + g];
        fb[i] = (double)Bs[buf][k0 + q][wn * 32 + i * 8 + g];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    if (st + 1 < nst) store(buf ^ 1);
    __syncthreads();
  }
  // D[m = g][n = 2 q + {0, 1}] of tile (i, j) -> ws[chunk][a][b]
  double* W = ws + chunk * (int64_t)((Ka + ATB_T - 1) / ATB_T * ATB_T) * ws_ld;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = a0 + wm * 32 + i * 8 + g, c = b0 + wn * 32 + j * 8 + 2 * q;
      *reinterpret_cast<double2*>(&W[r * ws_ld + c]) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

__global__ void atb_reduce_kernel(const double* __restrict__ ws, int64_t ws_ld, int64_t ka_pad, int nchunks,
                                  int64_t Ka, int64_t Kb, int symmetric, double* __restrict__ G, int64_t ldg,
                                  float* __restrict__ out32, int64_t ld32, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  int64_t tot = Ka * Kb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / Kb, j = t - (t / Kb) * Kb;
    int64_t si = i, sj = j;
    if (symmetric && i > j) { si = j; sj = i; }
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += ws[((int64_t)c * ka_pad + si) * ws_ld + sj];
    if (G) G[i * ldg + j] = s;
    if (out32) out32[i * ld32 + j] = (float)s;
  }
}

// ------------------------------------------------------------------ colsum
__global__ void colsum_partial_kernel(const float* __restrict__ Q, int64_t rows, int64_t wpad, int64_t ldq,
                                      int64_t rows_per_block, double* __restrict__ ws) {
  // blockDim (32, 8): x over columns, y over rows
  const int64_t r0 = blockIdx.x * rows_per_block;
  int64_t r1 = r0 + rows_per_block;
  if (r1 > rows) r1 = rows;
  __shared__ double red[8][33];
  for (int64_t c0 = 0; c0 < wpad; c0 += 32) {
    int64_t c = c0 + threadIdx.x;
    double s = 0.0;
    if (c < wpad)
      for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) s += (double)Q[r * ldq + c];
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && c < wpad) {
      double t = 0.0;
      for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
      ws[blockIdx.x * wpad + c] = t;
    }
    __syncthreads();
  }
}

__global__ void colsum_final_kernel(const double* __restrict__ ws, int nblocks, int64_t wpad, double* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < wpad; c += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += ws[b * wpad + c];
    out[c] = s;
  }
}

// rows per colsum block: >= 64, and at most ~8 blocks per SM worth of blocks
int64_t colsum_rows_per_block(int64_t rows) {
  int64_t r = round_up(ceil_div(rows > 0 ? rows : 1, 148 * 8), 64);
  return r < 64 ? 64 : r;
}

// ------------------------------------------------------------------ misc
__global__ void scale_rows_kernel(const float* __restrict__ in, int64_t ldi, float* __restrict__ out, int64_t ldo,
                                  int64_t rows, int64_t w4, const float* __restrict__ vec, float coef,
                                  const int* gate, const int32_t* __restrict__ in_map) {
  if (gate && *((volatile const int*)gate) == 0) return;
  // four independent 16-byte loads in flight per thread (one per trip ran the n x 400 passes of the
  // solver at 2.7 TB/s: 2.9 ms where the copy rate gives 1.3 ms)
  const int64_t tot = rows * w4, S = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t0 < tot; t0 += 4 * S) {
    float4 v[4];
    float sc[4];
    int64_t dst[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = t0 + u * S;
      dst[u] = -1;
      if (t < tot) {
        const int64_t i = row_of(t, w4), c = (t - i * w4) * 4;
        sc[u] = coef * (vec ? vec[i] : 1.f);
        const int64_t src = in_map ? (int64_t)in_map[i] : i;
        ISVD_ASSERT(src >= 0 && c + 3 < ldi && c + 3 < ldo);
        v[u] = *reinterpret_cast<const float4*>(in + src * ldi + c);
        dst[u] = i * ldo + c;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (dst[u] >= 0)
        *reinterpret_cast<float4*>(out + dst[u]) = make_float4(sc[u] * v[u].x, sc[u] * v[u].y, sc[u] * v[u].z, sc[u] * v[u].w);
  }
}

// out[out_map[i], :] = in[i, :]  (rows of `out` not in the map are left as they are)
__global__ void scatter_rows_kernel(const float* __restrict__ in, int64_t ldi, float* __restrict__ out, int64_t ldo,
                                    int64_t rows, int64_t w4, const int32_t* __restrict__ out_map) {
  const int64_t tot = rows * w4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row_of(t, w4), c = (t - i * w4) * 4;
    ISVD_ASSERT(out_map[i] >= 0 && c + 3 < ldo);
    *reinterpret_cast<float4*>(out + (int64_t)out_map[i] * ldo + c) = *reinterpret_cast<const float4*>(in + i * ldi + c);
  }
}

// inv[perm[t]] = t, then out[i] = inv[idx[i]]  (perm: a permutation of [0, n))
__global__ void invert_perm_kernel(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ inv) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    inv[perm[t]] = (int32_t)t;
}
__global__ void gather_idx_kernel(const int32_t* __restrict__ table, const int32_t* __restrict__ idx, int64_t m,
                                  int32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = table[idx[t]];
}

__global__ void scale_cols_kernel(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int64_t w4,
                                  const float* __restrict__ colvec) {
  const int64_t tot = rows * w4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row_of(t, w4), c = (t - i * w4) * 4;
    const float4 v = *reinterpret_cast<const float4*>(in + i * ldi + c);
    const float4 s = *reinterpret_cast<const float4*>(colvec + c);
    *reinterpret_cast<float4*>(out + i * ldo + c) = make_float4(s.x * v.x, s.y * v.y, s.z * v.z, s.w * v.w);
  }
}

__global__ void f64_to_f32_kernel(const double* __restrict__ G, int64_t ldg, float* __restrict__ out, int64_t ldo,
                                  int64_t rows, int64_t cols) {
  int64_t tot = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = row_of(t, cols), j = t - i * cols;
    out[i * ldo + j] = (float)G[i * ldg + j];
  }
}

__global__ void check_finite_kernel(const float* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                    DevStatus* status) {
  int64_t tot = rows * cols;
  int bad = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = row_of(t, cols), j = t - i * cols;
    if (!isfinite(A[i * lda + j])) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status->nonfinite, 1);
}

int grid_for(int64_t work, int threads, int cap) {
  int64_t b = (work + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

cudaError_t launch_gemm_tn(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int64_t M,
                           int64_t N, int64_t K, const float* row_scale, float alpha, bool upper_tri_b,
                           const int* gate, cudaStream_t st, const int32_t* out_map) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  size_t kres_smem = 0;
  static const char* kres_env = getenv("ISVD_GEMM_KRES");  // 0: the tiled kernel for short K too (A/B)
  if (!upper_tri_b && !(kres_env && atoi(kres_env) == 0) && lda % 4 == 0 && ldb % 4 == 0 &&
      ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) && gemm_kres_fits(N, K, &kres_smem)) {
    using KresFn = void (*)(const float*, int64_t, const float*, int64_t, float*, int64_t, int64_t, int, int,
                            const float*, float, const int*, const int32_t*);
    const int NP = (int)round_up(N, 32);
    // compile-time shapes: config 4 (d = 100, l = 400) and config 2 (d = 128, l = 256)
    KresFn fn = (K == 100 && NP == 416)   ? gemm_kres_kernel<100, 416>
                : (K == 128 && NP == 256) ? gemm_kres_kernel<128, 256>
                                          : gemm_kres_kernel<0, 0>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t ntile = ceil_div(M, kResBM);
    const int grid = (int)(ntile < sms ? ntile : sms);
    ++g_launches;
    fn<<<grid, (unsigned)(NP + 32), kres_smem, st>>>(A, lda, B, ldb, C, ldc, M, (int)N, (int)K, row_scale, alpha, gate,
                                                     out_map);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess && getenv("ISVD_TRACE")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, fn);
      fprintf(stderr, "gemm_kres: %s regs %d maxthr %d static smem %zu maxdyn %d threads %d smem %zu\n",
              cudaGetErrorString(le), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
              fa.maxDynamicSharedSizeBytes, NP + 32, kres_smem);
    }
    return le;
  }
  size_t kch_smem = 0;
  int kch_stages = 0;
  static const char* kch_env = getenv("ISVD_GEMM_KCHUNK");  // 0: the tiled kernel for long K (A/B)
  const int kc = (kch_env && atoi(kch_env) == 0) || lda % 4 || ldb % 4 || (uintptr_t)A % 16 || (uintptr_t)B % 16
                     ? 0
                     : gemm_kchunk_kc(N, K, &kch_smem, &kch_stages);
  if (kc) {
    using KchFn = void (*)(const float*, int64_t, const float*, int64_t, float*, int64_t, int64_t, int, int,
                           const float*, float, int, int, const int*, const int32_t*);
    const int NP = (int)round_up(N, 32);
    // compile-time shapes: config 4 (l = 400) and config 2 (l = 256)
    KchFn fn = kc == 20 ? (NP == 416 && K == 400 ? gemm_kchunk_kernel<20, 404, 416> : gemm_kchunk_kernel<20, 0, 0>)
                        : (NP == 256 && K == 256 ? gemm_kchunk_kernel<16, 260, 256> : gemm_kchunk_kernel<16, 0, 0>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t ntile = ceil_div(M, kResBM);
    const int grid = (int)(ntile < sms ? ntile : sms);
    ++g_launches;
    fn<<<grid, (unsigned)(NP + 32), kch_smem, st>>>(A, lda, B, ldb, C, ldc, M, (int)N, (int)K, row_scale, alpha,
                                                    upper_tri_b ? 1 : 0, kch_stages, gate, out_map);
    return cudaGetLastError();
  }
  if (N > 64 && round_up(N, 80) < round_up(N, 128)) {  // e.g. N = 400: 5 x 80 instead of 4 x 128
    // 16-deep K stages halve the CTA barriers for long K (Y R^-1: 12.0 -> 11.7 ms at config 4);
    // for short K (X G_j, K = d = 100) the 8-deep ones waste less on the ragged last stage
    dim3 grid((unsigned)ceil_div(N, 80), (unsigned)ceil_div(M, 128));
    ++g_launches;
    // 3 CTAs per SM (128 registers, a few bytes of spill) hide the per-tile prologue and the
    // barriers better than 2: X G_j 5.47 -> 5.04 ms, Y R^-1 11.65 -> 11.34 ms at config 4
    // (16 x 8 and 12 x 8 register tiles -- fewer shared-memory reads per FMA -- measured slower:
    //  X G_j 7.41 / 6.30 ms, Y R^-1 15.8 / 13.6 ms vs 5.04 / 11.3 ms; profiles/r02b_dense_check.txt)
    if (K >= 256)
      gemm_tn_kernel<128, 80, 16, 8, 8, 3><<<grid, 160, 0, st>>>(A, lda, B, ldb, C, ldc, M, N, K, row_scale, alpha,
                                                                upper_tri_b ? 1 : 0, gate, out_map);
    else
      gemm_tn_kernel<128, 80, 8, 8, 8, 3><<<grid, 160, 0, st>>>(A, lda, B, ldb, C, ldc, M, N, K, row_scale, alpha,
                                                               upper_tri_b ? 1 : 0, gate, out_map);
  } else if (N > 64) {
    dim3 grid((unsigned)ceil_div(N, 128), (unsigned)ceil_div(M, 128));
    ++g_launches; gemm_tn_kernel<128, 128, 8, 8, 8><<<grid, 256, 0, st>>>(A, lda, B, ldb, C, ldc, M, N, K, row_scale, alpha,
                                                           upper_tri_b ? 1 : 0, gate, out_map);
  } else {
    dim3 grid((unsigned)ceil_div(N, 64), (unsigned)ceil_div(M, 128));
    ++g_launches; gemm_tn_kernel<128, 64, 8, 8, 4><<<grid, 256, 0, st>>>(A, lda, B, ldb, C, ldc, M, N, K, row_scale, alpha,
                                                          upper_tri_b ? 1 : 0, gate, out_map);
  }
  return cudaGetLastError();
}

// ------------------------------------------------ A^T B, fp32 chunks (f32_stage)
// Register-tiled SIMT contraction over a chunk of <= kF32ChunkRows rows, fp32 FMA
// accumulation inside the chunk (relative error ~ sqrt(chunk) u_fp32 ~ 2e-6), fp32
// partial tiles reduced in fp64 across chunks in a fixed order.  Thread (tx, ty) owns
// rows ty*TM + 0..TM-1 and columns {tx*4 + 0..3, BN/2 + tx*4 + 0..3} of a BM x BN tile, so
// every shared-memory float4 read of a quarter-warp is conflict-free.  Tile shapes are
// picked per call by padding and register-tile size (d = 100, l = 400: 104 x 80, 8 x 8).
constexpr int kF32ChunkRows = 1024;
constexpr int kF32Stage = 16;

// 16-byte asynchronous global -> shared copy (LDGSTS); src_bytes = 0 zero-fills
ISVD_DEVICE void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}
ISVD_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
ISVD_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


// SCALE: a row scale is applied to A inside the loop (one FMUL per A element and row); callers
// that can pass a pre-scaled A use SCALE = false (the same fp32 products, about 11 % fewer
// FMA-pipe cycles).
template <int BM, int BN, int TM, int TN, int MINB = 1, bool SCALE = true>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
    atb_f32_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb, int64_t rows,
                   int64_t Ka, int64_t Kb, const float* __restrict__ row_scale, int tiles_b, int64_t rows_per_chunk,
                   float* __restrict__ ws, int64_t ws_lda, int64_t ws_ld, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  static_assert(TM == 4 || TM == 8, "rows per thread");
  static_assert(TN == 8 || TN == 16, "columns per thread");
  constexpr int TY = BM / TM, TX = BN / TN, NT = TX * TY;
  constexpr int QN = TN / 4, CS = BN / QN;  // thread column groups: tx*4 + q*CS, q < QN
  // rows per stage: 32 where two stages fit the 48 KB of static shared memory (half the CTA
  // barriers of 16-row stages), else 16; ring depth 3 where it fits, else 2
  constexpr int SR = 2 * (32 * (BM + BN) + 32) * 4 <= 48 * 1024 ? 32 : kF32Stage;
  constexpr int A4 = SR * BM / 4, B4 = SR * BN / 4;  // float4 per stage
  constexpr int kF32Ring = 3 * (SR * (BM + BN) + SR) * 4 <= 48 * 1024 ? 3 : 2;
  __shared__ __align__(16) float As[kF32Ring][SR][BM];
  __shared__ __align__(16) float Bs[kF32Ring][SR][BN];
  __shared__ __align__(16) float Ss[kF32Ring][SR];  // row scales of the stage (applied to A)
  const int tid = threadIdx.x;
  int tx, ty;
  thread_xy<TX>(tid, &tx, &ty);
  const int ti = blockIdx.x / tiles_b, tj = blockIdx.x - ti * tiles_b;
  const int64_t a0 = (int64_t)ti * BM, b0 = (int64_t)tj * BN;
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_chunk;
  const int64_t r_end = r_begin + rows_per_chunk < rows ? r_begin + rows_per_chunk : rows;
  // issue the copies of stage s (rows r_begin + 16 s ..) into ring slot s % kF32Ring; rows and
  // columns outside the operands are zero-filled
  auto issue = [&](int64_t s) {
    const int slot = (int)(s % kF32Ring);
    const int64_t r0 = r_begin + s * SR;
    for (int f = tid; f < A4 + B4; f += NT) {
      if (f < A4) {
        const int rr = f / (BM / 4), cc = (f % (BM / 4)) * 4;
        const int64_t gr = r0 + rr;
        const bool ok = gr < r_end && a0 + cc < Ka;
        cp_async16(&As[slot][rr][cc], ok ? A + gr * lda + a0 + cc : A, ok ? 16 : 0);
      } else {
        const int g = f - A4;
        const int rr = g / (BN / 4), cc = (g % (BN / 4)) * 4;
        const int64_t gr = r0 + rr;
        const bool ok = gr < r_end && b0 + cc < Kb;
        cp_async16(&Bs[slot][rr][cc], ok ? B + gr * ldb + b0 + cc : B, ok ? 16 : 0);
      }
    }
    if (SCALE && row_scale && tid < SR) {
      const int64_t gr = r0 + tid;
      Ss[slot][tid] = gr < r_end ? __ldg(row_scale + gr) : 0.f;
    }
  };
  float2 acc[TM][TN / 2];  // column pairs (FFMA2)
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  const int64_t nst = (r_end - r_begin + SR - 1) / SR;
#pragma unroll
  for (int s = 0; s < kF32Ring - 1; ++s) {
    if (s < nst) issue(s);
    cp_async_commit();
  }
  for (int64_t s = 0; s < nst; ++s) {
    cp_async_wait<kF32Ring - 2>();  // stage s landed (this thread's copies)
    __syncthreads();                // ... everyone's; and slot (s - 1) % ring is free
    if (s + kF32Ring - 1 < nst) issue(s + kF32Ring - 1);
    cp_async_commit();
    const int buf = (int)(s % kF32Ring);
#pragma unroll
    for (int kk = 0; kk < SR; ++kk) {
      float a[TM];
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        const float4 va = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM + i]);
        if (SCALE) {
          const float sc = row_scale ? Ss[buf][kk] : 1.f;
          a[i] = va.x * sc; a[i + 1] = va.y * sc; a[i + 2] = va.z * sc; a[i + 3] = va.w * sc;
        } else {
          a[i] = va.x; a[i + 1] = va.y; a[i + 2] = va.z; a[i + 3] = va.w;
        }
      }
      float b[TN];
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(&Bs[buf][kk][q * CS + tx * 4]);
        b[4 * q] = v.x; b[4 * q + 1] = v.y; b[4 * q + 2] = v.z; b[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN / 2; ++j) acc[i][j] = ffma2(make_float2(a[i], a[i]), make_float2(b[2 * j], b[2 * j + 1]), acc[i][j]);
    }
  }
  cp_async_wait<0>();
  float* W = ws + (int64_t)blockIdx.y * ws_lda * ws_ld;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    float* w = W + (a0 + ty * TM + i) * ws_ld + b0;
#pragma unroll
    for (int q = 0; q < QN; ++q)
      *reinterpret_cast<float4*>(w + q * CS + tx * 4) =
          make_float4(acc[i][2 * q].x, acc[i][2 * q].y, acc[i][2 * q + 1].x, acc[i][2 * q + 1].y);
  }
}

// One warp per group of chunks: warp g of a 256-thread CTA sums the chunks c = g (mod 8) of 32
// consecutive output entries in increasing order (four loads in flight per lane), and the eight group
// sums are combined in a fixed tree -- the same sums in the same order as one thread per entry with
// eight interleaved partial sums (round 1), but with 8x the loads in flight: the 40,000-entry
// reduction of X^T Z_j (2,392 chunks, 383 MB of partials) ran at 2.7 TB/s.
__global__ void __launch_bounds__(256)
    atb_f32_reduce_kernel(const float* __restrict__ ws, int64_t ws_lda, int64_t ws_ld, int nchunks, int64_t Ka,
                          int64_t Kb, int symmetric, double* __restrict__ G, int64_t ldg, float* __restrict__ out32,
                          int64_t ld32, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t tot = Ka * Kb;
  const int64_t cstride = ws_lda * ws_ld;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < tot; base += (int64_t)gridDim.x * 32) {
    const int64_t t = base + lane;
    double acc = 0.0;
    int64_t i = 0, j = 0;
    if (t < tot) {
      i = t / Kb;
      j = t - i * Kb;
      int64_t si = i, sj = j;
      if (symmetric && i > j) { si = j; sj = i; }
      const float* src = ws + si * ws_ld + sj;
      int c = grp;
      for (; c + 24 < nchunks; c += 32) {
        const float v0 = src[(int64_t)c * cstride], v1 = src[(int64_t)(c + 8) * cstride];
        const float v2 = src[(int64_t)(c + 16) * cstride], v3 = src[(int64_t)(c + 24) * cstride];
        acc += (double)v0;
        acc += (double)v1;
        acc += (double)v2;
        acc += (double)v3;
      }
      for (; c < nchunks; c += 8) acc += (double)src[(int64_t)c * cstride];
    }
    part[grp][lane] = acc;
    __syncthreads();
    if (grp == 0 && t < tot) {
      const double s = ((part[0][lane] + part[1][lane]) + (part[2][lane] + part[3][lane])) +
                       ((part[4][lane] + part[5][lane]) + (part[6][lane] + part[7][lane]));
      if (G) G[i * ldg + j] = s;
      if (out32) out32[i * ld32 + j] = (float)s;
    }
    __syncthreads();
  }
}

struct F32Tiling {
  int bm, bn, tm, tn;
  int64_t ta, tb, chunk_rows, chunks;
};

F32Tiling f32_tiling(int64_t rows, int64_t Ka, int64_t Kb, int num_sms) {
  // {BM, BN, TM}: 8 x 8 register tiles halve the shared-memory reads per FMA (the 4 x 8 tiles
  // are shared-memory-bound), so they win unless their padding costs more than ~1/3
  // {BM, BN, TM, TN}; cost = padded area x shared-memory floats per FMA ((TM + TN) / (TM TN)):
  // on B200 (128 FP32 lanes, 128 B/clk of shared memory per SM) small register tiles are
  // shared-memory-bound.  (8 x 16 tiles need 255 registers; at 2 CTAs per SM they measured
  // slower than 8 x 8 -- 0.95 vs 0.88 s per config-4 isvd -- and are not offered.)
  // (32 x 32: the symmetric Gram's small trailing diagonal block, e.g. 16 x 16 at l = 400)
  // (104 x 200 in 325-thread CTAs -- 8 % idle lanes instead of the 19 % of 104 x 80's 130 threads,
  // but 135 registers, one CTA per SM -- measured no faster: 6.45 vs 6.38 ms, round 2)
  const int cand[6][4] = {{64, 64, 4, 8}, {100, 80, 4, 8}, {128, 128, 4, 8}, {104, 80, 8, 8}, {128, 128, 8, 8},
                          {32, 32, 4, 8}};
  // Round 2: the cost also counts idle lanes of a partial last warp (104 x 80 x (8 x 8) is 130 threads:
  // its fifth warp issues every instruction for 2 threads) and weighs the shared-memory reads per FMA
  // as an overhead on the FMAs rather than the bound (ncu: FMA pipe 66 % active, LSU 27 %, barrier
  // stalls first).  At d = 100, l = 400 that picks 100 x 80 x (4 x 8), 250 threads, no padding:
  // X^T Z_j 6.67 -> 4.70 ms (profiles/r02e_dense_check.txt).
  F32Tiling t{64, 64, 4, 8, 0, 0, 0, 0};
  double best = -1;
  for (auto& c : cand) {
    const int thr = (c[0] / c[2]) * (c[1] / c[3]);
    const double lanes = (double)round_up(thr, 32) / thr;
    const double cost = (double)round_up(Ka, c[0]) * round_up(Kb, c[1]) * lanes *
                        (1.0 + (double)(c[2] + c[3]) / (c[2] * c[3]));
    if (best < 0 || cost < best) {
      best = cost;
      t.bm = c[0];
      t.bn = c[1];
      t.tm = c[2];
      t.tn = c[3];
    }
  }
  t.ta = ceil_div(Ka, t.bm);
  t.tb = ceil_div(Kb, t.bn);
  // enough CTAs to fill the GPU several times over, chunks of 64 .. kF32ChunkRows rows
  int64_t want = ceil_div(4LL * num_sms, t.ta * t.tb);
  int64_t cr = round_up(ceil_div(rows > 0 ? rows : 1, want), kF32Stage);
  if (cr > kF32ChunkRows) cr = kF32ChunkRows;
  if (cr < 64) cr = 64;
  t.chunk_rows = cr;
  t.chunks = rows > 0 ? ceil_div(rows, cr) : 1;
  return t;
}

static int64_t atb_chunks(int64_t rows, int64_t ntiles, int num_sms) {
  int64_t target = 8LL * num_sms;  // 64-thread CTAs, several resident per SM
  int64_t ch = ceil_div(target, ntiles);
  int64_t max_ch = ceil_div(rows, 256);  // at least 256 rows per chunk
  if (ch > max_ch) ch = max_ch;
  if (ch < 1) ch = 1;
  return ch;
}

static int64_t atb_ntiles(int64_t Ka, int64_t Kb, bool symmetric) {
  int64_t ta = ceil_div(Ka, ATB_T), tb = ceil_div(Kb, ATB_T);
  return symmetric ? ta * (ta + 1) / 2 : ta * tb;
}

cudaError_t launch_atb_f32_reduce(const float* ws32, int64_t ws_lda, int64_t ws_ld, int64_t chunks, int64_t Ka,
                                  int64_t Kb, bool symmetric, double* G, int64_t ldg, float* out32, int64_t ld32,
                                  int num_sms, const int* gate, cudaStream_t st) {
  ++g_launches;
  atb_f32_reduce_kernel<<<grid_for(Ka * Kb, 32, num_sms * 16), 256, 0, st>>>(
      ws32, ws_lda, ws_ld, (int)chunks, Ka, Kb, symmetric ? 1 : 0, G, ldg, out32, ld32, gate);
  return cudaGetLastError();
}

int64_t atb_ws_doubles(int64_t rows, int64_t Ka, int64_t Kb, int num_sms) {
  // the non-symmetric tile count is the smaller one, so its chunk count bounds both cases
  int64_t ch = atb_chunks(rows, atb_ntiles(Ka, Kb, Ka == Kb), num_sms);
  int64_t ch2 = atb_chunks(rows, atb_ntiles(Ka, Kb, false), num_sms);
  if (ch2 > ch) ch = ch2;
  const int64_t f64_path = ch * round_up(Ka, ATB_T) * round_up(Kb, ATB_T);
  F32Tiling t = f32_tiling(rows, Ka, Kb, num_sms);
  const int64_t f32_path = (t.chunks * t.ta * t.bm * t.tb * t.bn + 1) / 2;  // floats -> doubles
  return f64_path > f32_path ? f64_path : f32_path;
}

// the exact fp64 Grams on the FP64 tensor cores (mma.sync f64) unless ISVD_DMMA=0
static bool atb_dmma_enabled() {
  const char* v = getenv("ISVD_DMMA");
  return !(v && v[0] == '0');
}

cudaError_t launch_atb(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t rows, int64_t Ka, int64_t Kb,
                       const float* row_scale, bool symmetric, double* ws, double* G, int64_t ldg, float* out32,
                       int64_t ld32, int num_sms, const int* gate, cudaStream_t st,
                       bool f32_stage) {
  if (Ka <= 0 || Kb <= 0) return cudaSuccess;
  if (f32_stage) {
    F32Tiling t = f32_tiling(rows, Ka, Kb, num_sms);
    float* ws32 = reinterpret_cast<float*>(ws);
    const int64_t ws_lda = t.ta * t.bm, ws_ld = t.tb * t.bn;
    if (rows > 0) {
      dim3 grid((unsigned)(t.ta * t.tb), (unsigned)t.chunks);
      ++g_launches;
      // 4 x 16 register tiles at 100 x 80 (125-thread CTAs): 5 shared-memory float4 reads per 32 paired
      // FMAs instead of 3 per 16 -- the 4 x 8 form is bound by shared-memory wavefronts (a float4 read
      // costs a wavefront per quarter-warp: ~12 per warp and k-step against 32 FMA-pipe cycles).  The
      // same per-entry sums in the same order: X^T Z_j 4.70 -> 4.47 ms (profiles/r02h_dense_check.txt).
      // ISVD_ATB_TN16=0: the 4 x 8 form; 2: three CTAs per SM.
      static const char* tn16_env = getenv("ISVD_ATB_TN16");
      const int tn16 = tn16_env ? atoi(tn16_env) : 1;
#define ISVD_ATB_F32(BM_, BN_, TM_, TN_)                                                                \
  if (t.bm == BM_ && t.bn == BN_ && t.tm == TM_ && t.tn == TN_)                                          \
    atb_f32_kernel<BM_, BN_, TM_, TN_><<<grid, (BM_ / TM_) * (BN_ / TN_), 0, st>>>(                       \
        A, lda, B, ldb, rows, Ka, Kb, row_scale, (int)t.tb, t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      ISVD_ATB_F32(64, 64, 4, 8)
      else ISVD_ATB_F32(32, 32, 4, 8)
      else if (t.bm == 100 && t.bn == 80 && t.tm == 4 && t.tn == 8 && row_scale)  // 250 threads, full warps
        atb_f32_kernel<100, 80, 4, 8, 3><<<grid, 250, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, row_scale, (int)t.tb,
                                                              t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      else if (t.bm == 100 && t.bn == 80 && t.tm == 4 && t.tn == 8 && !row_scale && tn16 == 1)
        atb_f32_kernel<100, 80, 4, 16, 4, false><<<grid, 125, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, nullptr, (int)t.tb,
                                                                      t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      else if (t.bm == 100 && t.bn == 80 && t.tm == 4 && t.tn == 8 && !row_scale && tn16 == 2)
        atb_f32_kernel<100, 80, 4, 16, 3, false><<<grid, 125, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, nullptr, (int)t.tb,
                                                                      t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      else if (t.bm == 100 && t.bn == 80 && t.tm == 4 && t.tn == 8)  // X^T Z_j with a pre-scaled X: 4.7 ms
        atb_f32_kernel<100, 80, 4, 8, 4, false><<<grid, 250, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, nullptr, (int)t.tb,
                                                                     t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      else if (t.bm == 104 && t.bn == 80 && t.tm == 8 && row_scale)  // 4 CTAs per SM (96 registers): 8.2 -> 7.4 ms at config 4
        atb_f32_kernel<104, 80, 8, 8, 4><<<grid, 130, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, row_scale, (int)t.tb,
                                                              t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      else if (t.bm == 104 && t.bn == 80 && t.tm == 8)  // no row scale (X^T Z_j with a pre-scaled X)
        atb_f32_kernel<104, 80, 8, 8, 4, false><<<grid, 130, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, nullptr, (int)t.tb,
                                                                     t.chunk_rows, ws32, ws_lda, ws_ld, gate);
      else ISVD_ATB_F32(128, 128, 8, 8)
#undef ISVD_ATB_F32
    } else {
      cudaMemsetAsync(ws32, 0, sizeof(float) * ws_lda * ws_ld, st);
    }
    ++g_launches;
    atb_f32_reduce_kernel<<<grid_for(Ka * Kb, 32, num_sms * 16), 256, 0, st>>>(
        ws32, ws_lda, ws_ld, rows > 0 ? (int)t.chunks : 1, Ka, Kb, symmetric ? 1 : 0, G, ldg, out32, ld32, gate);
    return cudaGetLastError();
  }
  int64_t ta = ceil_div(Ka, ATB_T), tb = ceil_div(Kb, ATB_T);
  int64_t ntiles = atb_ntiles(Ka, Kb, symmetric);
  int64_t ch = atb_chunks(rows, ntiles, num_sms);
  int64_t rpc = rows > 0 ? round_up(ceil_div(rows, ch), ATB_R) : ATB_R;
  ch = rows > 0 ? ceil_div(rows, rpc) : 1;
  int64_t ka_pad = round_up(Ka, ATB_T), ws_ld = round_up(Kb, ATB_T);
  if (rows > 0) {
    dim3 grid((unsigned)ntiles, (unsigned)ch);
    ++g_launches;
    if (atb_dmma_enabled())
      atb_dmma_kernel<<<grid, ATBD_THREADS, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, row_scale, symmetric ? 1 : 0,
                                                     (int)ta, (int)tb, rpc, ws, ws_ld, gate);
    else
      atb_kernel<<<grid, ATB_THREADS, 0, st>>>(A, lda, B, ldb, rows, Ka, Kb, row_scale, symmetric ? 1 : 0,
                                               (int)ta, (int)tb, rpc, ws, ws_ld, gate, 0);
  } else {
    cudaMemsetAsync(ws, 0, sizeof(double) * ka_pad * ws_ld, st);
    ch = 1;
  }
  ++g_launches; atb_reduce_kernel<<<grid_for(Ka * Kb, 256, num_sms * 8), 256, 0, st>>>(ws, ws_ld, ka_pad, (int)ch, Ka, Kb,
                                                                         symmetric ? 1 : 0, G, ldg, out32, ld32, gate);
  return cudaGetLastError();
}

int64_t colsum_ws_doubles(int64_t rows, int64_t wpad) {
  return (ceil_div(rows, colsum_rows_per_block(rows)) + 1) * wpad;
}

cudaError_t launch_colsum(const float* Q, int64_t rows, int64_t wpad, int64_t ldq, double* ws, double* out,
                          cudaStream_t st) {
  const int64_t rpb = colsum_rows_per_block(rows);
  int64_t nb = ceil_div(rows, rpb);
  if (nb < 1) {
    cudaMemsetAsync(out, 0, sizeof(double) * wpad, st);
    return cudaGetLastError();
  }
  ++g_launches; colsum_partial_kernel<<<(unsigned)nb, dim3(32, 8), 0, st>>>(Q, rows, wpad, ldq, rpb, ws);
  ++g_launches; colsum_final_kernel<<<grid_for(wpad, 128, 64), 128, 0, st>>>(ws, (int)nb, wpad, out);
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int64_t wpad,
                              const float* vec, float coef, const int* gate, cudaStream_t st,
                              const int32_t* in_map) {
  if (rows <= 0) return cudaSuccess;
  ++g_launches;
  scale_rows_kernel<<<grid_for(rows * (wpad / 4), 256, 148 * 16), 256, 0, st>>>(in, ldi, out, ldo, rows, wpad / 4,
                                                                               vec, coef, gate, in_map);
  return cudaGetLastError();
}

cudaError_t launch_scale_cols(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int64_t wpad,
                              const float* colvec, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  ++g_launches;
  scale_cols_kernel<<<grid_for(rows * (wpad / 4), 256, 148 * 16), 256, 0, st>>>(in, ldi, out, ldo, rows, wpad / 4,
                                                                               colvec);
  return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const float* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int64_t wpad,
                               const int32_t* out_map, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  ++g_launches;
  scatter_rows_kernel<<<grid_for(rows * (wpad / 4), 256, 148 * 16), 256, 0, st>>>(in, ldi, out, ldo, rows, wpad / 4,
                                                                                 out_map);
  return cudaGetLastError();
}

cudaError_t launch_compose_inverse(const int32_t* perm, int64_t n, const int32_t* idx, int64_t m, int32_t* inv_ws,
                                   int32_t* out, cudaStream_t st) {
  if (n > 0) {
    ++g_launches;
    invert_perm_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(perm, n, inv_ws);
  }
  if (m > 0) {
    ++g_launches;
    gather_idx_kernel<<<grid_for(m, 256, 148 * 8), 256, 0, st>>>(inv_ws, idx, m, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* G, int64_t ldg, float* out, int64_t ldo, int64_t rows, int64_t cols,
                              cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  ++g_launches; f64_to_f32_kernel<<<grid_for(rows * cols, 256, 148 * 8), 256, 0, st>>>(G, ldg, out, ldo, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* A, int64_t lda, int64_t rows, int64_t cols, DevStatus* status,
                                cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  ++g_launches; check_finite_kernel<<<grid_for(rows * cols, 256, 148 * 8), 256, 0, st>>>(A, lda, rows, cols, status);
  return cudaGetLastError();
}

// ---- simulated ranks (test backend of the row-partitioned schedule, capi.cpp SimGroup) ----
// out[i] = sum_{q = 0..world-1} in_q[i], always in rank order: every logical rank runs this same
// kernel on the same inputs, so the all-reduced values are bitwise identical across ranks.
namespace {
__global__ void sum_ranks_kernel(RankPtrs p, int world, int64_t count, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < world; ++q) s += p.p[q][i];
    out[i] = s;
  }
}
}  // namespace

cudaError_t launch_sum_ranks(const RankPtrs& p, int world, int64_t count, double* out, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  ++g_launches; sum_ranks_kernel<<<grid_for(count, 256, 148 * 4), 256, 0, st>>>(p, world, count, out);
  return cudaGetLastError();
}

}  // namespace isvd
