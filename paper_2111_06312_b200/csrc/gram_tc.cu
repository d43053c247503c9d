// Tensor-core tall-skinny products C = (diag(s) A)^T B on tcgen05, 3xTF32, for
//   * the Grams G = Y^T Y of CholeskyQR (Alg. 2 right) of tall iterates, and
//   * the NC blocks X^T A_hat^j Q of M^T Q (Eq. 6) -- X^T diag(1/s) Zt_j.
//
// north_star: tensor cores only in these contractions, and only where 3xTF32 meets the
// tolerance.  Each operand value x is split x = hi + lo (hi = x with the low 13 mantissa bits
// cleared, exactly a TF32 value; lo = x - hi exactly); a product is hi*hi' + hi*lo' + lo*hi'
// (relative error ~2^-21).  The tensor core's fp32 accumulation truncates (measured:
// profiles/umma_mn_probe.cu variant 3; profiles/gram_tc_check.cu), so the error grows with the
// number of MMAs accumulated into one TMEM value.  Hence:
//   * a TMEM accumulator covers one CHUNK of 128 rows (16 k-steps x 3 MMAs), then it is drained;
//     two accumulators alternate so the MMAs of chunk c+1 run while chunk c is drained;
//   * the drained chunk is added (round-to-nearest fp32) into per-thread running sums in
//     registers; the CTA's sums over its row range are written as one fp32 partial;
//   * partials are summed in fp64 in a fixed order by atb_f32_reduce_kernel (dense.cu).
// The result is in the fp32-chunk numerics class of the SIMT path.
//
// One CTA (18 warps, 1 per SM: TMEM 2N columns, ~200 KB smem) computes a 128 x N tile over a
// contiguous row range, in 16-row steps:
//   * the producer warp TMA-loads (cp.async.bulk.tensor.2d, no swizzle) the raw row-major tiles
//     A[16 x 128] and B[16 x N] into a 3-deep ring (rows past the tensor are zero-filled);
//   * 16 converter warps rewrite each raw tile into the UMMA K-major no-swizzle canonical layout
//     (core matrices of 8 MN-rows x 4 K-values = 16 bytes per row, MN-groups 128 B apart,
//     K-groups E/8*128 B apart), split into hi / lo: a thread reads a 4 x 4 block (4 rows, one
//     float4 each), transposes it and stores four 4-value K-vectors into a 3-deep ring.  (The
//     MN-major operand form of kind::tf32, which would take the row-major tiles as they are,
//     produced no output in every descriptor variant tried -- profiles/umma_mn_probe.cu.)
//   * the MMA warp issues 2 k-steps x 3 tcgen05.mma.kind::tf32 (M = 128, N <= 256, K = 8) per
//     step, commits to the converted slot's "empty" barrier and, at the end of a chunk, to the
//     chunk accumulator's "full" barrier;
//   * the converter warps drain each finished chunk (tcgen05.ld.32x32b: warp w reads TMEM lanes
//     32 (w % 4) .. +31, column quarter w / 4) and release the accumulator.
// Operand descriptors and the instruction descriptor follow the sm_100 UMMA bit layouts.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "umma.cuh"

namespace isvd {
namespace {

constexpr int kTcM = 128;       // UMMA M (rows of the C tile = columns of A)
constexpr int kTcChunk = 128;   // rows per TMEM accumulation (truncation bound)

// Store the K-vector (rows k0..k0+3, k0 % 4 == 0) of MN-element c into the K-major layout.
ISVD_DEVICE void st_split(float* hi, float* lo, int k0, int c, int lbo_floats, float4 v) {
  const int off = (k0 >> 2) * lbo_floats + (c >> 3) * 32 + (c & 7) * 4;
  float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// Convert one 4 x 4 block (raw rows 4 kb .. +3, columns 4 cb .. +3, row-major with row stride
// W floats) into the K-major hi / lo layout of an E-wide operand.  Rows >= valid_rows and
// columns >= valid_cols are zero; row q is multiplied by sc[q].
// Bank map: the 16-byte store slot of (cb, j) within a 128-byte line is 4 (cb & 1) + j', with
// j' = (j + (cb >> 1)) & 3, so 8 consecutive blocks hit 8 distinct slots.
template <int E, int W>
ISVD_DEVICE void convert_block(const float* raw, float* hi, float* lo, int kb, int cb, int valid_rows,
                               int valid_cols, const float (&sc)[4]) {
  constexpr int LBO = E / 8 * 32;  // floats
  float4 v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = kb * 4 + q;
    v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < valid_rows && cb * 4 < valid_cols) {
      v[q] = *reinterpret_cast<const float4*>(raw + r * W + cb * 4);
      v[q].x *= sc[q]; v[q].y *= sc[q]; v[q].z *= sc[q]; v[q].w *= sc[q];
    }
  }
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const int j = (jj + (cb >> 1)) & 3;
    float4 kv;
    if (j == 0) kv = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
    else if (j == 1) kv = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
    else if (j == 2) kv = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
    else kv = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
    st_split(hi, lo, kb * 4, cb * 4 + j, LBO, kv);
  }
}

template <int N>
struct TcCfg {
  static constexpr int kStep = 16;                     // rows per pipeline step (2 MMAs of K = 8)
  static constexpr int kStepsPerChunk = kTcChunk / kStep;
  static constexpr int kRaw = 3;                       // TMA ring of raw row tiles
  static constexpr int kConv = 3;                      // ring of converted (K-major hi / lo) operands
  static constexpr int RAW_FL = kStep * (kTcM + N);    // raw A | raw B rows of one step
  static constexpr int A_FL = kStep * kTcM, B_FL = kStep * N;
  static constexpr int CONV_FL = 2 * A_FL + 2 * B_FL;  // A hi | A lo | B hi | B lo
  static constexpr size_t smem_bytes() { return (size_t)(kRaw * RAW_FL + kConv * CONV_FL) * sizeof(float); }
};

// Warp roles (warp specialisation; hand-offs through mbarriers, no CTA-wide barrier per step):
//   warps 0..15  converters + drainers: raw tile -> K-major hi / lo operands; every chunk, warp w
//                drains TMEM lane quadrant w % 4, column quarter w / 4 into its register sums
//   warp 16      TMA producer (lane 0)
//   warp 17      MMA issuer (lane 0)
// Measured at config 4 (Gram 2.45M x 400): 7.77 ms; 8 converter warps (168 registers, no spill)
// 9.2 ms; the CTA-barrier lockstep form 7.95 ms.  The conversion's shared-memory traffic
// (TMA write, transposing read/write of hi and lo, MMA operand reads: ~150 KB per 16-row step)
// is the limit, not the hand-offs.
constexpr int kTcConvWarps = 16;
constexpr int kTcWsThreads = (kTcConvWarps + 2) * 32;

template <int N>
__global__ void __launch_bounds__(kTcWsThreads, 1)
    tc_atb_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t Ka,
                  const float* __restrict__ rs, int64_t Kb, int64_t rows, int ta, int tb, int symmetric,
                  int64_t rows_per_cta, float* __restrict__ ws, int64_t ws_lda, int64_t ws_ld, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  using C = TcCfg<N>;
  static_assert(N % 16 == 0 && N >= 32 && N <= 256, "UMMA N");
  constexpr int KS = C::kStep;
  constexpr int LBO_A = kTcM / 8 * 32, LBO_B = N / 8 * 32;  // K-group (4 values) strides in floats
  constexpr int CT = kTcConvWarps * 32;                      // converter threads
  constexpr int NBLK_A = (KS / 4) * (kTcM / 4), NBLK = NBLK_A + (KS / 4) * (N / 4);
  constexpr int QTR = N / (kTcConvWarps / 4);               // columns drained per thread
  constexpr uint32_t kCols = 2 * N <= 256 ? 256 : 512;       // TMEM: two N-column accumulators
  static_assert(QTR % 4 == 0, "drain granularity");
  static_assert(NBLK_A <= CT, "A blocks in the first round");

  extern __shared__ __align__(1024) float sm[];
  float* const raw0 = sm;                          // raw slot i at raw0 + i * RAW_FL
  float* const conv0 = sm + C::kRaw * C::RAW_FL;   // conv slot i at conv0 + i * CONV_FL
  __shared__ __align__(8) uint64_t raw_full[C::kRaw], raw_empty[C::kRaw];
  __shared__ __align__(8) uint64_t conv_full[C::kConv], conv_empty[C::kConv];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // tile of this CTA (symmetric: only tiles holding some (i <= j))
  int ti = 0, tj = 0;
  {
    int t = blockIdx.x;
    for (int i = 0; i < ta; ++i)
      for (int j = 0; j < tb; ++j) {
        if (symmetric && (int64_t)i * kTcM > (int64_t)j * N + N - 1) continue;
        if (t-- == 0) { ti = i; tj = j; }
      }
  }
  const int64_t a0 = (int64_t)ti * kTcM, b0 = (int64_t)tj * N;
  const int a_cols = (int)(Ka - a0 < kTcM ? Ka - a0 : kTcM);  // valid columns of the tile
  const int b_cols = (int)(Kb - b0 < N ? Kb - b0 : N);
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r_end = r_begin + rows_per_cta < rows ? r_begin + rows_per_cta : rows;
  const int64_t nst = r_end > r_begin ? (r_end - r_begin + KS - 1) / KS : 0;
  const int64_t nch = (nst + C::kStepsPerChunk - 1) / C::kStepsPerChunk;

  if (tid == 0) {
    for (int i = 0; i < C::kRaw; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], kTcConvWarps);
    }
    for (int i = 0; i < C::kConv; ++i) {
      mbar_init(&conv_full[i], kTcConvWarps);
      mbar_init(&conv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kTcConvWarps);
    }
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

  if (warp == kTcConvWarps) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int64_t st = 0; st < nst; ++st) {
        const int slot = (int)(st % C::kRaw);
        if (st >= C::kRaw) mbar_wait(&raw_empty[slot], (uint32_t)((st / C::kRaw - 1) & 1));
        float* rawA = raw0 + slot * C::RAW_FL;
        mbar_expect_tx(&raw_full[slot], (uint32_t)C::RAW_FL * 4);
        const int r0 = (int)(r_begin + st * KS);
        tma_2d(rawA, &tmA, (int)a0, r0, &raw_full[slot]);
        tma_2d(rawA + C::A_FL, &tmB, (int)b0, r0, &raw_full[slot]);
      }
    }
  } else if (warp == kTcConvWarps + 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(kTcM, N);
      for (int64_t st = 0; st < nst; ++st) {
        const int cs = (int)(st % C::kConv);
        const int64_t ch = st / C::kStepsPerChunk;
        const bool first = (st % C::kStepsPerChunk) == 0;
        if (first && ch >= 2) mbar_wait(&acc_empty[ch & 1], (uint32_t)((ch / 2 - 1) & 1));  // drained
        mbar_wait(&conv_full[cs], (uint32_t)((st / C::kConv) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(ch & 1) * N;
        const uint32_t ah = smem_u32(conv0 + cs * C::CONV_FL), al = ah + C::A_FL * 4;
        const uint32_t bh = ah + 2 * C::A_FL * 4, bl = bh + C::B_FL * 4;
#pragma unroll
        for (int s = 0; s < KS / 8; ++s) {
          // one MMA (K = 8) spans two K-groups
          const uint32_t ka = (uint32_t)(2 * s) * LBO_A * 4, kb = (uint32_t)(2 * s) * LBO_B * 4;  // bytes
          const uint64_t dah = umma_desc(ah + ka, LBO_A * 4, 128), dal = umma_desc(al + ka, LBO_A * 4, 128);
          const uint64_t dbh = umma_desc(bh + kb, LBO_B * 4, 128), dbl = umma_desc(bl + kb, LBO_B * 4, 128);
          mma_tf32(d, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
          mma_tf32(d, dah, dbl, idesc, 1u);
          mma_tf32(d, dal, dbh, idesc, 1u);
        }
        umma_commit(&conv_empty[cs]);
        if ((st % C::kStepsPerChunk) == C::kStepsPerChunk - 1 || st == nst - 1) umma_commit(&acc_full[ch & 1]);
      }
    }
  } else {
    // ---------------------------------------------------------------- converters / drainers
    float acc[QTR];
#pragma unroll
    for (int q = 0; q < QTR; ++q) acc[q] = 0.f;
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32;
    const uint32_t col_q = (uint32_t)(warp >> 2) * QTR;  // column group of this warp
    int64_t drained = 0;
    auto drain = [&](int64_t c) {
      mbar_wait(&acc_full[c & 1], (uint32_t)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + (lane_base << 16) + (uint32_t)(c & 1) * N + col_q;
#pragma unroll
      for (int q0 = 0; q0 < QTR; q0 += 16) {
        uint32_t r[16];
#pragma unroll
        for (int q = 0; q < 16; q += 4)
          if (q0 + q < QTR)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r[q]), "=r"(r[q + 1]), "=r"(r[q + 2]), "=r"(r[q + 3])
                         : "r"(base + (uint32_t)(q0 + q)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q0 + q < QTR) acc[q0 + q] += __uint_as_float(r[q]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[c & 1]);
    };
    // blocks f = tid + i CT (A blocks first, all in round 0); row scales of the next step for them
    const bool is_a = tid < NBLK_A;
    const int kb = is_a ? tid / (kTcM / 4) : 0;
    float sc[4] = {1.f, 1.f, 1.f, 1.f};
    auto load_scale = [&](int64_t st) {
      if (!rs || !is_a) return;
      const int64_t k0 = r_begin + st * KS;
#pragma unroll
      for (int q = 0; q < 4; ++q) sc[q] = k0 + kb * 4 + q < r_end ? __ldg(rs + k0 + kb * 4 + q) : 0.f;
    };
    if (nst > 0) load_scale(0);
    const float one[4] = {1.f, 1.f, 1.f, 1.f};
    for (int64_t st = 0; st < nst; ++st) {
      const int rslot = (int)(st % C::kRaw), cs = (int)(st % C::kConv);
      const int64_t k0 = r_begin + st * KS;
      const int nr = (int)(r_end - k0 < KS ? r_end - k0 : KS);
      // the chunk that ended two steps ago: drain it (its accumulator is next written by chunk
      // + 2, which the MMA warp starts only after every warp arrived on acc_empty)
      if ((st % C::kStepsPerChunk) == 1 && st > C::kStepsPerChunk) drain(drained++);
      if (st >= C::kConv) mbar_wait(&conv_empty[cs], (uint32_t)((st / C::kConv - 1) & 1));
      mbar_wait(&raw_full[rslot], (uint32_t)((st / C::kRaw) & 1));
      {
        const float* rawA = raw0 + rslot * C::RAW_FL;
        float* const Ahi = conv0 + cs * C::CONV_FL;
#pragma unroll
        for (int i = 0; i < (NBLK + CT - 1) / CT; ++i) {
          const int f = tid + i * CT;
          if (f < NBLK_A) {
            convert_block<kTcM, kTcM>(rawA, Ahi, Ahi + C::A_FL, f / (kTcM / 4), f % (kTcM / 4), nr, a_cols, sc);
          } else if (f < NBLK) {
            const int g = f - NBLK_A;
            convert_block<N, N>(rawA + C::A_FL, Ahi + 2 * C::A_FL, Ahi + 2 * C::A_FL + C::B_FL, g / (N / 4),
                                g % (N / 4), nr, b_cols, one);
          }
        }
      }
      if (st + 1 < nst) load_scale(st + 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rslot]);
        mbar_arrive(&conv_full[cs]);
      }
    }
    while (drained < nch) drain(drained++);
    // epilogue: this thread's row of the tile, columns [col_q, col_q + QTR)
    const int64_t row = a0 + lane_base + lane;
    float* w = ws + ((int64_t)blockIdx.y * ws_lda + row) * ws_ld + b0 + col_q;
#pragma unroll
    for (int q = 0; q < QTR; q += 4)
      *reinterpret_cast<float4*>(w + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

// ----------------------------------------------------------------------------------------------
// Round 2: the same product with MN-major operands, no transposition.  The sm_100 smem descriptor
// has a layout type for 32-bit MN-major operands, SWIZZLE_128B_BASE32B (encoding 1: 32-byte atoms
// swizzled in a 128-byte span, Swizzle<2,5,2> on byte offsets), which TMA writes directly
// (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).  profiles/umma_mn_probe2.cu: exact with LBO = stride of
// the 32-column boxes and SBO = 512 B (4-row groups); the 16-byte-atom layouts the round-1 probe
// tried return zeros.  So a row-major tile of Y *is* a UMMA operand of Y^T Y:
//   * the producer TMA-loads, per 16-row step, ceil(128/32) boxes of A and ceil(N/32) boxes of B
//     (32 columns x 16 rows each) into a ring slot; the raw fp32 values are the hi operands as
//     loaded (the tensor core reads the top 19 bits: hi = x with the low 13 mantissa bits cleared,
//     profiles/umma_mn_probe.cu variant 3);
//   * 16 converter warps write lo = x - hi at the same offsets of the slot (an elementwise pass:
//     the layout needs no index arithmetic), and, for a row-scaled A, the scaled hi in place
//     (row k of a box is the 128-byte line k);
//   * the MMA warp issues 2 k-steps x 3 MMAs per step, each k-step 8 rows = 1024 B further into
//     every box;
//   * chunked TMEM accumulation, draining and the fp32 partials are as in tc_atb_kernel.
// Shared-memory traffic per step falls from ~150 KB (raw write, transposing read, hi + lo writes)
// to the raw write, one read and one lo write (~68 KB at N = 208), below the MMAs' own time.
template <int N>
struct TcMnCfg {
  static constexpr int kStep = 16;
  static constexpr int kStepsPerChunk = kTcChunk / kStep;
  static constexpr int kSlots = 4;
  static constexpr int A_BOX = kTcM / 32, B_BOX = (N + 31) / 32;  // 32-column boxes
  static constexpr int BOX_FL = 32 * kStep;                      // floats per box (16 rows x 128 B)
  static constexpr int A_FL = A_BOX * BOX_FL, B_FL = B_BOX * BOX_FL;
  static constexpr int SLOT_FL = 2 * A_FL + 2 * B_FL;            // A hi | A lo | B hi | B lo
  static constexpr size_t smem_bytes() { return (size_t)kSlots * SLOT_FL * sizeof(float) + 1024; }
};

template <int N>
__global__ void __launch_bounds__(kTcWsThreads, 1)
    tc_atb_mn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const float* __restrict__ rs, int64_t rows, int ta, int tb, int symmetric, int64_t rows_per_cta,
                     float* __restrict__ ws, int64_t ws_lda, int64_t ws_ld, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  using C = TcMnCfg<N>;
  static_assert(N % 16 == 0 && N >= 32 && N <= 256, "UMMA N");
  constexpr int KS = C::kStep;
  constexpr uint32_t LBO = C::BOX_FL * 4, SBO = 512;        // bytes: box stride, 4-row group stride
  constexpr int CT = kTcConvWarps * 32;
  constexpr int A_V4 = C::A_FL / 4, ALL_V4 = (C::A_FL + C::B_FL) / 4;
  constexpr int QTR = N / (kTcConvWarps / 4);
  constexpr uint32_t kCols = 2 * N <= 256 ? 256 : 512;
  static_assert(QTR % 4 == 0, "drain granularity");

  extern __shared__ uint8_t smraw[];
  float* const slot0 = reinterpret_cast<float*>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t raw_full[C::kSlots], conv_full[C::kSlots], slot_empty[C::kSlots];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int ti = 0, tj = 0;
  {
    int t = blockIdx.x;
    for (int i = 0; i < ta; ++i)
      for (int j = 0; j < tb; ++j) {
        if (symmetric && (int64_t)i * kTcM > (int64_t)j * N + N - 1) continue;
        if (t-- == 0) { ti = i; tj = j; }
      }
  }
  const int a0 = ti * kTcM, b0 = tj * N;
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r_end = r_begin + rows_per_cta < rows ? r_begin + rows_per_cta : rows;
  const int64_t nst = r_end > r_begin ? (r_end - r_begin + KS - 1) / KS : 0;
  const int64_t nch = (nst + C::kStepsPerChunk - 1) / C::kStepsPerChunk;

  if (tid == 0) {
    for (int i = 0; i < C::kSlots; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&conv_full[i], kTcConvWarps);
      mbar_init(&slot_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kTcConvWarps);
    }
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

  if (warp == kTcConvWarps) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int64_t st = 0; st < nst; ++st) {
        const int s = (int)(st % C::kSlots);
        if (st >= C::kSlots) mbar_wait(&slot_empty[s], (uint32_t)((st / C::kSlots - 1) & 1));
        float* A = slot0 + s * C::SLOT_FL;
        float* B = A + 2 * C::A_FL;
        mbar_expect_tx(&raw_full[s], (uint32_t)(C::A_FL + C::B_FL) * 4);
        const int r0 = (int)(r_begin + st * KS);
#pragma unroll
        for (int b = 0; b < C::A_BOX; ++b) tma_2d(A + b * C::BOX_FL, &tmA, a0 + 32 * b, r0, &raw_full[s]);
#pragma unroll
        for (int b = 0; b < C::B_BOX; ++b) tma_2d(B + b * C::BOX_FL, &tmB, b0 + 32 * b, r0, &raw_full[s]);
      }
    }
  } else if (warp == kTcConvWarps + 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(kTcM, N) | (1u << 15) | (1u << 16);  // A and B MN-major
      for (int64_t st = 0; st < nst; ++st) {
        const int s = (int)(st % C::kSlots);
        const int64_t ch = st / C::kStepsPerChunk;
        const bool first = (st % C::kStepsPerChunk) == 0;
        if (first && ch >= 2) mbar_wait(&acc_empty[ch & 1], (uint32_t)((ch / 2 - 1) & 1));
        mbar_wait(&conv_full[s], (uint32_t)((st / C::kSlots) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(ch & 1) * N;
        const uint32_t ah = smem_u32(slot0 + s * C::SLOT_FL), al = ah + C::A_FL * 4;
        const uint32_t bh = ah + 2 * C::A_FL * 4, bl = bh + C::B_FL * 4;
#pragma unroll
        for (int k = 0; k < KS / 8; ++k) {
          const uint32_t ko = (uint32_t)k * 8 * 128;  // 8 rows of 128 B into every box
          const uint64_t dah = umma_desc(ah + ko, LBO, SBO, 1), dal = umma_desc(al + ko, LBO, SBO, 1);
          const uint64_t dbh = umma_desc(bh + ko, LBO, SBO, 1), dbl = umma_desc(bl + ko, LBO, SBO, 1);
          mma_tf32(d, dah, dbh, idesc, (first && k == 0) ? 0u : 1u);
          mma_tf32(d, dah, dbl, idesc, 1u);
          mma_tf32(d, dal, dbh, idesc, 1u);
        }
        umma_commit(&slot_empty[s]);
        if ((st % C::kStepsPerChunk) == C::kStepsPerChunk - 1 || st == nst - 1) umma_commit(&acc_full[ch & 1]);
      }
    }
  } else {
    // ---------------------------------------------------------------- converters / drainers
    float acc[QTR];
#pragma unroll
    for (int q = 0; q < QTR; ++q) acc[q] = 0.f;
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32;
    const uint32_t col_q = (uint32_t)(warp >> 2) * QTR;
    int64_t drained = 0;
    auto drain = [&](int64_t c) {
      mbar_wait(&acc_full[c & 1], (uint32_t)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + (lane_base << 16) + (uint32_t)(c & 1) * N + col_q;
#pragma unroll
      for (int q0 = 0; q0 < QTR; q0 += 16) {
        uint32_t r[16];
#pragma unroll
        for (int q = 0; q < 16; q += 4)
          if (q0 + q < QTR)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r[q]), "=r"(r[q + 1]), "=r"(r[q + 2]), "=r"(r[q + 3])
                         : "r"(base + (uint32_t)(q0 + q)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q0 + q < QTR) acc[q0 + q] += __uint_as_float(r[q]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[c & 1]);
    };
    for (int64_t st = 0; st < nst; ++st) {
      const int s = (int)(st % C::kSlots);
      if ((st % C::kStepsPerChunk) == 1 && st > C::kStepsPerChunk) drain(drained++);
      // row scales of this step for the A vectors this thread converts (row k of a box = line k)
      mbar_wait(&raw_full[s], (uint32_t)((st / C::kSlots) & 1));
      float* const A = slot0 + s * C::SLOT_FL;
      const int64_t k0 = r_begin + st * KS;
#pragma unroll
      for (int i = 0; i < (ALL_V4 + CT - 1) / CT; ++i) {
        const int f = tid + i * CT;  // float4 index over [A raw | B raw]
        if (f < A_V4) {
          float4 v = reinterpret_cast<const float4*>(A)[f];
          if (rs) {
            const int k = (f % (C::BOX_FL / 4)) >> 3;  // 8 float4 per 128-byte line
            const float sc = k0 + k < r_end ? __ldg(rs + k0 + k) : 0.f;
            v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
            reinterpret_cast<float4*>(A)[f] = v;
          }
          const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          reinterpret_cast<float4*>(A + C::A_FL)[f] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        } else if (f < ALL_V4) {
          const int g = f - A_V4;
          float* const B = A + 2 * C::A_FL;
          const float4 v = reinterpret_cast<const float4*>(B)[g];
          const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          reinterpret_cast<float4*>(B + C::B_FL)[g] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv_full[s]);
    }
    while (drained < nch) drain(drained++);
    const int64_t row = a0 + lane_base + lane;
    float* w = ws + ((int64_t)blockIdx.y * ws_lda + row) * ws_ld + b0 + col_q;
#pragma unroll
    for (int q = 0; q < QTR; q += 4)
      *reinterpret_cast<float4*>(w + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

constexpr int kTcNs[] = {128, 160, 208, 256};  // instantiated tile widths

struct TcTiling {
  int n, ta, tb, tiles;
  int ta_run;            // M-tiles computed (symmetric: the last one may be left to a small kernel)
  int64_t diag0;         // >= 0: the diagonal block [diag0, Ka)^2 is computed by the caller instead
  int64_t parts, rows_per_cta;
};

// skip_diag: for a symmetric product whose last 128-row M-tile holds only a few valid rows, that
// tile contributes only the diagonal block [a0, Ka)^2 to the upper triangle (every other entry of
// those rows is mirrored from a column tile): leave it to the caller's small kernel.
TcTiling tc_tiling(int64_t rows, int64_t Ka, int64_t Kb, bool symmetric, int num_sms, bool skip_diag = false) {
  TcTiling t{};
  t.ta = (int)ceil_div(Ka, kTcM);
  const int64_t tb = ceil_div(Kb, 256);
  const int64_t need = round_up(ceil_div(Kb, tb), 16);
  t.n = 256;
  for (int n : kTcNs)
    if (n >= need) { t.n = n; break; }
  t.tb = (int)ceil_div(Kb, t.n);
  t.ta_run = t.ta;
  t.diag0 = -1;
  if (skip_diag && symmetric && t.ta > 1 && Ka - (int64_t)(t.ta - 1) * kTcM <= 64) {
    t.ta_run = t.ta - 1;
    t.diag0 = (int64_t)(t.ta - 1) * kTcM;
  }
  t.tiles = 0;
  for (int i = 0; i < t.ta_run; ++i)
    for (int j = 0; j < t.tb; ++j)
      if (!(symmetric && (int64_t)i * kTcM > (int64_t)j * t.n + t.n - 1)) ++t.tiles;
  // one wave of CTAs (1 per SM), row ranges a multiple of the chunk
  int64_t parts = std::max<int64_t>(1, num_sms / t.tiles);
  t.rows_per_cta = round_up(ceil_div(std::max<int64_t>(rows, 1), parts), kTcChunk);
  t.parts = ceil_div(std::max<int64_t>(rows, 1), t.rows_per_cta);
  return t;
}

template <int N>
cudaError_t tc_launch_n(const TcTiling& t, const float* A, int64_t lda, int64_t Ka, const float* rs, const float* B,
                        int64_t ldb, int64_t Kb, int64_t rows, bool symmetric, float* ws, int64_t ws_lda,
                        int64_t ws_ld, const int* gate, cudaStream_t st) {
  CUtensorMap tmA, tmB;
  dim3 grid((unsigned)t.tiles, (unsigned)t.parts);
  static const bool mn = [] {  // ISVD_TC_MN=0: the round-1 transposing kernel (A/B evidence)
    const char* e = getenv("ISVD_TC_MN");
    return !(e && atoi(e) == 0);
  }();
  if (mn) {
    using C = TcMnCfg<N>;
    if (!make_map(&tmA, A, rows, Ka, lda, 32, C::kStep, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
        !make_map(&tmB, B, rows, Kb, ldb, 32, C::kStep, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorInvalidValue;
    static bool attr_mn = false;
    if (!attr_mn) {
      cudaFuncSetAttribute(tc_atb_mn_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes());
      attr_mn = true;
    }
    ++g_launches;
    tc_atb_mn_kernel<N><<<grid, kTcWsThreads, C::smem_bytes(), st>>>(tmA, tmB, rs, rows, t.ta_run, t.tb,
                                                                      symmetric ? 1 : 0, t.rows_per_cta, ws, ws_lda,
                                                                      ws_ld, gate);
    return cudaGetLastError();
  }
  if (!make_map(&tmA, A, rows, Ka, lda, kTcM, TcCfg<N>::kStep, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map(&tmB, B, rows, Kb, ldb, N, TcCfg<N>::kStep, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  const size_t smem = TcCfg<N>::smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_atb_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  ++g_launches;
  tc_atb_kernel<N><<<grid, kTcWsThreads, smem, st>>>(tmA, tmB, Ka, rs, Kb, rows, t.ta_run, t.tb, symmetric ? 1 : 0,
                                                   t.rows_per_cta, ws, ws_lda, ws_ld, gate);
  return cudaGetLastError();
}

}  // namespace

bool tc_atb_supported(int64_t rows, int64_t Ka, int64_t Kb, int64_t lda, int64_t ldb) {
  return rows >= 65536 && Ka >= 1 && Kb >= 32 && Ka <= 1024 && Kb <= 1024 && lda % 4 == 0 && ldb % 4 == 0;
}

int64_t tc_atb_ws_floats(int64_t rows, int64_t Ka, int64_t Kb, bool symmetric, int num_sms) {
  TcTiling t = tc_tiling(rows, Ka, Kb, symmetric, num_sms);
  TcTiling u = tc_tiling(rows, Ka, Kb, symmetric, num_sms, true);  // fewer tiles -> possibly more parts
  return std::max(t.parts, u.parts) * ((int64_t)t.ta * kTcM) * ((int64_t)t.tb * t.n);
}

cudaError_t launch_tc_atb(const float* A, int64_t lda, int64_t Ka, const float* row_scale, const float* B,
                          int64_t ldb, int64_t Kb, int64_t rows, bool symmetric, float* ws32, int64_t* ws_lda,
                          int64_t* ws_ld, int64_t* parts, int num_sms, const int* gate, cudaStream_t st,
                          int64_t* diag0) {
  TcTiling t = tc_tiling(rows, Ka, Kb, symmetric, num_sms, diag0 != nullptr);
  if (diag0) *diag0 = t.diag0;
  *ws_lda = (int64_t)t.ta * kTcM;
  *ws_ld = (int64_t)t.tb * t.n;
  *parts = t.parts;
  switch (t.n) {
    case 128: return tc_launch_n<128>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st);
    case 160: return tc_launch_n<160>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st);
    case 208: return tc_launch_n<208>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st);
    default: return tc_launch_n<256>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st);
  }
}

}  // namespace isvd
