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
// One CTA (256 threads, 1 per SM: TMEM 2N columns, ~200 KB smem) computes a 128 x N tile over
// a contiguous row range:
//   * all threads stage 32 rows per step into shared memory in the UMMA K-major no-swizzle
//     canonical layout (core matrices of 8 MN-rows x 4 K-values = 16 bytes per row, MN-groups
//     128 B apart, K-groups E/8*128 B apart), split into hi / lo: each thread holds 4 x 4 blocks
//     (4 rows, one float4 each) in registers, transposes them and stores 4-value K-vectors.
//     The global loads of step t+1 are issued right after step t is stored, so one full step
//     of loads (~48 KB per SM) is in flight behind the MMAs.  (The MN-major operand form of
//     kind::tf32, which would take the row-major tiles as they are, produced no output on this
//     driver in every descriptor variant tried -- profiles/umma_mn_probe.cu.)
//   * one thread issues 4 k-steps x 3 tcgen05.mma.kind::tf32 (M = 128, N <= 256, K = 8) per
//     step and commits to the step buffer's mbarrier (gates refilling it) and, at the end of a
//     chunk, to the chunk's mbarrier (gates draining it);
//   * warp w drains TMEM lanes 32 (w % 4) .. +31 (rows of the tile), columns half w / 4, with
//     tcgen05.ld.32x32b.
// Operand descriptors and the instruction descriptor follow the sm_100 UMMA bit layouts.
#include <algorithm>

#include "common.cuh"

namespace isvd {
namespace {

constexpr int kTcM = 128;       // UMMA M (rows of the C tile = columns of A)
constexpr int kTcKB = 32;       // rows per pipeline step (4 MMAs of K = 8)
constexpr int kTcChunk = 128;   // rows per TMEM accumulation (truncation bound)
constexpr int kTcStepsPerChunk = kTcChunk / kTcKB;
constexpr int kTcThreads = 256;

ISVD_DEVICE uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SWIZZLE_NONE smem matrix descriptor: start, LBO = K-group stride, SBO = MN-group stride.
ISVD_DEVICE uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

ISVD_DEVICE void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

ISVD_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// Bounded wait: a commit that never arrives traps (kernel error) instead of hanging the GPU.
ISVD_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1u << 26)) __trap();
  }
}

ISVD_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

ISVD_DEVICE float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// Store the K-vector (rows k0..k0+3, k0 % 4 == 0) of MN-element c into the K-major layout.
ISVD_DEVICE void st_split(float* hi, float* lo, int k0, int c, int lbo_floats, float4 v) {
  const int off = (k0 >> 2) * lbo_floats + (c >> 3) * 32 + (c & 7) * 4;
  float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// A 4 x 4 block of one operand: rows k0 + 4 kb .. +3, columns c0 + 4 cb .. +3 (zero outside
// [0, r_end) x [0, cols)); row_scale multiplies each row when given.
ISVD_DEVICE void load_block(const float* __restrict__ src, int64_t ld, int64_t cols, const float* __restrict__ rs,
                            int64_t k0, int64_t r_end, int64_t c, int kb, float4 (&v)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t gr = k0 + kb * 4 + q;
    v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gr < r_end && c < cols) {
      v[q] = __ldg(reinterpret_cast<const float4*>(src + gr * ld + c));
      if (rs) {
        const float s = __ldg(rs + gr);
        v[q].x *= s; v[q].y *= s; v[q].z *= s; v[q].w *= s;
      }
    }
  }
}

// transpose: K-vector of column c + j = (v[0].j, v[1].j, v[2].j, v[3].j); rotate j by the
// block index to spread the 16-byte stores over the banks
template <int E>
ISVD_DEVICE void store_block(float* hi, float* lo, int kb, int cb, const float4 (&v)[4]) {
  constexpr int LBO = E / 8 * 32;  // floats
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const int j = (jj + cb) & 3;
    float4 kv;
    if (j == 0) kv = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
    else if (j == 1) kv = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
    else if (j == 2) kv = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
    else kv = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
    st_split(hi, lo, kb * 4, cb * 4 + j, LBO, kv);
  }
}

template <int N>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_atb_kernel(const float* __restrict__ A, int64_t lda, int64_t Ka, const float* __restrict__ rs,
                  const float* __restrict__ B, int64_t ldb, int64_t Kb, int64_t rows, int ta, int tb, int symmetric,
                  int64_t rows_per_cta, float* __restrict__ ws, int64_t ws_lda, int64_t ws_ld, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  static_assert(N % 16 == 0 && N >= 32 && N <= 256, "UMMA N");
  constexpr int A_FL = kTcKB * kTcM;  // floats per A hi (or lo) step buffer
  constexpr int B_FL = kTcKB * N;
  constexpr int LBO_A = kTcM / 8 * 32, LBO_B = N / 8 * 32;  // K-group (4 values) strides in floats
  constexpr int NB_BLK = (kTcKB / 4) * (N / 4);              // 4x4 blocks of B per step
  constexpr int B_PER_T = (NB_BLK + kTcThreads - 1) / kTcThreads;
  constexpr int HALF = N / 2;                                // columns drained per thread
  constexpr uint32_t kCols = 2 * N <= 256 ? 256 : 512;       // TMEM: two N-column accumulators
  static_assert((kTcKB / 4) * (kTcM / 4) == kTcThreads, "one A block per thread");
  static_assert(HALF % 8 == 0, "drain granularity");

  extern __shared__ __align__(1024) float sm[];
  // step buffer b: [A hi | A lo | B hi | B lo] at sm + b * STEP_FL
  constexpr int STEP_FL = 2 * A_FL + 2 * B_FL;
  __shared__ __align__(8) uint64_t mbar[2];  // step buffer b free again
  __shared__ __align__(8) uint64_t cbar[2];  // chunk accumulator b complete
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
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r_end = r_begin + rows_per_cta < rows ? r_begin + rows_per_cta : rows;
  const int64_t nst = r_end > r_begin ? (r_end - r_begin + kTcKB - 1) / kTcKB : 0;
  const int64_t nch = (nst + kTcStepsPerChunk - 1) / kTcStepsPerChunk;

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&cbar[0], 1);
    mbar_init(&cbar[1], 1);
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
  const uint32_t idesc = umma_idesc(kTcM, N);

  // operand columns of this thread's blocks: A block (kb_a, cb_a); B blocks f = tid + i * 256
  const int kb_a = tid / (kTcM / 4), cb_a = tid % (kTcM / 4);
  const float* Ab = A + a0;
  const float* Bb = B + b0;
  const int64_t a_cols = Ka - a0, b_cols = Kb - b0;
  float4 va[4], vb[B_PER_T][4];
  auto load_step = [&](int64_t k0) {
    load_block(Ab, lda, a_cols, rs, k0, r_end, cb_a * 4, kb_a, va);
#pragma unroll
    for (int i = 0; i < B_PER_T; ++i) {
      const int f = tid + i * kTcThreads;
      const int kb = f / (N / 4), cb = f - kb * (N / 4);
      if (f < NB_BLK) load_block(Bb, ldb, b_cols, nullptr, k0, r_end, cb * 4, kb, vb[i]);
    }
  };

  float acc[HALF];
#pragma unroll
  for (int q = 0; q < HALF; ++q) acc[q] = 0.f;
  const uint32_t lane_base = (uint32_t)(warp & 3) * 32;
  const uint32_t col_half = (uint32_t)(warp >> 2) * HALF;
  int64_t drained = 0;
  auto drain = [&](int64_t c) {
    mbar_wait(&cbar[c & 1], (uint32_t)((c >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = tmem + (lane_base << 16) + (uint32_t)(c & 1) * N + col_half;
#pragma unroll
    for (int q0 = 0; q0 < HALF; q0 += 32) {
      uint32_t r[32];
#pragma unroll
      for (int q = 0; q < 32; q += 8)
        if (q0 + q < HALF)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                       : "=r"(r[q]), "=r"(r[q + 1]), "=r"(r[q + 2]), "=r"(r[q + 3]), "=r"(r[q + 4]), "=r"(r[q + 5]),
                         "=r"(r[q + 6]), "=r"(r[q + 7])
                       : "r"(base + (uint32_t)(q0 + q)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q0 + q < HALF) acc[q0 + q] += __uint_as_float(r[q]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  };

  if (nst > 0) load_step(r_begin);
  for (int64_t st = 0; st < nst; ++st) {
    const int buf = (int)(st & 1);
    if (st >= 2) mbar_wait(&mbar[buf], (uint32_t)(((st - 2) >> 1) & 1));  // MMAs of step st-2 done
    // the chunk finished two steps ago is complete too: drain it (its accumulator is next
    // written by chunk + 2, whose MMAs are issued after this step's __syncthreads)
    if ((st % kTcStepsPerChunk) == 1 && st > kTcStepsPerChunk) drain(drained++);
    float* const Ahi = sm + buf * STEP_FL;
    float* const Alo = Ahi + A_FL;
    float* const Bhi = Ahi + 2 * A_FL;
    float* const Blo = Bhi + B_FL;
    store_block<kTcM>(Ahi, Alo, kb_a, cb_a, va);
#pragma unroll
    for (int i = 0; i < B_PER_T; ++i) {
      const int f = tid + i * kTcThreads;
      const int kb = f / (N / 4), cb = f - kb * (N / 4);
      if (f < NB_BLK) store_block<N>(Bhi, Blo, kb, cb, vb[i]);
    }
    if (st + 1 < nst) load_step(r_begin + (st + 1) * kTcKB);  // in flight behind this step's MMAs
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t c = st / kTcStepsPerChunk;
      const uint32_t d = tmem + (uint32_t)(c & 1) * N;
      const uint32_t ah = smem_u32(Ahi), al = smem_u32(Alo);
      const uint32_t bh = smem_u32(Bhi), bl = smem_u32(Blo);
      const bool first = (st % kTcStepsPerChunk) == 0;
#pragma unroll
      for (int s = 0; s < kTcKB / 8; ++s) {
        // one MMA (K = 8) spans two K-groups
        const uint32_t ka = (uint32_t)(2 * s) * LBO_A * 4, kb = (uint32_t)(2 * s) * LBO_B * 4;  // bytes
        const uint64_t dah = umma_desc(ah + ka, LBO_A * 4, 128), dal = umma_desc(al + ka, LBO_A * 4, 128);
        const uint64_t dbh = umma_desc(bh + kb, LBO_B * 4, 128), dbl = umma_desc(bl + kb, LBO_B * 4, 128);
        mma_tf32(d, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
        mma_tf32(d, dah, dbl, idesc, 1u);
        mma_tf32(d, dal, dbh, idesc, 1u);
      }
      umma_commit(&mbar[buf]);
      if ((st % kTcStepsPerChunk) == kTcStepsPerChunk - 1 || st == nst - 1) umma_commit(&cbar[c & 1]);
    }
  }
  while (drained < nch) drain(drained++);

  // epilogue: this thread's row of the tile, columns [col_half, col_half + HALF)
  const int64_t row = a0 + lane_base + lane;
  float* w = ws + ((int64_t)blockIdx.y * ws_lda + row) * ws_ld + b0 + col_half;
#pragma unroll
  for (int q = 0; q < HALF; q += 4)
    *reinterpret_cast<float4*>(w + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

constexpr int kTcNs[] = {128, 160, 208, 256};  // instantiated tile widths

struct TcTiling {
  int n, ta, tb, tiles;
  int64_t parts, rows_per_cta;
};

TcTiling tc_tiling(int64_t rows, int64_t Ka, int64_t Kb, bool symmetric, int num_sms) {
  TcTiling t{};
  t.ta = (int)ceil_div(Ka, kTcM);
  const int64_t tb = ceil_div(Kb, 256);
  const int64_t need = round_up(ceil_div(Kb, tb), 16);
  t.n = 256;
  for (int n : kTcNs)
    if (n >= need) { t.n = n; break; }
  t.tb = (int)ceil_div(Kb, t.n);
  t.tiles = 0;
  for (int i = 0; i < t.ta; ++i)
    for (int j = 0; j < t.tb; ++j)
      if (!(symmetric && (int64_t)i * kTcM > (int64_t)j * t.n + t.n - 1)) ++t.tiles;
  // one wave of CTAs (1 per SM), row ranges a multiple of the chunk
  int64_t parts = std::max<int64_t>(1, num_sms / t.tiles);
  t.rows_per_cta = round_up(ceil_div(std::max<int64_t>(rows, 1), parts), kTcChunk);
  t.parts = ceil_div(std::max<int64_t>(rows, 1), t.rows_per_cta);
  return t;
}

template <int N>
void tc_launch_n(const TcTiling& t, const float* A, int64_t lda, int64_t Ka, const float* rs, const float* B,
                 int64_t ldb, int64_t Kb, int64_t rows, bool symmetric, float* ws, int64_t ws_lda, int64_t ws_ld,
                 const int* gate, cudaStream_t st) {
  const size_t smem = (size_t)2 * (2 * kTcKB * kTcM + 2 * kTcKB * N) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_atb_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)t.tiles, (unsigned)t.parts);
  ++g_launches;
  tc_atb_kernel<N><<<grid, kTcThreads, smem, st>>>(A, lda, Ka, rs, B, ldb, Kb, rows, t.ta, t.tb, symmetric ? 1 : 0,
                                                   t.rows_per_cta, ws, ws_lda, ws_ld, gate);
}

}  // namespace

bool tc_atb_supported(int64_t rows, int64_t Ka, int64_t Kb, int64_t lda, int64_t ldb) {
  return rows >= 65536 && Ka >= 1 && Kb >= 32 && Ka <= 1024 && Kb <= 1024 && lda % 4 == 0 && ldb % 4 == 0;
}

int64_t tc_atb_ws_floats(int64_t rows, int64_t Ka, int64_t Kb, bool symmetric, int num_sms) {
  TcTiling t = tc_tiling(rows, Ka, Kb, symmetric, num_sms);
  return t.parts * ((int64_t)t.ta * kTcM) * ((int64_t)t.tb * t.n);
}

cudaError_t launch_tc_atb(const float* A, int64_t lda, int64_t Ka, const float* row_scale, const float* B,
                          int64_t ldb, int64_t Kb, int64_t rows, bool symmetric, float* ws32, int64_t* ws_lda,
                          int64_t* ws_ld, int64_t* parts, int num_sms, const int* gate, cudaStream_t st) {
  TcTiling t = tc_tiling(rows, Ka, Kb, symmetric, num_sms);
  *ws_lda = (int64_t)t.ta * kTcM;
  *ws_ld = (int64_t)t.tb * t.n;
  *parts = t.parts;
  switch (t.n) {
    case 128: tc_launch_n<128>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st); break;
    case 160: tc_launch_n<160>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st); break;
    case 208: tc_launch_n<208>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st); break;
    default: tc_launch_n<256>(t, A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, *ws_lda, *ws_ld, gate, st); break;
  }
  return cudaGetLastError();
}

}  // namespace isvd
