// Tensor-core Gram G = Y^T Y for CholeskyQR (Alg. 2 right), 3xTF32 on tcgen05.
//
// north_star: tensor cores only in the Gram contraction, and only if 3xTF32 meets the
// tolerance.  Each operand value x is split x = hi + lo (hi = x with the low 13 mantissa
// bits cleared, i.e. exactly representable in TF32; lo = x - hi exactly); the product is
// hi*hi' + hi*lo' + lo*hi' (relative error ~2^-21 per product), accumulated in fp32 in
// TMEM over a chunk of rows; chunk partials are summed in fp64 in a fixed order by
// atb_f32_reduce_kernel (dense.cu) -- the same numerics class as the fp32-chunk SIMT path,
// used for every Gram except the first pass of the CholeskyQR2 of Y = M Omega.
//
// One CTA computes a 128 x N tile of G over one chunk of rows:
//   * all 256 threads stage 32 rows of Y into shared memory, split into hi / lo, in the
//     UMMA K-major no-swizzle canonical layout (core matrices of 8 MN-rows x 4 K-values =
//     16 bytes per row, MN-groups 128 B apart, K-groups E/8*128 B apart): each thread loads a
//     4 x 4 block of Y (4 rows, one float4 each), transposes it in registers and stores
//     four 4-value K-vectors; double-buffered.  (The MN-major form of kind::tf32 was measured
//     to produce no output on this driver -- profiles/umma_probe.cu -- so the transpose is
//     done while staging.)
//   * one thread issues 4 k-steps x 3 tcgen05.mma.kind::tf32 (M = 128, N <= 256, K = 8)
//     per stage and commits to the stage's mbarrier, which gates refilling that buffer;
//   * the accumulator lives in TMEM (N fp32 columns x 128 lanes); the epilogue reads it
//     with tcgen05.ld.32x32b (warp w owns lanes 32 (w % 4) ...) and writes the fp32 partial.
// Operand descriptors and the instruction descriptor follow the sm_100 UMMA bit layouts.
#include "common.cuh"

namespace isvd {
namespace {

constexpr int kTcM = 128;      // UMMA M (rows of the G tile)
constexpr int kTcKB = 32;      // rows of Y per pipeline stage (4 MMAs of K = 8)
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

// Stage a 32-row x E-column slice of Y (columns [c0, c0 + E)) into the K-major hi/lo buffers.
template <int E>
ISVD_DEVICE void stage_operand(const float* __restrict__ Y, int64_t ld, int64_t k0, int64_t r_end, int64_t c0,
                               int64_t l, float* hi, float* lo, int tid) {
  constexpr int LBO = E / 8 * 32;  // floats
  for (int f = tid; f < (kTcKB / 4) * (E / 4); f += kTcThreads) {
    const int kb = f / (E / 4), cb = f - kb * (E / 4);
    const int c = cb * 4;
    float4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t gr = k0 + kb * 4 + q;
      v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < r_end && c0 + c < l) v[q] = __ldg(reinterpret_cast<const float4*>(Y + gr * ld + c0 + c));
    }
    // transpose: K-vector of column c + j = (v[0].j, v[1].j, v[2].j, v[3].j); rotate j by the
    // thread index to spread the 16-byte stores over the banks
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = (jj + cb) & 3;
      float4 kv;
      if (j == 0) kv = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
      else if (j == 1) kv = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
      else if (j == 2) kv = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
      else kv = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
      st_split(hi, lo, kb * 4, c + j, LBO, kv);
    }
  }
}

template <int N>
__global__ void __launch_bounds__(kTcThreads, 1)
    gram_tc_kernel(const float* __restrict__ Y, int64_t ld, int64_t rows, int64_t l, int tiles_n,
                   int64_t rows_per_chunk, float* __restrict__ ws, int64_t ws_lda, int64_t ws_ld, const int* gate) {
  if (gate && *((volatile const int*)gate) == 0) return;
  constexpr int A_FL = kTcKB * kTcM;  // floats per A hi/lo stage buffer
  constexpr int B_FL = kTcKB * N;
  constexpr int LBO_A = kTcM / 8 * 32, LBO_B = N / 8 * 32;  // K-group (4 values) strides in floats
  extern __shared__ __align__(1024) float sm[];
  float* Ahi[2] = {sm, sm + 2 * A_FL + 2 * B_FL};
  float* Alo[2] = {Ahi[0] + A_FL, Ahi[1] + A_FL};
  float* Bhi[2] = {Ahi[0] + 2 * A_FL, Ahi[1] + 2 * A_FL};
  float* Blo[2] = {Bhi[0] + B_FL, Bhi[1] + B_FL};
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ti = blockIdx.x / tiles_n, tj = blockIdx.x - ti * tiles_n;
  const int64_t a0 = (int64_t)ti * kTcM, b0 = (int64_t)tj * N;
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_chunk;
  const int64_t r_end = r_begin + rows_per_chunk < rows ? r_begin + rows_per_chunk : rows;
  constexpr uint32_t kCols = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;  // TMEM columns (pow2)

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
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

  const int64_t nst = (r_end - r_begin + kTcKB - 1) / kTcKB;
  for (int64_t st = 0; st < nst; ++st) {
    const int buf = (int)(st & 1);
    if (st >= 2) mbar_wait(&mbar[buf], (uint32_t)(((st - 2) >> 1) & 1));  // MMAs of stage st-2 done
    const int64_t k0 = r_begin + st * kTcKB;
    // stage rows [k0, k0 + 32): A = columns [a0, a0 + 128), B = columns [b0, b0 + N)
    stage_operand<kTcM>(Y, ld, k0, r_end, a0, l, Ahi[buf], Alo[buf], tid);
    stage_operand<N>(Y, ld, k0, r_end, b0, l, Bhi[buf], Blo[buf], tid);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = smem_u32(Ahi[buf]), al = smem_u32(Alo[buf]);
      const uint32_t bh = smem_u32(Bhi[buf]), bl = smem_u32(Blo[buf]);
#pragma unroll
      for (int s = 0; s < kTcKB / 8; ++s) {
        // one MMA (K = 8) spans two K-groups
        const uint32_t ka = (uint32_t)(2 * s) * LBO_A * 4, kb = (uint32_t)(2 * s) * LBO_B * 4;  // bytes
        const uint64_t dah = umma_desc(ah + ka, LBO_A * 4, 128), dal = umma_desc(al + ka, LBO_A * 4, 128);
        const uint64_t dbh = umma_desc(bh + kb, LBO_B * 4, 128), dbl = umma_desc(bl + kb, LBO_B * 4, 128);
        mma_tf32(tmem, dah, dbh, idesc, (st > 0 || s > 0) ? 1u : 0u);
        mma_tf32(tmem, dah, dbl, idesc, 1u);
        mma_tf32(tmem, dal, dbh, idesc, 1u);
      }
      umma_commit(&mbar[buf]);
    }
  }
  if (nst > 0) mbar_wait(&mbar[(nst - 1) & 1], (uint32_t)(((nst - 1) >> 1) & 1));  // all MMAs done
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (rows of the tile), columns split by w / 4
  const int lane_base = (warp & 3) * 32;
  const int64_t row = a0 + lane_base + lane;
  float* W = ws + (int64_t)blockIdx.y * ws_lda * ws_ld;
  for (int c = (warp >> 2) * 8; c < N; c += 16) {
    uint32_t r[8];
    const uint32_t taddr = tmem + ((uint32_t)lane_base << 16) + (uint32_t)c;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float* w = W + row * ws_ld + b0 + c;
    if (nst == 0) {
      for (int q = 0; q < 8; ++q) r[q] = 0u;
    }
    *reinterpret_cast<float4*>(w) =
        make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3]));
    *reinterpret_cast<float4*>(w + 4) =
        make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]), __uint_as_float(r[7]));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

}  // namespace

// Tile shape: M = 128, N = the largest multiple of 8 <= 256 that splits l into equal tiles.
static int tc_tile_n(int64_t l) {
  const int64_t tn = (l + 255) / 256;
  return (int)round_up(ceil_div(l, tn), 8);
}

bool gram_tc_supported(int64_t rows, int64_t l) {
  if (l < 128 || l > 1024 || rows < 65536) return false;
  const int n = tc_tile_n(l);
  return n == 200 || n == 256 || n == 128;  // instantiated shapes
}

int64_t gram_tc_ws_floats(int64_t rows, int64_t l, int64_t* chunks_out, int64_t* chunk_rows_out) {
  const int n = tc_tile_n(l);
  const int64_t ta = ceil_div(l, kTcM), tb = ceil_div(l, n);
  // rows per TMEM accumulation: the tensor core's fp32 accumulation truncates, so the error
  // grows ~linearly with the chunk (measured 3.8e-5 relative at 2048 rows)
  int64_t cr = 512;
  const int64_t chunks = ceil_div(rows, cr);
  if (chunks_out) *chunks_out = chunks;
  if (chunk_rows_out) *chunk_rows_out = cr;
  return chunks * (ta * kTcM) * (tb * n);
}

cudaError_t launch_gram_tc(const float* Y, int64_t ld, int64_t rows, int64_t l, float* ws32, int64_t* ws_lda,
                           int64_t* ws_ld, int64_t* chunks, const int* gate, cudaStream_t st) {
  const int n = tc_tile_n(l);
  const int64_t ta = ceil_div(l, kTcM), tb = ceil_div(l, n);
  int64_t cr = 0;
  gram_tc_ws_floats(rows, l, chunks, &cr);
  *ws_lda = ta * kTcM;
  *ws_ld = tb * n;
  const size_t smem = (size_t)2 * (2 * kTcKB * kTcM + 2 * kTcKB * n) * sizeof(float);
  dim3 grid((unsigned)(ta * tb), (unsigned)*chunks);
  ++g_launches;
#define ISVD_TC_LAUNCH(NN)                                                                                     \
  {                                                                                                            \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      cudaFuncSetAttribute(gram_tc_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
      attr = true;                                                                                             \
    }                                                                                                          \
    gram_tc_kernel<NN><<<grid, kTcThreads, smem, st>>>(Y, ld, rows, l, (int)tb, cr, ws32, *ws_lda, *ws_ld, gate); \
  }
  if (n == 200) ISVD_TC_LAUNCH(200)
  else if (n == 256) ISVD_TC_LAUNCH(256)
  else ISVD_TC_LAUNCH(128)
#undef ISVD_TC_LAUNCH
  return cudaGetLastError();
}

}  // namespace isvd
