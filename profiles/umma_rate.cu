// tcgen05.mma kind::tf32 issue-rate microbenchmark (one CTA per SM, operands static in smem):
//   M = 128, N in {208, 256}, K = 8 per MMA, K-major operands, SWIZZLE_NONE vs SWIZZLE_128B.
// Also checks that both layouts give the same D for the same logical A, B.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc \
//        profiles/umma_rate.cu -o build/umma_rate
#include <cstdio>
#include <vector>

#include "../paper_2111_06312_b200/csrc/gram_tc.cu"

namespace isvd {
thread_local int64_t g_launches = 0;
}
using namespace isvd;

constexpr int M = 128, KT = 32;  // K extent held in smem (4 MMAs of K = 8)

__host__ __device__ inline float a_val(int m, int k) { return 0.25f * ((m * 7 + k * 3) % 11) - 1.f; }
__host__ __device__ inline float b_val(int n, int k) { return 0.125f * ((n * 5 + k * 13) % 17) - 1.f; }

// byte offsets of element (mn, k) of an E x KT K-major operand
__device__ inline int off_none(int mn, int k, int E) {  // core matrices 8 x 16 B; MN groups 128 B, K groups E*16 B
  return (k >> 2) * (E * 16) + (mn >> 3) * 128 + (mn & 7) * 16 + (k & 3) * 4;
}
__device__ inline int off_sw128(int mn, int k) {  // rows of 32 K-values = 128 B, 8-row atoms of 1024 B
  return (mn >> 3) * 1024 + (mn & 7) * 128 + ((((k >> 2) ^ (mn & 7)) & 7) << 4) + (k & 3) * 4;
}

template <int N>
__global__ void rate(int layout, int iters, float* out, long long* cycles) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tbase;
  uint8_t* base = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* A = base;
  uint8_t* B = base + M * KT * 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int f = tid; f < M * KT; f += blockDim.x) {
    const int m = f / KT, k = f % KT;
    *(float*)(A + (layout ? off_sw128(m, k) : off_none(m, k, M))) = a_val(m, k);
  }
  for (int f = tid; f < N * KT; f += blockDim.x) {
    const int n = f / KT, k = f % KT;
    *(float*)(B + (layout ? off_sw128(n, k) : off_none(n, k, N))) = b_val(n, k);
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t idesc = umma_idesc(M, N);
  const uint32_t a = smem_u32(A), b = smem_u32(B);
  long long t0 = clock64();
  if (tid == 0) {
    for (int it = 0; it < iters; ++it) {
      if (it >= 2) mbar_wait(&bar[it & 1], (uint32_t)(((it - 2) >> 1) & 1));
      for (int s = 0; s < KT / 8; ++s) {
        uint64_t da, db;
        if (layout == 0) {
          da = umma_desc(a + s * 2 * M * 16, M * 16, 128);
          db = umma_desc(b + s * 2 * N * 16, N * 16, 128);
        } else {
          da = umma_desc(a + s * 32, 16, 1024) | (2ull << 61);
          db = umma_desc(b + s * 32, 16, 1024) | (2ull << 61);
        }
        // 3 MMAs per k-step as in 3xTF32 (same operands here); only the first iteration overwrites
        mma_tf32(tmem, da, db, idesc, (it == 0 && s == 0) ? 0u : 1u);
        mma_tf32(tmem + N, da, db, idesc, (it == 0 && s == 0) ? 0u : 1u);
        mma_tf32(tmem, da, db, idesc, 1u);
      }
      umma_commit(&bar[it & 1]);
    }
    mbar_wait(&bar[(iters - 1) & 1], (uint32_t)(((iters - 1) >> 1) & 1));
    if (iters >= 2) mbar_wait(&bar[(iters - 2) & 1], (uint32_t)(((iters - 2) >> 1) & 1));
  }
  __syncthreads();
  long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (blockIdx.x == 0 && warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 8; ++q) out[(warp * 32 + lane) * N + c0 + q] = __uint_as_float(r[q]);
    }
  }
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N>
void run(int layout, int iters) {
  float* d;
  long long* cyc;
  cudaMalloc(&d, M * N * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int smem = M * KT * 4 + N * KT * 4 + 2048;
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate<N><<<148, 128, smem>>>(layout, 2, d, cyc);  // warm-up + result check (2 iterations)
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h(M * N);
  cudaMemcpy(h.data(), d, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < KT; ++k) s += (double)a_val(m, k) * b_val(n, k);
      s *= 2 * 2;  // 2 iterations x (MMA 1 + MMA 3 into the same accumulator)
      maxerr = fmax(maxerr, fabs(h[m * N + n] - s));
    }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<N><<<148, 128, smem>>>(layout, iters, d, cyc);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = 148.0 * iters * (KT / 8) * 3;
  const double flops = mmas * 2.0 * M * N * 8;
  printf("N=%d layout=%s: %s  check max err %.2e   %.3f ms  %.1f ns/MMA/SM  %.1f TFLOP/s (tf32)\n", N,
         layout ? "SW128" : "NONE", cudaGetErrorString(e), maxerr, ms, ms * 1e6 / (mmas / 148), flops / (ms * 1e-3) / 1e12);
  cudaFree(d);
  cudaFree(cyc);
}

int main() {
  run<208>(0, 20000);
  run<208>(1, 20000);
  run<256>(0, 20000);
  run<256>(1, 20000);
  run<128>(0, 20000);
  run<128>(1, 20000);
  return 0;
}
