// tcgen05.mma kind::tf32 operand-layout probe: one 128 x 128 x 8 MMA per variant, checked on the host.
//   v0  MN-major SWIZZLE_NONE    (canonical ((T,1,m),(8,k)):((1,T,SBO),(1T,LBO)))
//   v1  MN-major SWIZZLE_128B    (canonical ((T,8,m),(8,k)):((1,T,LBO),(8T,SBO)), 1024 B atoms)
//   v2  MN-major SWIZZLE_128B with LBO / SBO exchanged
//   v3  K-major  SWIZZLE_NONE    (the layout gram_tc.cu uses) -- also probes TF32 truncation vs rounding:
//       A = 1 + 3*2^-12 (not representable in TF32): D = 8 if the TC truncates, 8 * (1 + 2^-10) if it rounds
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc \
//        profiles/umma_mn_probe.cu -o build/umma_mn_probe
#include <cmath>
#include <cstdio>

#include "../paper_2111_06312_b200/csrc/gram_tc.cu"

namespace isvd {
thread_local int64_t g_launches = 0;
}

using namespace isvd;

constexpr int M = 128, N = 128;

__host__ __device__ inline float a_val(int m, int k, int variant) {
  return variant == 3 ? 1.0f + 3.0f / 4096.0f : 1.0f + m / 128.0f + k / 1024.0f;
}
__host__ __device__ inline float b_val(int k, int n, int variant) {
  return variant == 3 ? 1.0f : (float)(k + 1) + n / 256.0f;
}

// byte offset of element (mn, k) for an MN-major SW128 tile with `mn_extent` elements along MN, 8 K rows
__device__ inline int sw128_off(int mn, int k, int lbo, int sbo) {
  const int atom = mn >> 5, w = mn & 31;
  const int chunk = (w >> 2) ^ (k & 7);
  return atom * lbo + (k >> 3) * sbo + (k & 7) * 128 + chunk * 16 + (w & 3) * 4;
}

__global__ void probe(float* out, int variant) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  float* A = (float*)base;                // 4 KB
  float* B = (float*)(base + 8 * M * 4);  // 4 KB
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool sw = variant == 1 || variant == 2;
  // SW128 strides: MN atoms (32 elements x 8 rows = 1024 B) adjacent, one K group
  const int lbo_sw = 1024, sbo_sw = (M / 32) * 1024;
  for (int f = tid; f < 8 * M; f += blockDim.x) {
    const int k = f / M, m = f % M;
    int off;
    if (variant == 0) off = ((m >> 2) * 32 + (k & 7) * 4 + (m & 3)) * 4;
    else if (sw) off = sw128_off(m, k, lbo_sw, sbo_sw);
    else off = ((m >> 3) * 32 + (m & 7) * 4 + (k & 3) + (k >> 2) * (M / 8 * 32)) * 4;
    *(float*)((uint8_t*)A + off) = a_val(m, k, variant);
  }
  for (int f = tid; f < 8 * N; f += blockDim.x) {
    const int k = f / N, n = f % N;
    int off;
    if (variant == 0) off = ((n >> 2) * 32 + (k & 7) * 4 + (n & 3)) * 4;
    else if (sw) off = sw128_off(n, k, lbo_sw, (N / 32) * 1024);
    else off = ((n >> 3) * 32 + (n & 7) * 4 + (k & 3) + (k >> 2) * (N / 8 * 32)) * 4;
    *(float*)((uint8_t*)B + off) = b_val(k, n, variant);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  uint32_t idesc = umma_idesc(M, N);
  if (variant <= 2) idesc |= (1u << 15) | (1u << 16);  // MN-major A and B
  uint64_t da, db;
  if (variant == 0) {
    da = umma_desc(smem_u32(A), 4096, 128);  // LBO = K-group stride (one group), SBO = MN-group stride
    db = umma_desc(smem_u32(B), 4096, 128);
  } else if (sw) {
    uint32_t la = lbo_sw, sa = sbo_sw, lb = lbo_sw, sb = (N / 32) * 1024;
    if (variant == 2) { uint32_t t = la; la = sa; sa = t; t = lb; lb = sb; sb = t; }
    da = umma_desc(smem_u32(A), la, sa) | (2ull << 61);
    db = umma_desc(smem_u32(B), lb, sb) | (2ull << 61);
  } else {
    da = umma_desc(smem_u32(A), M / 8 * 128, 128);
    db = umma_desc(smem_u32(B), N / 8 * 128, 128);
  }
  if (tid == 0) {
    mma_tf32(tmem, da, db, idesc, 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
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
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

static float tf32_trunc(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  float* d;
  cudaMalloc(&d, M * N * 4);
  static float h[M * N];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int variant = 0; variant < 4; ++variant) {
    cudaMemset(d, 0, M * N * 4);
    probe<<<1, 128, 64 * 1024>>>(d, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double maxrel = 0.0, maxrel_t = 0.0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0.0, st = 0.0;
        for (int k = 0; k < 8; ++k) {
          s += (double)a_val(m, k, variant) * b_val(k, n, variant);
          st += (double)tf32_trunc(a_val(m, k, variant)) * tf32_trunc(b_val(k, n, variant));
        }
        maxrel = fmax(maxrel, fabs(h[m * N + n] - s) / fabs(s));
        maxrel_t = fmax(maxrel_t, fabs(h[m * N + n] - st) / fabs(st));
      }
    printf("variant %d: %s  D[0][0]=%.7g D[5][77]=%.7g D[127][127]=%.7g  max rel err vs exact %.3e, vs tf32-truncated %.3e\n",
           variant, cudaGetErrorString(e), h[0], h[5 * N + 77], h[M * N - 1], maxrel, maxrel_t);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
