// Minimal tcgen05.mma kind::tf32 probe: one 128 x N x 8 MMA on constant operands.
#include <cstdio>

#include "../paper_2111_06312_b200/csrc/gram_tc.cu"

namespace isvd {
thread_local int64_t g_launches = 0;
}

using namespace isvd;

template <int N>
__global__ void probe(float* out, int variant) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  float* A = sm;             // 8 K-rows x 128 M
  float* B = sm + 8 * 128;   // 8 K-rows x N
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A[k][m] = 1 + m/128 ; B[k][n] = (k + 1)   -> D[m][n] = sum_k (1 + m/128)(k+1) = 36 (1 + m/128)
  for (int f = tid; f < 8 * 128; f += blockDim.x) {
    int k = f / 128, m = f % 128;
    int off = (k >> 3) * (128 / 4 * 32) + (m >> 2) * 32 + (k & 7) * 4 + (m & 3);
    if (variant == 2)  // K-major: core matrix = 8 MN-rows x 4 K (16 B), MN-groups of 8 at 128 B, K-groups at 16*128 B
      off = (k >> 2) * (128 / 8 * 32) + (m >> 3) * 32 + (m & 7) * 4 + (k & 3);
    A[off] = 1.0f + m / 128.0f;
  }
  for (int f = tid; f < 8 * N; f += blockDim.x) {
    int k = f / N, n = f % N;
    int off = (k >> 3) * (N / 4 * 32) + (n >> 2) * 32 + (k & 7) * 4 + (n & 3);
    if (variant == 2) off = (k >> 2) * (N / 8 * 32) + (n >> 3) * 32 + (n & 7) * 4 + (k & 3);
    B[off] = (float)(k + 1);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  uint32_t idesc = umma_idesc(128, N);
  if (variant == 2) idesc &= ~((1u << 15) | (1u << 16));  // K-major A and B
  uint32_t lboA = 128 / 4 * 128, lboB = N / 4 * 128, sbo = 128;
  if (variant == 1) { uint32_t t = lboA; lboA = sbo; sbo = t; lboB = 128; }  // swapped roles
  if (variant == 2) { lboA = 128 / 8 * 128; lboB = N / 8 * 128; sbo = 128; }
  if (variant == 3 && warp < 4) {  // TMEM store/load round trip, no MMA
    uint32_t v[8];
    for (int q = 0; q < 8; ++q) v[q] = __float_as_uint(1000.f * warp + lane + q / 8.f);
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  if (tid == 0 && variant != 3) {
    uint64_t da = umma_desc(smem_u32(A), lboA, variant == 1 ? 128 / 4 * 128 : sbo);
    uint64_t db = umma_desc(smem_u32(B), lboB, variant == 1 ? N / 4 * 128 : sbo);
    printf("tmem base %08x idesc %08x descA %016llx descB %016llx\n", tmem, idesc, (unsigned long long)da,
           (unsigned long long)db);
    mma_tf32(tmem, da, db, idesc, 0u);
    umma_commit(&bar);
  }
  if (variant != 3) mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    uint32_t r[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 8; ++q) out[(warp * 32 + lane) * 8 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * 4);
  for (int variant = 0; variant < 4; ++variant) {
    cudaMemset(d, 0, 128 * 8 * 4);
    cudaFuncSetAttribute(probe<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    probe<128><<<1, 128, 64 * 1024>>>(d, variant);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("variant %d: %s  D[0][0..3] = %g %g %g %g  D[64][0] = %g  D[127][7] = %g (expect 36, 54, 71.7)\n", variant,
           cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[64 * 8], h[127 * 8 + 7]);
  }
  return 0;
}
