// tcgen05.mma kind::tf32 with MN-major operands, round 2.  The round-1 probe (umma_mn_probe.cu)
// built MN-major tiles by hand in SWIZZLE_NONE / SWIZZLE_128B (16-B atoms) and got all zeros.  The
// sm_100 descriptor has a fifth layout type, SWIZZLE_128B_BASE32B (encoding 1): 32-byte swizzle atoms
// in a 128-byte span, which is the only MN-major layout for 32-bit operands.  TMA writes it directly
// (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B), so the tiles here are loaded straight from row-major global
// matrices, exactly as the Gram would: A(m, k) = Ag[k][m], B(n, k) = Bg[k][n], D = Ag^T Bg.
//
// Tile: 32 columns (128 B) x KR rows per TMA box; M = N = 128 -> 4 boxes per operand; KR = 32 rows
// -> 4 MMA k-steps of 8.  Canonical MN-major form (units of 16 B): ((8, n), (4, k)) : ((1, LBO), (8, SBO)),
// i.e. LBO = byte stride between 32-column boxes, SBO = byte stride between 4-row groups.
//   v0  layout 1, LBO = KR*128, SBO = 512
//   v1  layout 1, LBO / SBO swapped
//   v2  layout 2 (SWIZZLE_128B, TMA SWIZZLE_128B), LBO = KR*128, SBO = 1024
//   v3  layout 2, swapped
// It also dumps the smem image of the first box (v0) so the swizzle function can be checked.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2111_06312_b200/csrc \
//        profiles/umma_mn_probe2.cu -o build/umma_mn_probe2
#include <cmath>
#include <cstdio>
#include <cstring>

#include "umma.cuh"

namespace isvd {
thread_local int64_t g_launches = 0;
}
using namespace isvd;

constexpr int M = 128, N = 128, KR = 32;

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* out,
                      uint32_t* dump, int layout, uint32_t lbo, uint32_t sbo) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tbase;
  uint8_t* base = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* A = base;                    // 4 boxes x KR x 128 B = 16 KB
  uint8_t* B = base + 4 * KR * 128;     // 16 KB
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar_tma, 2 * 4 * KR * 128);
    for (int b = 0; b < 4; ++b) {
      tma_2d(A + b * KR * 128, &ta, 32 * b, 0, &bar_tma);
      tma_2d(B + b * KR * 128, &tb, 32 * b, 0, &bar_tma);
    }
  }
  mbar_wait(&bar_tma, 0);
  for (int i = tid; i < KR * 32; i += blockDim.x) dump[i] = ((uint32_t*)A)[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t idesc = umma_idesc(M, N) | (1u << 15) | (1u << 16);  // MN-major A and B
  if (tid == 0) {
    for (int ks = 0; ks < KR / 8; ++ks) {
      const uint64_t da = umma_desc(smem_u32(A) + ks * 8 * 128, lbo, sbo, layout);
      const uint64_t db = umma_desc(smem_u32(B) + ks * 8 * 128, lbo, sbo, layout);
      mma_tf32(tmem, da, db, idesc, ks > 0 ? 1u : 0u);
    }
    umma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
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

// exactly representable in TF32 (<= 11 significant bits) so D is exact
static float ag(int k, int m) { return (float)((k * 7 + m * 3) % 17 - 8) / 8.0f; }
static float bg(int k, int n) { return (float)((k * 5 + n * 11) % 13 - 6) / 4.0f; }

int main() {
  const int K = KR;
  static float hA[K * M], hB[K * N], h[M * N];
  static uint32_t hd[KR * 32];
  for (int k = 0; k < K; ++k) {
    for (int m = 0; m < M; ++m) hA[k * M + m] = ag(k, m);
    for (int n = 0; n < N; ++n) hB[k * N + n] = bg(k, n);
  }
  // dump tile: element index as payload, to read back the swizzle (box 0: columns 0..31, rows 0..KR-1)
  float *dA, *dB, *dAidx, *dout;
  uint32_t* ddump;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dAidx, sizeof(hA));
  cudaMalloc(&dout, sizeof(h));
  cudaMalloc(&ddump, sizeof(hd));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  {
    static uint32_t idx[K * M];
    for (int k = 0; k < K; ++k)
      for (int m = 0; m < M; ++m) idx[k * M + m] = (uint32_t)(k << 16 | m);
    cudaMemcpy(dAidx, idx, sizeof(idx), cudaMemcpyHostToDevice);
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  struct V { int layout; CUtensorMapSwizzle sw; uint32_t lbo, sbo; const char* name; } vs[] = {
      {1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, KR * 128, 512, "layout1 LBO=box SBO=512"},
      {1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 512, KR * 128, "layout1 swapped"},
      {2, CU_TENSOR_MAP_SWIZZLE_128B, KR * 128, 1024, "layout2 LBO=box SBO=1024"},
      {2, CU_TENSOR_MAP_SWIZZLE_128B, 1024, KR * 128, "layout2 swapped"},
  };
  int ok_any = 0;
  for (int v = 0; v < 4; ++v) {
    CUtensorMap ta, tb, tidx;
    bool ok = make_map(&ta, dA, K, M, M, 32, KR, vs[v].sw) && make_map(&tb, dB, K, N, N, 32, KR, vs[v].sw) &&
              make_map(&tidx, dAidx, K, M, M, 32, KR, vs[v].sw);
    if (!ok) { printf("v%d: tensor map encode failed\n", v); continue; }
    cudaMemset(dout, 0, sizeof(h));
    probe<<<1, 128, 64 * 1024>>>(ta, tb, dout, ddump, vs[v].layout, vs[v].lbo, vs[v].sbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("v%d: %s\n", v, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
    double maxerr = 0.0, maxref = 0.0;
    int nz = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += (double)hA[k * M + m] * hB[k * N + n];
        maxerr = fmax(maxerr, fabs(h[m * N + n] - s));
        maxref = fmax(maxref, fabs(s));
        nz += h[m * N + n] != 0.0f;
      }
    printf("v%d %-26s: nonzero %5d / %d  max |D - ref| %.3e (max |ref| %.3e)  D[0][0]=%g ref %g  D[77][5]=%g\n", v,
           vs[v].name, nz, M * N, maxerr, maxref, h[0], 0.0, h[77 * N + 5]);
    ok_any |= maxerr == 0.0;
    // swizzle map of the index tile
    if (v == 0 || v == 2) {
      probe<<<1, 128, 64 * 1024>>>(tidx, tb, dout, ddump, vs[v].layout, vs[v].lbo, vs[v].sbo);
      cudaDeviceSynchronize();
      cudaMemcpy(hd, ddump, sizeof(hd), cudaMemcpyDeviceToHost);
      printf("  smem image (word w -> (row k, col m)) of box 0, rows 0..7:\n");
      for (int r = 0; r < 8; ++r) {
        printf("   smem row %d:", r);
        for (int w = 0; w < 32; w += 4) {
          uint32_t x;
          memcpy(&x, &hd[r * 32 + w], 4);
          float f;
          memcpy(&f, &x, 4);
          // payload was written as float bits of an integer pattern: recover from the index tile
          printf(" [%2u,%2u]", x >> 16, x & 0xFFFF);
        }
        printf("\n");
      }
    }
  }
  printf(ok_any ? "MN-major tf32: EXACT in at least one variant\n" : "MN-major tf32: no exact variant\n");
  return 0;
}
