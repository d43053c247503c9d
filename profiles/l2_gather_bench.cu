// Microbenchmark: random-row gather bandwidth vs. footprint on B200 (decides the SpMM layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather_bench l2_gather_bench.cu
//   ./l2_gather_bench
// A warp reads 32 consecutive indices (coalesced) and each lane gathers one row of
// `row_bytes` from a table of `table_mb`; the sum is written per warp (negligible).
// Reports effective gather GB/s (gathered bytes / time) per (row_bytes, table_mb).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int NV4>  // float4 per gathered row
__global__ void gather(const float4* __restrict__ table, const uint32_t* __restrict__ idx, int64_t n_idx,
                       float* __restrict__ out, int evict_first_idx) {
  float4 acc = make_float4(0, 0, 0, 0);
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (int64_t e = tid; e < n_idx; e += stride) {
    uint32_t j;
    if (evict_first_idx)
      asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(j) : "l"(idx + e), "l"(pol));
    else
      j = __ldg(idx + e);
    const float4* p = table + (int64_t)j * NV4;
#pragma unroll
    for (int v = 0; v < NV4; ++v) {
      float4 x = __ldg(p + v);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
  }
  out[tid] = acc.x + acc.y + acc.z + acc.w;
}

template <int NV4>
void run(float4* table, size_t table_bytes, uint32_t* idx_d, std::vector<uint32_t>& idx_h, int64_t n_idx, float* out,
         int ef) {
  int64_t rows = table_bytes / (16 * NV4);
  for (int64_t e = 0; e < n_idx; ++e) idx_h[e] = (uint32_t)(((uint64_t)e * 2654435761ULL + (e >> 7) * 40503ULL) % rows);
  cudaMemcpy(idx_d, idx_h.data(), n_idx * 4, cudaMemcpyHostToDevice);
  int blocks = 148 * 8, threads = 256;
  gather<NV4><<<blocks, threads>>>(table, idx_d, n_idx, out, ef);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) gather<NV4><<<blocks, threads>>>(table, idx_d, n_idx, out, ef);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 3;
  double gb = (double)n_idx * 16 * NV4 / 1e9;
  printf("{\"row_bytes\": %d, \"table_MB\": %.0f, \"idx_evict_first\": %d, \"ms\": %.3f, \"gather_GBps\": %.0f}\n",
         16 * NV4, table_bytes / 1e6, ef, ms, gb / (ms / 1e3));
}

int main() {
  const int64_t n_idx = 64LL << 20;
  size_t max_table = 4096ULL << 20;
  float4* table;
  uint32_t* idx_d;
  float* out;
  cudaMalloc(&table, max_table);
  cudaMemset(table, 0, max_table);
  cudaMalloc(&idx_d, n_idx * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  std::vector<uint32_t> idx_h(n_idx);
  for (size_t mb : {16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 1024, 4096}) {
    size_t bytes = mb << 20;
    run<2>(table, bytes, idx_d, idx_h, n_idx, out, 0);
    run<2>(table, bytes, idx_d, idx_h, n_idx, out, 1);
    run<8>(table, bytes, idx_d, idx_h, n_idx, out, 0);
    run<100>(table, bytes, idx_d, idx_h, n_idx / 16, out, 0);
  }
  return 0;
}
