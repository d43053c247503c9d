// Microbenchmark (round 2): random-row gather bandwidth on B200 with enough loads in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather_bench2 l2_gather_bench2.cu
//   ./l2_gather_bench2 > r02_l2_gather_bench2.jsonl
//
// Why: the SpMM of the NC/NE products gathers one whole neighbour row per edge (config 4: 1600 B
// rows, 198 GB per step).  Round 1's bench (profiles/l2_gather_bench.cu) issued one row per loop
// trip per lane, a dependent index -> row chain with ~1 load in flight, so its "L2 ceiling" of
// 5.7 TB/s measured latency, not bandwidth.  Here a TEAM of TS threads reads
// one row of 16*TS bytes cooperatively (coalesced, like spmm_kernel) and every thread keeps MLP
// independent rows in flight (indices loaded first, then MLP row loads, then the adds).
// Sweeps row size (32 / 64 / 128 / 1600 B), MLP (4 / 8 / 16) and table size (L2-resident 16-120 MB,
// DRAM-resident 1-4 GB).  Reports gathered bytes / time (the SpMM's "Gv" rate).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

template <int TS, int MLP>
__global__ void __launch_bounds__(1024) gather_team(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                                                    int64_t n, float* __restrict__ out) {
  const int per_block = blockDim.x / TS;
  const int team = threadIdx.x / TS, c = threadIdx.x - team * TS;
  if (team >= per_block) return;
  const int64_t t0 = (int64_t)blockIdx.x * per_block + team, nt = (int64_t)gridDim.x * per_block;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t e = t0 * MLP; e + MLP <= n; e += nt * MLP) {
    uint32_t j[MLP];
#pragma unroll
    for (int u = 0; u < MLP; ++u) j[u] = __ldg(idx + e + u);
    float4 v[MLP];
#pragma unroll
    for (int u = 0; u < MLP; ++u) v[u] = __ldg(table + (int64_t)j[u] * TS + c);
#pragma unroll
    for (int u = 0; u < MLP; ++u) {
      acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
    }
  }
  const float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keeps the loads live
}

static uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <int TS, int MLP>
void run(const float4* table, size_t table_bytes, uint32_t* idx_d, int64_t n_idx, float* out, int sms) {
  const int64_t rows = (int64_t)(table_bytes / (16 * TS));
  std::vector<uint32_t> h(n_idx);
  uint64_t st = 12345 + TS * 7 + table_bytes;
  for (int64_t e = 0; e < n_idx; ++e) h[e] = (uint32_t)(splitmix(st) % (uint64_t)rows);
  cudaMemcpy(idx_d, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
  const int per_block = 1024 / TS;
  const int threads = per_block * TS;
  const int blocks = sms * (2048 / threads);
  gather_team<TS, MLP><<<blocks, threads>>>(table, idx_d, n_idx, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) gather_team<TS, MLP><<<blocks, threads>>>(table, idx_d, n_idx, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double gb = (double)n_idx * 16.0 * TS / 1e9;
  printf("{\"row_bytes\": %d, \"mlp\": %d, \"table_MB\": %.0f, \"ms\": %.3f, \"gather_GBps\": %.0f, \"err\": \"%s\"}\n",
         16 * TS, MLP, table_bytes / 1e6, ms, gb / (ms / 1e3), cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

template <int TS>
void sweep(const float4* table, uint32_t* idx_d, float* out, int sms) {
  // about 8 GB gathered per launch at 1600-B rows, fewer bytes (but >= 256M rows... capped) below
  const int64_t n_idx = std::min<int64_t>((int64_t)(8e9 / (16.0 * TS)), 256LL << 20);
  for (double mb : {16.0, 48.0, 96.0, 120.0, 1024.0, 4096.0}) {
    const size_t tb = (size_t)(mb * 1e6) / (16 * TS) * (16 * TS);
    run<TS, 4>(table, tb, idx_d, n_idx, out, sms);
    run<TS, 8>(table, tb, idx_d, n_idx, out, sms);
    run<TS, 16>(table, tb, idx_d, n_idx, out, sms);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t max_table = (size_t)4096e6 + 4096;
  float4* table = nullptr;
  uint32_t* idx = nullptr;
  float* out = nullptr;
  cudaMalloc(&table, max_table);
  cudaMemset(table, 0, max_table);
  cudaMalloc(&idx, (256LL << 20) * 4);
  cudaMalloc(&out, 1 << 24);
  sweep<2>(table, idx, out, sms);    // 32 B rows
  sweep<4>(table, idx, out, sms);    // 64 B
  sweep<8>(table, idx, out, sms);    // 128 B
  sweep<100>(table, idx, out, sms);  // 1600 B (config 4's l = 400 rows)
  return 0;
}
