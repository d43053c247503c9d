// Microbenchmark (round 2): can cold-row eviction hints keep the hub rows of a power-law gather in L2?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/hub_gather_bench profiles/hub_gather_bench.cu
//
// Config-4-like stream: a table of R = 2,449,029 rows of 1600 B (3.92 GB, the SpMM gather source);
// 41.5 % of the gathers hit the first H = 49,000 rows (78.4 MB, the "hub" prefix a degree relabel
// produces), uniformly, the rest hit the other rows uniformly (no temporal locality).  The index stream
// is made of batches of 8 rows of one class (so a team's batch is all-hub or all-cold), classes mixed
// at random.  A team of 100 threads gathers one row per load (16 B per thread), 8 rows in flight.
// Variants:
//   0  plain loads, no window
//   1  plain loads, persisting window on the hub prefix (launch attribute, hitRatio 1)
//   2  window + cold batches loaded with an L2::evict_first cache-hint policy (hub batches plain)
//   3  no window + cold batches evict_first, hub batches evict_last policy
// Reports gathered bytes / time (the "Gv" rate) and the time a 198 GB step would take.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int TS = 100, MLP = 8;

__device__ __forceinline__ float4 ld_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

template <int kMode>
__global__ void __launch_bounds__(1000) gather(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                                               int64_t nbatch, int H, float* __restrict__ out) {
  const int per_block = blockDim.x / TS;
  const int team = threadIdx.x / TS, c = threadIdx.x - team * TS;
  if (team >= per_block) return;
  uint64_t pol_first = 0, pol_last = 0;
  if (kMode >= 2) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t b = (int64_t)blockIdx.x * per_block + team; b < nbatch; b += (int64_t)gridDim.x * per_block) {
    uint32_t j[MLP];
#pragma unroll
    for (int u = 0; u < MLP; ++u) j[u] = __ldg(idx + b * MLP + u);
    float4 v[MLP];
    const bool cold = (int)j[0] >= H;  // a batch is all one class
    if (kMode >= 2 && cold) {
#pragma unroll
      for (int u = 0; u < MLP; ++u) v[u] = ld_hint(table + (int64_t)j[u] * TS + c, pol_first);
    } else if (kMode == 3) {
#pragma unroll
      for (int u = 0; u < MLP; ++u) v[u] = ld_hint(table + (int64_t)j[u] * TS + c, pol_last);
    } else {
#pragma unroll
      for (int u = 0; u < MLP; ++u) v[u] = __ldg(table + (int64_t)j[u] * TS + c);
    }
#pragma unroll
    for (int u = 0; u < MLP; ++u) {
      acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
    }
  }
  const float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main() {
  const int64_t R = 2449029, H = 49000;
  const size_t row_bytes = 16 * TS;
  const int64_t nbatch = 8'000'000;  // 64M gathers = 102 GB per pass
  int dev = 0, sms = 0, maxwin = 0, maxpersist = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxpersist);
  float4* table;
  uint32_t* idx;
  float* out;
  cudaMalloc(&table, R * row_bytes);
  cudaMemset(table, 0, R * row_bytes);
  cudaMalloc(&idx, nbatch * MLP * 4);
  cudaMalloc(&out, 1 << 24);
  std::vector<uint32_t> h(nbatch * MLP);
  uint64_t st = 7;
  for (int64_t b = 0; b < nbatch; ++b) {
    const bool hub = (splitmix(st) % 1000) < 415;
    for (int u = 0; u < MLP; ++u)
      h[b * MLP + u] = hub ? (uint32_t)(splitmix(st) % H) : (uint32_t)(H + splitmix(st) % (R - H));
  }
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const size_t win = std::min<size_t>((size_t)H * row_bytes, std::min<size_t>(maxwin, maxpersist));
  printf("{\"sms\": %d, \"max_window\": %d, \"max_persist\": %d, \"window_bytes\": %zu}\n", sms, maxwin, maxpersist, win);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms * 2);
      cfg.blockDim = dim3(1000);
      cudaLaunchAttribute attr[1];
      if (mode == 1 || mode == 2) {
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = table;
        attr[0].val.accessPolicyWindow.num_bytes = win;
        attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
      }
      void (*k)(const float4*, const uint32_t*, int64_t, int, float*) =
          mode == 0 || mode == 1 ? gather<0> : (mode == 2 ? gather<2> : gather<3>);
      cudaLaunchKernelEx(&cfg, k, (const float4*)table, (const uint32_t*)idx, nbatch, (int)H, out);  // warm
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k, (const float4*)table, (const uint32_t*)idx, nbatch, (int)H, out);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gb = (double)nbatch * MLP * row_bytes / 1e9;
      printf("{\"rep\": %d, \"mode\": %d, \"err\": \"%s\", \"ms\": %.3f, \"gather_TBps\": %.3f, \"ms_per_198GB\": %.2f}\n", rep,
             mode, cudaGetErrorString(err), ms, gb / ms, 198.0 / (gb / ms));
      cudaCtxResetPersistingL2Cache();
    }
  return 0;
}
