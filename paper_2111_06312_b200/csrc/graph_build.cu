// Device-side graph build for isvd_graph_create: degree relabelling order, fp64-derived scale
// vectors and the SpMM segment plan, computed from the device row_ptr (so the host neither sorts
// nor uploads O(n) arrays).  Results are identical to the host formulation they replace:
//   * order: stable sort by decreasing degree (CUB radix sort of 0xFFFFFFFF - degree, which is
//     stable) -- the same permutation as a stable counting sort;
//   * scales: 1/d, (d+1)^-1/2, (d+1)^-1, (d+1)^1/2 computed in fp64 (IEEE division / sqrt, as on
//     the host) and rounded to fp32 (reading O3);
//   * plan: rows of <= kSegEdges edges are one segment, longer rows ceil(d / kSegEdges) segments
//     whose partial sums go to consecutive slots, slots numbered in row order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace isvd {
namespace {

__global__ void degree_keys_kernel(const int64_t* __restrict__ rp, int64_t n, uint32_t* __restrict__ keys,
                                   int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = 0xFFFFFFFFu - (uint32_t)(rp[i + 1] - rp[i]);
    idx[i] = (int32_t)i;
  }
}

__global__ void relabel_maps_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ order, int64_t n,
                                    int32_t* __restrict__ new_of_old, int64_t* __restrict__ deg_new) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n; t += (int64_t)gridDim.x * blockDim.x) {
    if (t == n) {
      deg_new[n] = 0;
      continue;
    }
    const int32_t o = order[t];
    new_of_old[o] = (int32_t)t;
    deg_new[t] = rp[o + 1] - rp[o];
  }
}

ISVD_DEVICE void write_scales(int64_t i, double d, float* inv, float* s, float* s2, float* rs) {
  inv[i] = d > 0.0 ? (float)(1.0 / d) : 0.f;
  s[i] = (float)(1.0 / sqrt(d + 1.0));
  s2[i] = (float)(1.0 / (d + 1.0));
  rs[i] = (float)sqrt(d + 1.0);
}

// unweighted: d_i = number of stored edges (exact integer)
__global__ void scales_kernel(const int64_t* __restrict__ rp, int64_t n, float* __restrict__ inv,
                              float* __restrict__ s, float* __restrict__ s2, float* __restrict__ rs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    write_scales(i, (double)(rp[i + 1] - rp[i]), inv, s, s2, rs);
}

// weighted: d_i = sum_j A_ij in fp64, one warp per row (lane-strided sums, then a fixed
// xor tree: deterministic)
__global__ void scales_weighted_kernel(const int64_t* __restrict__ rp, const float* __restrict__ val, int64_t n,
                                       float* __restrict__ inv, float* __restrict__ s, float* __restrict__ s2,
                                       float* __restrict__ rs) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double d = 0.0;
    for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) d += (double)val[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) write_scales(i, d, inv, s, s2, rs);
  }
}

__global__ void plan_count_kernel(const int64_t* __restrict__ rp, int64_t n, int64_t* __restrict__ nseg,
                                  int32_t* __restrict__ nsplit, int32_t* __restrict__ nslot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) {
      nseg[n] = 0; nsplit[n] = 0; nslot[n] = 0;
      continue;
    }
    const int64_t d = rp[i + 1] - rp[i];
    const bool split = d > kSegEdges;
    const int64_t ns = split ? (d + kSegEdges - 1) / kSegEdges : 1;
    nseg[i] = ns;
    nsplit[i] = split ? 1 : 0;
    nslot[i] = split ? (int32_t)ns : 0;
  }
}

__global__ void plan_fill_kernel(const int64_t* __restrict__ rp, int64_t n, const int64_t* __restrict__ seg_off,
                                 const int32_t* __restrict__ split_off, const int32_t* __restrict__ slot_off,
                                 SpmmPlan p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = rp[i], e0 = rp[i + 1], d = e0 - b0;
    const int64_t s0 = seg_off[i];
    if (d <= kSegEdges) {
      p.seg_row[s0] = (int32_t)i;
      p.seg_beg[s0] = b0;
      p.seg_len[s0] = (int32_t)d;
      p.seg_slot[s0] = -1;
    } else {
      const int32_t ns = (int32_t)((d + kSegEdges - 1) / kSegEdges), slot0 = slot_off[i], r = split_off[i];
      p.split_row[r] = (int32_t)i;
      p.split_slot0[r] = slot0;
      p.split_nslot[r] = ns;
      for (int32_t t = 0; t < ns; ++t) {
        const int64_t b = b0 + (int64_t)t * kSegEdges;
        const int64_t e = b + kSegEdges < e0 ? b + kSegEdges : e0;
        p.seg_row[s0 + t] = (int32_t)i;
        p.seg_beg[s0 + t] = b;
        p.seg_len[s0 + t] = (int32_t)(e - b);
        p.seg_slot[s0 + t] = slot0 + t;
      }
    }
  }
}

__global__ void split_count_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                                   int64_t lo, int64_t hi, int64_t* __restrict__ cnt_loc, int64_t* __restrict__ cnt_rem) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i <= n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (i == n) {
      if (lane == 0) { cnt_loc[n] = 0; cnt_rem[n] = 0; }
      continue;
    }
    int64_t c = 0;
    for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) c += (ci[e] >= lo && ci[e] < hi) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) {
      cnt_loc[i] = c;
      cnt_rem[i] = (rp[i + 1] - rp[i]) - c;
    }
  }
}

// warp per row: stable partition of the row's edges (ballot + prefix popcount per 32-edge chunk)
__global__ void split_fill_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const float* __restrict__ val, int64_t n, int64_t lo, int64_t hi,
                                  const int64_t* __restrict__ rp_loc, const int64_t* __restrict__ rp_rem,
                                  int32_t* __restrict__ ci_loc, float* __restrict__ val_loc,
                                  int32_t* __restrict__ ci_rem, float* __restrict__ val_rem) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t pl = rp_loc[i], pr = rp_rem[i];
    for (int64_t b = rp[i]; b < rp[i + 1]; b += 32) {
      const int64_t e = b + lane;
      const bool valid = e < rp[i + 1];
      const int32_t j = valid ? ci[e] : 0;
      const bool loc = valid && j >= lo && j < hi;
      const unsigned ml = __ballot_sync(0xffffffffu, loc), mr = __ballot_sync(0xffffffffu, valid && !loc);
      const unsigned below = (1u << lane) - 1u;
      if (loc) {
        const int64_t d = pl + __popc(ml & below);
        ci_loc[d] = j;
        if (val) val_loc[d] = val[e];
      } else if (valid) {
        const int64_t d = pr + __popc(mr & below);
        ci_rem[d] = j;
        if (val) val_rem[d] = val[e];
      }
      pl += __popc(ml);
      pr += __popc(mr);
    }
  }
}

unsigned grid_n(int64_t n) { return (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n + 1, 256), 1), 148 * 16); }

}  // namespace

size_t graph_build_temp_bytes(int64_t n) {
  size_t a = 0, b = 0, c = 0, d = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(n + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, c, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n + 1));
  d = std::max(std::max(a, b), c);
  return d + 256;
}

cudaError_t launch_degree_order(const int64_t* rp, int64_t n, uint32_t* keys2, int32_t* idx, int32_t* order,
                                int32_t* new_of_old, int64_t* deg_tmp, int64_t* rp_new, void* temp, size_t temp_bytes,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; degree_keys_kernel<<<grid_n(n), 256, 0, st>>>(rp, n, keys2, idx);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys2, keys2 + n, idx, order, (int)n, 0, 32, st);
  if (e != cudaSuccess) return e;
  ++g_launches; relabel_maps_kernel<<<grid_n(n), 256, 0, st>>>(rp, order, n, new_of_old, deg_tmp);
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, deg_tmp, rp_new, (int)(n + 1), st);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_scales(const int64_t* rp, const float* val, int64_t n, float* inv, float* s, float* s2, float* rs,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  if (val) {
    const int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), 148 * 16);
    scales_weighted_kernel<<<(unsigned)blocks, 256, 0, st>>>(rp, val, n, inv, s, s2, rs);
  } else {
    scales_kernel<<<grid_n(n), 256, 0, st>>>(rp, n, inv, s, s2, rs);
  }
  return cudaGetLastError();
}

namespace {
// one warp per row: out[row, col_idx[e]] += (val ? val[e] : 1)  (duplicates sum, as in the CSR)
__global__ void dense_adj_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const float* __restrict__ val, int64_t n, int64_t ld, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5)
    for (int64_t e = rp[r] + lane; e < rp[r + 1]; e += 32) atomicAdd(out + r * ld + ci[e], val ? val[e] : 1.f);
}
}  // namespace

namespace {
__global__ void f32_to_u8_kernel(const float* __restrict__ in, int64_t n, int64_t ldi, uint8_t* __restrict__ out,
                                 int64_t ldo) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * ldo; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ldo, c = t - r * ldo;
    out[t] = c < n ? (uint8_t)fminf(in[r * ldi + c], 255.f) : 0;
  }
}
}  // namespace

cudaError_t launch_dense_to_u8(const float* in, int64_t n, int64_t ldi, uint8_t* out, int64_t ldo, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  f32_to_u8_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * ldo, 256), 148 * 32), 256, 0, st>>>(in, n, ldi, out, ldo);
  return cudaGetLastError();
}

cudaError_t launch_dense_adjacency(const int64_t* rp, const int32_t* ci, const float* val, int64_t n, int64_t ld,
                                   float* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float) * (size_t)n * ld, st);
  if (e != cudaSuccess) return e;
  const int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), 148 * 16);
  ++g_launches;
  dense_adj_kernel<<<(unsigned)blocks, 256, 0, st>>>(rp, ci, val, n, ld, out);
  return cudaGetLastError();
}

cudaError_t launch_plan_count(const int64_t* rp, int64_t n, int64_t* nseg, int32_t* nsplit, int32_t* nslot,
                              int64_t* seg_off, int32_t* split_off, int32_t* slot_off, void* temp, size_t temp_bytes,
                              cudaStream_t st) {
  ++g_launches; plan_count_kernel<<<grid_n(n), 256, 0, st>>>(rp, n, nseg, nsplit, nslot);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, nseg, seg_off, (int)(n + 1), st);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, nsplit, split_off, (int)(n + 1), st);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, nslot, slot_off, (int)(n + 1), st);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_split_count(const int64_t* rp, const int32_t* ci, int64_t n, int64_t lo, int64_t hi,
                               int64_t* cnt_loc, int64_t* cnt_rem, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(std::max<int64_t>(ceil_div((n + 1) * 32, 256), 1), 148 * 16);
  ++g_launches; split_count_kernel<<<(unsigned)blocks, 256, 0, st>>>(rp, ci, n, lo, hi, cnt_loc, cnt_rem);
  return cudaGetLastError();
}

cudaError_t launch_split_fill(const int64_t* rp, const int32_t* ci, const float* val, int64_t n, int64_t lo, int64_t hi,
                              const int64_t* rp_loc, const int64_t* rp_rem, int32_t* ci_loc, float* val_loc,
                              int32_t* ci_rem, float* val_rem, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), 148 * 16);
  ++g_launches;
  split_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(rp, ci, val, n, lo, hi, rp_loc, rp_rem, ci_loc, val_loc, ci_rem,
                                                      val_rem);
  return cudaGetLastError();
}

cudaError_t launch_exclusive_scan64(const int64_t* in, int64_t* out, int64_t n1, void* temp, size_t temp_bytes,
                                    cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n1, st);
}

cudaError_t launch_plan_fill(const int64_t* rp, int64_t n, const int64_t* seg_off, const int32_t* split_off,
                             const int32_t* slot_off, const SpmmPlan& p, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; plan_fill_kernel<<<grid_n(n), 256, 0, st>>>(rp, n, seg_off, split_off, slot_off, p);
  return cudaGetLastError();
}

}  // namespace isvd
