// Fused CSR SpMM step (K1): one application of T = D^-1 A (NE, Eq. 3)
// or of A_hat = S (A + I) S (NC, Eq. 6 / P:68) to an n x w block, with the
// Horner-chain term, the row scales and the rank-1 correction of Eq. 3
// (-lambda 1 1^T, applied matrix-free as <M2, <M1, G>>) fused into
// the epilogue.  Replaces the paper's tf.sparse.sparse_dense_matmul
// (SparseMatrixPF.dot), SumPF.dot and the lazy cache of
// ProductPF.
//
// Two work decompositions (B200):
//  * row-major gather source (small n; the whole iterate is L2-resident): a "team"
//    of w/4 threads owns one CSR segment; thread t owns columns [4t, 4t+4) and
//    gathers them with one 16-byte read-only load per neighbour, so every
//    neighbour row is read as one contiguous, coalesced span.
//  * slab-major gather source (large n: the iterate is far larger than the 126 MB
//    L2): columns are processed one group of 8-column slabs at a time so that the
//    slab being gathered (n x 32 B) stays L2-resident while the CSR streams past;
//    an item is (slab, segment) served by 2 threads (16 B each = one 32 B sector
//    per gathered row).  Segments are visited longest-first so a warp's 16 items
//    have similar lengths.
// In both, eight neighbours are in flight per thread (memory-level parallelism
// for the dependent index -> row gather), summed in fp32, and each block of
// eight is added into an fp64 accumulator (reading O15: fp64 row accumulation).
// Rows longer than kSegEdges edges are split into segments whose fp32 partials
// are combined by `spmm_fixup_kernel` in a fixed order: results are
// deterministic and hubs (max degree ~1.4e5 in config 4) do not serialise.
#include <cstdlib>

#include "common.cuh"

namespace isvd {
namespace {

struct Acc4 { double x, y, z, w; };

ISVD_DEVICE void acc_add(Acc4& a, float4 v) { a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w; }

// columns [col, col+4) of local row `row`
ISVD_DEVICE void spmm_epilogue(const SpmmArgs& a, int64_t row, int64_t col, Acc4 acc) {
  if (a.self_coef != 0.f) {
    float4 y = ldg4(a.Y + mat_off(a.ldy, a.ysr, row + a.row_offset, col));
    double sc = a.self_coef;
    acc.x += sc * y.x; acc.y += sc * y.y; acc.z += sc * y.z; acc.w += sc * y.w;
  }
  double p = a.post_coef;
  if (a.post_vec) p *= (double)a.post_vec[row];
  acc.x *= p; acc.y *= p; acc.z *= p; acc.w *= p;
  if (a.T) {
    double t = a.term_coef;
    if (a.term_vec) t *= (double)a.term_vec[row];
    float4 tv = *reinterpret_cast<const float4*>(a.T + mat_off(a.ldt, a.tsr, row, col));  // may alias out
    acc.x += t * tv.x; acc.y += t * tv.y; acc.z += t * tv.z; acc.w += t * tv.w;
  }
  if (a.colsum) {
    double r = a.rank1_coef;
    acc.x -= r * a.colsum[col]; acc.y -= r * a.colsum[col + 1];
    acc.z -= r * a.colsum[col + 2]; acc.w -= r * a.colsum[col + 3];
  }
  st4(a.out + mat_off(a.ldo, a.osr, row, col),
      make_float4((float)acc.x, (float)acc.y, (float)acc.z, (float)acc.w));
}

// Gather-sum of one segment for 4 columns: y points at column 4t of gather row 0 and
// `stride` is the distance between consecutive gather rows (ld, or 8 in a slab).
// col_idx entries carry a 2-bit hotness tag in bits 30-31 (kHotShift; 0 = cold,
// 3 = top 1 % by degree).  kHint: rows tagged >= hot_level are loaded with an L2
// evict_last policy, the rest evict_first, so the few hub rows that take ~40 % of
// the gathers of a power-law graph stay L2-resident under the stream of cold rows.
template <bool kHint>
ISVD_DEVICE Acc4 gather_segment(const int32_t* __restrict__ idx, int len, const float* __restrict__ y, int64_t stride,
                                unsigned hot_level, uint64_t keep, uint64_t stream) {
  Acc4 acc{0.0, 0.0, 0.0, 0.0};
  int e = 0;
  for (; e + 8 <= len; e += 8) {
    unsigned j[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) j[u] = (unsigned)__ldg(idx + e + u);
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float* p = y + (int64_t)(j[u] & kIdxMask) * stride;
      if (kHint) v[u] = ldg4_hint(p, (j[u] >> kHotShift) >= hot_level ? keep : stream);
      else v[u] = ldg4(p);
    }
    float4 s01 = f4add(v[0], v[1]), s23 = f4add(v[2], v[3]), s45 = f4add(v[4], v[5]), s67 = f4add(v[6], v[7]);
    acc_add(acc, f4add(f4add(s01, s23), f4add(s45, s67)));
  }
  if (e < len) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    for (; e < len; ++e) {
      unsigned j = (unsigned)__ldg(idx + e);
      const float* p = y + (int64_t)(j & kIdxMask) * stride;
      t = f4add(t, kHint ? ldg4_hint(p, (j >> kHotShift) >= hot_level ? keep : stream) : ldg4(p));
    }
    acc_add(acc, t);
  }
  return acc;
}

template <bool kHint>
__global__ void __launch_bounds__(1024) spmm_kernel(SpmmArgs a, const int32_t* __restrict__ seg_row,
                                                    const int64_t* __restrict__ seg_beg,
                                                    const int32_t* __restrict__ seg_len,
                                                    const int32_t* __restrict__ seg_slot, int64_t n_seg,
                                                    int teams, float* __restrict__ partial, unsigned hot_level) {
  const int TS = (int)(a.wpad >> 2);
  const int team = threadIdx.x / TS;
  const int c4 = threadIdx.x - team * TS;
  if (team >= teams) return;
  uint64_t keep = 0, stream = 0;
  if (kHint) {
    keep = l2_policy_evict_last();
    stream = l2_policy_evict_first();
  }
  const float* __restrict__ Yc = a.Y + 4 * (int64_t)c4;
  for (int64_t s = (int64_t)blockIdx.x * teams + team; s < n_seg; s += (int64_t)gridDim.x * teams) {
    const int64_t row = seg_row[s];
    Acc4 acc = gather_segment<kHint>(a.col_idx + seg_beg[s], seg_len[s], Yc, a.ldy, hot_level, keep, stream);
    const int slot = seg_slot[s];
    if (slot < 0) {
      spmm_epilogue(a, row, 4 * (int64_t)c4, acc);
    } else {
      st4(partial + (int64_t)slot * a.wpad + 4 * (int64_t)c4,
          make_float4((float)acc.x, (float)acc.y, (float)acc.z, (float)acc.w));
    }
  }
}

// Slab-major gather source: items (slab in [slab0, slab0 + nslab), segment rank), 2 threads each.
__global__ void __launch_bounds__(256) spmm_slab_kernel(SpmmArgs a, const int32_t* __restrict__ seg_order,
                                                        const int32_t* __restrict__ seg_row,
                                                        const int64_t* __restrict__ seg_beg,
                                                        const int32_t* __restrict__ seg_len,
                                                        const int32_t* __restrict__ seg_slot, int64_t n_seg,
                                                        int slab0, int nslab, float* __restrict__ partial) {
  const int half = threadIdx.x & 1;
  const int64_t n_items = n_seg * nslab;
  const int64_t stride_items = ((int64_t)gridDim.x * blockDim.x) >> 1;
  for (int64_t it = (((int64_t)blockIdx.x * blockDim.x) >> 1) + (threadIdx.x >> 1); it < n_items;
       it += stride_items) {
    const int sl = slab0 + (int)(it / n_seg);
    const int64_t s = __ldg(seg_order + (it - (it / n_seg) * n_seg));
    const int64_t row = __ldg(seg_row + s);
    const float* __restrict__ y = a.Y + (int64_t)sl * a.ysr * kSlab + 4 * half;
    Acc4 acc = gather_segment<false>(a.col_idx + __ldg(seg_beg + s), __ldg(seg_len + s), y, kSlab, 4u, 0, 0);
    const int64_t col = (int64_t)sl * kSlab + 4 * half;
    const int slot = __ldg(seg_slot + s);
    if (slot < 0) {
      spmm_epilogue(a, row, col, acc);
    } else {
      st4(partial + (int64_t)slot * a.wpad + col, make_float4((float)acc.x, (float)acc.y, (float)acc.z, (float)acc.w));
    }
  }
}

__global__ void __launch_bounds__(1024) spmm_fixup_kernel(SpmmArgs a, const int32_t* __restrict__ split_row,
                                                          const int32_t* __restrict__ split_slot0,
                                                          const int32_t* __restrict__ split_nslot, int64_t n_split,
                                                          int teams, const float* __restrict__ partial) {
  const int TS = (int)(a.wpad >> 2);
  const int team = threadIdx.x / TS;
  const int c4 = threadIdx.x - team * TS;
  if (team >= teams) return;
  for (int64_t r = (int64_t)blockIdx.x * teams + team; r < n_split; r += (int64_t)gridDim.x * teams) {
    const int64_t row = split_row[r];
    const int64_t s0 = split_slot0[r];
    const int ns = split_nslot[r];
    Acc4 acc{0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < ns; ++t) acc_add(acc, ldg4(partial + (s0 + t) * a.wpad + 4 * (int64_t)c4));
    spmm_epilogue(a, row, 4 * (int64_t)c4, acc);
  }
}

void team_shape(int64_t wpad, int* teams, int* threads) {
  int TS = (int)(wpad / 4);
  int R = TS >= 512 ? 1 : 512 / TS;
  if (R < 1) R = 1;
  *teams = R;
  *threads = TS * R;
}

cudaError_t launch_fixup(const SpmmPlan& plan, const SpmmArgs& a, const float* ws_partial, int num_sms,
                         cudaStream_t st) {
  if (plan.n_split_rows == 0) return cudaSuccess;
  int teams, threads;
  team_shape(a.wpad, &teams, &threads);
  int64_t fb = ceil_div(plan.n_split_rows, teams);
  int64_t cap = (int64_t)num_sms * 8;
  if (fb > cap) fb = cap;
  ++g_launches;
  spmm_fixup_kernel<<<(int)fb, threads, 0, st>>>(a, plan.split_row, plan.split_slot0, plan.split_nslot,
                                                 plan.n_split_rows, teams, ws_partial);
  return cudaGetLastError();
}

__global__ void tag_hot_kernel(int32_t* __restrict__ col_idx, int64_t nnz, const uint8_t* __restrict__ tag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    unsigned j = (unsigned)col_idx[e] & kIdxMask;
    col_idx[e] = (int32_t)(j | ((unsigned)tag[j] << kHotShift));
  }
}

}  // namespace

cudaError_t launch_tag_hot(int32_t* col_idx, int64_t nnz, const uint8_t* tag, cudaStream_t st) {
  if (nnz <= 0) return cudaSuccess;
  int64_t b = ceil_div(nnz, 256);
  if (b > 148 * 16) b = 148 * 16;
  ++g_launches;
  tag_hot_kernel<<<(int)b, 256, 0, st>>>(col_idx, nnz, tag);
  return cudaGetLastError();
}

int64_t spmm_ws_floats(const SpmmPlan& plan, int64_t wpad) { return plan.n_slots * wpad; }

cudaError_t launch_spmm(const SpmmPlan& plan, const SpmmArgs& a0, float* ws_partial, int num_sms, cudaStream_t st,
                        int64_t l2_budget) {
  if (plan.n_local == 0) return cudaSuccess;
  if (a0.ysr) {
    // slab-major gather source: groups of slabs whose footprint fits the L2 budget
    const int nsl = (int)(a0.wpad / kSlab);
    int64_t per_slab = a0.ysr * kSlab * (int64_t)sizeof(float);
    int group = (int)(l2_budget / (per_slab > 0 ? per_slab : 1));
    if (group < 1) group = 1;
    if (group > nsl) group = nsl;
    const int threads = 256;
    for (int s0 = 0; s0 < nsl; s0 += group) {
      int ns = nsl - s0 < group ? nsl - s0 : group;
      int64_t items = plan.n_seg * ns;
      int64_t blocks = ceil_div(items * 2, threads);
      int64_t cap = (int64_t)num_sms * 8;
      if (blocks > cap) blocks = cap;
      ++g_launches;
      spmm_slab_kernel<<<(int)blocks, threads, 0, st>>>(a0, plan.seg_order, plan.seg_row, plan.seg_beg, plan.seg_len,
                                                        plan.seg_slot, plan.n_seg, s0, ns, ws_partial);
    }
    return launch_fixup(plan, a0, ws_partial, num_sms, st);
  }
  // Column blocks: cb columns per pass (team of cb/4 threads).  A narrower block makes the
  // gathered row shorter, so more hub rows fit the L2 budget; each pass re-reads the CSR.
  int64_t cb = a0.wpad;
  if (const char* e = getenv("ISVD_SPMM_CB")) cb = atoll(e);
  else if (plan.col_block > 0) cb = plan.col_block;
  cb = round_up(cb < 4 ? 4 : cb, 4);
  if (cb > 4096) cb = 4096;
  if (cb > a0.wpad) cb = a0.wpad;
  for (int64_t c0 = 0; c0 < a0.wpad; c0 += cb) {
    SpmmArgs a = a0;
    a.wpad = (a0.wpad - c0) < cb ? (a0.wpad - c0) : cb;
    a.Y += c0;
    if (a.T) a.T += c0;
    if (a.colsum) a.colsum += c0;
    a.out += c0;
    // hottest tag level whose rows fit the L2 budget at this block width (4 = no hints)
    // Measured on B200 (profiles/r01_spmm_sweep.md): the hints did not beat the default
    // replacement policy at config 4, so they are opt-in (ISVD_SPMM_HOT=auto|1..3).
    unsigned lvl = 4;
    if (const char* e = getenv("ISVD_SPMM_HOT")) {
      if (e[0] == 'a') {
        for (int t = 1; t <= 3; ++t)
          if (plan.hot_count[t] > 0 && plan.hot_count[t] * a.wpad * 4 <= l2_budget) { lvl = (unsigned)t; break; }
      } else {
        lvl = (unsigned)atoi(e);
      }
    }
    int teams, threads;
    team_shape(a.wpad, &teams, &threads);
    int64_t blocks = ceil_div(plan.n_seg, teams);
    int per_sm = 2048 / threads;
    if (per_sm < 1) per_sm = 1;
    int64_t cap = (int64_t)num_sms * per_sm * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    // Experiment hook (profiles/spmm_sweep.py): persisting-L2 window over the first
    // ISVD_L2_WINDOW_MB of the gather source (hub rows first after a degree relabel).
    static const char* win_env = getenv("ISVD_L2_WINDOW_MB");
    if (win_env) {
      static bool limit_set = false;
      size_t want = (size_t)atoll(win_env) << 20;
      if (!limit_set) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        limit_set = true;
      }
      cudaStreamAttrValue v = {};
      v.accessPolicyWindow.base_ptr = (void*)a.Y;
      v.accessPolicyWindow.num_bytes = want;
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    ++g_launches;
    if (lvl <= 3)
      spmm_kernel<true><<<(int)blocks, threads, 0, st>>>(a, plan.seg_row, plan.seg_beg, plan.seg_len, plan.seg_slot,
                                                         plan.n_seg, teams, ws_partial, lvl);
    else
      spmm_kernel<false><<<(int)blocks, threads, 0, st>>>(a, plan.seg_row, plan.seg_beg, plan.seg_len, plan.seg_slot,
                                                          plan.n_seg, teams, ws_partial, lvl);
    cudaError_t e = launch_fixup(plan, a, ws_partial, num_sms, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace isvd
