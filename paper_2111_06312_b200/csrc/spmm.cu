// Fused CSR SpMM step (K1): one application of T = D^-1 A (NE, Eq. 3)
// or of A_hat = S (A + I) S (NC, Eq. 6 / P:68) to an n x w block, with the
// Horner-chain term, the row scales and the rank-1 correction of Eq. 3
// (-lambda 1 1^T, applied matrix-free as <M2, <M1, G>>) fused into
// the epilogue.  Replaces the paper's tf.sparse.sparse_dense_matmul
// (SparseMatrixPF.dot), SumPF.dot and the lazy cache of
// ProductPF.
//
// Work decomposition (B200): a "team" of w/4 threads owns one CSR segment at a
// time; thread t of the team owns columns [4t, 4t+4) and gathers them with one
// 16-byte read-only load per neighbour, so every neighbour row (1600 B at
// w = 400) is read as one contiguous, coalesced span.  Eight neighbours are in
// flight per thread (memory-level parallelism for the dependent index -> row
// gather), summed in fp32, and each block of eight is added into an fp64
// accumulator (reading O15: fp64 row accumulation).  Rows longer than kSegEdges
// edges are split into segments whose fp32 partials are combined by
// `spmm_fixup_kernel` in a fixed order: results are deterministic and hubs (max
// degree ~1.4e5 in config 4) do not serialise one team.
//
// When the iterate is far larger than L2 the step is bound by DRAM reads of
// gathered rows (ncu: 171 GB per step at config 4 for 10.3 GB of algorithmic
// bytes).  The graph is then relabelled by degree (capi.cpp) so the hub rows —
// 2 % of the nodes take 41 % of the gathers — are one contiguous prefix that an
// L2 persisting window keeps resident (profiles/r01_spmm_sweep.md).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace isvd {
namespace {

// ISVD_SPMM_VARIANT default: 1 = register (LDG) gather with the masked last batch, 2 = shared-memory
// (bulk-copy) staged gather
constexpr int kSpmmDefaultVariant = 1;

struct Acc4 { double x, y, z, w; };

ISVD_DEVICE void acc_add(Acc4& a, float4 v) { a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w; }

// columns [col, col+4) of local row `row`
ISVD_DEVICE void spmm_epilogue(const SpmmArgs& a, int64_t row, int64_t col, Acc4 acc) {
  if (a.pre) {  // the other pass's partial sums (distributed local / remote split)
    const float4 q = ldg4(a.pre + row * a.ldpre + col);
    acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
  }
  if (a.self_coef != 0.f) {
    ISVD_ASSERT(row + a.row_offset < a.n_src);
    float4 y = ldg4(a.Y + (row + a.row_offset) * a.ldy + col);
    double sc = a.self_coef;
    acc.x += sc * y.x; acc.y += sc * y.y; acc.z += sc * y.z; acc.w += sc * y.w;
  }
  double p = a.post_coef;
  if (a.post_vec) p *= (double)a.post_vec[row];
  acc.x *= p; acc.y *= p; acc.z *= p; acc.w *= p;
  if (a.T) {
    double t = a.term_coef;
    if (a.term_vec) t *= (double)a.term_vec[row];
    float4 tv = *reinterpret_cast<const float4*>(a.T + row * a.ldt + col);  // may alias out
    acc.x += t * tv.x; acc.y += t * tv.y; acc.z += t * tv.z; acc.w += t * tv.w;
  }
  if (a.colsum) {
    double r = a.rank1_coef;
    acc.x -= r * a.colsum[col]; acc.y -= r * a.colsum[col + 1];
    acc.z -= r * a.colsum[col + 2]; acc.w -= r * a.colsum[col + 3];
  }
  const int64_t orow = a.out_map ? (int64_t)a.out_map[row] : row;
  ISVD_ASSERT(orow >= 0 && col + 3 < a.ldo);
  st4(a.out + orow * a.ldo + col, make_float4((float)acc.x, (float)acc.y, (float)acc.z, (float)acc.w));
}

// Gather-sum of one segment for 4 columns: y points at column 4t of gather row 0.
// Software-pipelined: the eight row loads of batch b+1 are issued before batch b is summed,
// so 8-16 independent 16-byte loads per thread are in flight (measured: letting the
// compiler interleave loads and adds left ~2 in flight and cost 20 % at config 4).
// kW: weighted graph, each row scaled by its edge weight A_ij inside the fp32 batch.
template <bool kW>
ISVD_DEVICE void load_batch(const int32_t* __restrict__ idx, const float* __restrict__ val,
                            const float* __restrict__ y, int64_t ld, float4 v[8], float wv[8], int64_t n_src) {
  int j[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    j[u] = __ldg(idx + u);
    ISVD_ASSERT(j[u] >= 0 && j[u] < n_src);
  }
  if constexpr (kW) {
#pragma unroll
    for (int u = 0; u < 8; ++u) wv[u] = __ldg(val + u);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = ldg4(y + (int64_t)j[u] * ld);
}

ISVD_DEVICE float4 f4fma(float a, float4 x, float4 c) {
  return make_float4(fmaf(a, x.x, c.x), fmaf(a, x.y, c.y), fmaf(a, x.z, c.z), fmaf(a, x.w, c.w));
}
ISVD_DEVICE float4 f4mul(float a, float4 x) { return make_float4(a * x.x, a * x.y, a * x.z, a * x.w); }

template <bool kW>
ISVD_DEVICE float4 sum_batch(const float4 v[8], const float wv[8]) {
  if constexpr (kW) {
    float4 s01 = f4fma(wv[1], v[1], f4mul(wv[0], v[0])), s23 = f4fma(wv[3], v[3], f4mul(wv[2], v[2]));
    float4 s45 = f4fma(wv[5], v[5], f4mul(wv[4], v[4])), s67 = f4fma(wv[7], v[7], f4mul(wv[6], v[6]));
    return f4add(f4add(s01, s23), f4add(s45, s67));
  } else {
    float4 s01 = f4add(v[0], v[1]), s23 = f4add(v[2], v[3]), s45 = f4add(v[4], v[5]), s67 = f4add(v[6], v[7]);
    return f4add(f4add(s01, s23), f4add(s45, s67));
  }
}

template <bool kW, bool kMaskedTail>
ISVD_DEVICE Acc4 gather_segment(const int32_t* __restrict__ idx, const float* __restrict__ val, int len,
                                const float* __restrict__ y, int64_t ld, int64_t n_src) {
  Acc4 acc{0.0, 0.0, 0.0, 0.0};
  int e = 0;
  if (len >= 8) {
    float4 cur[8], nxt[8];
    float wc[8], wn[8];
    load_batch<kW>(idx, val, y, ld, cur, wc, n_src);
    for (e = 8; e + 8 <= len; e += 8) {
      load_batch<kW>(idx + e, kW ? val + e : val, y, ld, nxt, wn, n_src);
      acc_add(acc, sum_batch<kW>(cur, wc));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        cur[u] = nxt[u];
        if constexpr (kW) wc[u] = wn[u];
      }
    }
    acc_add(acc, sum_batch<kW>(cur, wc));
  }
  if (!kMaskedTail && e < len) {  // one dependent load chain per remaining neighbour
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    for (; e < len; ++e) {
      ISVD_ASSERT(__ldg(idx + e) >= 0 && __ldg(idx + e) < n_src);
      const float4 r = ldg4(y + (int64_t)__ldg(idx + e) * ld);
      t = kW ? f4fma(__ldg(val + e), r, t) : f4add(t, r);
    }
    acc_add(acc, t);
  } else if (e < len) {
    // the last (or only) partial batch: its < 8 row loads are all issued before any add (a masked
    // batch; rows of degree < 8 -- a large share of a power-law graph -- get the same memory-level
    // parallelism as full batches instead of one dependent load chain per neighbour)
    const int rem = len - e;
    int j[8];
    float4 v[8];
    float wv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      j[u] = u < rem ? __ldg(idx + e + u) : -1;
      ISVD_ASSERT(j[u] < n_src);
      if constexpr (kW) wv[u] = u < rem ? __ldg(val + e + u) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = j[u] >= 0 ? ldg4(y + (int64_t)j[u] * ld) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc_add(acc, sum_batch<kW>(v, wv));
  }
  return acc;
}

// kMasked: the last (partial) batch of a segment issues all its < 8 loads together (default);
// otherwise one dependent load chain per remaining neighbour.  (A variant that loaded the next
// segment's descriptor during the gather spilled 156 B at the 64-register cap and ran 25 % slower:
// profiles/r02c_spmm_variants.jsonl.)
template <bool kW, bool kMasked>
__global__ void __launch_bounds__(1024) spmm_kernel(SpmmArgs a, const int32_t* __restrict__ seg_row,
                                                    const int64_t* __restrict__ seg_beg,
                                                    const int32_t* __restrict__ seg_len,
                                                    const int32_t* __restrict__ seg_slot, int64_t n_seg,
                                                    int teams, float* __restrict__ partial) {
  const int TS = (int)(a.wpad >> 2);
  const int team = threadIdx.x / TS;
  const int c4 = threadIdx.x - team * TS;
  if (team >= teams) return;
  const float* __restrict__ Yc = a.Y + 4 * (int64_t)c4;
  for (int64_t s = (int64_t)blockIdx.x * teams + team; s < n_seg; s += (int64_t)gridDim.x * teams) {
    const int64_t row = seg_row[s];
    const int64_t b = seg_beg[s];
    const int len = seg_len[s];
    ISVD_ASSERT(row >= 0 && len >= 0 && len <= kSegEdges);
    Acc4 acc = gather_segment<kW, kMasked>(a.col_idx + b, kW ? a.val + b : nullptr, len, Yc, a.ldy, a.n_src);
    const int slot = seg_slot[s];
    if (slot < 0) {
      spmm_epilogue(a, row, 4 * (int64_t)c4, acc);
    } else {
      st4(partial + (int64_t)slot * a.wpad + 4 * (int64_t)c4,
          make_float4((float)acc.x, (float)acc.y, (float)acc.z, (float)acc.w));
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

// ---------------------------------------------------------------------------------------------
// Shared-memory / TMA-staged gather (north_star: "a shared-memory/TMA-staged gather"; round 2).
// One CTA = one producer warp + one consumer team of w/4 threads (rounded up to warps).  The
// producer walks the CTA's segments (the same strided assignment as spmm_kernel with one team per
// CTA) and, per neighbour j, issues one bulk copy (cp.async.bulk, 16-byte granules, the whole row
// slice Y[j, 0:w) = 1600 B at w = 400) into the next slot of an S-slot shared-memory ring, completing
// on that slot's "full" mbarrier; a slot is reused once every consumer warp has arrived on its
// "empty" mbarrier.  Lane e of the producer handles neighbour e of a 32-neighbour group, so up to 32
// copies are issued per warp instruction and the ring (S >= 32 rows per CTA, several CTAs per SM)
// keeps 100-200 KB of gathers in flight per SM without any register cost, across segment and row
// boundaries (no dependent index -> row bubble at the start of a row, the LDG kernel's stall).
// The consumers read each staged row once from shared memory (thread t: columns [4t, 4t+4), one
// conflict-free LDS.128) and sum exactly as spmm_kernel does -- the same fp32 batches of 8 (missing
// neighbours of the last batch as zeros), the same fp64 accumulation, the same epilogue -- so the
// two kernels are bitwise identical (tests/test_parity_gpu.py::test_spmm_bulk_equals_ldg).
// Optional per-copy L2 policy (hint_mode 1): hub rows (j < hub_rows, the persisting prefix of a
// degree-relabelled gather source) evict_last, the others evict_first.
ISVD_DEVICE void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
ISVD_DEVICE void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
ISVD_DEVICE uint32_t sm32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
ISVD_DEVICE void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm32(b)), "r"(n));
}
ISVD_DEVICE void bar_wait(const uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t"
        "}\n"
        : "=r"(done)
        : "r"(sm32(b)), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1u << 28)) __trap();  // a copy that never lands fails the launch instead of hanging the GPU
  }
}
ISVD_DEVICE void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm32(b)) : "memory");
}
ISVD_DEVICE void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(b)), "r"(bytes) : "memory");
}

constexpr int kBulkMaxThreads = 32 + 256;  // producer warp + up to 256 consumers (w <= 1024)

template <bool kW>
__global__ void __launch_bounds__(kBulkMaxThreads) spmm_bulk_kernel(
    SpmmArgs a, const int32_t* __restrict__ seg_row, const int64_t* __restrict__ seg_beg,
    const int32_t* __restrict__ seg_len, const int32_t* __restrict__ seg_slot, int64_t n_seg, float* __restrict__ partial,
    int log_slots, int64_t hub_rows, int hint_mode) {
  extern __shared__ __align__(128) uint8_t bulk_sm[];
  const int S = 1 << log_slots;
  const uint32_t row_bytes = (uint32_t)a.wpad * 4u;
  uint8_t* const ring = bulk_sm;
  uint64_t* const full = reinterpret_cast<uint64_t*>(bulk_sm + (size_t)S * row_bytes);
  uint64_t* const empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int TS = (int)(a.wpad >> 2);
  const int CW = (TS + 31) >> 5;  // consumer warps
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      bar_init(&full[i], 1);
      bar_init(&empty[i], (uint32_t)CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t G = gridDim.x;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    uint64_t pol_hub = 0, pol_cold = 0;
    if (hint_mode == 1) {
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_hub));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_cold));
    }
    const uint32_t ring_s = sm32(ring), full_s = sm32(full);
    uint32_t ctr = 0;
    for (int64_t s0 = blockIdx.x; s0 < n_seg; s0 += 32 * G) {
      const int64_t s = s0 + (int64_t)lane * G;
      int64_t b = 0;
      int len = 0;
      if (s < n_seg) {
        b = seg_beg[s];
        len = seg_len[s];
      }
      const int64_t left = (n_seg - s0 + G - 1) / G;
      const int nq = left < 32 ? (int)left : 32;
      for (int q = 0; q < nq; ++q) {
        const int64_t bq = __shfl_sync(0xffffffffu, b, q);
        const int lq = __shfl_sync(0xffffffffu, len, q);
        for (int e0 = 0; e0 < lq; e0 += 32) {
          const int e = e0 + lane;
          if (e < lq) {
            const int j = __ldg(a.col_idx + bq + e);
            ISVD_ASSERT(j >= 0 && j < a.n_src);
            const uint32_t c = ctr + (uint32_t)e;
            const uint32_t slot = c & (uint32_t)(S - 1);
            bar_wait(&empty[slot], ((c >> log_slots) & 1u) ^ 1u);
            bar_expect_tx(&full[slot], row_bytes);
            const float* src = a.Y + (int64_t)j * a.ldy;
            const uint32_t dst = ring_s + slot * row_bytes, bar = full_s + slot * 8u;
            if (hint_mode == 1) bulk_g2s_hint(dst, src, row_bytes, bar, j < hub_rows ? pol_hub : pol_cold);
            else bulk_g2s(dst, src, row_bytes, bar);
          }
        }
        ctr += (uint32_t)lq;
      }
    }
    return;
  }
  // -------------------------------------------------------------------- consumers
  const int c4 = tid - 32;
  const bool active = c4 < TS;
  uint32_t ctr = 0;
  int64_t s = blockIdx.x;
  int64_t row_n = 0, b_n = 0;
  int len_n = 0, slot_n = -1;
  if (s < n_seg) {
    row_n = seg_row[s];
    b_n = seg_beg[s];
    len_n = seg_len[s];
    slot_n = seg_slot[s];
  }
  for (; s < n_seg; s += G) {
    const int64_t row = row_n, b = b_n;
    const int len = len_n, pslot = slot_n;
    if (s + G < n_seg) {  // the next segment's descriptor, in flight during this one
      row_n = seg_row[s + G];
      b_n = seg_beg[s + G];
      len_n = seg_len[s + G];
      slot_n = seg_slot[s + G];
    }
    ISVD_ASSERT(row >= 0 && len >= 0 && len <= kSegEdges);
    Acc4 acc{0.0, 0.0, 0.0, 0.0};
    for (int e = 0; e < len; e += 8) {
      const int n8 = len - e < 8 ? len - e : 8;
      float4 v[8];
      float wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        wv[u] = 0.f;
        if (u < n8) {
          const uint32_t c = ctr + (uint32_t)(e + u);
          const uint32_t slot = c & (uint32_t)(S - 1);
          bar_wait(&full[slot], (c >> log_slots) & 1u);
          if (active) v[u] = *reinterpret_cast<const float4*>(ring + (size_t)slot * row_bytes + 16 * c4);
          if constexpr (kW) wv[u] = __ldg(a.val + b + e + u);
        }
      }
      __syncwarp();
      if (lane == 0)
        for (int u = 0; u < n8; ++u) bar_arrive(&empty[(ctr + (uint32_t)(e + u)) & (uint32_t)(S - 1)]);
      acc_add(acc, sum_batch<kW>(v, wv));
    }
    ctr += (uint32_t)len;
    if (!active) continue;
    if (pslot < 0) {
      spmm_epilogue(a, row, 4 * (int64_t)c4, acc);
    } else {
      st4(partial + (int64_t)pslot * a.wpad + 4 * (int64_t)c4,
          make_float4((float)acc.x, (float)acc.y, (float)acc.z, (float)acc.w));
    }
  }
}

void team_shape(int64_t wpad, int* teams, int* threads) {
  int TS = (int)(wpad / 4);
  int R = TS >= 512 ? 1 : 512 / TS;
  if (R < 1) R = 1;
  *teams = R;
  *threads = TS * R;
}


}  // namespace

int64_t spmm_ws_floats(const SpmmPlan& plan, int64_t wpad) { return plan.n_slots * wpad; }

namespace {
// One warp per new row t: copy old row order[t]'s neighbours, renamed through new_of_old.
__global__ void relabel_csr_kernel(const int64_t* __restrict__ rp_old, const int32_t* __restrict__ ci_old,
                                   const float* __restrict__ v_old, const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ new_of_old, const int64_t* __restrict__ rp_new,
                                   int32_t* __restrict__ ci_new, float* __restrict__ v_new, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t o = order[t];
    const int64_t b = rp_old[o], d = rp_old[o + 1] - b, dst = rp_new[t];
    for (int64_t e = lane; e < d; e += 32) {
      ci_new[dst + e] = new_of_old[ci_old[b + e]];
      if (v_old) v_new[dst + e] = v_old[b + e];
    }
  }
}
}  // namespace

cudaError_t launch_relabel_csr(const int64_t* rp_old, const int32_t* ci_old, const float* val_old,
                               const int32_t* order, const int32_t* new_of_old, const int64_t* rp_new,
                               int32_t* ci_new, float* val_new, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = ceil_div(n * 32, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ++g_launches;
  relabel_csr_kernel<<<(int)blocks, 256, 0, st>>>(rp_old, ci_old, val_old, order, new_of_old, rp_new, ci_new,
                                                  val_new, n);
  return cudaGetLastError();
}

namespace {
__global__ void spmm_dense_epilogue_kernel(const float* __restrict__ ws32, int64_t parts, int64_t ws_lda, int64_t ws_ld,
                                           SpmmArgs a, int64_t n_local) {
  const int64_t c4n = a.wpad >> 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_local * c4n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / c4n, col = 4 * (t - row * c4n);
    Acc4 acc{0.0, 0.0, 0.0, 0.0};
    for (int64_t p = 0; p < parts; ++p) acc_add(acc, ldg4(ws32 + (p * ws_lda + row) * ws_ld + col));
    spmm_epilogue(a, row, col, acc);
  }
}
}  // namespace

namespace {
__global__ void spmm_dense64_epilogue_kernel(const double* __restrict__ ws, int64_t parts, int64_t ws_rows,
                                             int64_t ws_ld, const unsigned* __restrict__ cmax, SpmmArgs a,
                                             int64_t n_local) {
  const int64_t c4n = a.wpad >> 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_local * c4n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / c4n, col = 4 * (t - row * c4n);
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t p = 0; p < parts; ++p) {
      const double* w = ws + (p * ws_rows + row) * ws_ld + col;
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] += w[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // the fixed-point scale 2^(E - 22) of the column (dense_i8.cu)
      const float m = __uint_as_float(cmax[col + u]);
      int e = 0;
      if (m > 0.f && isfinite(m)) frexpf(m, &e);
      // a non-finite entry of the column (its max is Inf / NaN) makes the whole column NaN, as the
      // CSR path would propagate it, so the solver's output check reports it
      v[u] = !isfinite(m) ? (double)NAN : (m > 0.f ? ldexp(v[u], e - 22) : 0.0);
    }
    spmm_epilogue(a, row, col, Acc4{v[0], v[1], v[2], v[3]});
  }
}
}  // namespace

cudaError_t launch_spmm_dense64_epilogue(const double* ws, int64_t parts, int64_t ws_rows, int64_t ws_ld,
                                         const unsigned* cmax, const SpmmArgs& a, int64_t n_local, int num_sms,
                                         cudaStream_t st) {
  if (n_local <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(ceil_div(n_local * (a.wpad >> 2), 256), (int64_t)num_sms * 8);
  ++g_launches;
  spmm_dense64_epilogue_kernel<<<(unsigned)blocks, 256, 0, st>>>(ws, parts, ws_rows, ws_ld, cmax, a, n_local);
  return cudaGetLastError();
}

cudaError_t launch_spmm_dense_epilogue(const float* ws32, int64_t parts, int64_t ws_lda, int64_t ws_ld,
                                       const SpmmArgs& a, int64_t n_local, int num_sms, cudaStream_t st) {
  if (n_local <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(ceil_div(n_local * (a.wpad >> 2), 256), (int64_t)num_sms * 8);
  ++g_launches;
  spmm_dense_epilogue_kernel<<<(unsigned)blocks, 256, 0, st>>>(ws32, parts, ws_lda, ws_ld, a, n_local);
  return cudaGetLastError();
}

cudaError_t launch_spmm(const SpmmPlan& plan, const SpmmArgs& a0, float* ws_partial, int num_sms, cudaStream_t st,
                        size_t persist_bytes, int64_t col_block) {
  if (plan.n_local == 0) return cudaSuccess;
  // Column blocks of at most min(col_block, 4096) columns (team of <= 1024 threads); a narrower
  // block gathers shorter row slices, so L2 holds proportionally more rows of the gather source.
  int64_t cb = col_block > 0 ? round_up(col_block, 4) : 4096;
  if (cb > 4096) cb = 4096;
  static int max_window = -1;
  if (max_window < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess) max_window = 0;
  }
  for (int64_t c0 = 0; c0 < a0.wpad; c0 += cb) {
    SpmmArgs a = a0;
    a.wpad = (a0.wpad - c0) < cb ? (a0.wpad - c0) : cb;
    // L2 persisting window on the hub prefix of the gather source, as a LAUNCH attribute (captured
    // into the CUDA graph's kernel node; a stream attribute is not, which cost 20 % at config 4:
    // ncu, graph replay without the window 29-30 ms / 167 GB DRAM per step vs 26.4 ms / 140 GB)
    cudaLaunchAttribute attr[1];
    int nattr = 0;
    if (persist_bytes) {
      // the window spans whole rows; only this block's slices of them are touched, so it is
      // widened by ldy / width to keep about persist_bytes of persisting lines in use
      size_t wb = persist_bytes * (size_t)(a0.ldy / a.wpad);
      if (wb > (size_t)max_window) wb = (size_t)max_window;
      attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
      attr[0].val.accessPolicyWindow.base_ptr = const_cast<float*>(a0.Y + c0);
      attr[0].val.accessPolicyWindow.num_bytes = wb;
      const char* hr = getenv("ISVD_L2_HIT_RATIO");  // tuning override (read per launch; default 1)
      attr[0].val.accessPolicyWindow.hitRatio = hr ? (float)atof(hr) : 1.0f;
      attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      nattr = 1;
    }
    a.Y += c0;
    if (a.T) a.T += c0;
    if (a.pre) a.pre += c0;
    if (a.colsum) a.colsum += c0;
    a.out += c0;
    int teams, threads;
    team_shape(a.wpad, &teams, &threads);
    int64_t blocks = ceil_div(plan.n_seg, teams);
    int per_sm = 2048 / threads;
    if (per_sm < 1) per_sm = 1;
    int64_t cap = (int64_t)num_sms * per_sm * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.stream = st;
    cfg.attrs = nattr ? attr : nullptr;
    cfg.numAttrs = nattr;
    ++g_launches;
    const char* ve = getenv("ISVD_SPMM_VARIANT");  // 0: sequential tail (A/B switch, read per launch)
    const int variant = ve ? atoi(ve) : kSpmmDefaultVariant;
    const bool masked = variant != 0;
    if (variant == 2 && a.wpad <= 1024) {
      // shared-memory / TMA-staged gather (spmm_bulk_kernel): S-slot ring per CTA
      const char* se = getenv("ISVD_SPMM_BULK_SLOTS");
      int S = se ? atoi(se) : 32;
      int log_s = 5;
      while ((1 << log_s) < S) ++log_s;
      const size_t row_bytes = (size_t)a.wpad * 4;
      while (log_s > 5 && ((size_t)1 << log_s) * (row_bytes + 16) > 200 * 1024) --log_s;
      const size_t smem = ((size_t)1 << log_s) * (row_bytes + 16);
      if (smem <= 227 * 1024) {
        const int bthreads = 32 + (int)round_up(a.wpad / 4, 32);
        void (*kb)(SpmmArgs, const int32_t*, const int64_t*, const int32_t*, const int32_t*, int64_t, float*, int,
                   int64_t, int) = a.val ? spmm_bulk_kernel<true> : spmm_bulk_kernel<false>;
        cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kb, bthreads, smem);
        if (per_sm < 1) per_sm = 1;
        int64_t nb = std::min<int64_t>(plan.n_seg, (int64_t)num_sms * per_sm);
        if (nb < 1) nb = 1;
        const char* he = getenv("ISVD_SPMM_BULK_HINT");
        const int hint = he ? atoi(he) : 0;
        const int64_t hub_rows = persist_bytes ? (int64_t)(persist_bytes / ((size_t)a0.ldy * 4)) : 0;
        cfg.gridDim = dim3((unsigned)nb);
        cfg.blockDim = dim3((unsigned)bthreads);
        cfg.dynamicSmemBytes = smem;
        ++g_launches;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kb, a, (const int32_t*)plan.seg_row, (const int64_t*)plan.seg_beg,
                                           (const int32_t*)plan.seg_len, (const int32_t*)plan.seg_slot, plan.n_seg,
                                           ws_partial, log_s, hub_rows, hint);
        if (e != cudaSuccess) return e;
        if (plan.n_split_rows > 0) {
          int64_t fb = ceil_div(plan.n_split_rows, teams);
          if (fb > cap) fb = cap;
          ++g_launches;
          spmm_fixup_kernel<<<(int)fb, threads, 0, st>>>(a, plan.split_row, plan.split_slot0, plan.split_nslot,
                                                         plan.n_split_rows, teams, ws_partial);
        }
        continue;
      }
    }
    void (*kern)(SpmmArgs, const int32_t*, const int64_t*, const int32_t*, const int32_t*, int64_t, int, float*) =
        a.val ? (masked ? spmm_kernel<true, true> : spmm_kernel<true, false>)
              : (masked ? spmm_kernel<false, true> : spmm_kernel<false, false>);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, (const int32_t*)plan.seg_row, (const int64_t*)plan.seg_beg,
                                       (const int32_t*)plan.seg_len, (const int32_t*)plan.seg_slot, plan.n_seg, teams,
                                       ws_partial);
    if (e != cudaSuccess) return e;
    if (plan.n_split_rows > 0) {
      int64_t fb = ceil_div(plan.n_split_rows, teams);
      if (fb > cap) fb = cap;
      ++g_launches;
      spmm_fixup_kernel<<<(int)fb, threads, 0, st>>>(a, plan.split_row, plan.split_slot0, plan.split_nslot,
                                                     plan.n_split_rows, teams, ws_partial);
    }
  }
  return cudaGetLastError();
}

}  // namespace isvd
