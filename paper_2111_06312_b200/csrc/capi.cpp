// C ABI of the isvd library (include/isvd.h): context, graph, operators,
// matrix-free products and the Alg. 1 solver driver.
//
// Host side only enqueues work: every arithmetic step of the path runs in the
// CUDA kernels of spmm.cu / dense.cu / smallmat.cu / omega.cu.  NCCL (over
// NVLink/NVSwitch) carries the two exchanges of the row-partitioned layout:
// an all-gather of each SpMM gather source and an fp64 all-reduce of the
// Gram / column-sum / X^T Z partials.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: phase ranges for nsys / ncu --nvtx

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/isvd.h"
#include "common.cuh"

using namespace isvd;

// graphs with at least this many rows (single rank) are relabelled by degree
constexpr int64_t kRelabelMinRows = 100000;

namespace isvd {
thread_local int64_t g_launches = 0;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// P logical ranks of the row-partitioned schedule on ONE device (a test backend, SURVEY 8(c)
// "simulation mode"): one context and one host thread per rank.  The collectives keep the real
// partitioned schedule (padded all-gathers, fp64 all-reduces, the sign-rule candidate gather)
// and move the data with one cudaMemcpyAsync per peer slice (all-gather) or one rank-ordered
// sum kernel (all-reduce).  Ordering across the ranks' streams uses events only -- no kernel
// ever waits on another rank's kernel: each collective is two host barriers, a cross-stream
// event wait on every peer's "ready" event, the copies / sum on the rank's own stream, and a
// wait on every peer's "done" event before the rank may overwrite what peers read.
struct isvd_sim_group_s {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void*> ptr;        // per rank: the buffer published for this collective
  std::vector<cudaEvent_t> ready, done;
  std::atomic<int> members{0};
  bool broken = false;  // a rank timed out: every later collective of the group fails
  // false on timeout (ISVD_SIM_TIMEOUT_S, default 120 s): a peer never reached this collective
  bool barrier() {
    static const double timeout_s = getenv("ISVD_SIM_TIMEOUT_S") ? atof(getenv("ISVD_SIM_TIMEOUT_S")) : 120.0;
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return generation != gen || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct isvd_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  bool dist = false;  // row-partitioned schedule on (NCCL id or simulated group given); partition follows `world`
  ncclComm_t comm = nullptr;
  isvd_sim_group_s* sim = nullptr;  // simulated ranks on one device (test backend), else null
  double* sim_tmp = nullptr;        // all-reduce staging of the simulated backend
  size_t sim_tmp_count = 0;
  std::vector<void*> sim_allocs;
  isvd_allocator alloc{};           // caller's device allocator (e.g. PyTorch's caching allocator)
  bool has_alloc = false;
  int num_sms = 148;
  std::string last_error;
  DevStatus* status = nullptr;  // device
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_join = nullptr;
  cudaStream_t work = nullptr;  // private non-blocking stream the solver runs (and is captured) on
  cudaStream_t side = nullptr;  // second private stream: NC dense terms overlapped with the SpMM chain
  cudaStream_t cstream = nullptr;  // collectives stream: all-gathers in flight during the local SpMM pass
  cudaEvent_t ev_fork = nullptr, ev_gath = nullptr;
  bool gather_pending = false;     // an all-gather on cstream the next remote pass must wait for
  std::vector<cudaEvent_t> ov_ev;  // fork/join events of the overlap (reused in order)
  size_t max_persist_l2 = 0;    // cudaDevAttrMaxPersistingL2CacheSize
  std::atomic<int> live_graphs{0};
  // SpMM accounting of the current isvd_svd call
  bool profiling = false;
  int spmm_steps = 0;
  double spmm_alg_bytes = 0.0;
  std::vector<cudaEvent_t> prof_events;  // pairs
  // ISVD_SVD_PROFILE phase brackets: (phase, start event index, end event index) into phase_ev
  std::vector<cudaEvent_t> phase_ev;
  std::vector<int> phase_tag;  // per pair: 0 products, 1 orth, 2 small, 3 comm
  // ISVD_SVD_PROFILE with the distributed split: (start, end) event pairs of every all-gather on the
  // collectives stream and of the local SpMM pass issued while it is in flight (overlap report)
  std::vector<cudaEvent_t> ag_ev, lp_ev;
  size_t n_ag = 0, n_lp = 0;
  // caching device allocator: buffers released by destroyed graphs / ops / workspaces are kept
  // (by exact rounded size) and handed out again, so rebuilding a graph + operator of the same
  // shape pays no cudaMalloc/cudaFree (they cost ~ms per GB-sized buffer); trimmed on OOM and
  // released by isvd_ctx_destroy
  std::mutex pool_mu;
  std::multimap<size_t, void*> pool_free;
  std::unordered_map<void*, size_t> pool_size;
};

struct isvd_graph_s {
  isvd_ctx ctx = nullptr;
  int64_t n = 0, row_begin = 0, n_local = 0, n_pad = 0, nnz = 0, max_deg = 0;
  int64_t* row_ptr = nullptr;  // device, rebased to 0
  int32_t* col_idx = nullptr;  // device
  float* val = nullptr;        // device edge weights (null: unweighted)
  // distributed local / remote split (world > 1): own-row columns and the rest, same row order
  bool split = false;
  int64_t nnz_loc = 0;
  int64_t *rp_loc = nullptr, *rp_rem = nullptr;
  int32_t *ci_loc = nullptr, *ci_rem = nullptr;
  float *val_loc = nullptr, *val_rem = nullptr;
  SpmmPlan plan_loc, plan_rem;
  float* inv_deg = nullptr;    // 1/d (0 for d = 0)
  float* s = nullptr;          // (d+1)^-1/2
  float* s2 = nullptr;         // (d+1)^-1
  float* rs = nullptr;         // (d+1)^1/2
  int32_t* new2old = nullptr;  // relabelled graphs: caller row of internal row i (device); else null
  // SURVEY 8(f) f3 comparison (ISVD_DENSE_A=1, single rank, n <= 32768): A as a dense fp32 n x ld_dense
  // matrix; every SpMM step of this graph then runs as a tcgen05 3xTF32 product A^T Y = A Y (A = A^T)
  float* dense = nullptr;
  int64_t ld_dense = 0;
  uint8_t* dense_u8 = nullptr;  // unweighted: A as bytes for the exact INT8 tensor-core product (dense_i8.cu)
  int64_t ld_u8 = 0;
  SpmmPlan plan;
  std::vector<void*> allocs;
  std::atomic<int> refs{0};
};

// Workspace of one op for one width: grown on demand, never freed until op destroy.
struct Workspace {
  int64_t wpad = 0;
  std::vector<DevBuf> bufs;
};

struct SolverWs {
  int64_t key_l = -1, key_k = -1;
  std::vector<void*> allocs;
  float *Qc = nullptr, *Qc2 = nullptr, *Yr = nullptr, *Yr2 = nullptr, *Rinv32 = nullptr, *Ub = nullptr,
        *Vb = nullptr, *Utmp = nullptr, *Vtmp = nullptr, *sgn = nullptr, *Rfold = nullptr, *Ub2 = nullptr;
  double *gram = nullptr, *Ra = nullptr, *Rb = nullptr, *Rc = nullptr, *Rab = nullptr, *Rfin = nullptr,
         *chol_ws = nullptr, *jac_ws = nullptr, *sigma = nullptr, *cand = nullptr, *cand_all = nullptr,
         *absmax_ws = nullptr;
  cudaGraphExec_t graph_exec = nullptr;  // the captured isvd for the argument set graph_key
  uint64_t graph_key = 0;
  bool graph_broken = false;
  int64_t graph_launches = 0, graph_spmm_steps = 0;
  double graph_alg_bytes = 0.0;
};

struct isvd_op_s {
  isvd_graph g = nullptr;
  isvd_op_kind kind = ISVD_OP_POWER_SUM;
  bool ahat_basis = false;  // NE over A_hat instead of T
  int terms = 0;
  std::vector<double> w;
  double lambda_ones = 0.0;
  double lambda_adj = 0.0;  // NE: coefficient of the +lambda A term (Eq. 3)
  const float* X = nullptr;
  int64_t d = 0, ldx = 0;
  bool own_x = false;
  float* Xrs = nullptr;  // NC: diag(1/s) X = diag((d+1)^1/2) X, the left operand of every X^T Zt_j
                         // (the same fp32 products the kernel would form; refreshed per call if X is borrowed)
  // product workspace (sized for the widest request so far)
  int64_t ws_wpad = 0;
  std::vector<void*> ws_allocs;
  float *full_a = nullptr, *full_b = nullptr, *full_c = nullptr, *ptmp = nullptr, *partial = nullptr;
  float* dense_ws = nullptr;  // f3 dense-A products: fp32 partial tiles of launch_tc_atb
  // the tensor-core probe of the exact first Gram flagged on an earlier call (e.g. config 4, whose
  // square Omega makes kappa(M Omega)^2 > 1e5 every time): later calls go straight to the exact Gram
  bool probe_failed = false;
  void* i8_ws = nullptr;      // f3 exact INT8 dense products: fp64 integer partials + column maxima
  uint8_t* i8_q = nullptr;    // ... and the byte slices of the fixed-point gather source
  double *colsum = nullptr, *colsum_ws = nullptr, *atb_ws = nullptr, *blk64 = nullptr;
  float* bt_ws = nullptr;  // split B operand of the tensor-core GEMM
  float* adjbuf = nullptr;  // NE with lambda_adj != 0: lambda_adj A Q (internal row order)
  float* loc_partial = nullptr;  // distributed split: local-pass row sums (n_local x wpad fp32)
  // NC label re-use: Y_train (internal row order, owned), width, ld, powers
  const float* Ylr = nullptr;
  int64_t ylr = 0, ldylr = 0;
  int lr_powers = 0;
  float* lrbuf = nullptr;  // X G_0 + sum_p B^p Y G'_p (internal row order)
  // implicit row gather (option (ii)): M_S = M[S, :] for sorted global rows S
  bool has_sub = false;
  int64_t sub_n = 0;       // |S| (global)
  int64_t sub_local = 0;   // rows of S in this rank's block
  int64_t sub_offset = 0;  // rows of S on lower ranks (global index of this rank's first subset row)
  int32_t* sub_caller = nullptr;  // device: caller-order local row of subset row i
  int32_t* sub_int = nullptr;     // device: internal (relabelled) local row of subset row i
  std::vector<void*> sub_allocs;
  float* sub_buf = nullptr;  // n_local x wpad: full-row product before the gather / after the scatter
  SolverWs sws;
};

// ------------------------------------------------------------------ helpers
namespace {
int64_t c_rows_local(const isvd_op_s* op);
int64_t r_rows_local(const isvd_op_s* op);

struct Fail {
  isvd_status st;
};

void set_err(isvd_ctx ctx, const std::string& m) {
  if (ctx) ctx->last_error = m;
}

#define CK(call)                                                                                              \
  do {                                                                                                        \
    cudaError_t e_ = (call);                                                                                  \
    if (e_ != cudaSuccess) {                                                                                  \
      set_err(ctx, std::string(#call) + ": " + cudaGetErrorString(e_));                                       \
      throw Fail{e_ == cudaErrorMemoryAllocation ? ISVD_ERR_OOM : ISVD_ERR_CUDA};                             \
    }                                                                                                         \
  } while (0)

#define NK(call)                                                                                              \
  do {                                                                                                        \
    ncclResult_t r_ = (call);                                                                                 \
    if (r_ != ncclSuccess) {                                                                                  \
      set_err(ctx, std::string(#call) + ": " + ncclGetErrorString(r_));                                       \
      throw Fail{ISVD_ERR_NCCL};                                                                              \
    }                                                                                                         \
  } while (0)

#define REQ(cond, code, msg)                                                                                  \
  do {                                                                                                        \
    if (!(cond)) {                                                                                            \
      set_err(ctx, msg);                                                                                      \
      throw Fail{code};                                                                                       \
    }                                                                                                         \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

void pool_trim(isvd_ctx ctx) {
  std::lock_guard<std::mutex> lk(ctx->pool_mu);
  for (auto& kv : ctx->pool_free) {
    ctx->pool_size.erase(kv.second);
    cudaFree(kv.second);
  }
  ctx->pool_free.clear();
}

void* dmalloc(isvd_ctx ctx, size_t bytes, std::vector<void*>& list) {
  void* p = nullptr;
  bytes = (bytes + 511) / 512 * 512;
  if (bytes == 0) bytes = 512;
  if (ctx->has_alloc) {  // the caller's allocator (it caches; the library keeps no pool then)
    p = ctx->alloc.alloc(bytes, ctx->stream, ctx->alloc.user);
    REQ(p != nullptr, ISVD_ERR_OOM, "the caller's allocator returned null");
    REQ(aligned16(p), ISVD_ERR_INVALID_ARG, "the caller's allocator returned a pointer that is not 16-byte aligned");
    list.push_back(p);
    CK(cudaMemsetAsync(p, 0, bytes, ctx->stream));
    return p;
  }
  {
    std::lock_guard<std::mutex> lk(ctx->pool_mu);
    auto it = ctx->pool_free.find(bytes);
    if (it != ctx->pool_free.end()) {
      p = it->second;
      ctx->pool_free.erase(it);
    }
  }
  if (!p) {
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      (void)cudaGetLastError();
      pool_trim(ctx);  // cached blocks of other sizes may be what is missing
      CK(cudaMalloc(&p, bytes));
    }
    std::lock_guard<std::mutex> lk(ctx->pool_mu);
    ctx->pool_size[p] = bytes;
  }
  list.push_back(p);
  // padding columns of every iterate must read as zero: workspaces start cleared (on the ctx
  // stream, so the clearing is ordered before every later use whatever stream kind it is)
  CK(cudaMemsetAsync(p, 0, bytes, ctx->stream));
  return p;
}

// return a dmalloc'd buffer to the context's cache (the device may still be using it: callers
// synchronise the stream before releasing, as they did before cudaFree)
void dfree(isvd_ctx ctx, void* p) {
  if (!p) return;
  if (ctx->has_alloc) {
    ctx->alloc.free(p, ctx->stream, ctx->alloc.user);
    return;
  }
  static const bool no_pool = getenv("ISVD_NO_POOL") && getenv("ISVD_NO_POOL")[0] == '1';
  std::lock_guard<std::mutex> lk(ctx->pool_mu);
  if (no_pool) {
    ctx->pool_size.erase(p);
    cudaFree(p);
    return;
  }
  auto it = ctx->pool_size.find(p);
  if (it == ctx->pool_size.end()) {
    cudaFree(p);
    return;
  }
  ctx->pool_free.insert({it->second, p});
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void partition(int64_t n, int world, int rank, int64_t* rb, int64_t* nl) {
  int64_t chunk = (n + world - 1) / world;
  int64_t b = std::min<int64_t>(n, chunk * rank);
  int64_t e = std::min<int64_t>(n, b + chunk);
  *rb = b;
  *nl = e - b;
}

// ------------------------------------------------------------ phase profiling
// Every phase of the solver is an NVTX range ("isvd:products" / "isvd:orth" / "isvd:small" /
// "isvd:comm"; host-side enqueue ranges, visible to nsys and `ncu --nvtx`).  With
// ISVD_SVD_PROFILE, CUDA events also bracket each phase on the solver's stream
// (isvd_svd_report ms_products / ms_orth / ms_small / ms_comm).
enum PhaseTag { kPhProducts = 0, kPhOrth = 1, kPhSmall = 2, kPhComm = 3 };
struct Phase {
  isvd_ctx ctx;
  size_t i = (size_t)-1;
  Phase(isvd_ctx c, PhaseTag tag) : ctx(c) {
    static const char* names[4] = {"isvd:products", "isvd:orth", "isvd:small", "isvd:comm"};
    nvtxRangePushA(names[tag]);
    if (!ctx->profiling) return;
    i = ctx->phase_tag.size();
    while (ctx->phase_ev.size() < 2 * i + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) { i = (size_t)-1; return; }
      ctx->phase_ev.push_back(e);
    }
    ctx->phase_tag.push_back((int)tag);
    cudaEventRecord(ctx->phase_ev[2 * i], ctx->stream);
  }
  ~Phase() {
    if (i != (size_t)-1) cudaEventRecord(ctx->phase_ev[2 * i + 1], ctx->stream);
    nvtxRangePop();
  }
};

// Next (start, end) event pair of a profiling list (created on demand); nullptr if unavailable.
cudaEvent_t* prof_pair(std::vector<cudaEvent_t>& v, size_t& n) {
  while (v.size() < 2 * n + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    v.push_back(e);
  }
  return &v[2 * n++];
}

// --------------------------------------------------------------- collectives
// In-place all-gather: rank p's `bytes_per_rank` bytes sit at recv + p * bytes_per_rank.
void coll_allgather(isvd_ctx ctx, void* recv, size_t bytes_per_rank) {
  if (!ctx->dist || bytes_per_rank == 0) return;
  Phase ph(ctx, kPhComm);
  char* r = static_cast<char*>(recv);
  if (ctx->comm) {
    NK(ncclAllGather(r + (size_t)ctx->rank * bytes_per_rank, r, bytes_per_rank, ncclChar, ctx->comm, ctx->stream));
    return;
  }
  isvd_sim_group_s* g = ctx->sim;
  const int me = ctx->rank;
  g->ptr[me] = recv;
  CK(cudaEventRecord(g->ready[me], ctx->stream));
  REQ(g->barrier(), ISVD_ERR_BUSY, "simulated ranks: a peer did not reach the collective (timeout)");
  for (int q = 0; q < g->world; ++q) {
    if (q == me) continue;
    CK(cudaStreamWaitEvent(ctx->stream, g->ready[q], 0));
    const char* src = static_cast<const char*>(g->ptr[q]) + (size_t)q * bytes_per_rank;
    CK(cudaMemcpyAsync(r + (size_t)q * bytes_per_rank, src, bytes_per_rank, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CK(cudaEventRecord(g->done[me], ctx->stream));
  REQ(g->barrier(), ISVD_ERR_BUSY, "simulated ranks: a peer did not reach the collective (timeout)");
  for (int q = 0; q < g->world; ++q)
    if (q != me) CK(cudaStreamWaitEvent(ctx->stream, g->done[q], 0));  // peers finished reading my buffer
}

// The stream the next consumer of an in-flight all-gather must wait on it (remote SpMM pass,
// end of every product).
void join_gather(isvd_ctx ctx) {
  if (!ctx->gather_pending) return;
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_gath, 0));
  ctx->gather_pending = false;
}

// All-gather of a full-height SpMM gather source (every rank's slice).  With the local / remote
// split it runs on the collectives stream: the next SpMM step's local pass (own rows only) runs
// meanwhile and its remote pass waits (join_gather).
void allgather_rows(isvd_ctx ctx, const isvd_graph_s* g, float* full, int64_t ld) {
  const size_t bytes = sizeof(float) * (size_t)g->n_pad * ld;
  if (!ctx->dist) return;
  if (!g->split) {
    coll_allgather(ctx, full, bytes);
    return;
  }
  join_gather(ctx);  // one all-gather in flight at a time
  CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_fork, 0));
  cudaStream_t main = ctx->stream;
  ctx->stream = ctx->cstream;
  cudaEvent_t* agp = ctx->profiling ? prof_pair(ctx->ag_ev, ctx->n_ag) : nullptr;
  if (agp) CK(cudaEventRecord(agp[0], ctx->cstream));
  try {
    coll_allgather(ctx, full, bytes);
  } catch (...) {
    ctx->stream = main;
    throw;
  }
  ctx->stream = main;
  if (agp) CK(cudaEventRecord(agp[1], ctx->cstream));
  CK(cudaEventRecord(ctx->ev_gath, ctx->cstream));
  ctx->gather_pending = true;
}

void allreduce_f64(isvd_ctx ctx, double* buf, size_t count) {
  if (!ctx->dist || count == 0) return;
  Phase ph(ctx, kPhComm);
  if (ctx->comm) {
    NK(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return;
  }
  isvd_sim_group_s* g = ctx->sim;
  const int me = ctx->rank;
  if (count > ctx->sim_tmp_count) {
    CK(cudaStreamSynchronize(ctx->stream));
    for (void* p : ctx->sim_allocs) dfree(ctx, p);
    ctx->sim_allocs.clear();
    ctx->sim_tmp = (double*)dmalloc(ctx, sizeof(double) * count, ctx->sim_allocs);
    ctx->sim_tmp_count = count;
  }
  g->ptr[me] = buf;
  CK(cudaEventRecord(g->ready[me], ctx->stream));
  REQ(g->barrier(), ISVD_ERR_BUSY, "simulated ranks: a peer did not reach the collective (timeout)");
  RankPtrs rp{};
  for (int q = 0; q < g->world; ++q) {
    rp.p[q] = static_cast<const double*>(g->ptr[q]);
    if (q != me) CK(cudaStreamWaitEvent(ctx->stream, g->ready[q], 0));
  }
  CK(launch_sum_ranks(rp, g->world, (int64_t)count, ctx->sim_tmp, ctx->stream));
  CK(cudaEventRecord(g->done[me], ctx->stream));
  REQ(g->barrier(), ISVD_ERR_BUSY, "simulated ranks: a peer did not reach the collective (timeout)");
  for (int q = 0; q < g->world; ++q)
    if (q != me) CK(cudaStreamWaitEvent(ctx->stream, g->done[q], 0));
  CK(cudaMemcpyAsync(buf, ctx->sim_tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
}

// recv (world x count doubles) <- every rank's send (count doubles), in rank order
void allgather_f64(isvd_ctx ctx, const double* send, double* recv, size_t count) {
  CK(cudaMemcpyAsync(recv + (size_t)ctx->rank * count, send, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  coll_allgather(ctx, recv, sizeof(double) * count);
}

// ------------------------------------------------------------------ op workspace
void ensure_op_ws(isvd_op op, int64_t wpad) {
  isvd_graph g = op->g;
  isvd_ctx ctx = g->ctx;
  if (wpad <= op->ws_wpad) return;
  CK(cudaStreamSynchronize(ctx->stream));
  for (void* p : op->ws_allocs) dfree(ctx, p);
  op->ws_allocs.clear();
  if (op->sws.graph_exec) {  // the captured solver referenced the freed buffers
    cudaGraphExecDestroy(op->sws.graph_exec);
    op->sws.graph_exec = nullptr;
  }
  int64_t n_full = g->n_pad * ctx->world;
  size_t full_bytes = sizeof(float) * (size_t)n_full * wpad;
  op->full_a = (float*)dmalloc(ctx, full_bytes, op->ws_allocs);
  op->full_b = (float*)dmalloc(ctx, full_bytes, op->ws_allocs);
  op->full_c = (float*)dmalloc(ctx, full_bytes, op->ws_allocs);
  // NC: one X G_j buffer per Horner term, so all L GEMMs can run ahead of the SpMM chain
  const int64_t nptmp = op->kind == ISVD_OP_STACKED_PROPAGATION ? std::max(op->terms, 1) : 1;
  op->ptmp = (float*)dmalloc(ctx, sizeof(float) * (size_t)nptmp * std::max<int64_t>(g->n_local, 1) * wpad,
                             op->ws_allocs);
  op->partial = (float*)dmalloc(
      ctx, sizeof(float) * (size_t)std::max({spmm_ws_floats(g->plan, wpad), spmm_ws_floats(g->plan_loc, wpad),
                                             spmm_ws_floats(g->plan_rem, wpad)}),
      op->ws_allocs);
  op->loc_partial = g->split ? (float*)dmalloc(ctx, sizeof(float) * (size_t)std::max<int64_t>(g->n_local, 1) * wpad,
                                               op->ws_allocs)
                             : nullptr;
  op->colsum = (double*)dmalloc(ctx, sizeof(double) * wpad, op->ws_allocs);
  op->colsum_ws = (double*)dmalloc(ctx, sizeof(double) * colsum_ws_doubles(g->n_local, wpad), op->ws_allocs);
  // Workspaces are sized for every width w <= wpad a later call may use (the tilings pick more
  // row parts for narrower products, so a narrower call can need more partial tiles than wpad)
  int64_t ka_nc = op->kind == ISVD_OP_STACKED_PROPAGATION ? op->d : 0;
  int64_t atb = 0, dense_f = 0, i8_b = 0, i8_q = 0;
  for (int64_t w = 4; w <= wpad; w += 4) {
    const int64_t ka = ka_nc ? ka_nc : w;
    atb = std::max({atb, atb_ws_doubles(g->n_local, ka, w, ctx->num_sms), atb_ws_doubles(g->n_local, w, w, ctx->num_sms),
                    (tc_atb_ws_floats(g->n_local, ka, w, false, ctx->num_sms) + 1) / 2,
                    (tc_atb_ws_floats(g->n_local, w, w, true, ctx->num_sms) + 1) / 2});
    if (op->lr_powers > 0)
      atb = std::max({atb, atb_ws_doubles(g->n_local, op->ylr, w, ctx->num_sms),
                      (tc_atb_ws_floats(g->n_local, op->ylr, w, false, ctx->num_sms) + 1) / 2});
    if (g->dense) dense_f = std::max(dense_f, tc_atb_ws_floats(g->n, g->n, w, false, ctx->num_sms));
    if (g->dense_u8) {
      int64_t qb = 0;
      i8_b = std::max(i8_b, dense_i8_ws_bytes(g->n, w, ctx->num_sms, &qb));
      i8_q = std::max(i8_q, qb);
    }
  }
  op->atb_ws = (double*)dmalloc(ctx, sizeof(double) * std::max<int64_t>(atb, 1), op->ws_allocs);
  op->dense_ws = g->dense ? (float*)dmalloc(ctx, sizeof(float) * (size_t)dense_f, op->ws_allocs) : nullptr;
  if (g->dense_u8) {
    op->i8_ws = dmalloc(ctx, (size_t)i8_b, op->ws_allocs);
    op->i8_q = (uint8_t*)dmalloc(ctx, (size_t)i8_q, op->ws_allocs);
  }
  op->bt_ws = (float*)dmalloc(ctx, sizeof(float) * tc_gemm_ws_floats(wpad, std::max<int64_t>(wpad, op->d)),
                              op->ws_allocs);
  op->adjbuf = op->lambda_adj != 0.0
                   ? (float*)dmalloc(ctx, sizeof(float) * (size_t)std::max<int64_t>(g->n_local, 1) * wpad, op->ws_allocs)
                   : nullptr;
  int64_t c = op->kind == ISVD_OP_STACKED_PROPAGATION ? c_rows_local(op) : 1;
  op->blk64 = (double*)dmalloc(ctx, sizeof(double) * c * wpad, op->ws_allocs);
  op->lrbuf = op->lr_powers > 0
                  ? (float*)dmalloc(ctx, sizeof(float) * (size_t)std::max<int64_t>(g->n_local, 1) * wpad, op->ws_allocs)
                  : nullptr;
  op->sub_buf = op->has_sub
                    ? (float*)dmalloc(ctx, sizeof(float) * (size_t)std::max<int64_t>(g->n_local, 1) * wpad, op->ws_allocs)
                    : nullptr;
  op->ws_wpad = wpad;
}

// north_star: "Tensor cores are used only in the Gram contraction, and only if 3xTF32 meets the
// tolerance."  By default the tcgen05 3xTF32 kernels therefore serve only the CholeskyQR Grams
// Y^T Y (ISVD_TC_GRAM=0 turns that off too).  ISVD_TC_PRODUCTS=1 additionally routes the other
// tall contractions -- the NC blocks X^T Z_j, the leaf GEMMs X G_j, the update Y R^-1 and the
// final U, V -- through the same 3xTF32 kernels (a measured alternative).
bool env_flag(const char* name, bool dflt) {
  const char* v = getenv(name);
  return v ? v[0] == '1' : dflt;
}
// read at every call (cheap) so a process can switch modes; the captured solver graph is keyed
// on them (graph_key)
bool tc_for_grams() { return env_flag("ISVD_TC_GRAM", true); }
bool tc_for_products() { return env_flag("ISVD_TC_PRODUCTS", false); }

bool use_tensor_cores(int64_t rows, int64_t Ka, int64_t Kb, int64_t lda, int64_t ldb, bool gram) {
  if (!(gram ? tc_for_grams() : tc_for_products())) return false;
  return tc_atb_supported(rows, Ka, Kb, lda, ldb);
}

// G (fp64, ldg) = (diag(row_scale) A)^T B over this rank's rows, fp32-class numerics: tcgen05
// 3xTF32 over 128-row TMEM chunks when supported, else SIMT fp32 over <= 1024-row chunks; fp64
// across chunks/parts in a fixed order either way.
void atb_fp32(isvd_op op, int64_t rows, const float* A, int64_t lda, int64_t Ka, const float* row_scale,
              const float* B, int64_t ldb, int64_t Kb, bool symmetric, double* G, int64_t ldg, const int* gate) {
  isvd_ctx ctx = op->g->ctx;
  if (use_tensor_cores(rows, Ka, Kb, lda, ldb, symmetric && A == B)) {
    int64_t ws_lda = 0, ws_ld = 0, parts = 0, diag0 = -1;
    float* ws32 = reinterpret_cast<float*>(op->atb_ws);
    CK(launch_tc_atb(A, lda, Ka, row_scale, B, ldb, Kb, rows, symmetric, ws32, &ws_lda, &ws_ld, &parts,
                     ctx->num_sms, gate, ctx->stream, symmetric ? &diag0 : nullptr));
    CK(launch_atb_f32_reduce(ws32, ws_lda, ws_ld, parts, Ka, Kb, symmetric, G, ldg, nullptr, 0, ctx->num_sms, gate,
                             ctx->stream));
    if (diag0 >= 0)  // the few trailing rows' diagonal block, SIMT fp32-chunk class (overwrites it)
      CK(launch_atb(A + diag0, lda, B + diag0, ldb, rows, Ka - diag0, Kb - diag0, row_scale, true, op->atb_ws,
                    G + diag0 * ldg + diag0, ldg, nullptr, 0, ctx->num_sms, gate, ctx->stream, true));
    return;
  }
  CK(launch_atb(A, lda, B, ldb, rows, Ka, Kb, row_scale, symmetric, op->atb_ws, G, ldg, nullptr, 0, ctx->num_sms,
                gate, ctx->stream, true));
}

// C[map(i), j] = alpha row_scale(i) (A B)[i, j], i < rows, j < N: the SIMT fp32 kernel (dense.cu),
// or with ISVD_TC_PRODUCTS=1 the tcgen05 3xTF32 tall GEMM (gemm_tc.cu).
void gemm_fp32(isvd_op op, const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
               int64_t rows, int64_t N, int64_t K, const float* row_scale, bool upper_tri_b, const int* gate,
               const int32_t* out_map = nullptr) {
  isvd_ctx ctx = op->g->ctx;
  const bool tc = tc_for_products() && tc_gemm_supported(rows, N, K, lda, ldc) &&
                  tc_gemm_ws_floats(N, K) <= tc_gemm_ws_floats(op->ws_wpad, std::max<int64_t>(op->ws_wpad, op->d));
  if (tc)
    CK(launch_tc_gemm(A, lda, B, ldb, C, ldc, rows, N, K, row_scale, 1.f, gate, ctx->stream, out_map, op->bt_ws,
                      ctx->num_sms));
  else
    CK(launch_gemm_tn(A, lda, B, ldb, C, ldc, rows, N, K, row_scale, 1.f, upper_tri_b, gate, ctx->stream, out_map));
}

SpmmArgs spmm_base(const isvd_graph_s* g, int64_t wpad) {
  SpmmArgs a{};
  a.col_idx = g->col_idx;
  a.val = g->val;
  a.row_offset = g->row_begin;
  a.post_coef = 1.f;
  a.term_coef = 1.f;
  a.wpad = wpad;
  a.n_src = g->n_pad * g->ctx->world;  // full-height gather sources (the caller's Q for n_local-row sources)
  return a;
}

void spmm(isvd_ctx ctx, isvd_op op, const SpmmArgs& a) {
  const isvd_graph_s* g = op->g;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    size_t i = 2 * (size_t)ctx->spmm_steps;
    while (ctx->prof_events.size() < i + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ctx->prof_events.push_back(e);
    }
    e0 = ctx->prof_events[i];
    e1 = ctx->prof_events[i + 1];
    CK(cudaEventRecord(e0, ctx->stream));
  }
  // relabelled graphs: the leading (hub) rows of the gather source stay L2-persisting
  size_t persist = 0;
  if (g->new2old) persist = std::min(ctx->max_persist_l2, (size_t)(g->n_pad * ctx->world) * a.wpad * sizeof(float));
  const char* persist_env = getenv("ISVD_L2_PERSIST_MB");  // tuning override (MB; 0 = off), read per call
  if (persist_env && g->new2old) persist = std::min(persist, (size_t)atoll(persist_env) << 20);
  static const char* cols_env = getenv("ISVD_SPMM_COLS");  // tuning override: column block width
  const int64_t col_block = cols_env ? atoll(cols_env) : 0;
  if (g->split && ctx->dist) {
    // local pass (columns of this rank's own rows: available before the all-gather completes)
    // -> raw fp32 row sums; remote pass after the all-gather, adding them in its epilogue
    SpmmArgs lo = a;
    lo.col_idx = g->ci_loc; lo.val = g->val_loc;
    lo.self_coef = 0.f; lo.post_vec = nullptr; lo.post_coef = 1.f; lo.T = nullptr; lo.term_vec = nullptr;
    lo.colsum = nullptr; lo.out = op->loc_partial; lo.ldo = a.wpad; lo.out_map = nullptr; lo.pre = nullptr;
    cudaEvent_t* lpp = (ctx->profiling && ctx->gather_pending) ? prof_pair(ctx->lp_ev, ctx->n_lp) : nullptr;
    if (lpp) CK(cudaEventRecord(lpp[0], ctx->stream));
    CK(launch_spmm(g->plan_loc, lo, op->partial, ctx->num_sms, ctx->stream, 0, col_block));
    if (lpp) CK(cudaEventRecord(lpp[1], ctx->stream));
    join_gather(ctx);
    SpmmArgs re = a;
    re.col_idx = g->ci_rem; re.val = g->val_rem;
    re.pre = op->loc_partial; re.ldpre = a.wpad;
    CK(launch_spmm(g->plan_rem, re, op->partial, ctx->num_sms, ctx->stream, 0, col_block));
  } else if (g->dense_u8 && !a.pre) {
    // f3 comparison, exact: A Y on the INT8 tensor cores over the fixed-point slices of Y
    int64_t parts = 0, ws_rows = 0, ws_ld = 0;
    const unsigned* cmax = nullptr;
    const double* pws = nullptr;
    CK(launch_dense_i8(g->dense_u8, g->ld_u8, g->n, a.Y, a.ldy, a.wpad, op->i8_q, op->i8_ws, ctx->num_sms,
                       ctx->stream, &parts, &ws_rows, &ws_ld, &cmax, &pws));
    CK(launch_spmm_dense64_epilogue(pws, parts, ws_rows, ws_ld, cmax, a, g->n_local, ctx->num_sms, ctx->stream));
  } else if (g->dense && !a.pre) {
    // f3 comparison: acc = A Y as a tensor-core product over the dense adjacency (A symmetric, so
    // A Y = A^T Y: the Gram kernel's row-contraction form), then the same epilogue
    int64_t ws_lda = 0, ws_ld = 0, parts = 0;
    CK(launch_tc_atb(g->dense, g->ld_dense, g->n, nullptr, a.Y, a.ldy, a.wpad, g->n, false, op->dense_ws, &ws_lda,
                     &ws_ld, &parts, ctx->num_sms, nullptr, ctx->stream));
    CK(launch_spmm_dense_epilogue(op->dense_ws, parts, ws_lda, ws_ld, a, g->n_local, ctx->num_sms, ctx->stream));
  } else {
    join_gather(ctx);
    CK(launch_spmm(g->plan, a, op->partial, ctx->num_sms, ctx->stream, persist, col_block));
  }
  if (e1) CK(cudaEventRecord(e1, ctx->stream));
  // algorithmic bytes of the step: CSR, scale vectors, the gather source read
  // once (all n rows), the epilogue operand T, the output
  double nl = (double)g->n_local, w = (double)a.wpad;
  double b = 8.0 * (nl + 1) + 4.0 * (double)g->nnz + 4.0 * (double)g->n * w + 4.0 * nl * w;
  if (a.val) b += 4.0 * (double)g->nnz;  // edge weights
  if (a.post_vec) b += 4.0 * nl;
  if (a.term_vec) b += 4.0 * nl;
  if (a.T) b += 4.0 * nl * w;
  ctx->spmm_alg_bytes += b;
  ctx->spmm_steps++;
}

// rows [row_begin, row_begin + n_local) of a full-height buffer
float* slice(const isvd_graph_s* g, float* full, int64_t ld) { return full + (size_t)g->row_begin * ld; }

// ----------------------------------------------------------------- NE products
// M Q = sum_c w_c T^c Q - lambda 1 (1^T Q), T = D^-1 A   (Eq. 3)
// Horner: H_C = w_C Q; H_c = w_c Q + D^-1 A H_{c+1}; M Q = D^-1 A H_1 - lambda 1 cs^T.
// user_order: Q and out are in the caller's row order (relabelled graphs map at the boundary).
// The +lambda_adj A Q term of Eq. 3's -lambda (1 1^T - A): one extra SpMM step over
// the full rows of Q into adjbuf (internal row order), added by the last Horner step's epilogue
// (SURVEY 8(f) f1).  A is symmetric, so M^T takes the same term.
void ne_adj_term(isvd_ctx ctx, isvd_op op, const float* qfull, int64_t ldq, int64_t wpad) {
  isvd_graph g = op->g;
  SpmmArgs a = spmm_base(g, wpad);
  a.Y = qfull; a.ldy = ldq;
  a.post_coef = (float)op->lambda_adj;
  a.out = op->adjbuf; a.ldo = wpad;
  spmm(ctx, op, a);
}

void ne_matmul(isvd_ctx ctx, isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad,
               bool user_order) {
  isvd_graph g = op->g;
  const int C = op->terms;
  const int32_t* omap = nullptr;
  CK(launch_colsum(Q, g->n_local, wpad, ldq, op->colsum_ws, op->colsum, ctx->stream));  // order-free
  allreduce_f64(ctx, op->colsum, wpad);
  if (user_order && g->new2old) {
    CK(launch_scale_rows(Q, ldq, op->ptmp, wpad, g->n_local, wpad, nullptr, 1.f, nullptr, ctx->stream, g->new2old));
    Q = op->ptmp;
    ldq = wpad;
    omap = g->new2old;
  }
  const float* src = Q;
  int64_t lds = ldq;
  if (ctx->dist) {
    CK(launch_scale_rows(Q, ldq, slice(g, op->full_a, wpad), wpad, g->n_local, wpad, nullptr, 1.f, nullptr,
                         ctx->stream));
    allgather_rows(ctx, g, op->full_a, wpad);
    src = op->full_a;
    lds = wpad;
  }
  if (op->adjbuf) ne_adj_term(ctx, op, src, lds, wpad);  // adjbuf = lambda_adj A Q
  float* bufs[2] = {op->full_b, op->full_c};
  for (int c = C - 1; c >= 1; --c) {
    float* dst_full = bufs[c & 1];
    SpmmArgs a = spmm_base(g, wpad);
    a.Y = src; a.ldy = lds;
    a.post_vec = g->inv_deg;
    a.post_coef = (c == C - 1) ? (float)op->w[C - 1] : 1.f;
    a.T = Q; a.ldt = ldq; a.term_coef = (float)op->w[c - 1];
    a.out = slice(g, dst_full, wpad); a.ldo = wpad;
    spmm(ctx, op, a);
    allgather_rows(ctx, g, dst_full, wpad);
    src = dst_full;
    lds = wpad;
  }
  SpmmArgs a = spmm_base(g, wpad);
  a.Y = src; a.ldy = lds;
  a.post_vec = g->inv_deg;
  a.post_coef = (C == 1) ? (float)op->w[0] : 1.f;
  a.colsum = op->colsum; a.rank1_coef = op->lambda_ones;
  if (op->adjbuf) { a.T = op->adjbuf; a.ldt = wpad; }
  a.out = out; a.ldo = ldo; a.out_map = omap;
  spmm(ctx, op, a);
}

// M^T Q = sum_c w_c (A D^-1)^c Q - lambda 1 (1^T Q)   (T^T = A D^-1 for symmetric A)
// Horner: Ht_C = D^-1 w_C Q; Ht_c = D^-1 (w_c Q + A Ht_{c+1}); M^T Q = A Ht_1 - lambda 1 cs^T.
void ne_matmul_T(isvd_ctx ctx, isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad,
                 bool user_order) {
  isvd_graph g = op->g;
  const int C = op->terms;
  const int32_t* omap = nullptr;
  CK(launch_colsum(Q, g->n_local, wpad, ldq, op->colsum_ws, op->colsum, ctx->stream));
  allreduce_f64(ctx, op->colsum, wpad);
  if (user_order && g->new2old) {
    CK(launch_scale_rows(Q, ldq, op->ptmp, wpad, g->n_local, wpad, nullptr, 1.f, nullptr, ctx->stream, g->new2old));
    Q = op->ptmp;
    ldq = wpad;
    omap = g->new2old;
  }
  if (op->adjbuf) {  // A^T = A (symmetric): the same lambda_adj A Q, gathered from Q's full rows
    const float* qf = Q;
    int64_t ldqf = ldq;
    if (ctx->dist) {
      CK(launch_scale_rows(Q, ldq, slice(g, op->full_b, wpad), wpad, g->n_local, wpad, nullptr, 1.f, nullptr,
                           ctx->stream));
      allgather_rows(ctx, g, op->full_b, wpad);
      qf = op->full_b;
      ldqf = wpad;
    }
    ne_adj_term(ctx, op, qf, ldqf, wpad);
  }
  CK(launch_scale_rows(Q, ldq, slice(g, op->full_a, wpad), wpad, g->n_local, wpad, g->inv_deg, (float)op->w[C - 1],
                       nullptr, ctx->stream));
  allgather_rows(ctx, g, op->full_a, wpad);
  const float* src = op->full_a;
  float* bufs[2] = {op->full_b, op->full_c};
  for (int c = C - 1; c >= 1; --c) {
    float* dst_full = bufs[c & 1];
    SpmmArgs a = spmm_base(g, wpad);
    a.Y = src; a.ldy = wpad;
    a.post_vec = g->inv_deg;
    a.T = Q; a.ldt = ldq; a.term_vec = g->inv_deg; a.term_coef = (float)op->w[c - 1];
    a.out = slice(g, dst_full, wpad); a.ldo = wpad;
    spmm(ctx, op, a);
    allgather_rows(ctx, g, dst_full, wpad);
    src = dst_full;
  }
  SpmmArgs a = spmm_base(g, wpad);
  a.Y = src; a.ldy = wpad;
  a.colsum = op->colsum; a.rank1_coef = op->lambda_ones;
  if (op->adjbuf) { a.T = op->adjbuf; a.ldt = wpad; }
  a.out = out; a.ldo = ldo; a.out_map = omap;
  spmm(ctx, op, a);
}

// NE over the symmetric basis A_hat ("replace T by A_hat, recovering a basis where L = R"):
// M = sum_c w_c A_hat^c - lambda_ones 1 1^T + lambda_adj A is symmetric, so M^T Q = M Q.
// Horner on pre-scaled iterates Ht = s H (A_hat H = s (A+I) Ht, as for NC):
//   Ht_C = s w_C Q;  Ht_c = w_c s Q + s^2 ((A+I) Ht_{c+1});  M Q = s ((A+I) Ht_1) - lambda 1 cs^T (+ lambda_adj A Q).
void ne_ahat_matmul(isvd_ctx ctx, isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad,
                    bool user_order) {
  isvd_graph g = op->g;
  const int C = op->terms;
  const int32_t* omap = nullptr;
  CK(launch_colsum(Q, g->n_local, wpad, ldq, op->colsum_ws, op->colsum, ctx->stream));
  allreduce_f64(ctx, op->colsum, wpad);
  if (user_order && g->new2old) {
    CK(launch_scale_rows(Q, ldq, op->ptmp, wpad, g->n_local, wpad, nullptr, 1.f, nullptr, ctx->stream, g->new2old));
    Q = op->ptmp;
    ldq = wpad;
    omap = g->new2old;
  }
  if (op->adjbuf) {  // lambda_adj A Q from Q's full rows (A symmetric)
    const float* qf = Q;
    int64_t ldqf = ldq;
    if (ctx->dist) {
      CK(launch_scale_rows(Q, ldq, slice(g, op->full_b, wpad), wpad, g->n_local, wpad, nullptr, 1.f, nullptr,
                           ctx->stream));
      allgather_rows(ctx, g, op->full_b, wpad);
      qf = op->full_b;
      ldqf = wpad;
    }
    ne_adj_term(ctx, op, qf, ldqf, wpad);
  }
  CK(launch_scale_rows(Q, ldq, slice(g, op->full_a, wpad), wpad, g->n_local, wpad, g->s, (float)op->w[C - 1], nullptr,
                       ctx->stream));
  allgather_rows(ctx, g, op->full_a, wpad);
  const float* src = op->full_a;
  float* bufs[2] = {op->full_b, op->full_c};
  for (int c = C - 1; c >= 1; --c) {
    float* dst_full = bufs[c & 1];
    SpmmArgs a = spmm_base(g, wpad);
    a.Y = src; a.ldy = wpad; a.self_coef = 1.f;
    a.post_vec = g->s2;
    a.T = Q; a.ldt = ldq; a.term_vec = g->s; a.term_coef = (float)op->w[c - 1];
    a.out = slice(g, dst_full, wpad); a.ldo = wpad;
    spmm(ctx, op, a);
    allgather_rows(ctx, g, dst_full, wpad);
    src = dst_full;
  }
  SpmmArgs a = spmm_base(g, wpad);
  a.Y = src; a.ldy = wpad; a.self_coef = 1.f;
  a.post_vec = g->s;
  a.colsum = op->colsum; a.rank1_coef = op->lambda_ones;
  if (op->adjbuf) { a.T = op->adjbuf; a.ldt = wpad; }
  a.out = out; a.ldo = ldo; a.out_map = omap;
  spmm(ctx, op, a);
}

// ---- overlap of the NC dense terms with the SpMM chain (single rank; opt-in) --------------
// The X G_j GEMMs of M G and the X^T Zt_j contractions of M^T Q are FP32-FMA-bound, the SpMM
// steps DRAM-bound; they are independent enough to run concurrently: the dense terms go to the
// context's second stream, joined by events (also inside a captured CUDA graph).  Measured at
// config 4: the isvd gains ~1 % (0.835 vs 0.846 s, within run-to-run noise) while each SpMM step
// stretches from 26.4 to 32.5 ms (shared SMs / DRAM, lower clocks under the power cap), so it is
// off by default (ISVD_OVERLAP=1 turns it on).
bool nc_overlap(isvd_ctx ctx, isvd_op op) {
  if (op->kind != ISVD_OP_STACKED_PROPAGATION || ctx->dist || !ctx->side || op->terms < 1 || op->lr_powers > 0)
    return false;
  const char* v = getenv("ISVD_OVERLAP");
  return v && v[0] == '1';
}
struct OnStream {  // route ctx->stream (used by every launcher wrapper) to another stream
  isvd_ctx c;
  cudaStream_t prev;
  OnStream(isvd_ctx c_, cudaStream_t st) : c(c_), prev(c_->stream) { c->stream = st; }
  ~OnStream() { c->stream = prev; }
};
void ev_record(isvd_ctx ctx, int i, cudaStream_t st) { CK(cudaEventRecord(ctx->ov_ev[i % ctx->ov_ev.size()], st)); }
void ev_wait(isvd_ctx ctx, int i, cudaStream_t st) { CK(cudaStreamWaitEvent(st, ctx->ov_ev[i % ctx->ov_ev.size()], 0)); }

// ----------------------------------------------------------------- NC products
// M G = sum_j A_hat^j X G_j  (Eq. 6), Horner from the deepest block, iterates stored
// pre-scaled (Yt = s Y) so the gather needs no per-neighbour scale:
//   Yt_L = s (X G_L);  Yt_j = s (X G_j) + s^2 ((A+I) Yt_{j+1});  out = X G_0 + s ((A+I) Yt_1).
// G (c rows) is never permuted; out rows are in the caller's order when user_order.
void nc_matmul(isvd_ctx ctx, isvd_op op, const float* G, int64_t ldgm, float* out, int64_t ldo, int64_t wpad,
               bool user_order) {
  isvd_graph g = op->g;
  const int L = op->terms;
  const int64_t d = op->d;
  const int32_t* omap = (user_order && g->new2old) ? g->new2old : nullptr;
  if (op->lr_powers > 0) {
    // label re-use blocks first: lrbuf = X G_0 + sum_p B^p (Y G'_p), Horner over p on
    // pre-scaled iterates, B Wt = s (A Wt) (no self term); L = 0: the sum goes straight to out
    const int P = op->lr_powers;
    const int64_t off = d * (L + 1), yw = op->ylr;
    auto gp = [&](int p) { return G + (size_t)(off + (int64_t)(p - 1) * yw) * ldgm; };
    float* wb[2] = {op->full_c, op->full_a};
    float* wt = wb[P & 1];
    gemm_fp32(op, op->Ylr, op->ldylr, gp(P), ldgm, slice(g, wt, wpad), wpad, g->n_local, wpad, yw, g->s, false,
              nullptr);
    allgather_rows(ctx, g, wt, wpad);
    for (int p = P - 1; p >= 1; --p) {
      gemm_fp32(op, op->Ylr, op->ldylr, gp(p), ldgm, op->ptmp, wpad, g->n_local, wpad, yw, nullptr, false, nullptr);
      float* dst = wb[p & 1];
      SpmmArgs a = spmm_base(g, wpad);
      a.Y = wt; a.ldy = wpad;
      a.post_vec = g->s2;
      a.T = op->ptmp; a.ldt = wpad; a.term_vec = g->s;
      a.out = slice(g, dst, wpad); a.ldo = wpad;
      spmm(ctx, op, a);
      allgather_rows(ctx, g, dst, wpad);
      wt = dst;
    }
    gemm_fp32(op, op->X, op->ldx, G, ldgm, op->ptmp, wpad, g->n_local, wpad, d, nullptr, false, nullptr);
    SpmmArgs a = spmm_base(g, wpad);
    a.Y = wt; a.ldy = wpad;
    a.post_vec = g->s;
    a.T = op->ptmp; a.ldt = wpad;
    if (L == 0) {
      a.out = out; a.ldo = ldo; a.out_map = omap;
      spmm(ctx, op, a);
      return;
    }
    a.out = op->lrbuf; a.ldo = wpad;
    spmm(ctx, op, a);
  }
  if (L == 0) {
    gemm_fp32(op, op->X, op->ldx, G, ldgm, out, ldo, g->n_local, wpad, d, nullptr, false, nullptr, omap);
    return;
  }
  float* bufs[2] = {op->full_a, op->full_b};
  float* cur = bufs[L & 1];
  if (nc_overlap(ctx, op)) {
    // side stream: all L+1 GEMMs in order (event L..0 after each); main: the SpMM chain, each
    // step waiting only for the GEMM it adds.  X G_j -> ptmp slot j (j < L).
    const cudaStream_t main = ctx->stream;
    auto tj = [&](int j) { return op->ptmp + (size_t)j * std::max<int64_t>(g->n_local, 1) * wpad; };
    ev_record(ctx, 15, main);
    CK(cudaStreamWaitEvent(ctx->side, ctx->ov_ev[15], 0));
    {
      OnStream on(ctx, ctx->side);
      gemm_fp32(op, op->X, op->ldx, G + (size_t)L * d * ldgm, ldgm, slice(g, cur, wpad), wpad, g->n_local, wpad, d,
                g->s, false, nullptr);
      ev_record(ctx, L, ctx->side);
      for (int j = L - 1; j >= 0; --j) {
        gemm_fp32(op, op->X, op->ldx, G + (size_t)j * d * ldgm, ldgm, tj(j), wpad, g->n_local, wpad, d, nullptr,
                  false, nullptr);
        ev_record(ctx, j, ctx->side);
      }
    }
    ev_wait(ctx, L, main);
    for (int j = L - 1; j >= 0; --j) {
      ev_wait(ctx, j, main);
      SpmmArgs a = spmm_base(g, wpad);
      a.Y = cur; a.ldy = wpad; a.self_coef = 1.f;
      a.T = tj(j); a.ldt = wpad;
      if (j >= 1) {
        float* dst = bufs[j & 1];
        a.post_vec = g->s2;
        a.term_vec = g->s;
        a.out = slice(g, dst, wpad); a.ldo = wpad;
        spmm(ctx, op, a);
        cur = dst;
      } else {
        a.post_vec = g->s;
        a.out = out; a.ldo = ldo; a.out_map = omap;
        spmm(ctx, op, a);
      }
    }
    return;
  }
  gemm_fp32(op, op->X, op->ldx, G + (size_t)L * d * ldgm, ldgm, slice(g, cur, wpad), wpad, g->n_local, wpad, d,
            g->s, false, nullptr);
  allgather_rows(ctx, g, cur, wpad);
  for (int j = L - 1; j >= 1; --j) {
    gemm_fp32(op, op->X, op->ldx, G + (size_t)j * d * ldgm, ldgm, op->ptmp, wpad, g->n_local, wpad, d, nullptr,
              false, nullptr);
    float* dst = bufs[j & 1];
    SpmmArgs a = spmm_base(g, wpad);
    a.Y = cur; a.ldy = wpad; a.self_coef = 1.f;
    a.post_vec = g->s2;
    a.T = op->ptmp; a.ldt = wpad; a.term_vec = g->s;
    a.out = slice(g, dst, wpad); a.ldo = wpad;
    spmm(ctx, op, a);
    allgather_rows(ctx, g, dst, wpad);
    cur = dst;
  }
  // X G_0 in internal row order; with a row map it goes through ptmp (the in-place
  // accumulation into `out` needs identical read and write rows).  With label re-use, lrbuf
  // already holds X G_0 plus the label blocks.
  float* t0 = op->lr_powers > 0 ? op->lrbuf : (omap ? op->ptmp : out);
  const int64_t ldt0 = (op->lr_powers > 0 || omap) ? wpad : ldo;
  if (op->lr_powers == 0)
    gemm_fp32(op, op->X, op->ldx, G, ldgm, t0, ldt0, g->n_local, wpad, d, nullptr, false, nullptr);
  SpmmArgs a = spmm_base(g, wpad);
  a.Y = cur; a.ldy = wpad; a.self_coef = 1.f;
  a.post_vec = g->s;
  a.T = t0; a.ldt = ldt0;  // may alias out: each element is read then written by one thread
  a.out = out; a.ldo = ldo; a.out_map = omap;
  spmm(ctx, op, a);
}

// Xrs = diag(1/s) X (P:182-193 with A_hat = S (A+I) S; 1/s = (d+1)^1/2 = g->rs)
void refresh_xrs(isvd_ctx ctx, isvd_op op) {
  isvd_graph g = op->g;
  CK(launch_scale_rows(op->X, op->ldx, op->Xrs, op->ldx, g->n_local, op->ldx, g->rs, 1.f, nullptr, ctx->stream,
                       nullptr));
}

// M^T Q: block j = X^T A_hat^j Q.  Zt_0 = s Q; Zt_{j+1} = s^2 ((A+I) Zt_j); block j = X^T diag(1/s) Zt_j.
// Q rows are in the caller's order when user_order (mapped by the first scaling pass).
void nc_matmul_T(isvd_ctx ctx, isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad,
                 bool user_order) {
  isvd_graph g = op->g;
  const int L = op->terms;
  const int64_t d = op->d;
  const int32_t* imap = (user_order && g->new2old) ? g->new2old : nullptr;
  float* bufs[2] = {op->full_a, op->full_b};
  if (!op->own_x) refresh_xrs(ctx, op);  // a borrowed X may have changed since the last call
  const float* Xrs = op->Xrs;
  // Zt_0 = s Q (internal row order), block 0 = X^T diag(1/s) Zt_0 = Xrs^T Zt_0
  CK(launch_scale_rows(Q, ldq, slice(g, bufs[0], wpad), wpad, g->n_local, wpad, g->s, 1.f, nullptr, ctx->stream,
                       imap));
  if (nc_overlap(ctx, op)) {
    // main: SpMM chain Zt_j -> Zt_{j+1} (event z_j = 2j after Zt_j is ready); side: block j as
    // soon as Zt_j is (event a_j = 2j+1 after it); SpMM j+2 overwrites Zt_j's buffer, so it
    // waits for block j.
    const cudaStream_t main = ctx->stream;
    auto block = [&](int j, const float* zt) {
      ev_wait(ctx, 2 * j, ctx->side);
      {
        OnStream on(ctx, ctx->side);
        atb_fp32(op, g->n_local, Xrs, op->ldx, d, nullptr, zt, wpad, wpad, false, op->blk64 + (size_t)j * d * wpad,
                 wpad, nullptr);
      }
      ev_record(ctx, 2 * j + 1, ctx->side);
    };
    ev_record(ctx, 0, main);
    block(0, slice(g, bufs[0], wpad));
    for (int j = 1; j <= L; ++j) {
      if (j >= 2) ev_wait(ctx, 2 * (j - 2) + 1, main);
      SpmmArgs a = spmm_base(g, wpad);
      a.Y = bufs[(j - 1) & 1]; a.ldy = wpad; a.self_coef = 1.f;
      a.post_vec = g->s2;
      a.out = slice(g, bufs[j & 1], wpad); a.ldo = wpad;
      spmm(ctx, op, a);
      ev_record(ctx, 2 * j, main);
      block(j, slice(g, bufs[j & 1], wpad));
    }
    ev_wait(ctx, 2 * L + 1, main);  // the last block (the side stream is in order)
    const int64_t c = d * (L + 1);
    CK(launch_f64_to_f32(op->blk64, wpad, out, ldo, c, wpad, ctx->stream));
    return;
  }
  atb_fp32(op, g->n_local, Xrs, op->ldx, d, nullptr, slice(g, bufs[0], wpad), wpad, wpad, false, op->blk64, wpad, nullptr);
  if (L > 0) allgather_rows(ctx, g, bufs[0], wpad);
  for (int j = 1; j <= L; ++j) {
    float* src = bufs[(j - 1) & 1];
    float* dst = bufs[j & 1];
    SpmmArgs a = spmm_base(g, wpad);
    a.Y = src; a.ldy = wpad; a.self_coef = 1.f;
    a.post_vec = g->s2;
    a.out = slice(g, dst, wpad); a.ldo = wpad;
    spmm(ctx, op, a);
    if (j < L) allgather_rows(ctx, g, dst, wpad);
    atb_fp32(op, g->n_local, Xrs, op->ldx, d, nullptr, slice(g, dst, wpad), wpad, wpad, false, op->blk64 + (size_t)j * d * wpad,
             wpad, nullptr);
  }
  if (op->lr_powers > 0) {
    // label re-use blocks: Zt_0 = s Q again; Zt_p = s^2 (A Zt_{p-1}) (B without the
    // self term, B^T = B); block p = Y^T diag(1/s) Zt_p
    float* zb[2] = {op->full_c, op->full_a};
    CK(launch_scale_rows(Q, ldq, slice(g, zb[0], wpad), wpad, g->n_local, wpad, g->s, 1.f, nullptr, ctx->stream,
                         imap));
    allgather_rows(ctx, g, zb[0], wpad);
    for (int p = 1; p <= op->lr_powers; ++p) {
      SpmmArgs a = spmm_base(g, wpad);
      a.Y = zb[(p - 1) & 1]; a.ldy = wpad;
      a.post_vec = g->s2;
      a.out = slice(g, zb[p & 1], wpad); a.ldo = wpad;
      spmm(ctx, op, a);
      if (p < op->lr_powers) allgather_rows(ctx, g, zb[p & 1], wpad);
      atb_fp32(op, g->n_local, op->Ylr, op->ldylr, op->ylr, g->rs, slice(g, zb[p & 1], wpad), wpad, wpad, false,
               op->blk64 + (size_t)(d * (L + 1) + (int64_t)(p - 1) * op->ylr) * wpad, wpad, nullptr);
    }
  }
  const int64_t c = c_rows_local(op);
  allreduce_f64(ctx, op->blk64, (size_t)c * wpad);
  CK(launch_f64_to_f32(op->blk64, wpad, out, ldo, c, wpad, ctx->stream));
}

void op_matmul(isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad, bool user_order) {
  isvd_ctx ctx = op->g->ctx;
  ensure_op_ws(op, wpad);
  Phase ph(ctx, kPhProducts);
  if (op->kind == ISVD_OP_POWER_SUM && op->ahat_basis) ne_ahat_matmul(ctx, op, Q, ldq, out, ldo, wpad, user_order);
  else if (op->kind == ISVD_OP_POWER_SUM) ne_matmul(ctx, op, Q, ldq, out, ldo, wpad, user_order);
  else nc_matmul(ctx, op, Q, ldq, out, ldo, wpad, user_order);
  join_gather(ctx);
}

void op_matmul_T(isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad, bool user_order) {
  isvd_ctx ctx = op->g->ctx;
  ensure_op_ws(op, wpad);
  Phase ph(ctx, kPhProducts);
  if (op->kind == ISVD_OP_POWER_SUM && op->ahat_basis) ne_ahat_matmul(ctx, op, Q, ldq, out, ldo, wpad, user_order);
  else if (op->kind == ISVD_OP_POWER_SUM) ne_matmul_T(ctx, op, Q, ldq, out, ldo, wpad, user_order);
  else nc_matmul_T(ctx, op, Q, ldq, out, ldo, wpad, user_order);
  join_gather(ctx);
}

// Implicit row gather (option (ii): "SVD of submatrix of M without explicitly
// computing M nor the submatrix"): M_S G = (M G)[S] and M_S^T H = M^T (scatter_S H), with the
// full-row product / scattered operand in sub_buf (zero outside S).  `caller_order`: the r-side
// rows of out / H are in the caller's order (API calls) or the solver's internal order.
void r_matmul(isvd_op op, const float* Q, int64_t ldq, float* out, int64_t ldo, int64_t wpad, bool caller_order) {
  if (!op->has_sub) return op_matmul(op, Q, ldq, out, ldo, wpad, caller_order);
  isvd_ctx ctx = op->g->ctx;
  ensure_op_ws(op, wpad);
  op_matmul(op, Q, ldq, op->sub_buf, wpad, wpad, caller_order);
  CK(launch_scale_rows(op->sub_buf, wpad, out, ldo, op->sub_local, wpad, nullptr, 1.f, nullptr, ctx->stream,
                       caller_order ? op->sub_caller : op->sub_int));
}
void r_matmul_T(isvd_op op, const float* H, int64_t ldh, float* out, int64_t ldo, int64_t wpad, bool caller_order) {
  if (!op->has_sub) return op_matmul_T(op, H, ldh, out, ldo, wpad, caller_order);
  isvd_ctx ctx = op->g->ctx;
  ensure_op_ws(op, wpad);
  CK(cudaMemsetAsync(op->sub_buf, 0, sizeof(float) * (size_t)std::max<int64_t>(op->g->n_local, 1) * wpad, ctx->stream));
  CK(launch_scatter_rows(H, ldh, op->sub_buf, wpad, op->sub_local, wpad, caller_order ? op->sub_caller : op->sub_int,
                         ctx->stream));
  op_matmul_T(op, op->sub_buf, wpad, out, ldo, wpad, caller_order);
}

void op_shape(const isvd_op_s* op, int64_t* r, int64_t* c) {
  *r = op->has_sub ? op->sub_n : op->g->n;
  *c = op->kind == ISVD_OP_POWER_SUM ? op->g->n : op->d * (op->terms + 1) + op->ylr * op->lr_powers;
}

// rows of the r-side (rows of M) held by this rank
int64_t r_rows_local(const isvd_op_s* op) { return op->has_sub ? op->sub_local : op->g->n_local; }

// rows of the c-side (columns of M) held by this rank
int64_t c_rows_local(const isvd_op_s* op) {
  return op->kind == ISVD_OP_POWER_SUM ? op->g->n_local : op->d * (op->terms + 1) + op->ylr * op->lr_powers;
}

template <typename F>
isvd_status guarded(isvd_ctx ctx, F&& f) {
  try {
    f();
    return ISVD_OK;
  } catch (const Fail& e) {
    return e.st;
  } catch (const std::bad_alloc&) {
    set_err(ctx, "host allocation failed");
    return ISVD_ERR_OOM;
  } catch (...) {
    set_err(ctx, "unexpected exception");
    return ISVD_ERR_INVALID_ARG;
  }
}

}  // namespace

// =================================================================== context
extern "C" {

int isvd_abi_version(void) { return ISVD_ABI_VERSION; }

const char* isvd_status_string(isvd_status s) {
  switch (s) {
    case ISVD_OK: return "ok";
    case ISVD_ERR_INVALID_ARG: return "invalid argument";
    case ISVD_ERR_SHAPE: return "shape mismatch";
    case ISVD_ERR_RANK: return "rank out of range";
    case ISVD_ERR_INDEX: return "index out of range";
    case ISVD_ERR_NONFINITE: return "non-finite value";
    case ISVD_ERR_OOM: return "out of memory";
    case ISVD_ERR_CUDA: return "CUDA error";
    case ISVD_ERR_NCCL: return "NCCL error";
    case ISVD_ERR_NOT_PD: return "Cholesky breakdown";
    case ISVD_ERR_BUSY: return "busy";
    case ISVD_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* isvd_last_error(isvd_ctx ctx) { return ctx ? ctx->last_error.c_str() : ""; }

isvd_status isvd_partition(int64_t n, int world, int rank, int64_t* row_begin, int64_t* n_local) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !row_begin || !n_local) return ISVD_ERR_INVALID_ARG;
  partition(n, world, rank, row_begin, n_local);
  return ISVD_OK;
}

isvd_status isvd_nccl_unique_id(void* id_out, size_t id_bytes) {
  if (!id_out || id_bytes < sizeof(ncclUniqueId)) return ISVD_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return ISVD_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return ISVD_OK;
}

namespace {
// Device, streams, events and status word of a new context (shared by both creation paths).
void ctx_init(isvd_ctx ctx, int device, void* stream, const isvd_allocator* alloc, int rank, int world) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  REQ(device >= 0 && device < ndev, ISVD_ERR_INVALID_ARG, "device out of range");
  if (alloc) {
    REQ(alloc->alloc && alloc->free, ISVD_ERR_INVALID_ARG, "allocator needs both alloc and free");
    ctx->alloc = *alloc;
    ctx->has_alloc = true;
  }
  ctx->device = device;
  DeviceGuard dg(device);
  ctx->stream = (cudaStream_t)stream;
  ctx->rank = rank;
  ctx->world = world;
  CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  REQ(major == 10, ISVD_ERR_UNSUPPORTED, "this library is built for sm_100a (B200) only");
  CK(cudaMalloc(&ctx->status, sizeof(DevStatus)));
  CK(cudaMemsetAsync(ctx->status, 0, sizeof(DevStatus), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaEventCreate(&ctx->ev0));
  CK(cudaEventCreate(&ctx->ev1));
  CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&ctx->work, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_gath, cudaEventDisableTiming));
  ctx->ov_ev.resize(16);
  for (auto& e : ctx->ov_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int persist = 0;
  CK(cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, device));
  ctx->max_persist_l2 = (size_t)persist;
}

isvd_status ctx_create_common(int device, void* stream, const isvd_allocator* alloc, const void* nccl_unique_id,
                              isvd_sim_group_s* sim, int rank, int world, isvd_ctx* out) {
  *out = nullptr;
  isvd_ctx ctx = new (std::nothrow) isvd_ctx_s();
  if (!ctx) return ISVD_ERR_OOM;
  isvd_status st = guarded(ctx, [&] {
    ctx_init(ctx, device, stream, alloc, rank, world);
    DeviceGuard dg(device);
    if (nccl_unique_id) {  // distributed mode (also world == 1: NCCL path with a 1-rank communicator)
      ctx->dist = true;
      ncclUniqueId id;
      memcpy(&id, nccl_unique_id, sizeof(id));
      NK(ncclCommInitRank(&ctx->comm, world, id, rank));
    } else if (sim) {
      ctx->dist = true;
      ctx->sim = sim;
    }
  });
  if (st != ISVD_OK) {
    fprintf(stderr, "isvd_ctx_create: %s\n", ctx->last_error.c_str());
    if (ctx->status) cudaFree(ctx->status);
    delete ctx;
    return st;
  }
  if (sim) sim->members++;
  *out = ctx;
  return ISVD_OK;
}
}  // namespace

isvd_status isvd_ctx_create(int device, void* stream, const isvd_allocator* alloc, const void* nccl_unique_id,
                            int rank, int world, isvd_ctx* out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return ISVD_ERR_INVALID_ARG;
  if (world > 1 && nccl_unique_id == nullptr) return ISVD_ERR_INVALID_ARG;
  return ctx_create_common(device, stream, alloc, nccl_unique_id, nullptr, rank, world, out);
}

isvd_status isvd_sim_group_create(int world, isvd_sim_group* out) {
  if (!out || world < 1 || world > kMaxSimRanks) return ISVD_ERR_INVALID_ARG;
  *out = nullptr;
  isvd_sim_group_s* g = new (std::nothrow) isvd_sim_group_s();
  if (!g) return ISVD_ERR_OOM;
  g->world = world;
  g->ptr.assign(world, nullptr);
  g->ready.assign(world, nullptr);
  g->done.assign(world, nullptr);
  for (int q = 0; q < world; ++q) {
    if (cudaEventCreateWithFlags(&g->ready[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done[q], cudaEventDisableTiming) != cudaSuccess) {
      (void)cudaGetLastError();
      for (int r = 0; r < world; ++r) {
        if (g->ready[r]) cudaEventDestroy(g->ready[r]);
        if (g->done[r]) cudaEventDestroy(g->done[r]);
      }
      delete g;
      return ISVD_ERR_CUDA;
    }
  }
  *out = g;
  return ISVD_OK;
}

isvd_status isvd_sim_group_destroy(isvd_sim_group g) {
  if (!g) return ISVD_ERR_INVALID_ARG;
  if (g->members.load() > 0) return ISVD_ERR_BUSY;
  for (int q = 0; q < g->world; ++q) {
    cudaEventDestroy(g->ready[q]);
    cudaEventDestroy(g->done[q]);
  }
  delete g;
  return ISVD_OK;
}

isvd_status isvd_ctx_create_sim(int device, void* stream, const isvd_allocator* alloc, isvd_sim_group group, int rank,
                                isvd_ctx* out) {
  if (!out || !group || rank < 0 || rank >= group->world) return ISVD_ERR_INVALID_ARG;
  return ctx_create_common(device, stream, alloc, nullptr, group, rank, group->world, out);
}

isvd_status isvd_ctx_destroy(isvd_ctx ctx) {
  if (!ctx) return ISVD_ERR_INVALID_ARG;
  if (ctx->live_graphs.load() > 0) return ISVD_ERR_BUSY;
  DeviceGuard dg(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (void* p : ctx->sim_allocs) dfree(ctx, p);
  if (ctx->sim) ctx->sim->members--;
  pool_trim(ctx);
  if (ctx->status) cudaFree(ctx->status);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->work) {
    cudaStreamSynchronize(ctx->work);
    cudaStreamDestroy(ctx->work);
  }
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->cstream) {
    cudaStreamSynchronize(ctx->cstream);
    cudaStreamDestroy(ctx->cstream);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_gath) cudaEventDestroy(ctx->ev_gath);
  for (cudaEvent_t e : ctx->ov_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->prof_events) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->phase_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ag_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->lp_ev) cudaEventDestroy(e);
  delete ctx;
  return ISVD_OK;
}

// ===================================================================== graph
namespace {
// SpMM segment plan of the CSR row_ptr `rp` (device) into p (device arrays owned by `allocs`).
void build_plan(isvd_ctx ctx, const int64_t* rp, int64_t n_local, SpmmPlan& p, std::vector<void*>& allocs, void* temp,
                size_t temp_bytes) {
  std::vector<void*> tmp;
  struct TmpFree {
    std::vector<void*>& v;
    isvd_ctx c;
    ~TmpFree() { for (void* q : v) dfree(c, q); }
  } tmp_free{tmp, ctx};
  int64_t* nseg = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), tmp);
  int64_t* seg_off = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), tmp);
  int32_t* cnt32 = (int32_t*)dmalloc(ctx, sizeof(int32_t) * 4 * (n_local + 1), tmp);
  int32_t *nsplit = cnt32, *nslot = cnt32 + (n_local + 1), *split_off = cnt32 + 2 * (n_local + 1),
          *slot_off = cnt32 + 3 * (n_local + 1);
  CK(launch_plan_count(rp, n_local, nseg, nsplit, nslot, seg_off, split_off, slot_off, temp, temp_bytes, ctx->stream));
  int64_t tot_seg = 0;
  int32_t tot_split = 0, tot_slot = 0;
  CK(cudaMemcpyAsync(&tot_seg, seg_off + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&tot_split, split_off + n_local, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&tot_slot, slot_off + n_local, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  p.n_local = n_local;
  p.n_seg = tot_seg;
  p.n_split_rows = tot_split;
  p.n_slots = tot_slot;
  auto d32 = [&](int64_t n) { return (int32_t*)dmalloc(ctx, sizeof(int32_t) * std::max<int64_t>(n, 1), allocs); };
  p.seg_row = d32(tot_seg);
  p.seg_len = d32(tot_seg);
  p.seg_slot = d32(tot_seg);
  p.split_row = d32(tot_split);
  p.split_slot0 = d32(tot_split);
  p.split_nslot = d32(tot_split);
  p.seg_beg = (int64_t*)dmalloc(ctx, sizeof(int64_t) * std::max<int64_t>(tot_seg, 1), allocs);
  CK(launch_plan_fill(rp, n_local, seg_off, split_off, slot_off, p, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}
}  // namespace

isvd_status isvd_graph_create(isvd_ctx ctx, int64_t n_global, int64_t row_begin, int64_t n_local,
                              const int64_t* row_ptr, const int32_t* col_idx, const float* values, uint32_t flags,
                              isvd_graph* out) {
  if (!ctx || !out) return ISVD_ERR_INVALID_ARG;
  *out = nullptr;
  isvd_graph g = new (std::nothrow) isvd_graph_s();
  if (!g) return ISVD_ERR_OOM;
  isvd_status st = guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    REQ(n_global >= 1 && n_global < (int64_t)INT32_MAX, ISVD_ERR_INVALID_ARG, "n must be in [1, 2^31-1)");
    REQ(row_ptr != nullptr, ISVD_ERR_INVALID_ARG, "row_ptr is null");
    REQ((flags & ~(uint32_t)(ISVD_PTR_DEVICE | ISVD_GRAPH_SYMMETRIC | ISVD_GRAPH_VALIDATE)) == 0,
        ISVD_ERR_INVALID_ARG, "unknown graph flag");
    REQ(flags & ISVD_GRAPH_SYMMETRIC, ISVD_ERR_UNSUPPORTED,
        "directed graphs need an explicit transpose (not built in this version); pass ISVD_GRAPH_SYMMETRIC");
    int64_t rb, nl;
    partition(n_global, ctx->world, ctx->rank, &rb, &nl);
    REQ(rb == row_begin && nl == n_local, ISVD_ERR_INVALID_ARG,
        "row partition must equal isvd_partition(n, world, rank)");
    const bool dev = flags & ISVD_PTR_DEVICE;
    // ISVD_TRACE=1: host-side phase times of the graph build on stderr
    static const bool trace = getenv("ISVD_TRACE") && getenv("ISVD_TRACE")[0] == '1';
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
      if (!trace) return;
      auto t = std::chrono::steady_clock::now();
      fprintf(stderr, "[isvd] graph_create %-10s %8.2f ms\n", name,
              std::chrono::duration<double, std::milli>(t - t_last).count());
      t_last = t;
    };
    std::vector<int64_t> rp(n_local + 1);
    if (dev) {  // on the ctx stream: ordered after the caller's producer on that stream
      CK(cudaMemcpyAsync(rp.data(), row_ptr, sizeof(int64_t) * (n_local + 1), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    } else {
      memcpy(rp.data(), row_ptr, sizeof(int64_t) * (n_local + 1));
    }
    const int64_t base = rp[0];
    for (auto& v : rp) v -= base;
    for (int64_t i = 0; i < n_local; ++i)
      REQ(rp[i + 1] >= rp[i], ISVD_ERR_INDEX, "row_ptr is not monotone");
    const int64_t nnz = rp[n_local];
    REQ(nnz == 0 || col_idx != nullptr, ISVD_ERR_INVALID_ARG, "col_idx is null");
    g->ctx = ctx;
    g->n = n_global;
    g->row_begin = row_begin;
    g->n_local = n_local;
    g->n_pad = (n_global + ctx->world - 1) / ctx->world;
    g->nnz = nnz;
    // CSR on the device (copied: the caller may free its arrays on return), with kIdxPad
    // readable zero entries after the last index (the gather prefetches one batch ahead)
    const bool relabel = !ctx->dist && n_local >= kRelabelMinRows;
    std::vector<void*> tmp;
    struct TmpFree {
      std::vector<void*>& v;
      isvd_ctx c;
      ~TmpFree() { for (void* q : v) dfree(c, q); }
    } tmp_free{tmp, ctx};
    g->row_ptr = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), g->allocs);
    g->col_idx = (int32_t*)dmalloc(ctx, sizeof(int32_t) * (nnz + kIdxPad), g->allocs);
    int32_t* ci_in = relabel ? (int32_t*)dmalloc(ctx, sizeof(int32_t) * std::max<int64_t>(nnz, 1), tmp) : g->col_idx;
    const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (nnz > 0) CK(cudaMemcpyAsync(ci_in, col_idx + base, sizeof(int32_t) * nnz, kind, ctx->stream));
    // edge weights: moved with their edges
    float* val_in = nullptr;
    if (values) {
      g->val = (float*)dmalloc(ctx, sizeof(float) * (nnz + kIdxPad), g->allocs);
      val_in = relabel ? (float*)dmalloc(ctx, sizeof(float) * std::max<int64_t>(nnz, 1), tmp) : g->val;
      if (nnz > 0) CK(cudaMemcpyAsync(val_in, values + base, sizeof(float) * nnz, kind, ctx->stream));
    }
    if (flags & ISVD_GRAPH_VALIDATE) {
      std::vector<int32_t> ci(nnz);
      if (nnz) CK(cudaMemcpyAsync(ci.data(), ci_in, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
      std::vector<float> vv(values ? nnz : 0);
      if (values && nnz)
        CK(cudaMemcpyAsync(vv.data(), val_in, sizeof(float) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      for (int64_t e = 0; e < nnz; ++e)
        REQ(ci[e] >= 0 && ci[e] < n_global, ISVD_ERR_INDEX, "col_idx outside [0, n)");
      for (float v : vv) REQ(std::isfinite(v) && v >= 0.f, ISVD_ERR_NONFINITE, "edge weights must be finite and >= 0");
    }
    phase("csr_upload");
    // Degree relabelling (single rank, large graphs; SURVEY 8(d2) "allowed optimisation"):
    // internal row t is caller row order[t], in decreasing degree, so the hub rows that take
    // most gathers form one contiguous prefix of every iterate, which the SpMM marks
    // L2-persisting.  A symmetric permutation of A: singular values are unchanged and every
    // caller-ordered input/output is mapped at the boundary (X, Omega, U, V, matmul I/O).
    // The order is computed on the host from the degrees; the index renaming runs on the GPU.
    int64_t maxd = 0;
    for (int64_t i = 0; i < n_local; ++i) maxd = std::max(maxd, rp[i + 1] - rp[i]);
    g->max_deg = maxd;
    // row_ptr of the caller's order on the device (the relabelling and the plan read it there)
    int64_t* d_rp_in = relabel ? (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), tmp) : g->row_ptr;
    CK(cudaMemcpyAsync(d_rp_in, rp.data(), sizeof(int64_t) * (n_local + 1), cudaMemcpyHostToDevice, ctx->stream));
    const size_t temp_bytes = graph_build_temp_bytes(n_local);
    void* temp = dmalloc(ctx, temp_bytes, tmp);
    if (relabel) {
      // stable sort by decreasing degree (device radix sort), maps, new row_ptr, renamed indices
      uint32_t* keys2 = (uint32_t*)dmalloc(ctx, sizeof(uint32_t) * 2 * n_local, tmp);
      int32_t* idx = (int32_t*)dmalloc(ctx, sizeof(int32_t) * n_local, tmp);
      int64_t* deg_tmp = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), tmp);
      int32_t* d_new_of_old = (int32_t*)dmalloc(ctx, sizeof(int32_t) * n_local, tmp);
      g->new2old = (int32_t*)dmalloc(ctx, sizeof(int32_t) * n_local, g->allocs);
      CK(launch_degree_order(d_rp_in, n_local, keys2, idx, g->new2old, d_new_of_old, deg_tmp, g->row_ptr, temp,
                             temp_bytes, ctx->stream));
      CK(launch_relabel_csr(d_rp_in, ci_in, val_in, g->new2old, d_new_of_old, g->row_ptr, g->col_idx, g->val,
                            n_local, ctx->stream));
      if (ctx->max_persist_l2 > 0) {
        static bool limit_set = false;  // process-wide L2 set-aside for persisting accesses
        if (!limit_set) {
          CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ctx->max_persist_l2));
          limit_set = true;
        }
      }
    }
    phase("relabel");
    // degrees (integers) -> scale vectors computed once in fp64, stored fp32 (reading O3)
    size_t nb = sizeof(float) * std::max<int64_t>(n_local, 1);
    g->inv_deg = (float*)dmalloc(ctx, nb, g->allocs);
    g->s = (float*)dmalloc(ctx, nb, g->allocs);
    g->s2 = (float*)dmalloc(ctx, nb, g->allocs);
    g->rs = (float*)dmalloc(ctx, nb, g->allocs);
    CK(launch_scales(g->row_ptr, g->val, n_local, g->inv_deg, g->s, g->s2, g->rs, ctx->stream));
    phase("scales");
    const char* dense_env = getenv("ISVD_DENSE_A");  // 1: exact INT8 (unweighted), 2: 3xTF32
    if (dense_env && dense_env[0] != '0' && !ctx->dist && n_local == n_global && n_global <= 32768 && !g->new2old &&
        n_global >= 1) {
      g->ld_dense = round_up(n_global, 4);
      g->dense = (float*)dmalloc(ctx, sizeof(float) * (size_t)n_global * g->ld_dense, g->allocs);
      CK(launch_dense_adjacency(g->row_ptr, g->col_idx, g->val, n_global, g->ld_dense, g->dense, ctx->stream));
      // ISVD_DENSE_A=1: the exact INT8 path for unweighted graphs; =2 forces the 3xTF32 path
      if (!g->val && dense_env[0] != '2') {
        g->ld_u8 = round_up(n_global, 16);
        g->dense_u8 = (uint8_t*)dmalloc(ctx, (size_t)n_global * g->ld_u8, g->allocs);
        CK(launch_dense_to_u8(g->dense, n_global, g->ld_dense, g->dense_u8, g->ld_u8, ctx->stream));
      }
    }
    // SpMM segment plan: rows of <= kSegEdges edges are one segment; longer rows are
    // split, their partial sums combined by the fixup pass in segment order (graph_build.cu)
    build_plan(ctx, g->row_ptr, n_local, g->plan, g->allocs, temp, temp_bytes);
    // distributed (world > 1): the local / remote split of every row's edges, so the local part
    // of each SpMM step runs while the all-gather of the gather source is in flight (SURVEY 8(e)
    // overlap item 1); ISVD_DIST_SPLIT=0 keeps the single pass after a blocking all-gather
    static const bool no_split = getenv("ISVD_DIST_SPLIT") && getenv("ISVD_DIST_SPLIT")[0] == '0';
    if (ctx->dist && ctx->world > 1 && !no_split && n_local > 0) {
      int64_t* cl = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), tmp);
      int64_t* cr = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), tmp);
      g->rp_loc = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), g->allocs);
      g->rp_rem = (int64_t*)dmalloc(ctx, sizeof(int64_t) * (n_local + 1), g->allocs);
      CK(launch_split_count(g->row_ptr, g->col_idx, n_local, row_begin, row_begin + n_local, cl, cr, ctx->stream));
      CK(launch_exclusive_scan64(cl, g->rp_loc, n_local + 1, temp, temp_bytes, ctx->stream));
      CK(launch_exclusive_scan64(cr, g->rp_rem, n_local + 1, temp, temp_bytes, ctx->stream));
      int64_t nl_e = 0, nr_e = 0;
      CK(cudaMemcpyAsync(&nl_e, g->rp_loc + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(&nr_e, g->rp_rem + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      g->nnz_loc = nl_e;
      g->ci_loc = (int32_t*)dmalloc(ctx, sizeof(int32_t) * (nl_e + kIdxPad), g->allocs);
      g->ci_rem = (int32_t*)dmalloc(ctx, sizeof(int32_t) * (nr_e + kIdxPad), g->allocs);
      if (g->val) {
        g->val_loc = (float*)dmalloc(ctx, sizeof(float) * (nl_e + kIdxPad), g->allocs);
        g->val_rem = (float*)dmalloc(ctx, sizeof(float) * (nr_e + kIdxPad), g->allocs);
      }
      CK(launch_split_fill(g->row_ptr, g->col_idx, g->val, n_local, row_begin, row_begin + n_local, g->rp_loc,
                           g->rp_rem, g->ci_loc, g->val_loc, g->ci_rem, g->val_rem, ctx->stream));
      build_plan(ctx, g->rp_loc, n_local, g->plan_loc, g->allocs, temp, temp_bytes);
      build_plan(ctx, g->rp_rem, n_local, g->plan_rem, g->allocs, temp, temp_bytes);
      g->split = true;
    }
    phase("plan");
  });
  if (st != ISVD_OK) {
    for (void* p : g->allocs) dfree(ctx, p);
    delete g;
    return st;
  }
  ctx->live_graphs++;
  *out = g;
  return ISVD_OK;
}

isvd_status isvd_graph_destroy(isvd_graph g) {
  if (!g) return ISVD_ERR_INVALID_ARG;
  if (g->refs.load() > 0) return ISVD_ERR_BUSY;
  DeviceGuard dg(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  for (void* p : g->allocs) dfree(g->ctx, p);
  g->ctx->live_graphs--;
  delete g;
  return ISVD_OK;
}

isvd_status isvd_graph_info(isvd_graph g, int64_t* n_global, int64_t* n_local, int64_t* nnz_local,
                            int64_t* max_degree) {
  if (!g) return ISVD_ERR_INVALID_ARG;
  if (n_global) *n_global = g->n;
  if (n_local) *n_local = g->n_local;
  if (nnz_local) *nnz_local = g->nnz;
  if (max_degree) *max_degree = g->max_deg;
  return ISVD_OK;
}

// ================================================================= operators
namespace {
// An owned device copy of a caller-ordered row block (n_local x ld fp32), rows in the graph's
// internal order (relabelled graphs gather them through new2old).
float* own_rows(isvd_ctx ctx, isvd_graph g, const float* src_in, int64_t ld, bool dev) {
  std::vector<void*> tmp;
  const size_t row_bytes = sizeof(float) * (size_t)ld;
  float* x = (float*)dmalloc(ctx, row_bytes * (size_t)std::max<int64_t>(g->n_local, 1), tmp);
  struct FreeOnThrow {  // the copy below may fail (bad pointer / alignment): do not leak x
    isvd_ctx c;
    float* p;
    ~FreeOnThrow() { if (p) dfree(c, p); }
  } guard{ctx, x};
  if (g->n_local > 0) {
    if (!g->new2old) {
      CK(cudaMemcpyAsync(x, src_in, row_bytes * (size_t)g->n_local, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    } else {
      const float* src = src_in;
      std::vector<void*> stage;
      if (!dev) {
        float* d = (float*)dmalloc(ctx, row_bytes * (size_t)g->n_local, stage);
        CK(cudaMemcpyAsync(d, src_in, row_bytes * (size_t)g->n_local, cudaMemcpyHostToDevice, ctx->stream));
        src = d;
      }
      REQ(aligned16(src), ISVD_ERR_INVALID_ARG, "row blocks must be 16-byte aligned");
      CK(launch_scale_rows(src, ld, x, ld, g->n_local, ld, nullptr, 1.f, nullptr, ctx->stream, g->new2old));
      CK(cudaStreamSynchronize(ctx->stream));
      for (void* q : stage) dfree(ctx, q);
    }
  }
  guard.p = nullptr;
  return x;
}
}  // namespace

isvd_status isvd_op_define(isvd_graph g, const isvd_op_desc* desc, isvd_op* out) {
  if (!g || !desc || !out) return ISVD_ERR_INVALID_ARG;
  isvd_ctx ctx = g->ctx;
  *out = nullptr;
  isvd_op op = new (std::nothrow) isvd_op_s();
  if (!op) return ISVD_ERR_OOM;
  isvd_status st = guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    op->g = g;
    op->kind = desc->kind;
    op->terms = desc->num_terms;
    REQ(desc->basis == ISVD_BASIS_DEFAULT || desc->basis == ISVD_BASIS_T_ROW || desc->basis == ISVD_BASIS_AHAT_SYM,
        ISVD_ERR_INVALID_ARG, "unknown basis");
    if (desc->kind == ISVD_OP_POWER_SUM) {
      op->ahat_basis = desc->basis == ISVD_BASIS_AHAT_SYM;
      REQ(desc->num_terms >= 1, ISVD_ERR_INVALID_ARG, "NE needs C >= 1 powers");
      REQ(desc->weights != nullptr, ISVD_ERR_INVALID_ARG, "NE weights are null");
      op->w.assign(desc->weights, desc->weights + desc->num_terms);
      for (double x : op->w) REQ(std::isfinite(x), ISVD_ERR_NONFINITE, "non-finite weight");
      REQ(std::isfinite(desc->lambda_ones) && std::isfinite(desc->lambda_adj), ISVD_ERR_NONFINITE,
          "non-finite lambda");
      op->lambda_ones = desc->lambda_ones;
      op->lambda_adj = desc->lambda_adj;
    } else if (desc->kind == ISVD_OP_STACKED_PROPAGATION) {
      REQ(desc->num_terms >= 0, ISVD_ERR_INVALID_ARG, "NC needs L >= 0");
      REQ(desc->basis != ISVD_BASIS_T_ROW, ISVD_ERR_UNSUPPORTED, "NC propagates with A_hat (Eq. 6, P:68) only");
      REQ(desc->d >= 1, ISVD_ERR_INVALID_ARG, "NC feature width d must be >= 1");
      REQ(desc->ldx >= desc->d && desc->ldx % 4 == 0, ISVD_ERR_INVALID_ARG, "ldx must be >= d and a multiple of 4");
      REQ(desc->X != nullptr || g->n_local == 0, ISVD_ERR_INVALID_ARG, "X is null");
      REQ((desc->x_flags & ~(uint32_t)(ISVD_PTR_DEVICE | ISVD_BORROW)) == 0, ISVD_ERR_INVALID_ARG, "bad x_flags");
      op->d = desc->d;
      op->ldx = desc->ldx;
      const bool dev = desc->x_flags & ISVD_PTR_DEVICE;
      if (dev && (desc->x_flags & ISVD_BORROW) && !g->new2old) {
        REQ(aligned16(desc->X), ISVD_ERR_INVALID_ARG, "X must be 16-byte aligned");
        op->X = desc->X;
      } else {
        op->X = own_rows(ctx, g, desc->X, desc->ldx, dev);
        op->own_x = true;
      }
      {
        std::vector<void*> tmp;
        op->Xrs = (float*)dmalloc(ctx, sizeof(float) * (size_t)desc->ldx * (size_t)std::max<int64_t>(g->n_local, 1), tmp);
        if (op->own_x) refresh_xrs(ctx, op);
      }
      if (desc->lr_powers > 0) {  // label re-use blocks
        REQ(desc->y >= 1 && desc->ldy >= desc->y && desc->ldy % 4 == 0, ISVD_ERR_INVALID_ARG,
            "label width y >= 1 and ldy >= y, a multiple of 4");
        REQ(desc->Y != nullptr || g->n_local == 0, ISVD_ERR_INVALID_ARG, "Y is null");
        REQ((desc->y_flags & ~(uint32_t)ISVD_PTR_DEVICE) == 0, ISVD_ERR_INVALID_ARG, "bad y_flags");
        op->Ylr = own_rows(ctx, g, desc->Y, desc->ldy, desc->y_flags & ISVD_PTR_DEVICE);
        op->ylr = desc->y;
        op->ldylr = desc->ldy;
        op->lr_powers = desc->lr_powers;
      }
    } else {
      REQ(false, ISVD_ERR_INVALID_ARG, "unknown op kind");
    }
    // implicit row gather (option (ii)): M_S = M[S, :], S sorted global row ids
    REQ(desc->n_rows >= 0 && (desc->n_rows == 0 || desc->rows != nullptr), ISVD_ERR_INVALID_ARG,
        "rows is null while n_rows > 0");
    if (desc->n_rows > 0) {
      const int64_t* S = desc->rows;
      for (int64_t i = 0; i < desc->n_rows; ++i) {
        REQ(S[i] >= 0 && S[i] < g->n, ISVD_ERR_INDEX, "row subset entry outside [0, n)");
        REQ(i == 0 || S[i] > S[i - 1], ISVD_ERR_INVALID_ARG, "row subset must be strictly increasing");
      }
      const int64_t* lo = std::lower_bound(S, S + desc->n_rows, g->row_begin);
      const int64_t* hi = std::lower_bound(S, S + desc->n_rows, g->row_begin + g->n_local);
      op->has_sub = true;
      op->sub_n = desc->n_rows;
      op->sub_offset = lo - S;
      op->sub_local = hi - lo;
      std::vector<int32_t> loc(std::max<int64_t>(op->sub_local, 1), 0);
      for (int64_t i = 0; i < op->sub_local; ++i) loc[i] = (int32_t)(lo[i] - g->row_begin);
      op->sub_caller = (int32_t*)dmalloc(ctx, sizeof(int32_t) * loc.size(), op->sub_allocs);
      CK(cudaMemcpyAsync(op->sub_caller, loc.data(), sizeof(int32_t) * loc.size(), cudaMemcpyHostToDevice,
                         ctx->stream));
      if (g->new2old) {  // internal row of each subset row: (new2old)^-1 composed with the caller rows
        op->sub_int = (int32_t*)dmalloc(ctx, sizeof(int32_t) * loc.size(), op->sub_allocs);
        std::vector<void*> tmp;
        int32_t* inv = (int32_t*)dmalloc(ctx, sizeof(int32_t) * std::max<int64_t>(g->n_local, 1), tmp);
        CK(launch_compose_inverse(g->new2old, g->n_local, op->sub_caller, op->sub_local, inv, op->sub_int,
                                  ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (void* q : tmp) dfree(ctx, q);
      } else {
        op->sub_int = op->sub_caller;
      }
      CK(cudaStreamSynchronize(ctx->stream));
    }
  });
  if (st != ISVD_OK) {  // give back whatever the op had already taken
    for (void* q : op->sub_allocs) dfree(ctx, q);
    if (op->own_x) dfree(ctx, (void*)op->X);
    dfree(ctx, op->Xrs);
    dfree(ctx, (void*)op->Ylr);
    delete op;
    return st;
  }
  g->refs++;
  *out = op;
  return ISVD_OK;
}

isvd_status isvd_op_shape(isvd_op op, int64_t* rows, int64_t* cols) {
  if (!op || !rows || !cols) return ISVD_ERR_INVALID_ARG;
  op_shape(op, rows, cols);
  return ISVD_OK;
}

static void free_solver_ws(isvd_ctx ctx, SolverWs& s) {
  if (s.graph_exec) cudaGraphExecDestroy(s.graph_exec);
  s.graph_exec = nullptr;
  for (void* p : s.allocs) dfree(ctx, p);
  s.allocs.clear();
  s.key_l = s.key_k = -1;
}

isvd_status isvd_op_destroy(isvd_op op) {
  if (!op) return ISVD_ERR_INVALID_ARG;
  DeviceGuard dg(op->g->ctx->device);
  cudaStreamSynchronize(op->g->ctx->stream);
  for (void* p : op->ws_allocs) dfree(op->g->ctx, p);
  free_solver_ws(op->g->ctx, op->sws);
  if (op->own_x) dfree(op->g->ctx, (void*)op->X);
  if (op->Xrs) dfree(op->g->ctx, op->Xrs);
  if (op->Ylr) dfree(op->g->ctx, (void*)op->Ylr);
  for (void* q : op->sub_allocs) dfree(op->g->ctx, q);
  op->g->refs--;
  delete op;
  return ISVD_OK;
}

static isvd_status check_dense(isvd_ctx ctx, const float* p, int64_t w, int64_t ld) {
  if (!p) { set_err(ctx, "null matrix pointer"); return ISVD_ERR_INVALID_ARG; }
  if (w < 1) { set_err(ctx, "width must be >= 1"); return ISVD_ERR_SHAPE; }
  if (ld < w || ld % 4 != 0 || !aligned16(p)) {
    set_err(ctx, "leading dimension must be >= width and a multiple of 4, pointer 16-byte aligned");
    return ISVD_ERR_INVALID_ARG;
  }
  if (ld < ((w + 3) / 4) * 4) { set_err(ctx, "leading dimension must be >= round_up(width, 4)"); return ISVD_ERR_INVALID_ARG; }
  return ISVD_OK;
}

isvd_status isvd_matmul(isvd_op op, const float* Q, int64_t w, int64_t ldq, float* out, int64_t ldo) {
  if (!op) return ISVD_ERR_INVALID_ARG;
  isvd_ctx ctx = op->g->ctx;
  isvd_status s;
  if ((s = check_dense(ctx, Q, w, ldq)) != ISVD_OK) return s;
  if ((s = check_dense(ctx, out, w, ldo)) != ISVD_OK) return s;
  if (Q == out) { set_err(ctx, "out must not alias Q"); return ISVD_ERR_INVALID_ARG; }
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    r_matmul(op, Q, ldq, out, ldo, round_up(w, 4), true);
  });
}

isvd_status isvd_matmul_T(isvd_op op, const float* Q, int64_t w, int64_t ldq, float* out, int64_t ldo) {
  if (!op) return ISVD_ERR_INVALID_ARG;
  isvd_ctx ctx = op->g->ctx;
  isvd_status s;
  if ((s = check_dense(ctx, Q, w, ldq)) != ISVD_OK) return s;
  if ((s = check_dense(ctx, out, w, ldo)) != ISVD_OK) return s;
  if (Q == out) { set_err(ctx, "out must not alias Q"); return ISVD_ERR_INVALID_ARG; }
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    r_matmul_T(op, Q, ldq, out, ldo, round_up(w, 4), true);
  });
}

// ==================================================================== solver
namespace {

// Everything a captured solver graph bakes in (FNV-1a over the argument values).  The graph writes
// U and V into the op's own buffers (copied out after each replay), so the caller's output
// pointers are not part of the key: a new pair of output tensors per call still replays.
uint64_t graph_key(const isvd_svd_params* p, int64_t l, int64_t ldk) {
  uint64_t h = 0xCBF29CE484222325ULL;
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xFF;
      h *= 0x100000001B3ULL;
    }
  };
  mix((uint64_t)p->k); mix((uint64_t)(uint32_t)p->oversampling); mix((uint64_t)p->power_iters); mix(p->seed);
  mix(p->flags); mix((uint64_t)(uintptr_t)p->omega); mix((uint64_t)l); mix((uint64_t)ldk);
  mix((uint64_t)tc_for_grams() | (uint64_t)tc_for_products() << 1);
  return h;
}

int64_t working_l(const isvd_op_s* op, const isvd_svd_params* p) {
  int64_t r, c;
  op_shape(op, &r, &c);
  int64_t l = p->oversampling < 0 ? 2LL * p->k : (int64_t)p->k + p->oversampling;
  return std::min(l, std::min(r, c));
}

void ensure_solver_ws(isvd_op op, int64_t l, int64_t k) {
  SolverWs& s = op->sws;
  if (s.key_l == l && s.key_k == k) return;
  isvd_ctx ctx = op->g->ctx;
  CK(cudaStreamSynchronize(ctx->stream));
  free_solver_ws(ctx, s);
  const int64_t ld = round_up(l, 4), ldk = round_up(k, 4);
  const int64_t rr = std::max<int64_t>(r_rows_local(op), 1), cr = std::max<int64_t>(c_rows_local(op), 1);
  auto f = [&](int64_t n) { return (float*)dmalloc(ctx, sizeof(float) * n, s.allocs); };
  auto d = [&](int64_t n) { return (double*)dmalloc(ctx, sizeof(double) * n, s.allocs); };
  s.Qc = f(cr * ld);
  s.Qc2 = f(cr * ld);
  s.Yr = f(rr * ld);
  s.Yr2 = f(rr * ld);
  s.Rinv32 = f(ld * ld);
  s.Rfold = f(ld * ld);
  s.Ub2 = f(l * ldk);
  s.Ub = f(l * ldk);
  s.Vb = f(l * ldk);
  s.Utmp = f(rr * ldk);
  s.Vtmp = f(cr * ldk);
  s.sgn = f(ldk);
  s.gram = d(l * l);
  s.Ra = d(l * l); s.Rb = d(l * l); s.Rc = d(l * l); s.Rab = d(l * l); s.Rfin = d(l * l);
  s.chol_ws = d(l * l);
  s.jac_ws = d(jacobi_ws_doubles((int)l));
  s.sigma = d(k);
  s.cand = d(3 * k);
  s.cand_all = d(3 * k * op->g->ctx->world);
  s.absmax_ws = d(absmax_ws_doubles(rr, (int)k));
  s.key_l = l;
  s.key_k = k;
}

// Gram precision classes of one CholeskyQR pass.
//   kGramF64:  fp64 FMA on the fp32 data (exact products, fp64 sums) -- input possibly
//              ill-conditioned (Y = M Omega), and the shifted third pass;
//   kGramFp32: fp32-class sums over short row chunks (128-row tcgen05 3xTF32 TMEM chunks, or
//              <= 1024-row SIMT chunks), fp64 across chunks: ~1e-6 relative (atb_fp32).
enum GramMode { kGramF64 = 0, kGramFp32 = 1 };

// One Cholesky pass (Alg. 2 right): G = Y^T Y (all-reduced when row-partitioned), R = chol(G), Yout = Y R^-1.
void cqr_pass(isvd_op op, const float* Y, float* Yout, int64_t rows, bool distributed, int64_t l, double* R64,
              GramMode mode, bool force_fail, const int* gate, const int* gemm_gate = nullptr) {
  isvd_ctx ctx = op->g->ctx;
  SolverWs& s = op->sws;
  const int64_t ld = round_up(l, 4);
  // Exact-Gram pass of a tall iterate (Y = M Omega): probe first with the tensor-core Gram, whose
  // fp32-class error is harmless unless kappa(Y)^2 is large; a probe-mode Cholesky flags a
  // breakdown or a pivot spread min r_kk^2 < 1e-5 max r_kk^2, and only then are the exact fp64
  // Gram and the (shift-capable) Cholesky recomputed, gated on that device flag (no host sync).
  // Saves the 22.6 ms exact Gram at config 4 when Y is well conditioned.  ISVD_GRAM_PROBE=0: off.
  static const bool probe_off = getenv("ISVD_GRAM_PROBE") && getenv("ISVD_GRAM_PROBE")[0] == '0';
  if (mode == kGramF64 && !gate && !probe_off && !op->probe_failed && l <= 512 &&
      use_tensor_cores(rows, l, l, ld, ld, true)) {
    int* flag = &ctx->status->need_exact_gram;
    CK(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    atb_fp32(op, rows, Y, ld, l, nullptr, Y, ld, l, true, s.gram, l, nullptr);
    if (distributed) allreduce_f64(ctx, s.gram, (size_t)l * l);
    CK(launch_chol_inv(s.gram, l, (int)l, ld, s.Rinv32, R64, s.chol_ws, ctx->status, force_fail, nullptr, ctx->stream,
                       1e-5, flag));
    CK(launch_atb(Y, ld, Y, ld, rows, l, l, nullptr, true, op->atb_ws, s.gram, l, nullptr, 0, ctx->num_sms, flag,
                  ctx->stream, false));
    if (distributed) allreduce_f64(ctx, s.gram, (size_t)l * l);  // (unused unless the flag is set)
    CK(launch_chol_inv(s.gram, l, (int)l, ld, s.Rinv32, R64, s.chol_ws, ctx->status, force_fail, flag, ctx->stream));
    gemm_fp32(op, Y, ld, s.Rinv32, ld, Yout, ld, rows, ld, l, nullptr, true, gemm_gate);
    return;
  }
  if (mode == kGramFp32)
    atb_fp32(op, rows, Y, ld, l, nullptr, Y, ld, l, true, s.gram, l, gate);
  else
    CK(launch_atb(Y, ld, Y, ld, rows, l, l, nullptr, true, op->atb_ws, s.gram, l, nullptr, 0, ctx->num_sms, gate,
                  ctx->stream, false));
  if (distributed) allreduce_f64(ctx, s.gram, (size_t)l * l);
  CK(launch_chol_inv(s.gram, l, (int)l, ld, s.Rinv32, R64, s.chol_ws, ctx->status, force_fail, gate, ctx->stream));
  gemm_fp32(op, Y, ld, s.Rinv32, ld, Yout, ld, rows, ld, l, nullptr, true, gemm_gate ? gemm_gate : gate);
}

// CholeskyQR2 (+ a third, device-gated pass after a shifted factorisation): result in Y.
// If Rout != null it receives R = R_3 R_2 R_1 (so that Y_in = Y_out R).
// exact_gram: pass 1 takes the fp64 Gram (input possibly ill-conditioned: Y = M Omega);
// otherwise Y = M Q with Q orthonormal (cond(Y) <= cond(M)) and pass 1 takes the fp32-class
// Gram, as does pass 2 (input orthonormal to ~1e-2 or better).
void cqr2(isvd_op op, float* Y, float* Y2, int64_t rows, bool distributed, int64_t l, bool force_fail, double* Rout,
          bool exact_gram) {
  isvd_ctx ctx = op->g->ctx;
  SolverWs& s = op->sws;
  const int64_t ld = round_up(l, 4);
  int* gate = &ctx->status->need_extra_pass;
  CK(cudaMemsetAsync(gate, 0, sizeof(int), ctx->stream));
  cqr_pass(op, Y, Y2, rows, distributed, l, Rout ? s.Ra : nullptr, exact_gram ? kGramF64 : kGramFp32, force_fail,
           nullptr);
  cqr_pass(op, Y2, Y, rows, distributed, l, Rout ? s.Rb : nullptr, kGramFp32, false, nullptr);
  cqr_pass(op, Y, Y2, rows, distributed, l, Rout ? s.Rc : nullptr, kGramF64, false, gate);
  CK(launch_scale_rows(Y2, ld, Y, ld, rows, ld, nullptr, 1.f, gate, ctx->stream));  // copy back iff pass 3 ran
  if (Rout) {
    CK(launch_trmm(s.Rb, s.Ra, s.Rab, (int)l, nullptr, ctx->stream));
    CK(launch_trmm(s.Rc, s.Rab, Rout, (int)l, gate, ctx->stream));
  }
}

}  // namespace

}  // extern "C"

extern "C" {

isvd_status isvd_sample_omega(isvd_op op, const isvd_svd_params* params, float* omega, int64_t ldo) {
  if (!op || !params || !omega) return ISVD_ERR_INVALID_ARG;
  isvd_ctx ctx = op->g->ctx;
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    int64_t r, c;
    op_shape(op, &r, &c);
    REQ(params->k >= 1 && params->k <= std::min(r, c), ISVD_ERR_RANK, "k must be in [1, min(r, c)]");
    int64_t l = working_l(op, params);
    REQ(ldo >= round_up(l, 4) && ldo % 4 == 0 && aligned16(omega), ISVD_ERR_INVALID_ARG, "bad omega ld");
    int64_t row0 = op->kind == ISVD_OP_POWER_SUM ? op->g->row_begin : 0;
    CK(launch_omega(params->seed, row0, c_rows_local(op), (int)l, ldo, omega, nullptr, ctx->stream));
  });
}

isvd_status isvd_embeddings(isvd_ctx ctx, int64_t rows, int64_t k, const float* M, int64_t ldm, const double* S,
                            float* out, int64_t ldo) {
  if (!ctx) return ISVD_ERR_INVALID_ARG;
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    REQ(rows >= 0 && k >= 1 && M && out && S, ISVD_ERR_INVALID_ARG, "null argument or bad shape");
    REQ(ldm >= round_up(k, 4) && ldo >= round_up(k, 4) && ldm % 4 == 0 && ldo % 4 == 0 && aligned16(M) &&
            aligned16(out),
        ISVD_ERR_INVALID_ARG, "ld must be a multiple of 4, >= round_up(k, 4), 16-byte aligned");
    std::vector<float> r(round_up(k, 4), 0.f);
    for (int64_t j = 0; j < k; ++j) {
      REQ(std::isfinite(S[j]) && S[j] >= 0.0, ISVD_ERR_NONFINITE, "singular values must be finite and >= 0");
      r[j] = (float)std::sqrt(S[j]);  // S^1/2 (Eq. 5), fp64 sqrt rounded once
    }
    std::vector<void*> tmp;
    struct Tmp {
      std::vector<void*>& v;
      isvd_ctx c;
      ~Tmp() { for (void* q : v) dfree(c, q); }
    } tmp_free{tmp, ctx};
    float* dr = (float*)dmalloc(ctx, sizeof(float) * r.size(), tmp);
    CK(cudaMemcpyAsync(dr, r.data(), sizeof(float) * r.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(launch_scale_cols(M, ldm, out, ldo, rows, round_up(k, 4), dr, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

isvd_status isvd_least_norm(isvd_ctx ctx, int64_t r_local, int64_t k, const float* U, int64_t ldu, const double* S,
                            int64_t r, int64_t c, int64_t v_rows, const float* V, int64_t ldv, int64_t ny,
                            const float* Y, int64_t ldy, const int32_t* rows, int64_t n_rows, float* W,
                            int64_t ldw) {
  if (!ctx) return ISVD_ERR_INVALID_ARG;
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    REQ(U && S && V && Y && W && k >= 1 && ny >= 1 && r_local >= 0 && v_rows >= 0 && r >= 1 && c >= 1,
        ISVD_ERR_INVALID_ARG, "null argument or bad shape");
    const int64_t kp = round_up(k, 4), nyp = round_up(ny, 4);
    for (int64_t ld_ : {ldu, ldv})
      REQ(ld_ >= kp && ld_ % 4 == 0, ISVD_ERR_INVALID_ARG, "ldu / ldv must be multiples of 4 >= round_up(k, 4)");
    for (int64_t ld_ : {ldy, ldw})
      REQ(ld_ >= nyp && ld_ % 4 == 0, ISVD_ERR_INVALID_ARG, "ldy / ldw must be multiples of 4 >= round_up(ny, 4)");
    REQ(aligned16(U) && aligned16(V) && aligned16(Y) && aligned16(W), ISVD_ERR_INVALID_ARG,
        "operands must be 16-byte aligned");
    for (int64_t j = 0; j < k; ++j) REQ(std::isfinite(S[j]), ISVD_ERR_NONFINITE, "non-finite singular value");
    REQ(!rows || (n_rows >= 0 && n_rows <= r_local), ISVD_ERR_INVALID_ARG, "bad row subset");
    std::vector<void*> tmp;
    struct Tmp {
      std::vector<void*>& v;
      isvd_ctx c;
      ~Tmp() { for (void* q : v) dfree(c, q); }
    } tmp_free{tmp, ctx};
    // labelled rows of U and Y (option (i))
    const float* Ua = U;
    const float* Ya = Y;
    int64_t nr = r_local, lda = ldu, ldb = ldy;
    if (rows) {
      nr = n_rows;
      float* u2 = (float*)dmalloc(ctx, sizeof(float) * std::max<int64_t>(nr, 1) * kp, tmp);
      float* y2 = (float*)dmalloc(ctx, sizeof(float) * std::max<int64_t>(nr, 1) * nyp, tmp);
      if (nr > 0) {
        CK(launch_scale_rows(U, ldu, u2, kp, nr, kp, nullptr, 1.f, nullptr, ctx->stream, rows));
        CK(launch_scale_rows(Y, ldy, y2, nyp, nr, nyp, nullptr, 1.f, nullptr, ctx->stream, rows));
      }
      Ua = u2; Ya = y2; lda = kp; ldb = nyp;
    }
    // T = U^T Y, exact fp64, then the sum over ranks
    double* ws = (double*)dmalloc(ctx, sizeof(double) * atb_ws_doubles(nr, k, ny, ctx->num_sms), tmp);
    double* T = (double*)dmalloc(ctx, sizeof(double) * k * ny, tmp);
    CK(launch_atb(Ua, lda, Ya, ldb, nr, k, ny, nullptr, false, ws, T, ny, nullptr, 0, ctx->num_sms, nullptr,
                  ctx->stream, false));
    allreduce_f64(ctx, T, (size_t)k * ny);
    // S^+ T on the host (k x ny, small), reading O24's cut
    std::vector<double> h((size_t)k * ny);
    CK(cudaMemcpyAsync(h.data(), T, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double smax = 0.0;
    for (int64_t j = 0; j < k; ++j) smax = std::max(smax, S[j]);
    const double tol = (double)std::max(r, c) * 2.220446049250313e-16 * smax;
    std::vector<float> t32((size_t)k * nyp, 0.f);
    for (int64_t i = 0; i < k; ++i) {
      const double inv = S[i] > tol ? 1.0 / S[i] : 0.0;
      for (int64_t j = 0; j < ny; ++j) t32[(size_t)i * nyp + j] = (float)(inv * h[(size_t)i * ny + j]);
    }
    float* dT = (float*)dmalloc(ctx, sizeof(float) * t32.size(), tmp);
    CK(cudaMemcpyAsync(dT, t32.data(), sizeof(float) * t32.size(), cudaMemcpyHostToDevice, ctx->stream));
    // W = V (S^+ T)
    if (v_rows > 0)
      CK(launch_gemm_tn(V, ldv, dT, nyp, W, ldw, v_rows, nyp, k, nullptr, 1.f, false, nullptr, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

isvd_status isvd_spectral_kernel(const double* S, int64_t k, double mu, double s_bar, double* out) {
  if (!S || !out || k < 0) return ISVD_ERR_INVALID_ARG;
  if (!std::isfinite(mu) || !std::isfinite(s_bar)) return ISVD_ERR_NONFINITE;
  constexpr int kGrid = 301;  // Omega = {0.5, 0.505, ..., 2.0}
  double w[kGrid], mx = -INFINITY;
  const double sc = std::exp(s_bar);
  for (int t = 0; t < kGrid; ++t) {
    const double x = 0.5 + 0.005 * t;
    w[t] = -(x - mu) * (x - mu) * sc;
    mx = std::max(mx, w[t]);
  }
  double z = 0.0;
  for (int t = 0; t < kGrid; ++t) z += (w[t] = std::exp(w[t] - mx));  // softmax, max-shifted
  for (int t = 0; t < kGrid; ++t) w[t] /= z;
  for (int64_t i = 0; i < k; ++i) {
    if (!(S[i] >= 0.0) || !std::isfinite(S[i])) return ISVD_ERR_NONFINITE;
    double acc = 0.0;
    for (int t = 0; t < kGrid; ++t) acc += std::pow(S[i], 0.5 + 0.005 * t) * w[t];
    out[i] = acc;
  }
  return ISVD_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ the solver body
namespace {

// CholeskyQR2 of a tall Y whose orthonormal factor is only ever consumed through products with
// small matrices (M^T Q, then Q U_B): the second pass's update Q2 = Q1 R2^-1 -- a full tall GEMM
// -- is not formed; Q1 is returned (in Y2) with Rfold = R2^-1, and consumers apply Rfold on the
// small side: M^T Q2 = (M^T Q1) Rfold, Q2 U_B = Q1 (Rfold U_B).  Exact in exact arithmetic;
// R2 = I + O(eps1) is perfectly conditioned, so nothing is lost in floating point.
// If the device flags a shifted factorisation, Q2 is formed after all (gated GEMM), the shifted
// third pass runs on it into Y2, and Rfold = I.  Returns the buffer holding the tall factor.
float* cqr2_deferred(isvd_op op, float* Y, float* Y2, int64_t rows, int64_t l, bool force_fail, bool exact_gram) {
  isvd_ctx ctx = op->g->ctx;
  SolverWs& s = op->sws;
  const int64_t ld = round_up(l, 4);
  int* gate = &ctx->status->need_extra_pass;
  CK(cudaMemsetAsync(gate, 0, sizeof(int), ctx->stream));
  cqr_pass(op, Y, Y2, rows, true, l, nullptr, exact_gram ? kGramF64 : kGramFp32, force_fail, nullptr);
  // pass 2: Gram + Cholesky of Q1; Q2 = Q1 R2^-1 only if a third pass will need it
  cqr_pass(op, Y2, Y, rows, true, l, nullptr, kGramFp32, false, nullptr, gate);
  CK(launch_select_rfold(s.Rinv32, s.Rfold, (int)l, ld, gate, ctx->stream));
  cqr_pass(op, Y, Y2, rows, true, l, nullptr, kGramF64, false, gate);
  return Y2;
}

void solver_body(isvd_op op, const isvd_svd_params* p, int64_t l, float* U, int64_t ldu, float* V, int64_t ldv) {
  isvd_graph g = op->g;
  isvd_ctx ctx = g->ctx;
  SolverWs& s = op->sws;
  const int64_t k = p->k;
  const int64_t ld = round_up(l, 4), ldk = round_up(k, 4);
  const bool ne = op->kind == ISVD_OP_POWER_SUM;
  const int64_t cr = c_rows_local(op), rr = r_rows_local(op);
  int64_t r_glob, c_glob;
  op_shape(op, &r_glob, &c_glob);
  const bool force = p->flags & ISVD_SVD_FORCE_CHOL_FAIL;
  CK(cudaMemsetAsync(ctx->status, 0, sizeof(DevStatus), ctx->stream));
  // Alg. 1 line 4: Q ~ N(0,1)^{c x l}
  // (NE on a relabelled graph: Omega's rows are node ids, mapped to the internal order)
  const int32_t* omap = ne ? g->new2old : nullptr;
  {
    Phase ph(ctx, kPhSmall);
    if (p->flags & ISVD_SVD_OMEGA_PROVIDED) {
      CK(launch_scale_rows(p->omega, ld, s.Qc, ld, cr, ld, nullptr, 1.f, nullptr, ctx->stream, omap));
    } else {
      CK(launch_omega(p->seed, ne ? g->row_begin : 0, cr, (int)l, ld, s.Qc, omap, ctx->stream));
    }
  }
  // r-side orthonormalisation: with a small c side (NC) the second CholeskyQR update is folded
  // into the small products (cqr2_deferred); otherwise the plain CholeskyQR2
  const bool fold = !ne && 4 * cr <= r_glob;  // NC: c = d (L + 1) rows, replicated on every rank
  float* q_r = s.Yr;  // buffer holding the r-side orthonormal factor (times Rfold when folding)
  auto orth_r = [&](bool exact) {
    Phase ph(ctx, kPhOrth);
    if (fold) {
      q_r = cqr2_deferred(op, s.Yr, s.Yr2, rr, l, force, exact);
    } else {
      cqr2(op, s.Yr, s.Yr2, rr, true, l, force, nullptr, exact);
      q_r = s.Yr;
    }
  };
  // W = M^T Q into Qc (Q = q_r Rfold when folding)
  auto mt_q = [&]() {
    if (fold) {
      r_matmul_T(op, q_r, ld, s.Qc2, ld, ld, false);
      Phase ph(ctx, kPhProducts);
      gemm_fp32(op, s.Qc2, ld, s.Rfold, ld, s.Qc, ld, cr, ld, l, nullptr, false, nullptr);
    } else {
      r_matmul_T(op, q_r, ld, s.Qc, ld, ld, false);
    }
  };
  // Alg. 1 lines 5-8
  for (int it = 0; it < p->power_iters; ++it) {
    r_matmul(op, s.Qc, ld, s.Yr, ld, ld, false);             // M Q       (r x l)
    orth_r(it == 0);                                         // orthonorm
    mt_q();                                                  // M^T Q     (c x l)
    Phase ph(ctx, kPhOrth);
    cqr2(op, s.Qc, s.Qc2, cr, ne, l, force, nullptr, true);  // orthonorm
  }
  // Alg. 1 line 9: Q <- orthonorm(M Q)
  r_matmul(op, s.Qc, ld, s.Yr, ld, ld, false);
  orth_r(p->power_iters == 0);
  // Alg. 1 line 10: B = (M^T Q)^T, taken as W = M^T Q = Q_W R  (CQR2 keeps R)
  mt_q();
  {
    Phase ph(ctx, kPhOrth);
    cqr2(op, s.Qc, s.Qc2, cr, ne, l, force, s.Rfin, true);
  }
  Phase ph(ctx, kPhSmall);
  // Alg. 1 line 11: svd(B) with B = R^T Q_W^T -> one-sided Jacobi on R^T
  CK(launch_jacobi_svd(s.Rfin, (int)l, (int)k, ldk, s.sigma, s.Ub, s.Vb, s.jac_ws, ctx->status, ctx->num_sms,
                       ctx->stream));
  // Alg. 1 line 12: U = Q U_B;  V = Q_W V_B;  truncate to k
  // (relabelled graphs: rows go back to the caller's order here)
  const float* ub = s.Ub;
  if (fold) {  // U = (Q1 Rfold) U_B = Q1 (Rfold U_B)
    gemm_fp32(op, s.Rfold, ld, s.Ub, ldk, s.Ub2, ldk, l, ldk, l, nullptr, false, nullptr);
    ub = s.Ub2;
  }
  // (a row subset's r-side rows are already in subset order)
  gemm_fp32(op, q_r, ld, ub, ldk, U, ldu, rr, ldk, l, nullptr, false, nullptr, op->has_sub ? nullptr : g->new2old);
  gemm_fp32(op, s.Qc, ld, s.Vb, ldk, V, ldv, cr, ldk, l, nullptr, false, nullptr, ne ? g->new2old : nullptr);
  // sign rule (reading O9)
  CK(launch_col_absmax(U, ldu, rr, (int)k, op->has_sub ? op->sub_offset : g->row_begin, s.absmax_ws, s.cand,
                       ctx->stream));
  const double* cand = s.cand;
  if (ctx->dist) {
    allgather_f64(ctx, s.cand, s.cand_all, 3 * k);
    cand = s.cand_all;
  }
  // sign flip of U and V; the flip of U also flags non-finite output entries (one pass over U)
  CK(launch_sign_flip(cand, ctx->world, (int)k, s.sgn, U, ldu, rr, V, ldv, cr, ctx->stream, ctx->status));
}

}  // namespace

extern "C" {

isvd_status isvd_svd(isvd_op op, const isvd_svd_params* p, float* U, int64_t ldu, double* S, float* V, int64_t ldv,
                     isvd_svd_report* rep) {
  if (!op) return ISVD_ERR_INVALID_ARG;
  isvd_ctx ctx = op->g->ctx;
  if (!p || !U || !S || !V) {
    set_err(ctx, "null argument");
    return ISVD_ERR_INVALID_ARG;
  }
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    int64_t r, c;
    op_shape(op, &r, &c);
    REQ(p->k >= 1 && p->k <= std::min(r, c), ISVD_ERR_RANK, "k must be in [1, min(r, c)]");
    REQ(p->power_iters >= 0, ISVD_ERR_INVALID_ARG, "power_iters must be >= 0");
    REQ((p->flags & ~(uint32_t)(ISVD_SVD_OMEGA_PROVIDED | ISVD_SVD_HOST_OUTPUT | ISVD_SVD_NO_GRAPH |
                                ISVD_SVD_FORCE_CHOL_FAIL | ISVD_SVD_PROFILE)) == 0,
        ISVD_ERR_INVALID_ARG, "unknown svd flag");
    REQ(!(p->flags & ISVD_SVD_OMEGA_PROVIDED) || p->omega, ISVD_ERR_INVALID_ARG, "omega is null");
    REQ(!(p->flags & ISVD_SVD_OMEGA_PROVIDED) || aligned16(p->omega), ISVD_ERR_INVALID_ARG,
        "omega must be 16-byte aligned (its rows are read as float4, ld = round_up(l, 4))");
    const int64_t l = working_l(op, p);
    REQ(l <= 1024, ISVD_ERR_UNSUPPORTED, "working width l > 1024 is not supported by the small-matrix kernels");
    const int64_t k = p->k, ldk = round_up(k, 4);
    const bool host_out = p->flags & ISVD_SVD_HOST_OUTPUT;
    REQ(ldu >= ldk && ldv >= ldk, ISVD_ERR_INVALID_ARG, "ldu and ldv must be >= round_up(k, 4)");
    if (!host_out) REQ(aligned16(U) && aligned16(V) && ldu % 4 == 0 && ldv % 4 == 0, ISVD_ERR_INVALID_ARG,
                       "U and V must be 16-byte aligned with ld a multiple of 4");
    ensure_op_ws(op, round_up(l, 4));
    ensure_solver_ws(op, l, k);
    SolverWs& s = op->sws;
    // The solver runs on the context's private stream, joined to the caller's stream by
    // events; without ISVD_SVD_NO_GRAPH / ISVD_SVD_PROFILE (and outside the simulated-rank
    // backend) the whole enqueue sequence is captured once per argument set into a CUDA graph
    // and replayed (one launch per isvd), writing U / V into the op's buffers.
    const bool use_graph = !(p->flags & (ISVD_SVD_NO_GRAPH | ISVD_SVD_PROFILE)) && !s.graph_broken && !ctx->sim;
    const bool staged = host_out || use_graph;
    float* Ud = staged ? s.Utmp : U;
    float* Vd = staged ? s.Vtmp : V;
    const int64_t lduu = staged ? ldk : ldu, ldvv = staged ? ldk : ldv;
    cudaStream_t user = ctx->stream;
    CK(cudaEventRecord(ctx->ev_join, user));
    CK(cudaStreamWaitEvent(ctx->work, ctx->ev_join, 0));
    struct StreamSwap {
      isvd_ctx c;
      cudaStream_t u;
      ~StreamSwap() { c->stream = u; c->profiling = false; }
    } swap_back{ctx, user};
    ctx->stream = ctx->work;
    ctx->profiling = p->flags & ISVD_SVD_PROFILE;
    ctx->phase_tag.clear();
    ctx->n_ag = ctx->n_lp = 0;
    const uint64_t key = graph_key(p, l, ldk) ^ (op->probe_failed ? 0x9E3779B97F4A7C15ULL : 0);
    int64_t launches = 0;
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    if (use_graph && (s.graph_exec == nullptr || s.graph_key != key)) {
      if (s.graph_exec) cudaGraphExecDestroy(s.graph_exec);
      s.graph_exec = nullptr;
      ctx->spmm_steps = 0;
      ctx->spmm_alg_bytes = 0.0;
      const int64_t l0 = g_launches;
      bool ok = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      if (ok) {
        try {
          solver_body(op, p, l, Ud, lduu, Vd, ldvv);
        } catch (const Fail&) {
          ok = false;
        }
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
        ok = ok && e == cudaSuccess && graph != nullptr &&
             cudaGraphInstantiate(&s.graph_exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
      }
      if (!ok) {  // some launch could not be captured: run eagerly for this op from now on
        (void)cudaGetLastError();
        if (s.graph_exec) cudaGraphExecDestroy(s.graph_exec);
        s.graph_exec = nullptr;
        s.graph_broken = true;
        ctx->last_error.clear();
      } else {
        s.graph_key = key;
        s.graph_launches = g_launches - l0;
        s.graph_spmm_steps = ctx->spmm_steps;
        s.graph_alg_bytes = ctx->spmm_alg_bytes;
      }
    }
    if (use_graph && s.graph_exec) {
      CK(cudaGraphLaunch(s.graph_exec, ctx->stream));
      launches = s.graph_launches;
      ctx->spmm_steps = s.graph_spmm_steps;
      ctx->spmm_alg_bytes = s.graph_alg_bytes;
    } else {
      ctx->spmm_steps = 0;
      ctx->spmm_alg_bytes = 0.0;
      const int64_t l0 = g_launches;
      solver_body(op, p, l, Ud, lduu, Vd, ldvv);
      launches = g_launches - l0;
    }
    const int64_t rr = r_rows_local(op), cr = c_rows_local(op);
    if (staged && !host_out) {  // the op's U / V buffers -> the caller's device outputs
      if (rr > 0)
        CK(cudaMemcpy2DAsync(U, ldu * sizeof(float), Ud, lduu * sizeof(float), ldk * sizeof(float), rr,
                             cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpy2DAsync(V, ldv * sizeof(float), Vd, ldvv * sizeof(float), ldk * sizeof(float), cr,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    DevStatus st;
    std::vector<double> sig(k);
    CK(cudaMemcpyAsync(sig.data(), s.sigma, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&st, ctx->status, sizeof(DevStatus), cudaMemcpyDeviceToHost, ctx->stream));
    if (host_out) {
      if (rr > 0)
        CK(cudaMemcpy2DAsync(U, ldu * sizeof(float), Ud, lduu * sizeof(float), k * sizeof(float), rr,
                             cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpy2DAsync(V, ldv * sizeof(float), Vd, ldvv * sizeof(float), k * sizeof(float), cr,
                           cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->comm) {  // a failed peer / network error surfaces here instead of as a hang later
      ncclResult_t aerr = ncclSuccess;
      NK(ncclCommGetAsyncError(ctx->comm, &aerr));
      REQ(aerr == ncclSuccess, ISVD_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(aerr));
    }
    CK(cudaEventRecord(ctx->ev_join, ctx->stream));
    CK(cudaStreamWaitEvent(user, ctx->ev_join, 0));
    // a probe that fell back on real data (not a forced breakdown) will fall back again on the next
    // call with the same operator: take the exact Gram directly from then on (a new graph key)
    const bool skipped_probe = op->probe_failed;
    if (st.probes_failed > 0 && !(p->flags & ISVD_SVD_FORCE_CHOL_FAIL)) op->probe_failed = true;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    if (rep) {
      rep->l = (int32_t)l;
      rep->ld = (int32_t)round_up(l, 4);
      rep->chol_fallbacks = st.chol_breakdown;
      rep->gram_probe_fallbacks = st.probes_failed;
      rep->gram_probe_skipped = skipped_probe ? 1 : 0;
      rep->jacobi_sweeps = st.jacobi_sweeps;
      rep->world = ctx->world;
      rep->kernel_launches = (int32_t)launches;
      rep->ms_total = ms;
      rep->spmm_steps = ctx->spmm_steps;
      rep->spmm_alg_bytes = ctx->spmm_alg_bytes;
      rep->ms_spmm = 0.0;
      rep->ms_products = rep->ms_orth = rep->ms_small = rep->ms_comm = 0.0;
      if (p->flags & ISVD_SVD_PROFILE) {
        for (int i = 0; i < ctx->spmm_steps; ++i) {
          float t = 0.f;
          CK(cudaEventElapsedTime(&t, ctx->prof_events[2 * i], ctx->prof_events[2 * i + 1]));
          rep->ms_spmm += t;
        }
        double* acc[4] = {&rep->ms_products, &rep->ms_orth, &rep->ms_small, &rep->ms_comm};
        for (size_t i = 0; i < ctx->phase_tag.size(); ++i) {
          float t = 0.f;
          CK(cudaEventElapsedTime(&t, ctx->phase_ev[2 * i], ctx->phase_ev[2 * i + 1]));
          *acc[ctx->phase_tag[i]] += t;
        }
        // all-gather / local-pass overlap: intervals relative to the call's start event; each
        // split all-gather is paired with the local pass issued while it was in flight
        rep->ms_allgather = rep->ms_allgather_hidden = 0.0;
        for (size_t i = 0; i < ctx->n_ag; ++i) {
          float a0 = 0.f, a1 = 0.f;
          CK(cudaEventElapsedTime(&a0, ctx->ev0, ctx->ag_ev[2 * i]));
          CK(cudaEventElapsedTime(&a1, ctx->ev0, ctx->ag_ev[2 * i + 1]));
          rep->ms_allgather += a1 - a0;
          if (i < ctx->n_lp) {
            float l0 = 0.f, l1 = 0.f;
            CK(cudaEventElapsedTime(&l0, ctx->ev0, ctx->lp_ev[2 * i]));
            CK(cudaEventElapsedTime(&l1, ctx->ev0, ctx->lp_ev[2 * i + 1]));
            rep->ms_allgather_hidden += std::max(0.f, std::min(a1, l1) - std::max(a0, l0));
          }
        }
      }
    }
    REQ(!st.chol_failed, ISVD_ERR_NOT_PD, "Cholesky of Q^T Q failed even after the shifted retries");
    REQ(!st.nonfinite, ISVD_ERR_NONFINITE, "non-finite value in the solver output");
    for (int64_t i = 0; i < k; ++i) S[i] = sig[i];
  });
}

}  // extern "C"
