#!/usr/bin/env python
"""Benchmark of the implicit randomized SVD hot path (arXiv 2111.06312) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--impl isvd|reference]

One "step" is one rank-k implicit SVD (Alg. 1) of the
config's implicit design matrix: every product M Q / M^T Q, every CholeskyQR2,
the small SVD and the final U, V -- the whole hot path.  The default workload
is config 4 (NC design matrix [X | AX | A^2X | A^3X] of a 2.45M-node power-law
graph, k = 256, l = 400, q = 2): the configuration the metric's HBM-bandwidth
clause and the 1/2/4/8-GPU scaling are quoted on.
Inputs are synthetic (synth/), resident in HBM when the timed region starts,
and larger than the 126 MB L2 (no flush needed).

For N > 1 the driver launches one process per GPU with torchrun; rows are
partitioned (strong scaling: one isvd of the same matrix over N GPUs).
Rank 0 prints ONE JSON line.

`--impl reference` times the fp64 CPU oracle (oracle/, the reference arm of this
tier) on a bounded sample of the same workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rank-k implicit SVD time (s); fused SpMM HBM GB/s vs ~8 TB/s B200 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="isvd", choices=["isvd", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ oracle arm
class ColumnParallel:
    """Harness adapter (not oracle arithmetic): the oracle operator's products applied to column
    chunks in a thread pool.  Columns of M.G and M^T.H are independent and scipy's sparse kernels
    release the GIL, so this spreads the oracle's own per-column computation over the host cores;
    BLAS inside each chunk runs single-threaded (no oversubscription).  Accumulates the time spent
    in products (`t_products`)."""

    def __init__(self, op, workers):
        self.op, self.workers = op, max(1, int(workers))
        self.t_products = 0.0

    @property
    def shape(self):
        return self.op.shape

    def _par(self, fn, M):
        import numpy as np
        from concurrent.futures import ThreadPoolExecutor
        from threadpoolctl import threadpool_limits

        t0 = time.perf_counter()
        chunks = [c for c in np.array_split(np.arange(M.shape[1]), self.workers) if c.size]
        with threadpool_limits(1), ThreadPoolExecutor(len(chunks)) as ex:
            parts = list(ex.map(lambda c: fn(np.ascontiguousarray(M[:, c])), chunks))
        out = np.concatenate(parts, axis=1)
        self.t_products += time.perf_counter() - t0
        return out

    def matmul(self, G):
        return self._par(self.op.matmul, G)

    def matmul_T(self, H):
        return self._par(self.op.matmul_T, H)


# full oracle isvd of config 4 on the GPU box's 16 cores (round 2, profiles/r02_oracle_full_cfg4.json)
FULL_ORACLE_CFG4_S = 477.06


def oracle_isvd_timed(cfg, g, X, sp, full=None):
    """The fp64 oracle's Alg. 1 (oracle/) on the host cores, timed from Omega in to U, s, V out:
    its own Omega (reading O11), definition-level products (column chunks in parallel,
    ColumnParallel), Householder QR (LAPACK, all cores), LAPACK SVD of B, U = Q U_B.

    full (default: configs with n <= 1M): one complete oracle isvd, value = the measured time.
    Otherwise (config 4, whose full run takes ~8 minutes on the 16-core GPU host,
    FULL_ORACLE_CFG4_S): the bounded sample is one full-width (l = 400) oracle application
    M.Omega -- the same column-chunked products, all L = 3 SpMM steps and 4 dense terms -- and
    value = its time x (2q + 2) applications (products only; the QRs and the SVD of B add ~10 %)."""
    from threadpoolctl import threadpool_info

    from oracle import NCOperator, NEOperator, adjacency, isvd, philox_omega

    A = adjacency(g.n, g.row_ptr, g.col_idx)
    ref = NEOperator(A, sp["weights"], sp["lambda_ones"]) if cfg["op"] == "NE" else NCOperator(A, X, sp["L"])
    cores = os.cpu_count() or 1
    par = ColumnParallel(ref, cores)
    if full is None:
        full = cfg["n"] <= 1_000_000
    blas = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
    nb = max(blas) if blas else 1
    t0 = time.perf_counter()
    om = philox_omega(sp["seed"], 0, ref.shape[1], sp["l"])
    if full:
        U, s, V, _ = isvd(par, sp["k"], om, sp["q"])
        value = time.perf_counter() - t0
        sample = (f"one full fp64 oracle isvd of {cfg['name']} (Alg. 1: Omega, {2 * sp['q'] + 2} products, "
                  f"{2 * sp['q'] + 2} Householder QRs, LAPACK SVD of B, U/V) measured: {value:.2f} s; products on "
                  f"{cores} threads (column chunks, {par.t_products:.2f} s), QR/SVD on {nb} BLAS threads")
        return value, cores, sample, s
    par.matmul(om)
    t = time.perf_counter() - t0
    apps = 2 * sp["q"] + 2
    value = t * apps
    sample = (f"bounded sample: one full-width (l = {sp['l']}) fp64 oracle application M.Omega of {cfg['name']} "
              f"(Omega + {sp.get('L', 0)} SpMM steps + dense terms, {cores} threads, column chunks) measured "
              f"{t:.1f} s, x {apps} applications = {value:.0f} s (products only; QR / SVD of B excluded).  One full "
              f"oracle isvd of this config measured {FULL_ORACLE_CFG4_S:.0f} s on the same 16-core host "
              "(profiles/r02_oracle_full_cfg4.json; `bench.py --impl reference` runs it in full)")
    return value, cores, sample, None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import get_config, make_features, make_graph, solver_params

    cfg = get_config(args.config)
    g = make_graph(cfg)
    X = make_features(cfg["n"], cfg["d"], cfg["seed"]) if cfg["op"] == "NC" else None
    sp = solver_params(cfg)
    # each step is one FULL oracle isvd (the verdict of round 1 asked for it at every config); config 4
    # takes ~8 minutes on the GPU host, so it runs once there, and at most 5 times elsewhere
    runs = 1 if cfg["n"] > 1_000_000 else max(1, min(args.steps, 5))
    times = []
    cores, sample = 1, ""
    for _ in range(runs):
        v, cores, sample, _ = oracle_isvd_timed(cfg, g, X, sp, full=True)
        times.append(v)
    v = statistics.median(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": runs,
        "warmup": 0, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "n": cfg["n"], "m": cfg["m"], "k": sp["k"], "l": sp["l"], "q": sp["q"]},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "oracle",
                         "sample": sample + f"; {runs} run(s), median (--steps {args.steps} --warmup {args.warmup} "
                                            "requested; at most 5 runs, config 4 once, no warm-up)"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ GPU arm
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(workload):
    """dram read+write bytes per SpMM launch from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "spmm_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if d.get("workload") == workload:
            return d.get("dram_bytes_per_launch")
    return None


def gather_floor(g, sp, world, alg_bytes_per_launch, avg_launch_ms):
    """A floor for one SpMM step of a relabelled single-GPU graph: the gathers of
    rows outside the 79 MB persisting hub window must come from DRAM at <= 6.3 TB/s (measured random
    1600-B row gathers, profiles/r02_l2_gather_bench2.jsonl) and the rest of the algorithmic bytes
    (CSR, scales, epilogue operand, output) at the measured copy peak.  Row sums of the degree
    sequence give the hub share exactly."""
    import numpy as np

    l = sp["l"]
    ld = (l + 3) // 4 * 4
    if world != 1 or 4 * g.n * ld < 8 * 126e6 or not avg_launch_ms:  # gather source must dwarf L2
        return None
    rows_in_window = int(79e6 // (4 * ld))
    deg = np.sort(np.diff(g.row_ptr))[::-1]
    hub_share = float(deg[:rows_in_window].sum() / deg.sum())
    cold = 4.0 * ld * float(deg[rows_in_window:].sum())
    rest = alg_bytes_per_launch - 4.0 * g.n * ld
    peak, _ = load_peaks()
    floor_ms = (cold / 6.3e12 + rest / (peak * 1e9)) * 1e3
    out = {"floor_ms": floor_ms, "achieved_ms": avg_launch_ms, "frac": floor_ms / avg_launch_ms,
           "hub_share_of_gathers": hub_share, "cold_gather_GB": cold / 1e9,
           "basis": "cold-row gathers at the measured 6.3 TB/s random-1600B-row DRAM rate + the other algorithmic "
                    "bytes at the measured copy peak (DESIGN.md §6)"}
    if l == 400 and g.n > 2_000_000:
        # the same gather mix as a pure-gather microbenchmark on this hardware (config 4 only):
        # profiles/hub_gather_bench.cu, 41.5 % of 1600-B row gathers on a 78 MB hub prefix with the
        # persisting window, the rest uniform over 3.9 GB: 24.7 ms per 198 GB (4 nnz l bytes)
        gv = 4.0 * ld * float(deg.sum())
        mix_ms = 24.7 * gv / 198e9
        out["measured_gather_mix"] = {"ms": mix_ms, "frac": mix_ms / avg_launch_ms,
                                      "source": "profiles/hub_gather_bench.cu (profiles/r02e_spmm_sorted_hint.jsonl)"}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_2111_06312_b200 import _build

    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()
    import paper_2111_06312_b200 as isvd
    from synth import get_config, make_features, make_graph, solver_params

    cfg = get_config(args.config)
    sp = solver_params(cfg)
    g = make_graph(cfg)
    X = make_features(cfg["n"], cfg["d"], cfg["seed"]) if cfg["op"] == "NC" else None

    nid = None
    if world > 1:
        obj = [isvd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    ctx = isvd.Context(local_rank, rank=rank, world=world, nccl_id=nid)
    rb, nl = isvd.partition(g.n, world, rank)
    rp, ci = g.row_slice(rb, rb + nl)
    Xl = None if X is None else np.ascontiguousarray(X[rb : rb + nl])

    def make_op(device_resident=True):
        if device_resident:
            graph = isvd.Graph(ctx, g.n, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
            if cfg["op"] == "NE":
                return isvd.NE(graph, sp["weights"], sp["lambda_ones"]), graph
            return isvd.NC(graph, torch.from_numpy(Xl).cuda(), sp["L"]), graph
        graph = isvd.Graph(ctx, g.n, rp_pin, ci_pin)
        if cfg["op"] == "NE":
            return isvd.NE(graph, sp["weights"], sp["lambda_ones"]), graph
        return isvd.NC(graph, X_pin, sp["L"]), graph

    p = -1 if cfg["p"] is None else cfg["p"]
    op, graph = make_op(True)
    torch.cuda.synchronize()

    # outputs allocated once, outside the timed region (a fresh torch.zeros per call would put a
    # cudaMalloc and a fill of U -- 2.5 GB at config 4 -- inside every timed step)
    kk4 = (sp["k"] + 3) // 4 * 4
    out_uv = (torch.zeros(max(op.r_rows(), 1), kk4, dtype=torch.float32, device="cuda"),
              torch.zeros(max(op.c_rows(), 1), kk4, dtype=torch.float32, device="cuda"))

    def step(profile=False):
        return op.svd(sp["k"], p, sp["q"], sp["seed"], profile=profile, out=out_uv)

    # headline: the default product path (the solver captured once as a CUDA graph and replayed)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    stream = ctx.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # working sets smaller than twice the 126 MB L2 (configs 0, 1, 3): flush L2 between timed isvds
    # (a 512 MB write, outside the per-step events); config 2 / 4 iterates exceed L2 on their own
    ws_bytes = 4 * cfg["n"] * sp["l"]
    flush = ws_bytes < 2 * 126 * 2 ** 20
    if flush:
        junk = torch.empty(128 * 2 ** 20, dtype=torch.float32, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        results = []
        with torch.cuda.stream(stream):
            for a, b in evs:
                junk.fill_(1.0)
                a.record(stream)
                r_ = step()
                b.record(stream)
                results.append(r_.kernel_launches)
        torch.cuda.synchronize()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        del junk
    else:
        e0.record(stream)
        results = [step().kernel_launches for _ in range(args.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms = None
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = sum(step_ms) / args.steps if flush else e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    launches = sum(results)

    # roofline pass (separate, after the headline): the same isvd run eagerly with every SpMM step
    # bracketed by CUDA events on the library's stream (ISVD_SVD_PROFILE) and per-phase times
    prof_runs = max(1, min(3, args.steps))
    prof = [step(profile=True) for _ in range(prof_runs)]
    spmm_ms = sum(r.ms_spmm for r in prof)
    spmm_n = sum(r.spmm_steps for r in prof)
    spmm_bytes = sum(r.spmm_alg_bytes for r in prof)
    phases = {k_: statistics.median(r.phases[k_] for r in prof) for k_ in prof[0].phases}
    # distributed split: all-gather time on the collectives stream and the part hidden behind the
    # local SpMM passes (CUDA-event intervals of the profiled pass)
    allgather = ({"ms": statistics.median(r.ms_allgather for r in prof),
                  "hidden_ms": statistics.median(r.ms_allgather_hidden for r in prof)} if world > 1 else None)
    ms_prof = statistics.median(r.ms_total for r in prof)

    # ---- variant: tensor cores for every tall contraction (ISVD_TC_PRODUCTS=1), not only the
    # Gram as north_star specifies -- reported beside the headline, never as it
    variants = {}
    if not args.no_variants:
        prev = os.environ.get("ISVD_TC_PRODUCTS")
        os.environ["ISVD_TC_PRODUCTS"] = "1"
        for _ in range(args.warmup):
            step(profile=False)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step(profile=False)
        e1.record(stream)
        torch.cuda.synchronize()
        tv = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tv, op=dist.ReduceOp.MAX)
        variants["tc_products"] = {"value": float(tv.item()) / 1e3, "unit": "s",
                                   "what": "ISVD_TC_PRODUCTS=1: tcgen05 3xTF32 also for X^T Z_j, X G_j, Y R^-1, "
                                           "final U/V (north_star keeps tensor cores to the Gram)"}
        if prev is None:
            del os.environ["ISVD_TC_PRODUCTS"]
        else:
            os.environ["ISVD_TC_PRODUCTS"] = prev
    # ---- variant: NC with M materialised (M = M . I through the library, once),
    # then the same isvd of the explicit n x c matrix (an NC operator with L = 0).  A measured
    # comparison of what "never formed" costs; the matrix-free path stays the contract.
    if not args.no_variants and cfg["op"] == "NC" and world == 1:
        c = op.shape[1]
        eye = torch.eye(c, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        e0.record(stream)
        Mx = op.matmul(eye)
        e1.record(stream)
        torch.cuda.synchronize()
        t_mat = e0.elapsed_time(e1) / 1e3
        del eye
        opm = isvd.NC(graph, Mx, 0)
        for _ in range(args.warmup):
            opm.svd(sp["k"], p, sp["q"], sp["seed"])
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            opm.svd(sp["k"], p, sp["q"], sp["seed"])
        e1.record(stream)
        torch.cuda.synchronize()
        variants["materialised_M"] = {
            "value": e0.elapsed_time(e1) / args.steps / 1e3, "unit": "s", "materialise_s": t_mat,
            "what": "NC with M = [X|AX|A^2X|A^3X] formed once (M . I) and the isvd run on the explicit "
                    "n x c matrix (SURVEY 8(f) f3, comparison only; north_star: M never materialised)"}
        opm.close()
        del Mx
    # ---- variants: NE with A held dense (n <= 32768), every SpMM step on tensor cores
    # plus the same fp64 epilogue: the exact INT8 product (ISVD_DENSE_A=1) and 3xTF32 (=2).  Comparison
    # only (same flush policy as the headline).
    if not args.no_variants and cfg["op"] == "NE" and world == 1 and cfg["n"] <= 32768:
        for dmode, dname, what in (
                ("1", "dense_A_i8", "exact INT8 tensor-core product of the binary A with 3-byte fixed-point slices "
                                    "of the gather source (dense_i8.cu)"),
                ("2", "dense_A_tf32", "tcgen05 3xTF32 row contraction A^T Y (gram_tc.cu)")):
            os.environ["ISVD_DENSE_A"] = dmode
            try:
                gd = isvd.Graph(ctx, g.n, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
            finally:
                del os.environ["ISVD_DENSE_A"]
            opd = isvd.NE(gd, sp["weights"], sp["lambda_ones"])
            for _ in range(args.warmup):
                opd.svd(sp["k"], p, sp["q"], sp["seed"])
            torch.cuda.synchronize()
            junk = torch.empty(128 * 2 ** 20, dtype=torch.float32, device="cuda") if flush else None
            tot = 0.0
            with torch.cuda.stream(stream):
                for _ in range(args.steps):
                    if junk is not None:
                        junk.fill_(1.0)
                    e0.record(stream)
                    opd.svd(sp["k"], p, sp["q"], sp["seed"])
                    e1.record(stream)
                    torch.cuda.synchronize()
                    tot += e0.elapsed_time(e1)
            rd = opd.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            variants[dname] = {
                "value": tot / args.steps / 1e3, "unit": "s", "spmm_step_ms": rd.ms_spmm / max(rd.spmm_steps, 1),
                "what": "NE with A held dense (formed at graph creation), every SpMM step as the " + what +
                        " + the same fp64 epilogue (SURVEY 8(f) f3, comparison only)"}
            del junk
            opd.close()
            gd.close()
    op.close()
    graph.close()

    # ---- end-to-end through the public API with host buffers (pinned), H2D + D2H inside
    rp_pin = torch.from_numpy(rp).pin_memory().numpy()
    ci_pin = torch.from_numpy(ci).pin_memory().numpy()
    X_pin = None if Xl is None else torch.from_numpy(Xl).pin_memory().numpy()
    h2d = rp_pin.nbytes + ci_pin.nbytes + (0 if X_pin is None else X_pin.nbytes)
    e2e_times, e2e_create = [], []
    d2h = 0
    host_out = None
    for i in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        op2, graph2 = make_op(False)
        torch.cuda.synchronize()
        tc = time.perf_counter()
        if host_out is None:  # page-locked result buffers, allocated once like the pinned inputs
            host_out = op2.host_buffers(sp["k"])
        r = op2.svd(sp["k"], p, sp["q"], sp["seed"], host_output=True, out=host_out)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        d2h = r.U.nbytes + r.V.nbytes + r.S.nbytes
        op2.close()
        graph2.close()
        if i > 0:  # first is a warm-up (allocator, pinned pages)
            e2e_times.append(t1 - t0)
            e2e_create.append(tc - t0)
    te = torch.tensor([statistics.median(e2e_times) if e2e_times else float("nan")], dtype=torch.float64,
                      device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _ = oracle_isvd_timed(cfg, g, X, sp)
        cpu = {"value": v, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        peak, peak_src = load_peaks()
        achieved = spmm_bytes / (spmm_ms / 1e3) / 1e9 if spmm_ms > 0 else None
        per_launch_bytes = spmm_bytes / spmm_n if spmm_n else None
        line = {
            "metric": METRIC,
            "value": ms_max / 1e3,
            "unit": "s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {
                "workload": cfg["name"], "op": cfg["op"], "n": cfg["n"], "m": cfg["m"], "k": sp["k"], "l": sp["l"],
                "q": sp["q"], "parallelism": f"rows-{world}",
                "l2": ("L2 flushed (512 MB write) before every timed isvd, per-step events" if flush
                       else "inputs larger than L2 (no flush)"),
                "accumulate": "fp32 storage, fp64 accumulation",
            },
            "step_ms": [round(x, 3) for x in step_ms] if step_ms else None,
            "roofline": {
                "bound": "hbm", "kernel": "spmm_kernel (+fixup): fused CSR SpMM step",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "peak_source": peak_src,
                "alg_bytes_per_launch": per_launch_bytes, "launches": spmm_n,
                "avg_launch_ms": spmm_ms / spmm_n if spmm_n else None,
                "share_of_step": (spmm_ms / prof_runs) / ms_prof if ms_prof > 0 else None,
                "measured_on": f"separate profiled pass ({prof_runs} eager isvds, CUDA events around every SpMM "
                               "step on the library stream), after the headline",
                "traffic": load_traffic(cfg["name"]),
                "traffic_source": "ncu --set full capture of this kernel at this config (profiles/spmm_traffic.json)",
                "gather_floor": gather_floor(g, sp, world, per_launch_bytes, spmm_ms / spmm_n if spmm_n else None),
            },
            "phases_ms": phases,
            "allgather": allgather,
            "cpu_baseline": cpu,
            "e2e": {"value": float(te.item()), "unit": "s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "graph_op_create_s": statistics.median(e2e_create) if e2e_create else None},
            "gpu_launches": launches,
            "variants": variants,
            "solver": {"jacobi_sweeps": prof[-1].jacobi_sweeps, "chol_fallbacks": prof[-1].chol_fallbacks,
                       "launches_per_isvd": results[-1]},
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
