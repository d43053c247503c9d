"""World-size-2 CPU (gloo) test of the row-partitioned layout the library uses for P > 1.

Only one GPU exists for this build, so the multi-rank schedule of csrc/capi.cpp is
modelled here step by step in numpy on each rank, with torch.distributed (gloo)
standing in for NCCL:
  * rows [p*ceil(n/P), ...) per rank, from the library's own isvd_partition (C ABI);
  * every SpMM gather source is all-gathered into a padded full-height buffer
    (uniform counts n_pad = ceil(n/P) rows per rank) before the step;
  * column sums, Gram matrices and X^T Z partials are all-reduced (fp64);
  * l x l math is replicated; the sign rule all-gathers per-rank candidates.
The result must equal the single-process oracle (fp64) and be identical on both ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class RankModel:
    """One rank's view: local CSR rows with global column ids, padded all-gathers."""

    def __init__(self, g, rank, world):
        from paper_2111_06312_b200 import partition

        self.n, self.rank, self.world = g.n, rank, world
        self.rb, self.nl = partition(g.n, world, rank)
        self.n_pad = -(-g.n // world)
        rp, ci = g.row_slice(self.rb, self.rb + self.nl)
        self.rp, self.ci = rp, ci.astype(np.int64)
        self.deg = np.diff(rp).astype(np.float64)

    def allgather_rows(self, local):
        """Padded uniform-count all-gather -> the first n rows of the full buffer."""
        w = local.shape[1]
        buf = np.zeros((self.n_pad, w))
        buf[: self.nl] = local
        parts = [torch.zeros(self.n_pad, w, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(parts, torch.from_numpy(buf))
        return torch.cat(parts).numpy()[: self.n]

    def allreduce(self, x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    def gather_step(self, Yfull, self_coef=0.0):
        """sum over local rows' neighbours (global ids) of the full buffer (+ own row)."""
        out = np.zeros((self.nl, Yfull.shape[1]))
        for i in range(self.nl):
            out[i] = Yfull[self.ci[self.rp[i] : self.rp[i + 1]]].sum(axis=0)
        if self_coef:
            out += self_coef * Yfull[self.rb : self.rb + self.nl]
        return out

    # ---- NE (Eq. 3), Horner as in ne_matmul / ne_matmul_T
    def ne_matmul(self, Q, w, lam):
        inv = np.where(self.deg > 0, 1.0 / np.maximum(self.deg, 1), 0.0)[:, None]
        cs = self.allreduce(Q.sum(axis=0))
        src = self.allgather_rows(Q)
        C = len(w)
        for c in range(C - 1, 0, -1):
            coef = w[C - 1] if c == C - 1 else 1.0
            H = coef * inv * self.gather_step(src) + w[c - 1] * Q
            src = self.allgather_rows(H)
        coef = w[0] if C == 1 else 1.0
        return coef * inv * self.gather_step(src) - lam * cs[None, :]

    def ne_matmul_T(self, Q, w, lam):
        inv = np.where(self.deg > 0, 1.0 / np.maximum(self.deg, 1), 0.0)[:, None]
        cs = self.allreduce(Q.sum(axis=0))
        C = len(w)
        src = self.allgather_rows(w[C - 1] * inv * Q)
        for c in range(C - 1, 0, -1):
            src = self.allgather_rows(inv * (self.gather_step(src) + w[c - 1] * Q))
        return self.gather_step(src) - lam * cs[None, :]

    # ---- NC (Eq. 6), pre-scaled iterates as in nc_matmul / nc_matmul_T
    def nc_matmul(self, Xl, G, L):
        d = Xl.shape[1]
        s = (1.0 / np.sqrt(self.deg + 1.0))[:, None]
        cur = self.allgather_rows(s * (Xl @ G[L * d : (L + 1) * d]))
        for j in range(L - 1, 0, -1):
            nxt = s * (Xl @ G[j * d : (j + 1) * d]) + s * s * self.gather_step(cur, 1.0)
            cur = self.allgather_rows(nxt)
        return Xl @ G[:d] + s * self.gather_step(cur, 1.0)

    def nc_matmul_T(self, Xl, Q, L):
        s = (1.0 / np.sqrt(self.deg + 1.0))[:, None]
        blocks = [Xl.T @ Q]
        Zt = s * Q
        for j in range(1, L + 1):
            Zt = s * s * self.gather_step(self.allgather_rows(Zt), 1.0)
            blocks.append(Xl.T @ (Zt / s))
        return self.allreduce(np.vstack(blocks))

    def cqr2(self, Y, distributed=True):
        for _ in range(2):
            G = Y.T @ Y
            if distributed:
                G = self.allreduce(G)
            R = np.linalg.cholesky(G).T
            Y = np.linalg.solve(R.T, Y.T).T
        return Y


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import NCOperator, NEOperator, adjacency, philox_omega
        from synth.graphs import powerlaw_graph

        g = powerlaw_graph(301, 900, 2.5, seed=5)  # n not a multiple of world: ragged last block
        m = RankModel(g, rank, world)
        A = adjacency(g.n, g.row_ptr, g.col_idx)
        rng = np.random.default_rng(0)
        res = {}
        # NE products
        w, lam = [0.2] * 5, 1.0 / g.n
        Q = rng.standard_normal((g.n, 6))
        ref = NEOperator(A, w, lam)
        sl = slice(m.rb, m.rb + m.nl)
        res["ne"] = np.abs(m.ne_matmul(Q[sl], w, lam) - ref.matmul(Q)[sl]).max()
        res["neT"] = np.abs(m.ne_matmul_T(Q[sl], w, lam) - ref.matmul_T(Q)[sl]).max()
        # NC products
        X = rng.standard_normal((g.n, 4))
        refc = NCOperator(A, X, 3)
        G = rng.standard_normal((16, 6))
        res["nc"] = np.abs(m.nc_matmul(X[sl], G, 3) - refc.matmul(G)[sl]).max()
        res["ncT"] = np.abs(m.nc_matmul_T(X[sl], Q[sl], 3) - refc.matmul_T(Q)).max()
        # distributed Alg. 1 (NC): partitioned r-side, replicated c-side, Omega keyed by global index
        k, l, iters = 3, 6, 2
        Qc = philox_omega(1, 0, 16, l).astype(np.float64)
        for _ in range(iters):
            Qr = m.cqr2(m.nc_matmul(X[sl], Qc, 3))
            Qc = m.cqr2(m.nc_matmul_T(X[sl], Qr, 3), distributed=False)
        Qr = m.cqr2(m.nc_matmul(X[sl], Qc, 3))
        W = m.nc_matmul_T(X[sl], Qr, 3)
        s = np.linalg.svd(W.T, compute_uv=False)[:k]
        res["s"] = s
        from oracle import isvd as oracle_isvd

        _, s_ref, _, _ = oracle_isvd(refc, k, philox_omega(1, 0, 16, l), iters)
        res["s_err"] = np.abs(s - s_ref).max() / s_ref[0]
        # replicated small math identical on every rank
        allS = [torch.zeros(k, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allS, torch.from_numpy(s))
        res["ranks_equal"] = all(torch.equal(allS[0], t) for t in allS)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_row_partitioned_schedule_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = out[r]
        for key in ("ne", "neT", "nc", "ncT"):
            assert res[key] < 1e-11, (r, key, res[key])
        assert res["s_err"] < 1e-10, res["s_err"]
        assert res["ranks_equal"]
