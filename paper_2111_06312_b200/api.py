"""Thin Python binding over the isvd C ABI (include/isvd.h).

Argument marshalling only: every arithmetic step of the path runs in the
CUDA kernels of ``libisvd.so``.  PyTorch supplies device memory (tensors
whose ``data_ptr`` is passed down), the CUDA stream and, for world > 1, the
process group used to broadcast the NCCL unique id.

Names follow the paper: ``NE`` is the network-embedding design matrix of
Eq. 3, ``NC`` the node-classification design
matrix of Eq. 6 (lines 182-193), ``svd`` is Alg. 1 (lines 834-863).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check

__all__ = ["Context", "SimGroup", "Graph", "NE", "NC", "SvdResult", "embeddings", "least_norm", "spectral_kernel",
           "nccl_unique_id", "partition", "padded", "round_up"]


def round_up(x: int, m: int = 4) -> int:
    return (x + m - 1) // m * m


def padded(rows: int, w: int, device, dtype=torch.float32) -> torch.Tensor:
    """A rows x w view with leading dimension round_up(w, 4) (zero padding), as the ABI wants."""
    return torch.zeros(max(rows, 1), round_up(w), dtype=dtype, device=device)[:rows, :w]


def _ld(t: torch.Tensor) -> int:
    return t.stride(0)


def _as_abi(t: torch.Tensor, device) -> torch.Tensor:
    """Return t itself if it satisfies the ABI layout (fp32, row stride % 4 == 0, unit column
    stride, 16-byte aligned, on `device`), else a padded copy."""
    ok = (t.dtype == torch.float32 and t.device == device and t.dim() == 2 and t.stride(1) == 1
          and t.stride(0) % 4 == 0 and t.stride(0) >= round_up(t.shape[1]) and t.data_ptr() % 16 == 0)
    if ok:
        return t
    out = padded(t.shape[0], t.shape[1], device)
    out.copy_(t)
    return out


def partition(n: int, world: int, rank: int):
    """Rows [row_begin, row_begin + n_local) owned by `rank` (isvd_partition)."""
    lib = _lib.load()
    rb, nl = C.c_int64(), C.c_int64()
    check(lib.isvd_partition(n, world, rank, C.byref(rb), C.byref(nl)), "isvd_partition")
    return rb.value, nl.value


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    check(lib.isvd_nccl_unique_id(buf, 128), "isvd_nccl_unique_id")
    return buf.raw


def _torch_allocator(device_index: int) -> "_lib.Allocator":
    """isvd_allocator over PyTorch's caching allocator (north_star: PyTorch supplies device memory).
    A failed allocation returns NULL, which the library reports as ISVD_ERR_OOM."""

    def alloc(nbytes, stream, user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device_index, int(stream or 0))
        except Exception:  # out of memory (or any failure) -> NULL, never an exception across the ABI
            return None

    def free(ptr, stream, user):
        if ptr:
            torch.cuda.caching_allocator_delete(int(ptr))

    a = _lib.Allocator()
    a.alloc = _lib.ALLOC_FN(alloc)
    a.free = _lib.FREE_FN(free)
    a.user = None
    return a


class SimGroup:
    """isvd_sim_group: `world` logical ranks of the row-partitioned schedule on ONE device (a test
    backend).  Each rank needs its own Context(sim_group=..., rank=r) driven by its own thread."""

    def __init__(self, world: int):
        self.lib = _lib.load()
        self.world = int(world)
        h = C.c_void_p()
        check(self.lib.isvd_sim_group_create(self.world, C.byref(h)), "isvd_sim_group_create")
        self.h = h

    def close(self):
        if self.h:
            check(self.lib.isvd_sim_group_destroy(self.h), "isvd_sim_group_destroy")
            self.h = None


class Context:
    """isvd_ctx: device, stream, device memory and (world > 1) the rank group.

    allocator: "torch" (default: every device buffer from PyTorch's caching allocator) or None
    (the library's own cudaMalloc cache).  nccl_id: NCCL distributed mode; sim_group: simulated
    ranks on one device (test backend of the same schedule)."""

    def __init__(self, device: int = 0, stream: "torch.cuda.Stream | None" = None, rank: int = 0, world: int = 1,
                 nccl_id: "bytes | None" = None, sim_group: "SimGroup | None" = None, allocator="torch"):
        self.lib = _lib.load()
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.rank, self.world = rank, world
        self._alloc = _torch_allocator(device) if allocator == "torch" else None
        ap = C.byref(self._alloc) if self._alloc is not None else None
        h = C.c_void_p()
        if sim_group is not None:
            self.world = sim_group.world
            check(self.lib.isvd_ctx_create_sim(device, C.c_void_p(self.stream.cuda_stream), ap, sim_group.h, rank,
                                               C.byref(h)), "isvd_ctx_create_sim")
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            check(self.lib.isvd_ctx_create(device, C.c_void_p(self.stream.cuda_stream), ap, idbuf, rank, world,
                                           C.byref(h)), "isvd_ctx_create")
        self.h = h

    def close(self):
        if self.h:
            check(self.lib.isvd_ctx_destroy(self.h), "isvd_ctx_destroy", self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Graph:
    """isvd_graph: this rank's rows of the symmetric adjacency A in CSR; `values` are the
    edge weights A_ij (None: unweighted, every A_ij = 1)."""

    def __init__(self, ctx: Context, n: int, row_ptr, col_idx, values=None, validate: bool = False):
        self.ctx = ctx
        lib = ctx.lib
        self.n = int(n)
        self.row_begin, self.n_local = partition(self.n, ctx.world, ctx.rank)
        flags = _lib.ISVD_GRAPH_SYMMETRIC | (_lib.ISVD_GRAPH_VALIDATE if validate else 0)
        if isinstance(row_ptr, torch.Tensor) and row_ptr.is_cuda:
            rp = row_ptr.to(torch.int64).contiguous()
            ci = col_idx.to(torch.int32).contiguous()
            vv = None if values is None else torch.as_tensor(values, device=rp.device).to(torch.float32).contiguous()
            flags |= _lib.ISVD_PTR_DEVICE
            keep = (rp, ci, vv)
            prp, pci = rp.data_ptr(), ci.data_ptr()
            pv = 0 if vv is None else vv.data_ptr()
        else:
            rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
            ci = np.ascontiguousarray(col_idx, dtype=np.int32)
            vv = None if values is None else np.ascontiguousarray(values, dtype=np.float32)
            keep = (rp, ci, vv)
            prp, pci = rp.ctypes.data, ci.ctypes.data
            pv = 0 if vv is None else vv.ctypes.data
        if len(keep[0]) != self.n_local + 1:
            raise ValueError(f"row_ptr must have n_local + 1 = {self.n_local + 1} entries for rank {ctx.rank}")
        h = C.c_void_p()
        check(lib.isvd_graph_create(ctx.h, self.n, self.row_begin, self.n_local, C.c_void_p(prp), C.c_void_p(pci),
                                    C.c_void_p(pv or None), flags, C.byref(h)), "isvd_graph_create", ctx.h)
        self.h = h

    def info(self):
        a = [C.c_int64() for _ in range(4)]
        check(self.ctx.lib.isvd_graph_info(self.h, *[C.byref(x) for x in a]), "isvd_graph_info", self.ctx.h)
        return dict(n=a[0].value, n_local=a[1].value, nnz_local=a[2].value, max_degree=a[3].value)

    def close(self):
        if self.h:
            check(self.ctx.lib.isvd_graph_destroy(self.h), "isvd_graph_destroy", self.ctx.h)
            self.h = None


@dataclass
class SvdResult:
    U: object       # n_local x k (torch cuda tensor, or numpy with host_output)
    S: np.ndarray   # k, fp64, non-increasing
    V: object       # NE: n_local x k; NC: c x k
    l: int
    chol_fallbacks: int
    jacobi_sweeps: int
    kernel_launches: int
    ms_total: float
    spmm_steps: int = 0
    ms_spmm: float = 0.0
    spmm_alg_bytes: float = 0.0
    phases: "dict | None" = None  # profile=True: ms by phase (products / orth / small / comm)
    gram_probe_fallbacks: int = 0  # first-pass tensor-core Gram probes that fell back to the exact Gram
    gram_probe_skipped: int = 0  # 1: the probe was skipped (an earlier call on this op fell back)
    ms_allgather: float = 0.0  # profile=True, distributed split: all-gather time on the collectives stream
    ms_allgather_hidden: float = 0.0  # ... the part concurrent with the local SpMM pass


class _Operator:
    def __init__(self, graph: Graph, desc: _lib.OpDesc, keep=(), rows=None):
        self.graph = graph
        self.ctx = graph.ctx
        self._r_local = graph.n_local
        if rows is not None:  # implicit row gather M[S, :] (option (ii))
            S = np.ascontiguousarray(rows, dtype=np.int64)
            desc.rows = S.ctypes.data_as(C.POINTER(C.c_int64))
            desc.n_rows = S.size
            keep = tuple(keep) + (S,)
            lo, hi = graph.row_begin, graph.row_begin + graph.n_local
            self._r_local = int(np.count_nonzero((S >= lo) & (S < hi)))
        self._keep = keep
        h = C.c_void_p()
        check(self.ctx.lib.isvd_op_define(graph.h, C.byref(desc), C.byref(h)), "isvd_op_define", self.ctx.h)
        self.h = h
        r, c = C.c_int64(), C.c_int64()
        check(self.ctx.lib.isvd_op_shape(h, C.byref(r), C.byref(c)), "isvd_op_shape", self.ctx.h)
        self.shape = (r.value, c.value)

    # rows of the operand of M . Q held by this rank (NE: partitioned; NC: all c)
    def c_rows(self) -> int:
        raise NotImplementedError

    # r-side rows held by this rank (rows of M . Q, of U): n_local, or this rank's subset rows
    def r_rows(self) -> int:
        return self._r_local

    def close(self):
        if self.h:
            check(self.ctx.lib.isvd_op_destroy(self.h), "isvd_op_destroy", self.ctx.h)
            self.h = None

    def matmul(self, Q: torch.Tensor, out: "torch.Tensor | None" = None) -> torch.Tensor:
        """M . Q (SymbolicPF.dot)."""
        dev = self.ctx.device
        Q = _as_abi(Q, dev)
        w = Q.shape[1]
        if out is None:
            out = padded(self.r_rows(), w, dev)
        check(self.ctx.lib.isvd_matmul(self.h, C.c_void_p(Q.data_ptr()), w, _ld(Q), C.c_void_p(out.data_ptr()),
                                       _ld(out)), "isvd_matmul", self.ctx.h)
        return out

    def matmul_T(self, Q: torch.Tensor, out: "torch.Tensor | None" = None) -> torch.Tensor:
        """M^T . Q (SymbolicPF.T().dot)."""
        dev = self.ctx.device
        Q = _as_abi(Q, dev)
        w = Q.shape[1]
        if out is None:
            out = padded(self.c_rows(), w, dev)
        check(self.ctx.lib.isvd_matmul_T(self.h, C.c_void_p(Q.data_ptr()), w, _ld(Q), C.c_void_p(out.data_ptr()),
                                         _ld(out)), "isvd_matmul_T", self.ctx.h)
        return out

    def _params(self, k, oversampling, power_iters, seed, flags=0, omega=None):
        p = _lib.SvdParams()
        p.k, p.oversampling, p.power_iters, p.seed, p.flags = int(k), int(oversampling), int(power_iters), int(seed), flags
        p.omega = omega.data_ptr() if omega is not None else None
        return p

    def working_width(self, k: int, oversampling: int) -> int:
        r, c = self.shape
        l = 2 * k if oversampling < 0 else k + oversampling
        return min(l, r, c)

    def sample_omega(self, k: int, oversampling: int, seed: int) -> torch.Tensor:
        """The Omega Alg. 1 starts from, this rank's rows, from the library's generator."""
        l = self.working_width(k, oversampling)
        om = padded(self.c_rows(), l, self.ctx.device)
        p = self._params(k, oversampling, 0, seed)
        check(self.ctx.lib.isvd_sample_omega(self.h, C.byref(p), C.c_void_p(om.data_ptr()), _ld(om)),
              "isvd_sample_omega", self.ctx.h)
        return om

    def host_buffers(self, k: int):
        """Page-locked host arrays (U, V) for svd(host_output=True, out=...): the library's device-to-host copies
        run at full DMA speed and a repeated call pays no allocation."""
        kk = max(round_up(k), 4)
        U = torch.zeros(max(self.r_rows(), 1), kk, dtype=torch.float32, pin_memory=True).numpy()
        V = torch.zeros(max(self.c_rows(), 1), kk, dtype=torch.float32, pin_memory=True).numpy()
        return U, V

    def svd(self, k: int, oversampling: int = -1, power_iters: int = 2, seed: int = 0, host_output: bool = False,
            omega: "torch.Tensor | None" = None, force_chol_fail: bool = False, profile: bool = False,
            out=None) -> SvdResult:
        """Rank-k implicit SVD (Alg. 1) -> U (n_local x k), S (k), V."""
        dev = self.ctx.device
        kk = max(round_up(k), 4)
        flags = 0
        if host_output:
            flags |= _lib.ISVD_SVD_HOST_OUTPUT
            if out is not None:  # caller-owned host arrays (ideally page-locked, see host_buffers())
                U, V = out
                for a, rows in ((U, self.r_rows()), (V, self.c_rows())):
                    if (not isinstance(a, np.ndarray) or a.dtype != np.float32 or a.ndim != 2
                            or a.shape[0] < rows or a.shape[1] < k or a.strides[1] != 4
                            or not a.flags.writeable):
                        raise ValueError("host output must be a writeable float32 row-major array of >= rows x k")
                pu, pv, ldu, ldv = U.ctypes.data, V.ctypes.data, U.strides[0] // 4, V.strides[0] // 4
            else:
                U, V = self.host_buffers(k)
                pu, pv, ldu, ldv = U.ctypes.data, V.ctypes.data, kk, kk
        else:
            if out is not None:
                U, V = out
            else:
                U = torch.zeros(max(self.r_rows(), 1), kk, dtype=torch.float32, device=dev)
                V = torch.zeros(max(self.c_rows(), 1), kk, dtype=torch.float32, device=dev)
            pu, pv, ldu, ldv = U.data_ptr(), V.data_ptr(), U.stride(0), V.stride(0)
        if omega is not None:
            flags |= _lib.ISVD_SVD_OMEGA_PROVIDED
            omega = _as_abi(omega, dev)
        if force_chol_fail:
            flags |= _lib.ISVD_SVD_FORCE_CHOL_FAIL
        if profile:
            flags |= _lib.ISVD_SVD_PROFILE
        p = self._params(k, oversampling, power_iters, seed, flags, omega)
        S = np.zeros(max(int(k), 1), dtype=np.float64)
        rep = _lib.SvdReport()
        check(self.ctx.lib.isvd_svd(self.h, C.byref(p), C.c_void_p(pu), ldu,
                                    S.ctypes.data_as(C.POINTER(C.c_double)), C.c_void_p(pv), ldv, C.byref(rep)),
              "isvd_svd", self.ctx.h)
        U = U[: self.r_rows(), :k]
        V = V[: self.c_rows(), :k]
        S = S[:k]
        phases = None
        if profile:
            phases = dict(products=rep.ms_products, orth=rep.ms_orth, small=rep.ms_small, comm=rep.ms_comm)
        return SvdResult(U, S, V, rep.l, rep.chol_fallbacks, rep.jacobi_sweeps, rep.kernel_launches, rep.ms_total,
                         rep.spmm_steps, rep.ms_spmm, rep.spmm_alg_bytes, phases, rep.gram_probe_fallbacks,
                         rep.gram_probe_skipped, rep.ms_allgather, rep.ms_allgather_hidden)


class NE(_Operator):
    """M = sum_{c=1..C} w_c B^c - lambda_ones 1 1^T + lambda_adj A   (Eq. 3),
    B = T = D^-1 A (basis "T") or B = A_hat (basis "Ahat", the symmetric variant of P:158)."""

    def __init__(self, graph: Graph, weights, lambda_ones: float, lambda_adj: float = 0.0, basis: str = "T",
                 rows=None):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        d = _lib.OpDesc()
        d.kind = _lib.ISVD_OP_POWER_SUM
        d.num_terms = int(w.size)
        d.weights = w.ctypes.data_as(C.POINTER(C.c_double))
        d.lambda_ones = float(lambda_ones)
        d.lambda_adj = float(lambda_adj)
        if basis not in ("T", "Ahat"):
            raise ValueError("basis must be 'T' or 'Ahat'")
        d.basis = _lib.ISVD_BASIS_T_ROW if basis == "T" else _lib.ISVD_BASIS_AHAT_SYM
        super().__init__(graph, d, keep=(w,), rows=rows)

    def c_rows(self) -> int:
        return self.graph.n_local


class NC(_Operator):
    """M = [X | A_hat X | ... | A_hat^L X],  A_hat = (D+I)^-1/2 (A+I) (D+I)^-1/2   (Eq. 6).

    rows (NE and NC): sorted global row ids S -> the op is M[S, :] (implicit row gather).

    X: this rank's rows (n_local x d), a CUDA tensor (borrowed when already in ABI layout)
    or a host numpy array (copied).  Label re-use: Y_train (this rank's n_local x y
    rows, copied) and P powers append the blocks B Y, ..., B^P Y, B = A_hat - (D+I)^-1."""

    def __init__(self, graph: Graph, X, L: int, Y_train=None, P: int = 0, rows=None):
        d = _lib.OpDesc()
        d.kind = _lib.ISVD_OP_STACKED_PROPAGATION
        d.num_terms = int(L)
        if isinstance(X, torch.Tensor):
            Xt = _as_abi(X, graph.ctx.device)
            d.X, d.d, d.ldx = Xt.data_ptr(), Xt.shape[1], _ld(Xt)
            d.x_flags = _lib.ISVD_PTR_DEVICE | _lib.ISVD_BORROW
            keep = (Xt,)
        else:
            Xn = np.asarray(X, dtype=np.float32)
            ldx = round_up(Xn.shape[1])
            if Xn.flags.c_contiguous and ldx == Xn.shape[1]:
                Xp = Xn  # already in ABI layout (e.g. a pinned host buffer): copied once by the library
            else:
                Xp = np.zeros((Xn.shape[0], ldx), dtype=np.float32)
                Xp[:, : Xn.shape[1]] = Xn
            d.X, d.d, d.ldx, d.x_flags = Xp.ctypes.data, Xn.shape[1], ldx, 0
            keep = (Xp,)
        self.y, self.P = 0, 0
        if Y_train is not None and P > 0:
            if isinstance(Y_train, torch.Tensor):
                Yt = _as_abi(Y_train, graph.ctx.device)
                d.Y, d.y, d.ldy, d.y_flags = Yt.data_ptr(), Yt.shape[1], _ld(Yt), _lib.ISVD_PTR_DEVICE
            else:
                Yn = np.asarray(Y_train, dtype=np.float32)
                Yt = np.zeros((Yn.shape[0], round_up(Yn.shape[1])), dtype=np.float32)
                Yt[:, : Yn.shape[1]] = Yn
                d.Y, d.y, d.ldy, d.y_flags = Yt.ctypes.data, Yn.shape[1], Yt.shape[1], 0
            d.lr_powers = int(P)
            keep = keep + (Yt,)
            self.y, self.P = int(d.y), int(P)
        self.d, self.L = int(d.d), int(L)
        super().__init__(graph, d, keep=keep, rows=rows)

    def c_rows(self) -> int:
        return self.d * (self.L + 1) + self.y * self.P


# ------------------------------------------------------------------ after the SVD


def embeddings(ctx: Context, M: torch.Tensor, S) -> torch.Tensor:
    """L = U S^1/2 (or R = V S^1/2): Eq. 5, P:161-167 (isvd_embeddings)."""
    M = _as_abi(M, ctx.device)
    rows, k = M.shape
    Sd = np.ascontiguousarray(S, dtype=np.float64)[:k]
    out = padded(rows, k, ctx.device)
    check(ctx.lib.isvd_embeddings(ctx.h, rows, k, C.c_void_p(M.data_ptr()), _ld(M),
                                  Sd.ctypes.data_as(C.POINTER(C.c_double)), C.c_void_p(out.data_ptr()), _ld(out)),
          "isvd_embeddings", ctx.h)
    return out


def least_norm(ctx: Context, U: torch.Tensor, S, V: torch.Tensor, Y: torch.Tensor, shape, rows=None) -> torch.Tensor:
    """W* = V S^+ U^T Y (Eq. 7), right to left; `rows` = labelled local rows;
    `shape` = (r, c) of M (isvd_least_norm)."""
    U = _as_abi(U, ctx.device)
    V = _as_abi(V, ctx.device)
    Y = _as_abi(Y, ctx.device)
    k, ny = U.shape[1], Y.shape[1]
    Sd = np.ascontiguousarray(S, dtype=np.float64)[:k]
    W = padded(V.shape[0], ny, ctx.device)
    idx = None
    if rows is not None:
        idx = torch.as_tensor(rows, dtype=torch.int32, device=ctx.device).contiguous()
    check(ctx.lib.isvd_least_norm(ctx.h, U.shape[0], k, C.c_void_p(U.data_ptr()), _ld(U),
                                  Sd.ctypes.data_as(C.POINTER(C.c_double)), int(shape[0]), int(shape[1]),
                                  V.shape[0], C.c_void_p(V.data_ptr()), _ld(V), ny, C.c_void_p(Y.data_ptr()), _ld(Y),
                                  C.c_void_p(idx.data_ptr() if idx is not None else 0),
                                  0 if idx is None else idx.numel(), C.c_void_p(W.data_ptr()), _ld(W)),
          "isvd_least_norm", ctx.h)
    return W


def spectral_kernel(S, mu: float, s_bar: float) -> np.ndarray:
    """Gaussian spectral reweighting of S (Eq. 9, discretised as P:1057-1065)."""
    lib = _lib.load()
    Sd = np.ascontiguousarray(S, dtype=np.float64)
    out = np.zeros_like(Sd)
    check(lib.isvd_spectral_kernel(Sd.ctypes.data_as(C.POINTER(C.c_double)), Sd.size, float(mu), float(s_bar),
                                   out.ctypes.data_as(C.POINTER(C.c_double))), "isvd_spectral_kernel")
    return out
