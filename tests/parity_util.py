"""Helpers shared by the GPU parity tests: build the library objects for a config,
run the oracle on the same seeded inputs, and the parity metrics of SURVEY 8(c).

Only tests import this module.  The oracle side never sees a value produced by
the CUDA path: it draws its own Omega (oracle.philox_omega) from the seed.
"""
from __future__ import annotations

import functools

import numpy as np

from synth import get_config, make_features, make_graph, solver_params


@functools.lru_cache(maxsize=None)
def config_inputs(i: int):
    cfg = get_config(i)
    g = make_graph(cfg)
    X = make_features(cfg["n"], cfg["d"], cfg["seed"]) if cfg["op"] == "NC" else None
    return cfg, g, X, solver_params(cfg)


def oracle_op(cfg, g, X, sp):
    from oracle import NCOperator, NEOperator, adjacency

    A = adjacency(g.n, g.row_ptr, g.col_idx)
    if cfg["op"] == "NE":
        return NEOperator(A, sp["weights"], sp["lambda_ones"])
    return NCOperator(A, X, sp["L"])


def gpu_op(ctx, cfg, g, X, sp, device_inputs=True):
    import torch

    import paper_2111_06312_b200 as isvd

    rb, nl = isvd.partition(g.n, ctx.world, ctx.rank)
    rp, ci = g.row_slice(rb, rb + nl)
    if device_inputs:
        rp = torch.from_numpy(rp).to(ctx.device)
        ci = torch.from_numpy(ci).to(ctx.device)
    graph = isvd.Graph(ctx, g.n, rp, ci)
    if cfg["op"] == "NE":
        return isvd.NE(graph, sp["weights"], sp["lambda_ones"])
    Xl = X[rb : rb + nl]
    if device_inputs:
        Xl = torch.from_numpy(np.ascontiguousarray(Xl)).to(ctx.device)
    return isvd.NC(graph, Xl, sp["L"])


def rel_fro(Y, Yref) -> float:
    Y = np.asarray(Y, dtype=np.float64)
    return float(np.linalg.norm(Y - Yref) / np.linalg.norm(Yref))


def worst_col_rel(Y, Yref) -> float:
    Y = np.asarray(Y, dtype=np.float64)
    num = np.linalg.norm(Y - Yref, axis=0)
    den = np.linalg.norm(Yref, axis=0)
    return float((num / np.maximum(den, 1e-300)).max())


def sin_theta(Ug, Uref) -> float:
    """sin of the largest principal angle between span(Ug) (re-orthonormalised in fp64) and span(Uref)."""
    Q, _ = np.linalg.qr(np.asarray(Ug, dtype=np.float64))
    Uref = np.asarray(Uref, dtype=np.float64)
    R = Uref - Q @ (Q.T @ Uref)
    return float(np.linalg.norm(R, 2))


def sigma_rel(s, sref) -> float:
    s = np.asarray(s, dtype=np.float64)
    sref = np.asarray(sref, dtype=np.float64)
    floor = 1e-6 * sref[0]
    err = np.where(sref >= floor, np.abs(s - sref) / np.maximum(sref, 1e-300), np.abs(s - sref) / (1e-4 * sref[0]))
    return float(err.max())


def gap_index(s_all, k, thresh=1e-2) -> int:
    """k' = largest index <= k with relative gap (s_k' - s_k'+1)/s_k' >= thresh (reading O20)."""
    for kk in range(k, 0, -1):
        if (s_all[kk - 1] - s_all[kk]) / s_all[kk - 1] >= thresh:
            return kk
    return 0
