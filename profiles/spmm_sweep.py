"""Sweep the SpMM column-block width and L2 hot-row hints on one config (GPU box).

    python profiles/spmm_sweep.py [--config 4]

Prints the average fused-SpMM step time (CUDA events around every step inside one
isvd, ISVD_SVD_PROFILE) and the whole isvd time for each setting.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--cb", default="0,200,100,48")
    ap.add_argument("--hot", default="auto,4")
    ap.add_argument("--relabel", action="store_true", help="relabel nodes by degree (hubs first)")
    ap.add_argument("--window", default="", help="comma list of persisting-L2 window sizes (MB)")
    args = ap.parse_args()
    import torch

    import paper_2111_06312_b200 as isvd
    from synth import get_config, make_features, make_graph, solver_params

    cfg = get_config(args.config)
    sp = solver_params(cfg)
    g = make_graph(cfg)
    import numpy as np

    X = make_features(cfg["n"], cfg["d"], cfg["seed"]) if cfg["op"] == "NC" else None
    if args.relabel:
        order = np.argsort(-g.degrees(), kind="stable")  # new id t -> old node order[t]
        perm = np.empty(g.n, dtype=np.int64)
        perm[order] = np.arange(g.n)
        g = g.permuted(perm)
        if X is not None:
            X = np.ascontiguousarray(X[order])
    ctx = isvd.Context(0)
    graph = isvd.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    if cfg["op"] == "NC":
        op = isvd.NC(graph, torch.from_numpy(X).cuda(), sp["L"])
    else:
        op = isvd.NE(graph, sp["weights"], sp["lambda_ones"])
    p = -1 if cfg["p"] is None else cfg["p"]
    ref = None
    if args.window:
        os.environ["ISVD_L2_WINDOW_MB"] = args.window
    for cb in args.cb.split(","):
        for hot in args.hot.split(","):
            os.environ.pop("ISVD_SPMM_CB", None)
            os.environ.pop("ISVD_SPMM_HOT", None)
            if cb != "0":
                os.environ["ISVD_SPMM_CB"] = cb
            if hot != "auto":
                os.environ["ISVD_SPMM_HOT"] = hot
            op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            r = op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            if ref is None:
                ref = r.S
            print(json.dumps({"cb": cb, "hot": hot, "spmm_ms": r.ms_spmm / r.spmm_steps, "isvd_ms": r.ms_total,
                              "alg_GBps": r.spmm_alg_bytes / (r.ms_spmm / 1e3) / 1e9,
                              "max_rel_S_vs_first": float(abs(r.S - ref).max() / ref[0])}), flush=True)


if __name__ == "__main__":
    main()
