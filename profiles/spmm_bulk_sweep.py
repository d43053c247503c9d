"""SpMM step time: register gather (ISVD_SPMM_VARIANT=1) vs the shared-memory staged bulk-copy gather
(variant 2) with ring sizes ISVD_SPMM_BULK_SLOTS and per-copy L2 hints ISVD_SPMM_BULK_HINT, from the
profiled eager isvd (CUDA events around every SpMM step on the library stream).
GPU box:  python profiles/spmm_bulk_sweep.py --config 4 > gpurun_out/spmm_bulk.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETTINGS = [
    {"ISVD_SPMM_VARIANT": "1"},
    {"ISVD_SPMM_VARIANT": "2", "ISVD_SPMM_BULK_SLOTS": "32", "ISVD_SPMM_BULK_HINT": "0"},
    {"ISVD_SPMM_VARIANT": "2", "ISVD_SPMM_BULK_SLOTS": "64", "ISVD_SPMM_BULK_HINT": "0"},
    {"ISVD_SPMM_VARIANT": "2", "ISVD_SPMM_BULK_SLOTS": "32", "ISVD_SPMM_BULK_HINT": "1"},
    {"ISVD_SPMM_VARIANT": "2", "ISVD_SPMM_BULK_SLOTS": "64", "ISVD_SPMM_BULK_HINT": "1"},
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_2111_06312_b200 as isvd
    from synth import get_config, make_features, make_graph, solver_params

    cfg = get_config(args.config)
    sp = solver_params(cfg)
    g = make_graph(cfg)
    ctx = isvd.Context(0)
    graph = isvd.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    if cfg["op"] == "NC":
        X = make_features(cfg["n"], cfg["d"], cfg["seed"])
        op = isvd.NC(graph, torch.from_numpy(X).cuda(), sp["L"])
    else:
        op = isvd.NE(graph, sp["weights"], sp["lambda_ones"])
    p = -1 if cfg["p"] is None else cfg["p"]
    ref = None
    keys = sorted({k for s in SETTINGS for k in s})
    for rep in range(args.reps):
        for s in SETTINGS:
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update(s)
            op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            r = op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            if ref is None:
                ref = r.S
            print(json.dumps({"config": args.config, "setting": s, "rep": rep,
                              "spmm_ms": r.ms_spmm / r.spmm_steps, "isvd_ms_eager": r.ms_total,
                              "S_bitwise_equal_first": bool((r.S == ref).all())}), flush=True)


if __name__ == "__main__":
    main()
