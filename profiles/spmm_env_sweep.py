"""SpMM step time (profiled eager isvd, CUDA events around every SpMM step) for a list of environment
settings of the library, plus the graph-replay isvd time, in one process.
GPU box:  python profiles/spmm_env_sweep.py --config 4 --settings '[{"ISVD_SPMM_HINT": "0"}, {"ISVD_SPMM_HINT": "1"}]'
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
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--settings", required=True)
    args = ap.parse_args()
    settings = json.loads(args.settings)
    import torch

    import paper_2111_06312_b200 as isvd
    from synth import get_config, make_features, make_graph, solver_params

    cfg = get_config(args.config)
    sp = solver_params(cfg)
    g = make_graph(cfg)
    ctx = isvd.Context(0)
    graph = isvd.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    if cfg["op"] == "NC":
        op = isvd.NC(graph, torch.from_numpy(make_features(cfg["n"], cfg["d"], cfg["seed"])).cuda(), sp["L"])
    else:
        op = isvd.NE(graph, sp["weights"], sp["lambda_ones"])
    p = -1 if cfg["p"] is None else cfg["p"]
    keys = sorted({k for s in settings for k in s})
    ref = None
    for rep in range(args.reps):
        for s in settings:
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update(s)
            op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            r = op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            ref = r.S if ref is None else ref
            print(json.dumps({"config": args.config, "setting": s, "rep": rep, "spmm_ms": r.ms_spmm / r.spmm_steps,
                              "isvd_ms_eager": r.ms_total, "S_equal_first": bool((r.S == ref).all())}), flush=True)


if __name__ == "__main__":
    main()
