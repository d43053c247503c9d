"""Config-4 SpMM step time for each spmm_kernel variant (ISVD_SPMM_VARIANT: bit 0 masked tail
batch, bit 1 next-descriptor prefetch) in one process, plus the default graph-replay isvd time.
GPU box:  python profiles/spmm_variant_sweep.py [--config 4] > gpurun_out/r02c_spmm_variants.jsonl
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
    for rep in range(2):
        for v in ("0", "1", "2", "3"):
            os.environ["ISVD_SPMM_VARIANT"] = v
            op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            r = op.svd(sp["k"], p, sp["q"], sp["seed"], profile=True)
            if ref is None:
                ref = r.S
            print(json.dumps({"config": args.config, "variant": int(v), "rep": rep,
                              "spmm_ms": r.ms_spmm / r.spmm_steps, "isvd_ms_eager": r.ms_total,
                              "max_rel_S_vs_first": float(abs(r.S - ref).max() / ref[0])}), flush=True)
    os.environ.pop("ISVD_SPMM_VARIANT")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op.svd(sp["k"], p, sp["q"], sp["seed"])
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(3):
        op.svd(sp["k"], p, sp["q"], sp["seed"])
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    print(json.dumps({"config": args.config, "what": "graph replay, default variant", "isvd_ms": e0.elapsed_time(e1) / 3}),
          flush=True)


if __name__ == "__main__":
    main()
