"""Config-4 SpMM step time vs the L2 persisting window (size, hit ratio) and the graph-replay
isvd time, in ONE process (the graph is generated once).  GPU box:

    python profiles/spmm_window_sweep.py > gpurun_out/r02_window_sweep.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2111_06312_b200 as isvd
    from synth import get_config, make_features, make_graph, solver_params

    cfg = get_config(4)
    sp = solver_params(cfg)
    g = make_graph(cfg)
    X = make_features(cfg["n"], cfg["d"], cfg["seed"])
    ctx = isvd.Context(0)
    graph = isvd.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    op = isvd.NC(graph, torch.from_numpy(X).cuda(), sp["L"])

    def graph_mode(reps=3):
        op.svd(sp["k"], -1, sp["q"], sp["seed"])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        for _ in range(reps):
            op.svd(sp["k"], -1, sp["q"], sp["seed"])
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    print(json.dumps({"what": "graph replay, default window", "isvd_ms": graph_mode()}), flush=True)
    for hr in ("1.0", "0.8"):
        for mb in ("79", "72", "64", "48", "0"):
            os.environ["ISVD_L2_PERSIST_MB"] = mb
            os.environ["ISVD_L2_HIT_RATIO"] = hr
            op.svd(sp["k"], -1, sp["q"], sp["seed"], profile=True)
            r = op.svd(sp["k"], -1, sp["q"], sp["seed"], profile=True)
            print(json.dumps({"window_MB": int(mb), "hit_ratio": float(hr), "spmm_ms": r.ms_spmm / r.spmm_steps,
                              "isvd_ms_eager": r.ms_total, "phases": r.phases}), flush=True)
    os.environ.pop("ISVD_L2_PERSIST_MB")
    os.environ.pop("ISVD_L2_HIT_RATIO")
    print(json.dumps({"what": "graph replay, default window (again)", "isvd_ms": graph_mode()}), flush=True)


if __name__ == "__main__":
    main()
