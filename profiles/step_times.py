"""Per-step isvd times of one config (graph replay), with and without an L2 flush before each step,
to check the stability of bench.py's headline.   GPU box: python profiles/step_times.py --config 3
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--smi-ms", type=int, default=0, help="run nvidia-smi -lms this period during the timing")
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
    stream = ctx.stream
    for _ in range(3):
        op.svd(sp["k"], p, sp["q"], sp["seed"])
    junk = torch.empty(128 * 2 ** 20, dtype=torch.float32, device="cuda")
    smi = None
    if args.smi_ms:
        import subprocess

        smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                                "--format=csv,noheader", "-lms", str(args.smi_ms)], stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    for flush in (False, True, False):
        ms, host = [], []
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                if flush:
                    junk.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                t0 = time.perf_counter()
                r = op.svd(sp["k"], p, sp["q"], sp["seed"])
                host.append((time.perf_counter() - t0) * 1e3)
                b.record(stream)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
        print(json.dumps({"config": args.config, "flush": flush, "event_ms": [round(x, 3) for x in ms],
                          "host_ms": [round(x, 3) for x in host], "lib_ms_total": r.ms_total,
                          "launches": r.kernel_launches, "smi_ms": args.smi_ms}), flush=True)
    if smi:
        smi.terminate()


if __name__ == "__main__":
    main()
