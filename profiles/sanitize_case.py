"""Small isvd runs for compute-sanitizer (memcheck / racecheck / synccheck): configs 0 and 1
through the C ABI, default path (CUDA graph) and eager (profile) path, plus the products.

    compute-sanitizer --tool memcheck python profiles/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2111_06312_b200 as isvd
    from synth import get_config, make_graph, solver_params

    ctx = isvd.Context(0)
    for i in (0, 1):
        cfg = get_config(i)
        g = make_graph(cfg)
        sp = solver_params(cfg)
        graph = isvd.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
        op = isvd.NE(graph, sp["weights"], sp["lambda_ones"])
        Q = torch.randn(g.n, sp["l"], device="cuda")
        op.matmul(Q)
        op.matmul_T(Q)
        a = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"])
        b = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"], profile=True)
        torch.cuda.synchronize()
        print(f"cfg{i}: S[0] {a.S[0]:.6f} eager==graph {np.array_equal(a.S, b.S)} launches {a.kernel_launches}")
        op.close()
        graph.close()
    ctx.close()


if __name__ == "__main__":
    main()
