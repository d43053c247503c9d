import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2111_06312_b200 as isvd
from synth import get_config, make_graph, make_features
cfg = get_config(4); g = make_graph(cfg)
X = make_features(cfg['n'], cfg['d'], cfg['seed'])
ctx = isvd.Context(0)
rp = torch.from_numpy(g.row_ptr).pin_memory().numpy(); ci = torch.from_numpy(g.col_idx).pin_memory().numpy()
Xp = torch.from_numpy(np.ascontiguousarray(X)).pin_memory().numpy()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gr = isvd.Graph(ctx, g.n, rp, ci); t1 = time.perf_counter()
    op = isvd.NC(gr, Xp, 3); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"graph {1e3*(t1-t0):.1f} ms  op {1e3*(t2-t1):.1f} ms", flush=True)
    op.close(); gr.close()
