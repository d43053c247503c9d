"""The five BASELINE.json configs as concrete, seeded synthetic workloads.

Shapes come from BASELINE.json `configs`; the generator recipes and the
readings of unstated details (ledger O5, O6, O17, O18 in SURVEY.md 8(c)) are
restated in DESIGN.md.  Solver parameters:

* NE (Eq. 3): weights w_c = 1/C (configs text),
  lambda_ones = 1/n, lambda_adj = 0.
* NC (Eq. 6): L = 3 blocks after X.
* l = min(k + p, c) when the oversampling p is given, else min(2k, c)
  (Alg. 1 draws c x 2k; ledger O6).
"""
from __future__ import annotations

CONFIGS = [
    dict(index=0, name="cfg0_ne_powerlaw", op="NE", graph="powerlaw", n=2708, m=5429, gamma=2.5, seed=0,
         C=5, k=32, p=10, q=2, stands_in_for="Cora counts (PAPER.md line 430)"),
    dict(index=1, name="cfg1_ne_sbm", op="NE", graph="sbm", n=3890, m=76584, blocks=50, ratio=20.0, seed=1,
         C=10, k=64, p=16, q=4, stands_in_for="PPI scale (PAPER.md line 426)"),
    dict(index=2, name="cfg2_nc_powerlaw", op="NC", graph="powerlaw", n=169343, m=1166243, gamma=2.5, seed=2,
         L=3, d=128, k=128, p=None, q=2, stands_in_for="ogbn-ArXiv counts (PAPER.md line 433)"),
    dict(index=3, name="cfg3_ne_uniform", op="NE", graph="uniform", n=4267, m=1334889, seed=3,
         C=10, k=128, p=32, q=6, stands_in_for="ogbl-DDI counts (PAPER.md line 434)"),
    dict(index=4, name="cfg4_nc_powerlaw_large", op="NC", graph="powerlaw", n=2449029, m=61859140, gamma=2.2,
         seed=4, L=3, d=100, k=256, p=None, q=2, stands_in_for="none (no paper counterpart)"),
]


def get_config(i: int) -> dict:
    return dict(CONFIGS[i])


def op_cols(cfg: dict) -> int:
    """c = number of columns of M."""
    return cfg["n"] if cfg["op"] == "NE" else cfg["d"] * (cfg["L"] + 1)


def solver_params(cfg: dict) -> dict:
    """k, l, q, seed and operator parameters for a config."""
    c = op_cols(cfg)
    r = cfg["n"]
    k = cfg["k"]
    if cfg["p"] is None:
        l = min(2 * k, c, r)
    else:
        l = min(k + cfg["p"], c, r)
    out = dict(k=k, l=l, q=cfg["q"], seed=cfg["seed"], rows=r, cols=c)
    if cfg["op"] == "NE":
        C = cfg["C"]
        out.update(C=C, weights=[1.0 / C] * C, lambda_ones=1.0 / cfg["n"], lambda_adj=0.0)
    else:
        out.update(L=cfg["L"], d=cfg["d"])
    return out
