"""Invariants of the seeded synthetic inputs (SURVEY 8(d2) recipes; no GPU)."""
import numpy as np
import pytest

from synth import get_config, make_features, make_graph, solver_params
from synth.configs import op_cols
from synth.graphs import connected_components, sbm_graph


def _check_graph(g, m):
    n = g.n
    assert g.row_ptr[0] == 0 and g.row_ptr[-1] == 2 * m and g.m == m
    assert g.col_idx.dtype == np.int32 and g.row_ptr.dtype == np.int64
    rows = np.repeat(np.arange(n), g.degrees())
    cols = g.col_idx.astype(np.int64)
    assert (cols >= 0).all() and (cols < n).all()
    assert not (rows == cols).any(), "self loop"
    key = rows * n + cols
    assert (np.diff(key) > 0).all(), "rows sorted, no duplicates"
    rkey = np.sort(cols * n + rows)
    assert np.array_equal(rkey, key), "symmetric"
    assert g.degrees().min() >= 1, "no isolated nodes (reading O3)"


@pytest.mark.parametrize("i", [0, 1, 2, 3])
def test_config_graphs(i):
    cfg = get_config(i)
    g = make_graph(cfg)
    assert g.n == cfg["n"]
    _check_graph(g, cfg["m"])
    assert connected_components(g) == 1
    g2 = make_graph(cfg)
    assert np.array_equal(g.row_ptr, g2.row_ptr) and np.array_equal(g.col_idx, g2.col_idx)


def test_powerlaw_tail_is_heavy():
    g = make_graph(get_config(2))
    d = np.sort(g.degrees())[::-1]
    assert d[0] > 50 * np.median(d)
    # top 1 % of nodes hold a large share of endpoints (~18 % expected)
    assert 0.10 < d[: g.n // 100].sum() / d.sum() < 0.30


def test_sbm_block_ratio():
    cfg = get_config(1)
    g = sbm_graph(cfg["n"], cfg["m"], cfg["blocks"], cfg["ratio"], cfg["seed"])
    # intra fraction expected 20 N_in / (20 N_in + N_out) = 0.2872 of draws
    from synth import streams

    perm = streams.permutation(cfg["seed"], "blocks", cfg["n"])
    sizes = np.full(50, cfg["n"] // 50)
    sizes[: cfg["n"] % 50] += 1
    block = np.empty(cfg["n"], dtype=np.int64)
    start = 0
    for b, s in enumerate(sizes):
        block[perm[start : start + s]] = b
        start += s
    rows = np.repeat(np.arange(g.n), g.degrees())
    intra = (block[rows] == block[g.col_idx]).mean()
    assert 0.26 < intra < 0.31


def test_features_standard_normal_and_deterministic():
    X = make_features(5000, 16, 2)
    assert X.dtype == np.float32 and X.shape == (5000, 16)
    z = X.astype(np.float64).ravel()
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1) < 0.02
    assert np.array_equal(X, make_features(5000, 16, 2))


def test_solver_params():
    p = [solver_params(get_config(i)) for i in range(5)]
    assert [x["l"] for x in p] == [42, 80, 256, 160, 400]  # reading O6
    assert [x["q"] for x in p] == [2, 4, 2, 6, 2]
    assert op_cols(get_config(4)) == 400 and op_cols(get_config(2)) == 512
    assert p[0]["lambda_ones"] == 1 / 2708 and p[0]["weights"] == [0.2] * 5
