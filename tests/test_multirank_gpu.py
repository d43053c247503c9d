"""The library's own row-partitioned (multi-rank) schedule, executed on ONE GPU.

SURVEY 8(e) partitions the graph rows over P ranks: every SpMM gather source is all-gathered
(uniform padded counts, ragged last block), Gram / column-sum / X^T Z partials are all-reduced
in fp64, the l x l math is replicated, and the sign rule gathers its candidates.  This build has
one B200, so the P ranks run as the simulated-rank backend of the C ABI
(isvd_sim_group_create / isvd_ctx_create_sim): one context, one CUDA stream and one host thread
per rank, the same capi.cpp schedule as the NCCL path, with each collective done as one
cudaMemcpyAsync per peer slice (all-gather) or a rank-ordered sum kernel (all-reduce), ordered
by events and host barriers only (no kernel waits on another rank).

Checked against the fp64 oracle at P in {2, 3, 8} on config 0 (NE), config 2 (NC) and a ragged
graph (n = 1001, so the last block is short) for both families: products (every row and column),
the full isvd (sigma, subspaces), S bitwise identical on every rank, the replicated NC V bitwise
identical on every rank, and the P-rank result bitwise reproducible.
"""
import threading

import numpy as np
import pytest

from parity_util import (assert_product, check_isvd_arrays, config_inputs, oracle_isvd_result, oracle_op)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def run_ranks(P, fn, timeout=900):
    """fn(rank, ctx) on P simulated ranks, one thread and one stream each; returns the results."""
    import paper_2111_06312_b200 as isvd

    grp = isvd.SimGroup(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [isvd.Context(0, stream=streams[r], rank=r, sim_group=grp) for r in range(P)]
    out, errs = [None] * P, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                out[r] = fn(r, ctxs[r])
                streams[r].synchronize()
        except BaseException as e:  # noqa: BLE001 -- reported below
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a simulated rank did not finish (collective mismatch?)"
    assert not errs, errs
    torch.cuda.synchronize()
    for c in ctxs:
        c.close()
    grp.close()
    return out


# ------------------------------------------------------------------ cases


def _ragged(kind):
    """n = 1001 power-law graph (ragged last block at every P > 1), NE C = 5 or NC L = 3, d = 16."""
    from synth.graphs import make_features, powerlaw_graph

    g = powerlaw_graph(1001, 4000, 2.5, 11)
    if kind == "NE":
        cfg = {"op": "NE", "p": 8, "name": "ragged-NE"}
        sp = {"weights": np.full(5, 0.2), "lambda_ones": 1.0 / g.n, "k": 16, "l": 24, "q": 2, "seed": 5}
        return cfg, g, None, sp
    X = make_features(g.n, 16, 12)
    cfg = {"op": "NC", "p": None, "name": "ragged-NC"}
    sp = {"L": 3, "k": 16, "l": 32, "q": 2, "seed": 6}
    return cfg, g, X, sp


def _case(name):
    if name.startswith("ragged"):
        return _ragged(name.split("-")[1])
    return config_inputs(int(name[3:]))


_oracle_cache = {}


def _oracle(name, cfg, g, X, sp):
    if name.startswith("cfg"):
        return oracle_isvd_result(int(name[3:]))
    if name not in _oracle_cache:
        from oracle import isvd, philox_omega

        ref = oracle_op(cfg, g, X, sp)
        om = philox_omega(sp["seed"], 0, ref.shape[1], sp["l"])
        _oracle_cache[name] = isvd(ref, sp["k"], om, sp["q"])
    return _oracle_cache[name]


def _rank_op(ctx, cfg, g, X, sp):
    import paper_2111_06312_b200 as isvd

    rb, nl = isvd.partition(g.n, ctx.world, ctx.rank)
    rp, ci = g.row_slice(rb, rb + nl)
    graph = isvd.Graph(ctx, g.n, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    if cfg["op"] == "NE":
        return isvd.NE(graph, sp["weights"], sp["lambda_ones"]), graph, rb, nl
    Xl = torch.from_numpy(np.ascontiguousarray(X[rb : rb + nl])).cuda()
    return isvd.NC(graph, Xl, sp["L"]), graph, rb, nl


CASES = ["cfg0", "cfg2", "ragged-NE", "ragged-NC"]


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("name", CASES)
def test_multirank_products_and_isvd(name, P):
    cfg, g, X, sp = _case(name)
    ref = oracle_op(cfg, g, X, sp)
    r, c = ref.shape
    l = sp["l"]
    rng = np.random.default_rng(90 + P)
    Gc = rng.standard_normal((c, l)).astype(np.float32)   # operand of M . G (c rows)
    Hr = rng.standard_normal((r, l)).astype(np.float32)   # operand of M^T . H (r rows)
    p = -1 if cfg["p"] is None else cfg["p"]
    ne = cfg["op"] == "NE"

    def fn(rank, ctx):
        op, graph, rb, nl = _rank_op(ctx, cfg, g, X, sp)
        gin = Gc[rb : rb + nl] if ne else Gc  # NE: c side row-partitioned; NC: replicated
        Y = op.matmul(torch.from_numpy(np.ascontiguousarray(gin)).cuda()).cpu().numpy()
        W = op.matmul_T(torch.from_numpy(np.ascontiguousarray(Hr[rb : rb + nl])).cuda()).cpu().numpy()
        res = op.svd(sp["k"], p, sp["q"], sp["seed"])
        res2 = op.svd(sp["k"], p, sp["q"], sp["seed"])
        det = (np.array_equal(res.S, res2.S) and torch.equal(res.U, res2.U) and torch.equal(res.V, res2.V))
        o = dict(rb=rb, nl=nl, Y=Y, W=W, S=res.S.copy(), U=res.U.cpu().numpy(), V=res.V.cpu().numpy(), det=det,
                 l=res.l)
        op.close()
        graph.close()
        return o

    outs = run_ranks(P, fn)
    assert [o["rb"] for o in outs] == sorted(o["rb"] for o in outs)
    assert sum(o["nl"] for o in outs) == g.n
    # products: row blocks in rank order make the global result
    Y = np.concatenate([o["Y"] for o in outs])
    print(assert_product(Y, ref.matmul(Gc.astype(np.float64)), f"{name} P={P} M.G"))
    Wref = ref.matmul_T(Hr.astype(np.float64))
    if ne:
        W = np.concatenate([o["W"] for o in outs])
    else:  # replicated c x l: every rank holds the same, bitwise
        W = outs[0]["W"]
        assert all(np.array_equal(o["W"], W) for o in outs), "replicated M^T H differs across ranks"
    print(assert_product(W, Wref, f"{name} P={P} M^T.H"))
    # isvd: replicated l x l math -> bitwise identical S on every rank (and V for NC)
    for o in outs:
        assert o["det"], "the P-rank isvd is not bitwise reproducible"
        assert o["l"] == l
        assert np.array_equal(o["S"], outs[0]["S"]), "singular values differ across ranks"
    U = np.concatenate([o["U"] for o in outs]).astype(np.float64)
    if ne:
        V = np.concatenate([o["V"] for o in outs]).astype(np.float64)
    else:
        V = outs[0]["V"].astype(np.float64)
        assert all(np.array_equal(o["V"], outs[0]["V"]) for o in outs), "replicated V differs across ranks"
    print(check_isvd_arrays(U, outs[0]["S"], V, _oracle(name, cfg, g, X, sp), sp["k"], f"{name} P={P}"))


def test_multirank_equals_single_rank_to_rounding():
    """Config 2 at P = 3 against the single-GPU path: same Omega (global-index keyed), so the
    results agree to reduction-order rounding (SURVEY 8(e) determinism across P)."""
    import paper_2111_06312_b200 as isvd

    cfg, g, X, sp = config_inputs(2)
    with isvd.Context(0) as ctx1:
        op1, graph1, _, _ = _rank_op(ctx1, cfg, g, X, sp)
        r1 = op1.svd(sp["k"], -1, sp["q"], sp["seed"])
        S1, V1 = r1.S.copy(), r1.V.cpu().numpy()
        op1.close()
        graph1.close()

    def fn(rank, ctx):
        op, graph, _, _ = _rank_op(ctx, cfg, g, X, sp)
        res = op.svd(sp["k"], -1, sp["q"], sp["seed"])
        o = (res.S.copy(), res.V.cpu().numpy())
        op.close()
        graph.close()
        return o

    S3, V3 = run_ranks(3, fn)[0]
    assert np.max(np.abs(S3 - S1) / S1) <= 1e-5
    from parity_util import sin_theta

    assert sin_theta(V3.astype(np.float64), V1.astype(np.float64)) <= 1e-3


def test_multirank_least_norm_allreduce():
    """Eq. 7's U^T Y is all-reduced over the ranks (isvd_least_norm): W* from P = 3 simulated ranks
    equals the oracle formula on the assembled U (config 2, one-hot labels)."""
    from oracle import least_norm as o_ln
    from parity_util import rel_fro

    import paper_2111_06312_b200 as isvd

    cfg, g, X, sp = config_inputs(2)
    rng = np.random.default_rng(31)
    ny = 5
    Yl = np.zeros((g.n, ny), dtype=np.float32)
    Yl[np.arange(g.n), rng.integers(0, ny, g.n)] = 1.0

    def fn(rank, ctx):
        op, graph, rb, nl = _rank_op(ctx, cfg, g, X, sp)
        res = op.svd(sp["k"], -1, sp["q"], sp["seed"])
        W = isvd.least_norm(ctx, res.U, res.S, res.V, torch.from_numpy(Yl[rb : rb + nl]).cuda(), op.shape)
        o = dict(U=res.U.cpu().numpy(), S=res.S.copy(), V=res.V.cpu().numpy(), W=W.cpu().numpy())
        op.close()
        graph.close()
        return o

    outs = run_ranks(3, fn)
    U = np.concatenate([o["U"] for o in outs]).astype(np.float64)
    Wref = o_ln(U, outs[0]["S"], outs[0]["V"].astype(np.float64), Yl, shape=(g.n, X.shape[1] * (sp["L"] + 1)))
    for o in outs:
        assert rel_fro(o["W"], Wref) <= 1e-5
        assert np.array_equal(o["W"], outs[0]["W"])


@pytest.mark.parametrize("where", ["spread", "first_block"])
def test_multirank_row_subset(where):
    """Implicit row gather on P = 3 simulated ranks: S spread over every rank, or S
    inside rank 0's block only (ranks 1 and 2 hold ZERO r-side rows: empty Grams, empty GEMMs,
    empty sign-rule candidates).  Against the oracle's RowSubsetOperator."""
    from oracle import RowSubsetOperator, isvd, philox_omega

    import paper_2111_06312_b200 as isvd_mod

    cfg, g, X, sp = _ragged("NC")
    rng = np.random.default_rng(5)
    if where == "spread":
        S = np.sort(rng.choice(g.n, 300, replace=False)).astype(np.int64)
    else:
        S = np.sort(rng.choice(300, 120, replace=False)).astype(np.int64)  # rank 0 owns rows < 334
    ref = RowSubsetOperator(oracle_op(cfg, g, X, sp), S)

    def fn(rank, ctx):
        rb, nl = isvd_mod.partition(g.n, ctx.world, ctx.rank)
        rp, ci = g.row_slice(rb, rb + nl)
        graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
        op = isvd_mod.NC(graph, torch.from_numpy(np.ascontiguousarray(X[rb : rb + nl])).cuda(), sp["L"], rows=S)
        res = op.svd(sp["k"], -1, sp["q"], sp["seed"])
        o = dict(U=res.U.cpu().numpy(), S=res.S.copy(), V=res.V.cpu().numpy(), r=op.r_rows())
        op.close()
        graph.close()
        return o

    outs = run_ranks(3, fn)
    assert sum(o["r"] for o in outs) == S.size
    U = np.concatenate([o["U"] for o in outs]).astype(np.float64)
    om = philox_omega(sp["seed"], 0, ref.shape[1], sp["l"])
    print(check_isvd_arrays(U, outs[0]["S"], outs[0]["V"].astype(np.float64), isvd(ref, sp["k"], om, sp["q"]),
                            sp["k"], f"subset {where} P=3"))
    for o in outs:
        assert np.array_equal(o["S"], outs[0]["S"]) and np.array_equal(o["V"], outs[0]["V"])


@pytest.mark.skipif(__import__("os").environ.get("ISVD_DIST_SPLIT") == "0", reason="already the child run")
def test_multirank_blocking_allgather_path():
    """The default distributed SpMM step splits every row's edges into local / remote parts so the
    local pass overlaps the all-gather on the collectives stream; ISVD_DIST_SPLIT=0 keeps the
    single pass after a blocking all-gather.  Both must meet parity: the P = 3 cases re-run in a
    child process with the switch off (it is read once per process)."""
    import os
    import subprocess
    import sys

    here = os.path.abspath(__file__)
    ids = [f"{here}::test_multirank_products_and_isvd[cfg2-3]", f"{here}::test_multirank_products_and_isvd[ragged-NE-3]",
           f"{here}::test_multirank_row_subset[first_block]"]
    env = dict(os.environ, ISVD_DIST_SPLIT="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *ids], env=env,
                       cwd=os.path.dirname(os.path.dirname(here)), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout, r.stdout[-2000:]


def test_multirank_more_ranks_than_rows():
    """P = 8 simulated ranks on an n = 5 graph: ranks 5..7 own no rows (zero-row CSR, empty
    gather-source slices, empty Grams and sign-rule candidates), NE and NC, against the oracle."""
    from oracle import NCOperator, NEOperator, adjacency, isvd, philox_omega
    from synth.graphs import edges_to_graph

    import paper_2111_06312_b200 as isvd_mod

    g = edges_to_graph(5, [(0, 1), (1, 2), (2, 3), (3, 4), (0, 4), (1, 3)])
    A = adjacency(g.n, g.row_ptr, g.col_idx)
    X = np.random.default_rng(1).standard_normal((5, 2)).astype(np.float32)
    w = np.full(3, 1 / 3)

    def fn(rank, ctx):
        rb, nl = isvd_mod.partition(g.n, ctx.world, ctx.rank)
        rp, ci = g.row_slice(rb, rb + nl)
        graph = isvd_mod.Graph(ctx, g.n, rp, ci)
        ne = isvd_mod.NE(graph, w, 0.2)
        a = ne.svd(2, 2, 1, 3)
        Xl = torch.from_numpy(np.ascontiguousarray(X[rb : rb + nl])).cuda() if nl > 0 else np.zeros((0, 2), np.float32)
        nc = isvd_mod.NC(graph, Xl, 1)
        b = nc.svd(2, 2, 1, 4)
        o = dict(Sa=a.S.copy(), Ua=a.U.cpu().numpy(), Va=a.V.cpu().numpy(), Sb=b.S.copy(), Ub=b.U.cpu().numpy(),
                 Vb=b.V.cpu().numpy(), nl=nl)
        nc.close()
        ne.close()
        graph.close()
        return o

    outs = run_ranks(8, fn)
    assert [o["nl"] for o in outs] == [1, 1, 1, 1, 1, 0, 0, 0]
    ref = NEOperator(A, w, 0.2)
    Ua = np.concatenate([o["Ua"] for o in outs]).astype(np.float64)
    Va = np.concatenate([o["Va"] for o in outs]).astype(np.float64)
    print(check_isvd_arrays(Ua, outs[0]["Sa"], Va, isvd(ref, 2, philox_omega(3, 0, 5, 4), 1), 2, "NE n=5 P=8"))
    refc = NCOperator(A, X, 1)
    Ub = np.concatenate([o["Ub"] for o in outs]).astype(np.float64)
    print(check_isvd_arrays(Ub, outs[0]["Sb"], outs[0]["Vb"].astype(np.float64),
                            isvd(refc, 2, philox_omega(4, 0, 4, 4), 1), 2, "NC n=5 P=8"))


def test_multirank_allgather_overlaps_local_pass():
    """Event trace of the distributed split (SURVEY 8(e) overlap item 1): with ISVD_SVD_PROFILE every
    all-gather of an SpMM gather source is bracketed by CUDA events on the collectives stream and the
    local SpMM pass issued meanwhile by events on the solver stream; the report gives the summed
    all-gather time and the part of it concurrent with a local pass.  At P = 2 on config 2 (one GPU:
    the peer-slice copies of the simulated backend share it with the SpMM) the all-gathers must be
    measured and partly hidden; results stay identical to the unprofiled call."""
    cfg, g, X, sp = _case("cfg2")

    def fn(r, ctx):
        op, graph, rb, nl = _rank_op(ctx, cfg, g, X, sp)
        res = op.svd(sp["k"], -1, sp["q"], sp["seed"], profile=True)
        ref = op.svd(sp["k"], -1, sp["q"], sp["seed"])
        out = {"ag": res.ms_allgather, "hidden": res.ms_allgather_hidden, "S": res.S, "S0": ref.S}
        op.close()
        graph.close()
        return out

    outs = run_ranks(2, fn)
    for r, o in enumerate(outs):
        print(f"rank {r}: all-gather {o['ag']:.3f} ms, hidden {o['hidden']:.3f} ms")
        assert o["ag"] > 0.0
        assert 0.0 < o["hidden"] <= o["ag"] + 1e-3
        assert np.array_equal(o["S"], o["S0"])
