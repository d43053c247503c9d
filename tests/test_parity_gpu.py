"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Acceptance (BASELINE.json north_star): single products M Q / M^T Q within 1e-5
relative (Frobenius), top-k singular values within 1e-4 relative, subspace
principal angles below 1e-3 rad.  Every input is seeded and synthetic (synth/);
the oracle draws its own Omega from the seed (oracle.philox_omega), so no oracle
input comes from the CUDA path.
"""
import numpy as np
import pytest

from parity_util import (ANGLE_TOL, PROD_TOL, SIG_TOL, assert_product, check_isvd, config_inputs, gpu_op,
                         oracle_isvd_result, oracle_op, rel_fro, sigma_rel, sin_theta, worst_col_rel)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_06312_b200 as isvd

    c = isvd.Context(0)
    yield c


_ops = {}


def _op(ctx, i):
    if i not in _ops:
        cfg, g, X, sp = config_inputs(i)
        _ops[i] = (gpu_op(ctx, cfg, g, X, sp), oracle_op(cfg, g, X, sp), cfg, sp)
    return _ops[i]


def _to_np(t):
    return t.detach().cpu().numpy().astype(np.float64)


# ----------------------------------------------------------------------- Omega


@pytest.mark.parametrize("i", [0, 1, 2, 3])
def test_omega_stream_matches_oracle(ctx, i):
    """Reading O11: the library's Philox/Box-Muller Omega equals the oracle's own
    implementation of the same stream (<= 1 fp32 ulp where libm rounding differs)."""
    from oracle import philox_omega

    op, _, cfg, sp = _op(ctx, i)
    om = _to_np(op.sample_omega(sp["k"], -1 if cfg["p"] is None else cfg["p"], sp["seed"])).astype(np.float32)
    ref = philox_omega(sp["seed"], 0, op.c_rows(), sp["l"])
    assert om.shape == ref.shape
    ulp = np.abs(om.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1
    assert (ulp != 0).mean() < 1e-4


# -------------------------------------------------------------------- products


def _q_inputs(op, sp, cfg, kind, side):
    """side 'c': operand of M . Q (c rows); 'r': operand of M^T . Q (r rows)."""
    from oracle import philox_omega

    rows = op.c_rows() if side == "c" else op.graph.n_local
    if kind == "omega":
        return philox_omega(sp["seed"] + 17, 0, rows, sp["l"])
    rng = np.random.default_rng(1000 + cfg["index"])
    Q, _ = np.linalg.qr(rng.standard_normal((rows, sp["l"])))
    return Q.astype(np.float32)


@pytest.mark.parametrize("i", [0, 1, 3, 2])
@pytest.mark.parametrize("kind", ["omega", "orthonormal"])
def test_products(ctx, i, kind):
    op, ref, cfg, sp = _op(ctx, i)
    Qc = _q_inputs(op, sp, cfg, kind, "c")
    Y = _to_np(op.matmul(torch.from_numpy(Qc).cuda()))
    Yref = ref.matmul(Qc.astype(np.float64))
    print(assert_product(Y, Yref, f"cfg{i} M.Q {kind}"))
    Qr = _q_inputs(op, sp, cfg, kind, "r")
    W = _to_np(op.matmul_T(torch.from_numpy(Qr).cuda()))
    Wref = ref.matmul_T(Qr.astype(np.float64))
    print(assert_product(W, Wref, f"cfg{i} M^T.Q {kind}"))


def _col_parallel(fn, M, cols, workers=None):
    """Apply the oracle product `fn` to column chunks of M in threads (columns of every product are
    independent; scipy's sparse kernels release the GIL).  Harness only: the oracle's arithmetic
    per column is unchanged."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    workers = workers or min(len(cols), os.cpu_count() or 1)
    chunks = np.array_split(np.asarray(cols), workers)
    with ThreadPoolExecutor(workers) as ex:
        parts = list(ex.map(lambda c: fn(M[:, c].astype(np.float64)), chunks))
    return np.concatenate(parts, axis=1), np.concatenate(chunks)


def test_products_config4_sampled_columns(ctx):
    """Config 4 at full size in the bench's launch configuration (width l = 400, the relabelled
    graph with its hub/split segments and L2 window): the oracle computes 64 of the 400 output
    columns -- 60 random ones plus the last float4 (396..399) -- checked on every row (all hub,
    split-fixup and ragged-tail rows included) and every sampled column."""
    op, ref, cfg, sp = _op(ctx, 4)
    from oracle import philox_omega

    l = sp["l"]
    rng = np.random.default_rng(404)
    cols = np.sort(np.concatenate([rng.choice(l - 4, 60, replace=False), np.arange(l - 4, l)]))
    G = philox_omega(99, 0, op.c_rows(), l)
    Y = _to_np(op.matmul(torch.from_numpy(G).cuda())[:, torch.from_numpy(cols).cuda()])
    Yref, _ = _col_parallel(ref.matmul, G, cols)
    print(assert_product(Y, Yref, "cfg4 M.G sampled"))
    Q = rng.standard_normal((op.graph.n_local, l)).astype(np.float32)
    W = _to_np(op.matmul_T(torch.from_numpy(Q).cuda())[:, torch.from_numpy(cols).cuda()])
    Wref, _ = _col_parallel(ref.matmul_T, Q, cols)
    print(assert_product(W, Wref, "cfg4 M^T.Q sampled"))


def test_duality_config4_full_width(ctx):
    """<H, M G> = <M^T H, G> at full size and full width (property at any size)."""
    op, _, cfg, sp = _op(ctx, 4)
    gen = torch.Generator(device="cuda").manual_seed(5)
    G = torch.randn(op.c_rows(), sp["l"], device="cuda", generator=gen)
    H = torch.randn(op.graph.n_local, sp["l"], device="cuda", generator=gen)
    MG = op.matmul(G)
    MtH = op.matmul_T(H)
    lhs = (H.double() * MG.double()).sum().item()
    rhs = (MtH.double() * G.double()).sum().item()
    scale = (H.double().norm() * MG.double().norm()).item()
    assert abs(lhs - rhs) <= 1e-5 * scale


# ----------------------------------------------------------------- full isvd


def _check_isvd(res, oref, k, label):
    return check_isvd(res, oref, k, label)


def _oracle_result(i):
    return oracle_isvd_result(i)


@pytest.mark.parametrize("i", [0, 1, 3, 2])
def test_isvd_parity(ctx, i):
    op, _, cfg, sp = _op(ctx, i)
    p = -1 if cfg["p"] is None else cfg["p"]
    res = op.svd(sp["k"], p, sp["q"], sp["seed"])
    assert res.l == sp["l"]
    print(_check_isvd(res, _oracle_result(i), sp["k"], f"cfg{i}"), "launches", res.kernel_launches,
          "ms", res.ms_total, "sweeps", res.jacobi_sweeps)
    # determinism: same seed, same world -> bitwise identical
    res2 = op.svd(sp["k"], p, sp["q"], sp["seed"])
    assert np.array_equal(res.S, res2.S)
    assert torch.equal(res.U, res2.U) and torch.equal(res.V, res2.V)


def test_isvd_host_output_equals_device_output(ctx):
    op, _, cfg, sp = _op(ctx, 0)
    a = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"])
    b = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"], host_output=True)
    assert np.array_equal(a.S, b.S)
    assert np.array_equal(_to_np(a.U), b.U.astype(np.float64))
    assert np.array_equal(_to_np(a.V), b.V.astype(np.float64))


def test_cholesky_fallback_still_in_parity(ctx):
    """Fault injection (ISVD_SVD_FORCE_CHOL_FAIL): every first Cholesky takes the shifted
    path and the third CholeskyQR pass runs; the result must still meet parity."""
    op, _, cfg, sp = _op(ctx, 0)
    res = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"], force_chol_fail=True)
    assert res.chol_fallbacks > 0
    _check_isvd(res, _oracle_result(0), sp["k"], "cfg0/fallback")


def test_cholesky_fallback_nc_deferred_update_in_parity(ctx):
    """NC (small c side): the r-side CholeskyQR2 defers its second update into the small
    products (Rfold); a forced shifted factorisation must form Q2, run the third pass and
    switch Rfold to I -- and still meet parity."""
    op, _, cfg, sp = _op(ctx, 2)
    res = op.svd(sp["k"], -1 if cfg["p"] is None else cfg["p"], sp["q"], sp["seed"], force_chol_fail=True)
    assert res.chol_fallbacks > 0
    # the first tall pass probes with the tensor-core Gram; the forced breakdown must take the
    # gated exact-Gram path (gram_probe_fallbacks) and still meet parity
    assert res.gram_probe_fallbacks > 0
    _check_isvd(res, _oracle_result(2), sp["k"], "cfg2/fallback")
    clean = op.svd(sp["k"], -1 if cfg["p"] is None else cfg["p"], sp["q"], sp["seed"])
    assert clean.gram_probe_fallbacks == 0  # config 2's M Omega is well conditioned: the probe holds


# ------------------------------------------------------------ edge cases


def _tiny_case(ctx, n, edges, C=None, lam=None, L=None, d=3, w=3, seed=0):
    import paper_2111_06312_b200 as isvd
    from oracle import NCOperator, NEOperator, adjacency, uniform_weights
    from synth.graphs import edges_to_graph

    g = edges_to_graph(n, edges)
    A = adjacency(g.n, g.row_ptr, g.col_idx)
    graph = isvd.Graph(ctx, n, g.row_ptr, g.col_idx)
    rng = np.random.default_rng(seed)
    if L is None:
        w_ = uniform_weights(C)
        return isvd.NE(graph, w_, lam), NEOperator(A, w_, lam), rng
    X = rng.standard_normal((n, d)).astype(np.float32)
    return isvd.NC(graph, torch.from_numpy(X).cuda(), L), NCOperator(A, X, L), rng


@pytest.mark.parametrize("C", [1, 2, 5])
def test_ne_isolated_node_and_ragged_width(ctx, C):
    """Isolated node (T row = 0, reading O3), width 3 (not a multiple of 4), n = 7."""
    op, ref, rng = _tiny_case(ctx, 7, [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5)], C=C, lam=1 / 7)
    Q = rng.standard_normal((7, 3)).astype(np.float32)
    assert_product(_to_np(op.matmul(torch.from_numpy(Q).cuda())), ref.matmul(Q.astype(np.float64)))
    assert_product(_to_np(op.matmul_T(torch.from_numpy(Q).cuda())), ref.matmul_T(Q.astype(np.float64)))


@pytest.mark.parametrize("L", [0, 1, 3])
def test_nc_small_and_degenerate(ctx, L):
    """L = 0 is X itself; ragged width 5."""
    op, ref, rng = _tiny_case(ctx, 9, [(i, (i + 1) % 9) for i in range(9)] + [(0, 4)], L=L, d=3)
    G = rng.standard_normal((3 * (L + 1), 5)).astype(np.float32)
    assert_product(_to_np(op.matmul(torch.from_numpy(G).cuda())), ref.matmul(G.astype(np.float64)))
    H = rng.standard_normal((9, 5)).astype(np.float32)
    assert_product(_to_np(op.matmul_T(torch.from_numpy(H).cuda())), ref.matmul_T(H.astype(np.float64)))


def test_hub_rows_are_split_and_exact(ctx):
    """A star with a hub of degree 3000 (> one 512-edge segment): split-row fixup path."""
    n = 3001
    op, ref, rng = _tiny_case(ctx, n, [(0, j) for j in range(1, n)] + [(j, j + 1) for j in range(1, n - 1)],
                              C=3, lam=1 / n)
    Q = rng.standard_normal((n, 12)).astype(np.float32)
    assert_product(_to_np(op.matmul(torch.from_numpy(Q).cuda())), ref.matmul(Q.astype(np.float64)))
    assert_product(_to_np(op.matmul_T(torch.from_numpy(Q).cuda())), ref.matmul_T(Q.astype(np.float64)))


def test_errors_are_reported_not_raised_across_abi(ctx):
    import paper_2111_06312_b200 as isvd
    from paper_2111_06312_b200._lib import IsvdError

    op, _, cfg, sp = _op(ctx, 0)
    with pytest.raises(IsvdError, match="RANK"):
        op.svd(op.shape[1] + 1, 0, 1, 0)
    with pytest.raises(IsvdError, match="RANK"):
        op.svd(0, 0, 1, 0)
    with pytest.raises(IsvdError):
        isvd.Graph(ctx, 3, np.array([0, 1, 0, 1]), np.array([1], dtype=np.int32))  # non-monotone row_ptr


def test_permutation_invariance_through_library(ctx):
    """Relabelling nodes leaves the singular values unchanged (north_star); NE with
    Omega' = P Omega supplied through ISVD_SVD_OMEGA_PROVIDED."""
    import paper_2111_06312_b200 as isvd

    op, _, cfg, sp = _op(ctx, 0)
    _, g, _, _ = config_inputs(0)
    perm = np.random.default_rng(7).permutation(g.n)
    gp = g.permuted(perm)
    opp = isvd.NE(isvd.Graph(ctx, gp.n, gp.row_ptr, gp.col_idx), sp["weights"], sp["lambda_ones"])
    om = op.sample_omega(sp["k"], cfg["p"], sp["seed"])
    omp = torch.empty_like(om)
    omp[torch.from_numpy(perm).cuda()] = om
    a = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"])
    b = opp.svd(sp["k"], cfg["p"], sp["q"], sp["seed"], omega=omp)
    assert sigma_rel(b.S, a.S) <= 1e-5
    Ua = _to_np(a.U)
    Ub = _to_np(b.U)[perm]
    assert sin_theta(Ub[:, :16], Ua[:, :16]) <= 1e-3


@pytest.mark.slow
def test_isvd_config4_exact(ctx):
    """Config 4: l = c = 400 makes Alg. 1 exact (reading O6), so the oracle is the exact SVD of
    M = [X | AX | A^2X | A^3X], taken through its 400 x 400 Gram in fp64.
    Checked: top-k singular values, the V subspace and the U subspace on every row."""
    from oracle.isvd_oracle import exact_svd_tall, nc_blocks

    op, ref, cfg, sp = _op(ctx, 4)
    res = op.svd(sp["k"], -1, sp["q"], sp["seed"])
    s, V, s_all, Ufun = exact_svd_tall(nc_blocks(ref), sp["k"])
    assert sigma_rel(res.S, s) <= SIG_TOL
    Vg = _to_np(res.V)
    assert sin_theta(Vg, V) <= ANGLE_TOL
    # U on ALL rows, in chunks: largest principal angle between span(U_gpu) and span(U_ref) from
    # k x k accumulations, sin^2 = lambda_max(I - M M^T), M = U_ref^T Q, Q = U_gpu R^-1 (R^T R =
    # U_gpu^T U_gpu in fp64) -- the sine form of parity_util.sin_theta without forming Q.
    Ugpu = res.U
    k = sp["k"]
    G = np.zeros((k, k))
    Cx = np.zeros((k, k))
    n = op.graph.n_local
    for r0 in range(0, n, 200_000):
        rows = np.arange(r0, min(n, r0 + 200_000))
        Ug = _to_np(Ugpu[r0 : r0 + len(rows)])
        Ur = Ufun(rows)
        G += Ug.T @ Ug
        Cx += Ur.T @ Ug
    R = np.linalg.cholesky(G).T
    Mx = np.linalg.solve(R.T, Cx.T).T  # U_ref^T U_gpu R^-1
    sin2 = np.linalg.eigvalsh(np.eye(k) - Mx @ Mx.T).max()
    sinU = float(np.sqrt(max(sin2, 0.0)))
    print("cfg4 exact: sin theta U (all rows)", sinU)
    assert sinU <= ANGLE_TOL


@pytest.mark.parametrize("i", [0, 2])
def test_distributed_schedule_world1_nccl(i):
    """The NCCL row-partitioned schedule (all-gathers, fp64 all-reduces, candidate all-gather of
    the sign rule) through a 1-rank communicator: same parity bar as the single-GPU path."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2111_06312_b200 as isvd

    cfg, g, X, sp = config_inputs(i)
    c = isvd.Context(0, rank=0, world=1, nccl_id=isvd.nccl_unique_id())
    op = gpu_op(c, cfg, g, X, sp)
    p = -1 if cfg["p"] is None else cfg["p"]
    res = op.svd(sp["k"], p, sp["q"], sp["seed"])
    _check_isvd(res, _oracle_result(i), sp["k"], f"cfg{i}/nccl")
    ref = oracle_op(cfg, g, X, sp)
    from oracle import philox_omega

    Qc = philox_omega(7, 0, op.c_rows(), sp["l"])
    assert_product(_to_np(op.matmul(torch.from_numpy(Qc).cuda())), ref.matmul(Qc.astype(np.float64)))


# ------------------------------------------------ tensor-core products (opt-in mode)


@pytest.mark.skipif(__import__("os").environ.get("ISVD_TC_PRODUCTS") == "1", reason="already the child run")
def test_tc_products_mode_parity():
    """ISVD_TC_PRODUCTS=1 routes X^T Z_j, X G_j, Y R^-1 and the final U, V through the tcgen05
    3xTF32 kernels (the default keeps tensor cores to the Gram, as north_star says).  Config 2
    (NC, n = 169343 >= the tensor-core row threshold) must meet the same parity bars: the
    product and isvd tests are re-run in a child process with the flag set (it is read once per
    process by the library)."""
    import os
    import subprocess
    import sys

    here = os.path.abspath(__file__)
    ids = [f"{here}::test_products[omega-2]", f"{here}::test_products[orthonormal-2]",
           f"{here}::test_isvd_parity[2]", f"{here}::test_distributed_schedule_world1_nccl[2]"]
    env = dict(os.environ, ISVD_TC_PRODUCTS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *ids], env=env,
                       cwd=os.path.dirname(os.path.dirname(here)), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "4 passed" in r.stdout, r.stdout[-2000:]


@pytest.mark.skipif(__import__("os").environ.get("ISVD_ALT_PATHS") == "1", reason="already the child run")
def test_alternative_kernel_paths_parity():
    """The switchable alternatives stay in parity: DFMA exact Gram (ISVD_DMMA=0), pairwise
    cooperative Jacobi (ISVD_JACOBI_PAIRWISE=1), SIMT Grams (ISVD_TC_GRAM=0), no allocator cache
    (ISVD_NO_POOL=1), NC dense terms overlapped on a second stream (ISVD_OVERLAP=1), the exact
    first Gram without the tensor-core probe (ISVD_GRAM_PROBE=0), the SpMM's sequential tail instead
    of the masked last batch (ISVD_SPMM_VARIANT=0) -- all at once, configs 2 (NC, l = 256)
    and 3 (NE, l = 160), in a child process (some switches are read once per process)."""
    import os
    import subprocess
    import sys

    here = os.path.abspath(__file__)
    ids = [f"{here}::test_isvd_parity[2]", f"{here}::test_isvd_parity[3]", f"{here}::test_products[orthonormal-2]"]
    env = dict(os.environ, ISVD_ALT_PATHS="1", ISVD_DMMA="0", ISVD_JACOBI_PAIRWISE="1", ISVD_TC_GRAM="0",
               ISVD_NO_POOL="1", ISVD_OVERLAP="1", ISVD_GRAM_PROBE="0", ISVD_SPMM_VARIANT="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *ids], env=env,
                       cwd=os.path.dirname(os.path.dirname(here)), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout, r.stdout[-2000:]


def test_allocator_cache_reuse_is_exact(ctx):
    """Graphs and operators rebuilt from the context's buffer cache give bitwise-identical
    results (workspaces are re-zeroed on reuse)."""
    import paper_2111_06312_b200 as isvd

    cfg, g, X, sp = config_inputs(0)
    p = -1 if cfg["p"] is None else cfg["p"]
    outs = []
    for _ in range(3):
        graph = isvd.Graph(ctx, g.n, g.row_ptr, g.col_idx)
        op = isvd.NE(graph, sp["weights"], sp["lambda_ones"])
        r = op.svd(sp["k"], p, sp["q"], sp["seed"])
        outs.append((r.S.copy(), _to_np(r.U)))
        op.close()
        graph.close()
    for S, U in outs[1:]:
        assert np.array_equal(S, outs[0][0])
        assert np.array_equal(U, outs[0][1])


# --------------------------------------------- paper-exact NE: +lambda A, Fig. 1 weights


@pytest.mark.parametrize("i", [0, 1])
def test_ne_paper_exact_lambda_adj_and_fig1_weights(ctx, i):
    """Eq. 3 as printed: M = sum_c w_c T^c - lambda (1 1^T - A) with the Fig. 1 triangular weights
     -- the +lambda A term is one extra SpMM of Q in the library.  Products and the isvd
    against the oracle's NEOperator(lambda_adj = lambda)."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import NEOperator, adjacency, context_weights, isvd, philox_omega

    cfg, g, X, sp = config_inputs(i)
    C = len(sp["weights"])
    w = context_weights(C)
    lam = sp["lambda_ones"]
    A = adjacency(g.n, g.row_ptr, g.col_idx)
    ref = NEOperator(A, w, lam, lambda_adj=lam)
    graph = isvd_mod.Graph(ctx, g.n, g.row_ptr, g.col_idx)
    op = isvd_mod.NE(graph, w, lam, lambda_adj=lam)
    rng = np.random.default_rng(77 + i)
    Q = rng.standard_normal((g.n, sp["l"])).astype(np.float32)
    Y = _to_np(op.matmul(torch.from_numpy(Q).cuda()))
    assert_product(Y, ref.matmul(Q.astype(np.float64)))
    W = _to_np(op.matmul_T(torch.from_numpy(Q).cuda()))
    assert_product(W, ref.matmul_T(Q.astype(np.float64)))
    p = -1 if cfg["p"] is None else cfg["p"]
    res = op.svd(sp["k"], p, sp["q"], sp["seed"])
    om = philox_omega(sp["seed"], 0, ref.shape[1], sp["l"])
    print(_check_isvd(res, isvd(ref, sp["k"], om, sp["q"]), sp["k"], f"cfg{i}/paper-exact"))
    op.close()
    graph.close()


# --------------------------------------------- Eq. 5 embeddings and Eq. 7 W* on the device (f1)


@pytest.mark.parametrize("i", [0, 2])
def test_embeddings_and_least_norm_match_oracle(ctx, i):
    """From the library's own SVD: L = U S^1/2 (Eq. 5) and W* = V S^+ U^T Y (Eq. 7) on one-hot
    synthetic labels, all rows and a labelled subset, against the oracle formulas
    applied to the same U, S, V (fp32 U/V promoted to fp64): W* within 1e-5 relative."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import embeddings as o_emb
    from oracle import least_norm as o_ln

    op, _, cfg, sp = _op(ctx, i)
    p = -1 if cfg["p"] is None else cfg["p"]
    res = op.svd(sp["k"], p, sp["q"], sp["seed"])
    U, V, S = _to_np(res.U), _to_np(res.V), res.S
    L = _to_np(isvd_mod.embeddings(ctx, res.U, S))
    Lo, _ = o_emb(U, S, V)
    assert rel_fro(L, Lo) <= 1e-6
    rng = np.random.default_rng(21 + i)
    n = U.shape[0]
    ny = 7
    Y = np.zeros((n, ny), dtype=np.float32)
    Y[np.arange(n), rng.integers(0, ny, n)] = 1.0
    shape = op.shape
    W = _to_np(isvd_mod.least_norm(ctx, res.U, S, res.V, torch.from_numpy(Y).cuda(), shape))
    assert rel_fro(W, o_ln(U, S, V, Y, shape=shape)) <= PROD_TOL
    rows = np.sort(rng.choice(n, size=max(1, n // 10), replace=False)).astype(np.int32)
    Wr = _to_np(isvd_mod.least_norm(ctx, res.U, S, res.V, torch.from_numpy(Y).cuda(), shape, rows=rows))
    assert rel_fro(Wr, o_ln(U, S, V, Y, rows=rows, shape=shape)) <= PROD_TOL


def test_materialised_nc_equals_implicit(ctx):
    """SURVEY 8(f) f3 (comparison path): M formed through the library (M . I) and the isvd of the
    explicit matrix (an NC operator with L = 0) meets the same parity bars against the oracle of
    the implicit operator (implicit = explicit, oracle S3)."""
    import paper_2111_06312_b200 as isvd_mod

    op, _, cfg, sp = _op(ctx, 2)
    c = op.shape[1]
    Mx = op.matmul(torch.eye(c, dtype=torch.float32, device="cuda"))
    opm = isvd_mod.NC(op.graph, Mx, 0)
    assert opm.shape == op.shape
    p = -1 if cfg["p"] is None else cfg["p"]
    res = opm.svd(sp["k"], p, sp["q"], sp["seed"])
    print(_check_isvd(res, _oracle_result(2), sp["k"], "cfg2/materialised"))
    opm.close()


@pytest.mark.parametrize("n,d,widths", [(1000, 100, (400, 132, 416, 200)), (777, 128, (256, 260)), (64, 36, (132,)),
                                         (4097, 16, (400,)), (130, 124, (388,)),
                                         # K-chunked streaming form (d >= 160; chunks of 40 or 32 k-steps)
                                         (1000, 200, (400, 132)), (333, 192, (256, 300)), (9600, 160, (416,))])
def test_k_resident_gemm_shapes(ctx, n, d, widths):
    """The K-resident (d <= 128) and K-chunked (d >= 160) persistent SIMT GEMMs (widths 132 .. 416; the
    triangular K-chunked form is the CholeskyQR apply of every isvd test with l >= 160): an NC operator with
    L = 0 is M = X, so M G = X G is that kernel alone.  Compile-time shapes (d = 100 / l = 400,
    d = 128 / l = 256), run-time shapes, ragged last row tiles (n not a multiple of 64), a single
    partial tile, more tiles than SMs, a last warp with padding columns; every entry against the
    fp64 product."""
    import paper_2111_06312_b200 as isvd_mod

    rng = np.random.default_rng(n + d)
    rp = np.arange(n + 1, dtype=np.int64)
    ci = ((np.arange(n) + 1) % n).astype(np.int32)  # a ring: the graph is unused at L = 0
    X = rng.standard_normal((n, d)).astype(np.float32)
    graph = isvd_mod.Graph(ctx, n, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    op = isvd_mod.NC(graph, torch.from_numpy(X).cuda(), 0)
    for w in widths:
        G = rng.standard_normal((d, w)).astype(np.float32)
        out = _to_np(op.matmul(torch.from_numpy(G).cuda()))
        ref = X.astype(np.float64) @ G.astype(np.float64)
        assert out.shape == ref.shape
        mag = np.abs(X).astype(np.float64) @ np.abs(G).astype(np.float64)
        assert np.max(np.abs(out - ref) / mag) <= 4e-7, (n, d, w)
        assert_product(out, ref)
    op.close()
    graph.close()


# --------------------------------------------- label re-use NC operator


@pytest.mark.parametrize("L,P", [(3, 2), (0, 2), (2, 1)])
def test_label_reuse_products_and_isvd(ctx, L, P):
    """M_LR = [X | ... | A_hat^L X | B Y_train | ... | B^P Y_train], B = A_hat - (D+I)^-1
    on config 2's graph with synthetic one-hot labels on 30 % of the nodes: products within 1e-5 of
    the oracle, and the isvd meets the parity bars."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import NCOperator, adjacency, isvd, philox_omega

    cfg, g, X, sp = config_inputs(2)
    rng = np.random.default_rng(40 + L + P)
    ny = 8
    Y = np.zeros((g.n, ny), dtype=np.float32)
    lab = rng.random(g.n) < 0.3
    Y[np.where(lab)[0], rng.integers(0, ny, lab.sum())] = 1.0
    ref = NCOperator(adjacency(g.n, g.row_ptr, g.col_idx), X, L, Y_train=Y, P=P)
    graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    op = isvd_mod.NC(graph, torch.from_numpy(np.ascontiguousarray(X)).cuda(), L, Y_train=Y, P=P)
    assert op.shape == ref.shape
    c = op.shape[1]
    Gm = rng.standard_normal((c, 24)).astype(np.float32)
    assert_product(_to_np(op.matmul(torch.from_numpy(Gm).cuda())), ref.matmul(Gm.astype(np.float64)))
    Q = rng.standard_normal((g.n, 24)).astype(np.float32)
    assert_product(_to_np(op.matmul_T(torch.from_numpy(Q).cuda())), ref.matmul_T(Q.astype(np.float64)))
    if L == 3:
        k = 64
        res = op.svd(k, -1, sp["q"], sp["seed"])
        om = philox_omega(sp["seed"], 0, c, res.l)
        print(_check_isvd(res, isvd(ref, k, om, sp["q"]), k, f"LR L={L} P={P}"))
    op.close()
    graph.close()


def test_non_finite_input_is_reported_not_returned(ctx):
    """A NaN in X propagates through every product; the solver must report it instead of returning
    garbage: the Cholesky breakdown check fires first (ISVD_ERR_NOT_PD after the shifted
    retries), and the output check fused into the sign flip of U (ISVD_ERR_NONFINITE) backs it up."""
    import paper_2111_06312_b200 as isvd_mod

    cfg, g, X, sp = config_inputs(2)
    Xn = np.ascontiguousarray(X).copy()
    Xn[17, 3] = np.nan
    graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    op = isvd_mod.NC(graph, torch.from_numpy(Xn).cuda(), sp["L"])
    with pytest.raises(RuntimeError) as e:
        op.svd(sp["k"], -1 if cfg["p"] is None else cfg["p"], sp["q"], sp["seed"])
    msg = str(e.value)
    assert "ISVD_ERR_NOT_PD" in msg or "ISVD_ERR_NONFINITE" in msg, msg
    op.close()
    graph.close()


@pytest.mark.parametrize("k,p", [(64, 100), (96, 96), (96, 98)])
def test_tc_gram_partial_last_tile(ctx, k, p):
    """Config 2 (n = 169,343, tcgen05 Gram engaged) at l = 164 and l = 192, where the symmetric
    Gram leaves the last 128-row tile's diagonal block ([128, l)^2, 36 and 64 rows) to the SIMT
    kernel, and at l = 194 (66 rows), where the tensor-core kernel computes that tile itself."""
    from oracle import isvd, philox_omega

    op, ref, cfg, sp = _op(ctx, 2)
    res = op.svd(k, p, sp["q"], sp["seed"])
    assert res.l == k + p
    om = philox_omega(sp["seed"], 0, ref.shape[1], k + p)
    print(_check_isvd(res, isvd(ref, k, om, sp["q"]), k, f"cfg2 l={k + p}"))


# --------------------------------------------- weighted A and the A_hat NE basis


def _edge_weights(g, seed):
    """Symmetric synthetic weights in [0.5, 2): a counter-based hash of the unordered pair."""
    from synth.streams import mix64

    rows = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    cols = g.col_idx.astype(np.int64)
    lo, hi = np.minimum(rows, cols), np.maximum(rows, cols)
    h = mix64((lo * np.int64(g.n) + hi + np.int64(seed) * np.int64(0x9E3779B9)).astype(np.uint64))
    return (0.5 + 1.5 * (h >> np.uint64(11)).astype(np.float64) / 2.0 ** 53).astype(np.float32)


@pytest.mark.parametrize("i,basis", [(0, "T"), (0, "Ahat"), (1, "Ahat"), (3, "Ahat")])
def test_ne_basis_and_weights(ctx, i, basis):
    """NE over T or A_hat, on the config's graph unweighted and with edge weights:
    products against the oracle's NEOperator on every row / column, and the isvd (Alg. 1)."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import NEOperator, adjacency, isvd, philox_omega

    cfg, g, X, sp = config_inputs(i)
    p = -1 if cfg["p"] is None else cfg["p"]
    for weighted in (False, True):
        vals = _edge_weights(g, 3 + i) if weighted else None
        A = adjacency(g.n, g.row_ptr, g.col_idx, vals)
        ref = NEOperator(A, sp["weights"], sp["lambda_ones"], basis=basis)
        graph = isvd_mod.Graph(ctx, g.n, g.row_ptr, g.col_idx, values=vals, validate=True)
        op = isvd_mod.NE(graph, sp["weights"], sp["lambda_ones"], basis=basis)
        rng = np.random.default_rng(500 + i)
        Q = rng.standard_normal((g.n, sp["l"])).astype(np.float32)
        tag = f"cfg{i} {basis} weighted={weighted}"
        print(assert_product(_to_np(op.matmul(torch.from_numpy(Q).cuda())), ref.matmul(Q.astype(np.float64)),
                             tag + " M.Q"))
        print(assert_product(_to_np(op.matmul_T(torch.from_numpy(Q).cuda())), ref.matmul_T(Q.astype(np.float64)),
                             tag + " M^T.Q"))
        res = op.svd(sp["k"], p, sp["q"], sp["seed"])
        om = philox_omega(sp["seed"], 0, g.n, sp["l"])
        print(_check_isvd(res, isvd(ref, sp["k"], om, sp["q"]), sp["k"], tag))
        op.close()
        graph.close()


def test_nc_weighted_config2(ctx):
    """NC (Eq. 6) on config 2's graph with edge weights: A_hat from the weighted degrees.
    Products on every row / column and the isvd against the oracle."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import NCOperator, adjacency, isvd, philox_omega

    cfg, g, X, sp = config_inputs(2)
    vals = _edge_weights(g, 9)
    ref = NCOperator(adjacency(g.n, g.row_ptr, g.col_idx, vals), X, sp["L"])
    graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(),
                           values=torch.from_numpy(vals).cuda())
    op = isvd_mod.NC(graph, torch.from_numpy(np.ascontiguousarray(X)).cuda(), sp["L"])
    rng = np.random.default_rng(71)
    G = rng.standard_normal((op.shape[1], sp["l"])).astype(np.float32)
    print(assert_product(_to_np(op.matmul(torch.from_numpy(G).cuda())), ref.matmul(G.astype(np.float64)), "M.G w"))
    H = rng.standard_normal((g.n, sp["l"])).astype(np.float32)
    print(assert_product(_to_np(op.matmul_T(torch.from_numpy(H).cuda())), ref.matmul_T(H.astype(np.float64)),
                         "M^T.H w"))
    res = op.svd(sp["k"], -1, sp["q"], sp["seed"])
    om = philox_omega(sp["seed"], 0, op.shape[1], sp["l"])
    print(_check_isvd(res, isvd(ref, sp["k"], om, sp["q"]), sp["k"], "cfg2 weighted"))
    op.close()
    graph.close()


def test_weighted_config4_relabelled_sampled_columns(ctx):
    """Weights through the degree relabelling of a large graph (config 4, the weights move with
    their edges): M.G on 8 sampled columns (incl. the last float4) against the oracle, every row."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import NCOperator, adjacency, philox_omega

    cfg, g, X, sp = config_inputs(4)
    vals = _edge_weights(g, 4)
    ref = NCOperator(adjacency(g.n, g.row_ptr, g.col_idx, vals), X, sp["L"])
    graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(),
                           values=torch.from_numpy(vals).cuda())
    op = isvd_mod.NC(graph, torch.from_numpy(np.ascontiguousarray(X)).cuda(), sp["L"])
    cols = np.array([3, 101, 250, 396, 397, 398, 399])
    G = philox_omega(77, 0, op.shape[1], sp["l"])
    Y = _to_np(op.matmul(torch.from_numpy(G).cuda())[:, torch.from_numpy(cols).cuda()])
    Yref, _ = _col_parallel(ref.matmul, G, cols)
    print(assert_product(Y, Yref, "cfg4 weighted M.G"))
    op.close()
    graph.close()


def test_isvd_wide_working_width_l600(ctx):
    """l > 512 takes the single-CTA Cholesky with its global-memory matrix and the 1024-entry
    scratch (l in (512, 1024] overflowed a 512-entry shared array): config 1's graph,
    k = 300, p = 300 -> l = 600, q = 1, against the oracle."""
    from oracle import isvd, philox_omega

    op, ref, cfg, sp = _op(ctx, 1)
    res = op.svd(300, 300, 1, 42)
    assert res.l == 600
    om = philox_omega(42, 0, ref.shape[1], 600)
    print(_check_isvd(res, isvd(ref, 300, om, 1), 300, "cfg1 l=600"))


def test_solver_on_a_nonblocking_caller_stream():
    """workspaces are cleared / copied on the ctx stream, so a caller on a non-blocking
    torch stream gets the same (bitwise) result as on the default stream."""
    import paper_2111_06312_b200 as isvd_mod

    cfg, g, X, sp = config_inputs(2)
    outs = []
    for use_side in (False, True):
        st = torch.cuda.Stream() if use_side else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            c = isvd_mod.Context(0, stream=st)
            op = gpu_op(c, cfg, g, X, sp)
            r = op.svd(sp["k"], -1, sp["q"], sp["seed"])
            outs.append((r.S.copy(), r.U.cpu().numpy()))
            op.close()
            op.graph.close()
            c.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_library_allocator_and_torch_allocator_agree():
    """Device memory from PyTorch's caching allocator (the default binding) or from the library's
    own cudaMalloc cache: bitwise-identical results (config 0)."""
    import paper_2111_06312_b200 as isvd_mod

    cfg, g, X, sp = config_inputs(0)
    outs = []
    for alloc in ("torch", None):
        c = isvd_mod.Context(0, allocator=alloc)
        op = gpu_op(c, cfg, g, X, sp)
        r = op.svd(sp["k"], cfg["p"], sp["q"], sp["seed"])
        outs.append((r.S.copy(), _to_np(r.U)))
        op.close()
        op.graph.close()
        c.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_spectral_kernel_on_a_gpu_spectrum(ctx):
    """Eq. 9 (discretised P:1057-1065) applied to the library's own singular values of
    config 2: isvd_spectral_kernel equals the oracle's literal formula (f4 on the -m gpu path)."""
    from oracle import spectral_kernel as o_sk

    import paper_2111_06312_b200 as isvd_mod

    op, _, cfg, sp = _op(ctx, 2)
    res = op.svd(sp["k"], -1, sp["q"], sp["seed"])
    S = res.S / res.S[0] * 1.9  # spread the spectrum over Eq. 9's (0, 2] range
    for mu, sb in ((1.0, 0.0), (1.5, 3.0), (0.7, -2.0)):
        assert np.allclose(isvd_mod.spectral_kernel(S, mu, sb), o_sk(S, mu, sb), rtol=1e-12, atol=0)


# --------------------------------------------- implicit row gather (option (ii))


@pytest.mark.parametrize("i", [0, 2, 4])
def test_row_subset_operator(ctx, i):
    """M_S = M[S, :] for a 30 % labelled-node subset S (P:209-210 option (ii)) without forming M or
    the submatrix: products (caller order, every row / column) against the oracle's
    RowSubsetOperator and, for configs 0 and 2, the isvd (Alg. 1 of M_S).  Config 4 (relabelled
    graph): the subset rows go through the relabelling maps; products on 8 columns."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import RowSubsetOperator, isvd, philox_omega

    cfg, g, X, sp = config_inputs(i)
    rng = np.random.default_rng(600 + i)
    S = np.sort(rng.choice(g.n, int(0.3 * g.n), replace=False)).astype(np.int64)
    graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    if cfg["op"] == "NE":
        op = isvd_mod.NE(graph, sp["weights"], sp["lambda_ones"], rows=S)
    else:
        op = isvd_mod.NC(graph, torch.from_numpy(np.ascontiguousarray(X)).cuda(), sp["L"], rows=S)
    ref = RowSubsetOperator(oracle_op(cfg, g, X, sp), S)
    assert op.shape == ref.shape and op.r_rows() == S.size
    w = 8 if i == 4 else sp["l"]
    G = rng.standard_normal((op.shape[1], w)).astype(np.float32)
    H = rng.standard_normal((S.size, w)).astype(np.float32)
    if i == 4:
        Yref, _ = _col_parallel(ref.matmul, G, np.arange(w))
        Wref, _ = _col_parallel(ref.matmul_T, H, np.arange(w))
    else:
        Yref, Wref = ref.matmul(G.astype(np.float64)), ref.matmul_T(H.astype(np.float64))
    print(assert_product(_to_np(op.matmul(torch.from_numpy(G).cuda())), Yref, f"cfg{i} subset M_S.G"))
    print(assert_product(_to_np(op.matmul_T(torch.from_numpy(H).cuda())), Wref, f"cfg{i} subset M_S^T.H"))
    if i != 4:
        p = -1 if cfg["p"] is None else cfg["p"]
        l = min(sp["l"], *op.shape)
        res = op.svd(sp["k"], p, sp["q"], sp["seed"])
        om = philox_omega(sp["seed"], 0, op.shape[1], res.l)
        print(_check_isvd(res, isvd(ref, sp["k"], om, sp["q"]), sp["k"], f"cfg{i} subset"))
        assert res.l == l
    op.close()
    graph.close()


# --------------------------------------------- degenerate inputs


def test_edgeless_graph_both_families(ctx):
    """nnz = 0 (every node isolated): NE's T is 0 (reading O3), so M = -lambda 1 1^T (rank 1,
    sigma_1 = lambda n); NC's A_hat is I, so M = [X | X | X | X].  Products and the isvd (k = 1 for
    NE: the only nonzero singular value; k = l = 3 = rank(M) for NC) against the oracle."""
    import paper_2111_06312_b200 as isvd_mod
    from oracle import NCOperator, NEOperator, adjacency, isvd, philox_omega

    n = 6
    rp = np.zeros(n + 1, dtype=np.int64)
    ci = np.zeros(0, dtype=np.int32)
    A = adjacency(n, rp, ci)
    graph = isvd_mod.Graph(ctx, n, rp, ci)
    ne = isvd_mod.NE(graph, [0.5, 0.5], 0.25)
    ref = NEOperator(A, [0.5, 0.5], 0.25)
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((n, 4)).astype(np.float32)
    assert_product(_to_np(ne.matmul(torch.from_numpy(Q).cuda())), ref.matmul(Q.astype(np.float64)))
    assert_product(_to_np(ne.matmul_T(torch.from_numpy(Q).cuda())), ref.matmul_T(Q.astype(np.float64)))
    res = ne.svd(1, 3, 1, 7)
    assert abs(res.S[0] - 0.25 * n) <= 1e-6 * 0.25 * n
    X = rng.standard_normal((n, 3)).astype(np.float32)
    nc = isvd_mod.NC(graph, torch.from_numpy(X).cuda(), 3)
    refc = NCOperator(A, X, 3)
    G = rng.standard_normal((12, 5)).astype(np.float32)
    assert_product(_to_np(nc.matmul(torch.from_numpy(G).cuda())), refc.matmul(G.astype(np.float64)))
    assert_product(_to_np(nc.matmul_T(torch.from_numpy(Q).cuda())), refc.matmul_T(Q.astype(np.float64)))
    r2 = nc.svd(3, 0, 1, 11)  # l = 3 = rank(M): Y = M Omega has full column rank
    om = philox_omega(11, 0, 12, 3)
    _check_isvd(r2, isvd(refc, 3, om, 1), 3, "edgeless NC")
    nc.close()
    ne.close()
    graph.close()


def test_single_node_graph(ctx):
    """n = 1: NE with C = 1, lambda = 0 is T = [0]; NC (L = 2) of a single node is [x | x | x]
    (A_hat = [1]).  k = 1 isvd of the NC op against its exact SVD."""
    import paper_2111_06312_b200 as isvd_mod

    rp = np.zeros(2, dtype=np.int64)
    ci = np.zeros(0, dtype=np.int32)
    graph = isvd_mod.Graph(ctx, 1, rp, ci)
    x = np.array([[3.0, 4.0]], dtype=np.float32)
    nc = isvd_mod.NC(graph, torch.from_numpy(x).cuda(), 2)
    assert nc.shape == (1, 6)
    res = nc.svd(1, 0, 1, 0)
    assert abs(res.S[0] - np.sqrt(3 * 25.0)) <= 1e-5 * np.sqrt(75.0)
    nc.close()
    graph.close()


# ------------------------------------- SpMM variants: register (LDG) gather vs shared-memory staged gather


def _with_spmm_variant(v, fn):
    import os

    old = os.environ.get("ISVD_SPMM_VARIANT")
    os.environ["ISVD_SPMM_VARIANT"] = str(v)  # read per launch by launch_spmm
    try:
        out = fn()
        torch.cuda.synchronize()
        return out
    finally:
        if old is None:
            del os.environ["ISVD_SPMM_VARIANT"]
        else:
            os.environ["ISVD_SPMM_VARIANT"] = old


@pytest.mark.parametrize("i", [0, 1, 2, 3, 4])
def test_spmm_bulk_equals_ldg(ctx, i):
    """The shared-memory / bulk-copy staged gather (ISVD_SPMM_VARIANT=2, spmm_bulk_kernel) forms the
    same fp32 batches of 8 and the same fp64 sums as the register gather (variant 1), so M.Q and
    M^T.Q are bitwise equal on every config (hub-split segments, relabelled config 4, ragged widths),
    and -- transitively -- in parity with the oracle wherever variant 1 is."""
    op, _, cfg, sp = _op(ctx, i)
    gen = torch.Generator(device="cuda").manual_seed(1000 + i)
    G = torch.randn(op.c_rows(), sp["l"], device="cuda", generator=gen)
    H = torch.randn(op.graph.n_local, sp["l"], device="cuda", generator=gen)
    for f in (lambda: op.matmul(G), lambda: op.matmul_T(H)):
        a = _with_spmm_variant(1, f)
        b = _with_spmm_variant(2, f)
        assert torch.equal(a, b), float((a - b).abs().max())


def test_spmm_bulk_equals_ldg_weighted_and_split(ctx):
    """Bitwise equality of the two gathers on a weighted graph (config 2 with edge weights, the
    kW kernels) and on a star whose hub row is split into several segments (fixup path)."""
    import paper_2111_06312_b200 as isvd_mod

    cfg, g, X, sp = config_inputs(2)
    vals = _edge_weights(g, 9)
    graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(),
                           values=torch.from_numpy(vals).cuda())
    op = isvd_mod.NC(graph, torch.from_numpy(np.ascontiguousarray(X)).cuda(), sp["L"])
    gen = torch.Generator(device="cuda").manual_seed(7)
    G = torch.randn(op.shape[1], sp["l"], device="cuda", generator=gen)
    H = torch.randn(g.n, sp["l"], device="cuda", generator=gen)
    for f in (lambda: op.matmul(G), lambda: op.matmul_T(H)):
        assert torch.equal(_with_spmm_variant(1, f), _with_spmm_variant(2, f))
    op.close()
    graph.close()
    n = 3001
    op2, _, rng = _tiny_case(ctx, n, [(0, j) for j in range(1, n)] + [(j, j + 1) for j in range(1, n - 1)],
                             C=3, lam=1 / n)
    Q = torch.from_numpy(rng.standard_normal((n, 12)).astype(np.float32)).cuda()
    for f in (lambda: op2.matmul(Q), lambda: op2.matmul_T(Q)):
        assert torch.equal(_with_spmm_variant(1, f), _with_spmm_variant(2, f))


# ------------------------------ dense-A NE products on tensor cores (comparison variant)


@pytest.mark.parametrize("mode", ["i8", "tf32"])
@pytest.mark.parametrize("i", [0, 1, 3])
def test_dense_adjacency_products_and_isvd(ctx, i, mode):
    """ISVD_DENSE_A at graph creation: A is held dense (n <= 32768) and every SpMM step runs on tensor
    cores plus the same fp64 epilogue.  mode i8 (ISVD_DENSE_A=1, unweighted): the exact INT8 product of
    the binary A with the 3-byte fixed-point slices of Y (dense_i8.cu) -- every bar of this suite.
    mode tf32 (ISVD_DENSE_A=2): the 3xTF32 row contraction of gram_tc.cu -- at config 3 (C = 10,
    q = 6, 625 neighbours, M Q cancelling against the rank-1 term) its truncating fp32 accumulation
    meets north_star's Frobenius bar but not the per-column one, so only the former is asserted there."""
    import os

    import paper_2111_06312_b200 as isvd_mod

    cfg, g, X, sp = config_inputs(i)
    ref = oracle_op(cfg, g, X, sp)
    os.environ["ISVD_DENSE_A"] = "1" if mode == "i8" else "2"
    try:
        graph = isvd_mod.Graph(ctx, g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda())
    finally:
        del os.environ["ISVD_DENSE_A"]
    op = isvd_mod.NE(graph, sp["weights"], sp["lambda_ones"])
    rng = np.random.default_rng(300 + i)
    Q = rng.standard_normal((g.n, sp["l"])).astype(np.float32)
    for tag, Y, Yref in ((f"cfg{i} {mode} M.Q", op.matmul(torch.from_numpy(Q).cuda()), ref.matmul(Q.astype(np.float64))),
                         (f"cfg{i} {mode} M^T.Q", op.matmul_T(torch.from_numpy(Q).cuda()),
                          ref.matmul_T(Q.astype(np.float64)))):
        Y = _to_np(Y)
        if i == 3 and mode == "tf32":
            e = rel_fro(Y, Yref)
            print(tag, f"fro {e:.2e} (worst col {worst_col_rel(Y, Yref):.2e})")
            assert e <= PROD_TOL
        else:
            print(assert_product(Y, Yref, tag))
    p = -1 if cfg["p"] is None else cfg["p"]
    res = op.svd(sp["k"], p, sp["q"], sp["seed"])
    print(check_isvd(res, oracle_isvd_result(i), sp["k"], f"cfg{i} {mode} isvd"))
    op.close()
    graph.close()


def test_gram_probe_sticky_skip_config4(ctx):
    """Config 4 (l = c = 400, square Omega): kappa(M Omega)^2 is too large for the tensor-core probe
    of the first Gram, which falls back to the exact fp64 Gram; the op remembers it and later calls
    take the exact Gram directly (no probe), with bitwise-identical results (the exact path is the
    same kernels either way)."""
    op, _, cfg, sp = _op(ctx, 4)
    r1 = op.svd(sp["k"], -1, sp["q"], sp["seed"])
    r2 = op.svd(sp["k"], -1, sp["q"], sp["seed"])
    assert r1.gram_probe_fallbacks > 0 or r1.gram_probe_skipped == 1
    assert r2.gram_probe_skipped == 1 and r2.gram_probe_fallbacks == 0
    assert np.array_equal(r1.S, r2.S)
    assert torch.equal(r1.U, r2.U)


@pytest.mark.parametrize("mode", ["1", "2"])
def test_dense_adjacency_tiny_isolated_ragged(ctx, mode):
    """Dense-A paths (INT8 exact / 3xTF32) on a 7-node graph with an isolated node (zero row of T,
    reading O3), width 3 (ragged: one 16-row / 64-byte tile, zero-filled beyond n and w), and on a
    130-node cycle plus chords (two 128-row output tiles, the second with 2 rows), both directions."""
    import os

    import paper_2111_06312_b200 as isvd_mod
    from oracle import NEOperator, adjacency, uniform_weights
    from synth.graphs import edges_to_graph

    for n, edges, w in ((7, [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5)], 3),
                        (130, [(i, (i + 1) % 130) for i in range(130)] + [(i, (i + 17) % 130) for i in range(0, 130, 3)],
                         20)):
        g = edges_to_graph(n, edges)
        os.environ["ISVD_DENSE_A"] = mode
        try:
            graph = isvd_mod.Graph(ctx, n, g.row_ptr, g.col_idx)
        finally:
            del os.environ["ISVD_DENSE_A"]
        wts = uniform_weights(3)
        op = isvd_mod.NE(graph, wts, 1.0 / n)
        ref = NEOperator(adjacency(g.n, g.row_ptr, g.col_idx), wts, 1.0 / n)
        Q = np.random.default_rng(n).standard_normal((n, w)).astype(np.float32)
        print(assert_product(_to_np(op.matmul(torch.from_numpy(Q).cuda())), ref.matmul(Q.astype(np.float64)),
                             f"dense{mode} n={n} M.Q"))
        print(assert_product(_to_np(op.matmul_T(torch.from_numpy(Q).cuda())), ref.matmul_T(Q.astype(np.float64)),
                             f"dense{mode} n={n} M^T.Q"))
        Qn = Q.copy()
        Qn[1, 0] = np.nan  # a non-finite input must not come back as finite data
        assert not np.isfinite(_to_np(op.matmul(torch.from_numpy(Qn).cuda()))).all()
        op.close()
        graph.close()


def test_products_after_a_wider_call_config2(ctx):
    """An operator first used at width 256 and then at narrower widths (160, 100, 36) reuses its
    workspaces, which are sized for every width up to the widest seen (the tilings of a narrower
    product can need more row parts); every product still meets the bar."""
    op, ref, cfg, sp = _op(ctx, 2)
    rng = np.random.default_rng(2024)
    for w in (256, 160, 100, 36):
        H = rng.standard_normal((op.graph.n_local, w)).astype(np.float32)
        print(assert_product(_to_np(op.matmul_T(torch.from_numpy(H).cuda())), ref.matmul_T(H.astype(np.float64)),
                             f"cfg2 M^T.H w={w}"))
        G = rng.standard_normal((op.c_rows(), w)).astype(np.float32)
        print(assert_product(_to_np(op.matmul(torch.from_numpy(G).cuda())), ref.matmul(G.astype(np.float64)),
                             f"cfg2 M.G w={w}"))
