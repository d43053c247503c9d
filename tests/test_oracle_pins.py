"""Pins of the fp64 oracle against things other than itself (no GPU).

Each test names the passage / closed form it checks.  P:n = PAPER.md line n,
S:n = SPEC.md line n (test ideas only).  These must pass before the CUDA path
is compared against the oracle.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import (
    NCOperator,
    NEOperator,
    adjacency,
    context_weights,
    exact_svd,
    isvd,
    orthonorm_cholesky,
    orthonorm_qr,
    philox4x32_10,
    philox_omega,
    sign_fix,
    sym_norm_adj,
    transition,
    uniform_weights,
)
from oracle.isvd_oracle import DenseOperator
from synth.graphs import edges_to_graph, powerlaw_graph


def _A(n, edges):
    g = edges_to_graph(n, edges)
    return adjacency(g.n, g.row_ptr, g.col_idx)


def _complete(n):
    return _A(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def _cycle(n):
    return _A(n, [(i, (i + 1) % n) for i in range(n)])


def _random_connected(n, extra, rng):
    edges = {(i, int(rng.integers(0, i))) for i in range(1, n)}  # random tree
    extra = min(extra, n * (n - 1) // 2 - (n - 1))
    while len(edges) < n - 1 + extra:
        u, v = (int(x) for x in rng.integers(0, n, 2))
        if u != v and (u, v) not in edges and (v, u) not in edges:
            edges.add((u, v))
    return _A(n, sorted(edges))


# --------------------------------------------------------------------- Omega


def test_philox_known_answer_vectors(golden):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    for row in golden("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in row]
        out = philox4x32_10(np.array(v[:4]), (v[4], v[5]))
        assert [int(x) for x in out] == v[6:]


def test_omega_slices_are_consistent_and_standard_normal():
    """Counter-based: any row block equals the slice of the full matrix (P-invariance of
    the row partition); moments of N(0,1)."""
    full = philox_omega(7, 0, 1000, 37)
    part = philox_omega(7, 313, 101, 37)
    assert np.array_equal(full[313:414], part)
    z = philox_omega(11, 0, 20000, 50).astype(np.float64).ravel()
    assert abs(z.mean()) < 5 * 1 / np.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5 * np.sqrt(2.0 / z.size)
    assert abs((z ** 3).mean()) < 5 * np.sqrt(15.0 / z.size)
    assert abs((z ** 4).mean() - 3.0) < 5 * np.sqrt(96.0 / z.size)


# ----------------------------------------------------------- graph matrices


def test_transition_path_graph():
    """T = D^-1 A on the path 0-1-2."""
    T = transition(_A(3, [(0, 1), (1, 2)])).toarray()
    assert np.array_equal(T, [[0, 1, 0], [0.5, 0, 0.5], [0, 1, 0]])


def test_transition_isolated_node_row_is_zero():
    """0^-1 := 0 leaves the isolated node's row zero (reading O3)."""
    T = transition(_A(4, [(0, 1), (1, 2)])).toarray()
    assert np.array_equal(T[3], np.zeros(4))
    assert np.allclose(T[:3].sum(axis=1), 1.0)


def test_ahat_single_and_two_nodes():
    """A_hat of one node = [1]; of two connected nodes = [[.5,.5],[.5,.5]]."""
    assert np.array_equal(sym_norm_adj(_A(1, [])).toarray(), [[1.0]])
    assert np.allclose(sym_norm_adj(_A(2, [(0, 1)])).toarray(), [[0.5, 0.5], [0.5, 0.5]], atol=1e-15)


def test_ahat_path_graph_hand_values(golden):
    """Middle row of A_hat on the path 0-1-2, derived by hand in tests/golden/path3_hand.txt."""
    rows = {r[0]: [float(x) for x in r[1:]] for r in golden("path3_hand.txt")}
    Ah = sym_norm_adj(_A(3, [(0, 1), (1, 2)])).toarray()
    assert np.allclose(Ah[1], rows["nc_ahat_row1"], rtol=0, atol=1e-15)
    assert np.allclose(Ah, Ah.T, atol=0)


# ---------------------------------------------------------- context weights


def test_context_weights_fig1(golden):
    """C=3 -> [3,2,1]/6 exactly as Fig. 1's code."""
    rows = golden("fig1_context_weights.txt")
    C = int(rows[0][1])
    want = [float(Fraction(x)) for x in rows[1]]
    assert np.array_equal(context_weights(C), want)


def test_context_weights_closed_forms():
    """C=1 -> [1]; C=10 -> (11-q)/55; uniform 1/C sums to 1."""
    assert np.array_equal(context_weights(1), [1.0])
    assert np.allclose(context_weights(10), [(11 - q) / 55 for q in range(1, 11)], rtol=0, atol=1e-16)
    assert abs(uniform_weights(7).sum() - 1.0) < 1e-15
    with pytest.raises(ValueError):
        context_weights(0)


# -------------------------------------------------------------- NE operator


def test_ne_path_graph_hand_values(golden):
    """Eq. 3 on the path 0-1-2, C=2 uniform, lambda=1/3: rank 1, hand-derived entries and sigma."""
    rows = {r[0]: [float(x) for x in r[1:]] for r in golden("path3_hand.txt")}
    op = NEOperator(_A(3, [(0, 1), (1, 2)]), uniform_weights(2), 1.0 / 3.0)
    M = op.dense()
    assert np.allclose(M, np.tile(rows["ne_M_row"], (3, 1)), rtol=0, atol=1e-15)
    U, s, V, _ = isvd(op, 1, philox_omega(5, 0, 3, 3), iterations=1)
    assert abs(s[0] - rows["ne_sigma1"][0]) < 1e-15
    assert np.allclose(U[:, 0], np.full(3, 1 / np.sqrt(3)), atol=1e-14)
    assert np.allclose(V[:, 0], np.array([-1.0, 2.0, -1.0]) / np.sqrt(6), atol=1e-14)


@pytest.mark.parametrize("C", [1, 5, 10])
def test_ne_null_vector(C):
    """T 1 = 1 (row-stochastic) and sum w = 1 => M 1 = (sum w - lambda n) 1 = 0."""
    rng = np.random.default_rng(C)
    for t in range(20):
        n = 30
        op = NEOperator(_random_connected(n, 25, rng), uniform_weights(C), 1.0 / n)
        assert np.abs(op.matmul(np.ones((n, 1)))).max() < 1e-14
        op2 = NEOperator(_random_connected(n, 25, rng), context_weights(C), 1.0 / n)
        assert np.abs(op2.matmul(np.ones((n, 1)))).max() < 1e-14


@pytest.mark.parametrize("C,weights", [(1, "u"), (5, "u"), (10, "u"), (3, "t"), (10, "t")])
def test_ne_complete_graph_spectrum(C, weights):
    """K_n: T = (J - I)/(n-1) has eigenvalues 1 (on 1) and -1/(n-1) (mult. n-1), so
    sigma(M) = |sum_c w_c (-1/(n-1))^c| (mult. n-1) and 0 -- computed by Alg. 1 with l = n."""
    w = uniform_weights(C) if weights == "u" else context_weights(C)
    for n in range(5, 13):
        op = NEOperator(_complete(n), w, 1.0 / n)
        mu = -1.0 / (n - 1)
        want = abs(sum(w[c - 1] * mu ** c for c in range(1, C + 1)))
        _, s, _, s_all = isvd(op, n - 1, philox_omega(n, 0, n, n), iterations=1)
        assert np.allclose(s, want, rtol=1e-12, atol=1e-15)
        assert abs(s_all[-1]) < 1e-13


@pytest.mark.parametrize("C", [1, 5, 10])
def test_ne_cycle_spectrum(C):
    """Cycle C_n: T = (P + P^T)/2 with eigenvalues cos(2 pi j / n), so the singular values
    are {|sum_c w_c cos(2 pi j/n)^c| : j = 1..n-1} plus 0 (the 1-direction)."""
    w = uniform_weights(C)
    for n in range(6, 17):
        op = NEOperator(_cycle(n), w, 1.0 / n)
        lam = np.cos(2 * np.pi * np.arange(1, n) / n)
        want = np.sort(np.abs([sum(w[c - 1] * x ** c for c in range(1, C + 1)) for x in lam]))[::-1]
        _, _, _, s_all = isvd(op, n - 1, philox_omega(100 + n, 0, n, n), iterations=2)
        assert np.allclose(s_all[: n - 1], want, rtol=0, atol=1e-13)
        assert s_all[n - 1] < 1e-13


def test_ne_degenerate_c1_lambda0_is_T():
    """build_ne with lambda = 0, C = 1 is T itself."""
    rng = np.random.default_rng(3)
    A = _random_connected(12, 10, rng)
    op = NEOperator(A, [1.0], 0.0)
    G = rng.standard_normal((12, 4))
    assert np.allclose(op.matmul(G), transition(A) @ G, rtol=0, atol=1e-15)


def test_ne_lambda_adj_term():
    """Eq. 3's -lambda(1 - A) = -lambda 1 1^T + lambda A (P:145, P:254 'row1.T @ row1 - A')."""
    A = _A(4, [(0, 1), (1, 2), (2, 3)])
    lam = 0.05
    op = NEOperator(A, context_weights(3), lam, lam)
    T = transition(A).toarray()
    want = sum(w * np.linalg.matrix_power(T, c) for c, w in zip(range(1, 4), context_weights(3)))
    want = want - lam * (np.ones((4, 4)) - A.toarray())
    assert np.allclose(op.dense(), want, rtol=0, atol=1e-15)


# -------------------------------------------------------------- NC operator


def test_nc_path_graph_hand_values(golden):
    """Eq. 6 with X = e_0, L = 1 on the path graph: sigma^2 are the roots of the
    characteristic polynomial derived by hand (tests/golden/path3_hand.txt)."""
    rows = {r[0]: [float(x) for x in r[1:]] for r in golden("path3_hand.txt")}
    op = NCOperator(_A(3, [(0, 1), (1, 2)]), np.array([[1.0], [0.0], [0.0]]), 1)
    want = np.sort(np.sqrt(np.roots(rows["nc_sigma_sq_poly"])))[::-1]
    _, s, _, _ = isvd(op, 2, philox_omega(1, 0, 2, 2), iterations=2)
    assert np.allclose(s, want, rtol=1e-14, atol=0)


def test_nc_L0_is_X_and_shape():
    """L = 0 gives X; L = 2, d = 3 on 5 nodes has shape (5, 9), F = d + dL."""
    rng = np.random.default_rng(0)
    A = _random_connected(5, 2, rng)
    X = rng.standard_normal((5, 3))
    assert np.array_equal(NCOperator(A, X, 0).dense(), X)
    assert NCOperator(A, X, 2).shape == (5, 9)


def test_nc_complete_graph_closed_form():
    """K_n: A_hat = J/n, so A_hat^j X = 1 mean(X) for every j >= 1."""
    rng = np.random.default_rng(1)
    for n in (4, 7, 10):
        X = rng.standard_normal((n, 3))
        M = NCOperator(_complete(n), X, 3).dense()
        mean = np.tile(X.mean(axis=0), (n, 1))
        assert np.allclose(M[:, :3], X, atol=0)
        for j in (1, 2, 3):
            assert np.allclose(M[:, 3 * j : 3 * j + 3], mean, rtol=0, atol=1e-14)


# ---------------------------------------------- implicit vs explicit, duality


def _explicit_ne(A, w, lam_ones, lam_adj):
    Ad = A.toarray()
    d = Ad.sum(axis=1)
    T = np.divide(Ad, d[:, None], out=np.zeros_like(Ad), where=d[:, None] > 0)
    M = sum(wc * np.linalg.matrix_power(T, c + 1) for c, wc in enumerate(w))
    return M - lam_ones * np.ones_like(Ad) + lam_adj * Ad


def _explicit_nc(A, X, L):
    Ad = A.toarray()
    n = Ad.shape[0]
    s = 1.0 / np.sqrt(Ad.sum(axis=1) + 1.0)
    Ah = s[:, None] * (Ad + np.eye(n)) * s[None, :]
    return np.hstack([np.linalg.matrix_power(Ah, j) @ X for j in range(L + 1)])


def test_implicit_equals_explicit_and_transpose_duality():
    """north_star: implicit M.x equals explicit M.x; duality <H, M G> = <M^T H, G>."""
    rng = np.random.default_rng(42)
    graphs = [_A(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5), (2, 3)])]  # two triangles
    graphs += [_random_connected(int(rng.integers(3, 13)), int(rng.integers(0, 8)), rng) for _ in range(20)]
    for A in graphs:
        n = A.shape[0]
        for C in (1, 3, 5):
            w = rng.random(C)
            lo, la = rng.random(), rng.random() * (C == 3)
            op = NEOperator(A, w, lo, la)
            Me = _explicit_ne(A, w, lo, la)
            G = rng.standard_normal((n, 3))
            H = rng.standard_normal((n, 3))
            assert np.allclose(op.matmul(G), Me @ G, rtol=0, atol=1e-12)
            assert np.allclose(op.matmul_T(H), Me.T @ H, rtol=0, atol=1e-12)
            assert abs(np.sum(H * op.matmul(G)) - np.sum(op.matmul_T(H) * G)) < 1e-12
        X = rng.standard_normal((n, 2))
        for L in (0, 1, 3):
            op = NCOperator(A, X, L)
            Me = _explicit_nc(A, X, L)
            G = rng.standard_normal((2 * (L + 1), 3))
            H = rng.standard_normal((n, 3))
            assert np.allclose(op.matmul(G), Me @ G, rtol=0, atol=1e-12)
            assert np.allclose(op.matmul_T(H), Me.T @ H, rtol=0, atol=1e-12)
            assert abs(np.sum(H * op.matmul(G)) - np.sum(op.matmul_T(H) * G)) < 1e-12


# ------------------------------------------------------ orthonormalisation


def test_orthonorm_qr_matches_cholesky_and_spans():
    """Alg. 2: both routines give Q^T Q = I and span(Q) = span(Y) (footnote P:884); the
    thin QR factor with diag(R) > 0 is unique, so they agree."""
    rng = np.random.default_rng(9)
    for shape in [(200, 12), (50, 50), (1000, 42)]:
        Y = rng.standard_normal(shape) @ np.diag(np.logspace(0, 2, shape[1]))
        Q1 = orthonorm_qr(Y)
        Q2 = orthonorm_cholesky(Y)
        assert np.abs(Q1.T @ Q1 - np.eye(shape[1])).max() < 1e-13
        assert np.abs(Q1 - Q2).max() < 1e-10
        # span: Y = Q R with R upper triangular, positive diagonal
        R = Q1.T @ Y
        assert np.abs(np.tril(R, -1)).max() < 1e-10 * np.abs(R).max()
        assert (np.diag(R) > 0).all()
        assert np.abs(Q1 @ R - Y).max() < 1e-10 * np.abs(Y).max()


def test_cholesky_fails_on_duplicated_column():
    """Q with a duplicated column has a singular Gram: Cholesky breaks down."""
    rng = np.random.default_rng(2)
    Y = rng.standard_normal((20, 4))
    Y[:, 3] = Y[:, 1]
    with pytest.raises(np.linalg.LinAlgError):
        orthonorm_cholesky(Y)


# ------------------------------------------------------------------- Alg. 1


def test_exact_svd_special_matrices():
    """Identity -> s = 1; diag(3,2,1,0) -> (3,2) with basis vectors."""
    _, s, _, _ = exact_svd(np.eye(5), 5)
    assert np.allclose(s, 1.0, atol=1e-15)
    U, s, V, _ = exact_svd(np.diag([3.0, 2.0, 1.0, 0.0]), 2)
    assert np.allclose(s, [3, 2], atol=1e-15)
    assert np.allclose(np.abs(U), np.eye(4)[:, :2]) and np.allclose(np.abs(V), np.eye(4)[:, :2])
    U, s, V, _ = isvd(DenseOperator(np.diag([3.0, 2.0, 1.0, 0.0])), 2, philox_omega(3, 0, 4, 4), iterations=2)
    assert np.allclose(s, [3, 2], atol=1e-14)
    assert np.allclose(np.abs(U), np.eye(4)[:, :2], atol=1e-14)


def test_isvd_exact_when_l_covers_rank():
    """If k >= rank(M) the error is 0; Alg. 1 on an exact rank-20 50 x 40 matrix
    recovers the dense spectrum and reconstructs M."""
    rng = np.random.default_rng(4)
    M = rng.standard_normal((50, 20)) @ rng.standard_normal((20, 40))
    U, s, V, _ = isvd(DenseOperator(M), 20, philox_omega(4, 0, 40, 24), iterations=1)
    _, s_ex, _, _ = exact_svd(M, 20)
    assert np.allclose(s, s_ex, rtol=1e-12)
    assert np.abs(U @ np.diag(s) @ V.T - M).max() < 1e-10 * np.abs(M).max()
    assert np.abs(U.T @ U - np.eye(20)).max() < 1e-12 and np.abs(V.T @ V - np.eye(20)).max() < 1e-12


def test_eckart_young_tail_identity():
    """||M - U_k S_k V_k^T||_F^2 = sum_{j>k} sigma_j^2 for the exact SVD (Eckart-Young);
    Alg. 1's randomized factors can only do worse (>= tail)."""
    rng = np.random.default_rng(5)
    A = _random_connected(40, 60, rng)
    op = NEOperator(A, uniform_weights(5), 1.0 / 40)
    M = op.dense()
    fro2 = np.sum(M * M)
    for k in (1, 5, 10, 20):
        U, s, V, s_all = exact_svd(M, k)
        res = np.sum((M - U @ np.diag(s) @ V.T) ** 2)
        assert abs(res - np.sum(s_all[k:] ** 2)) < 1e-10 * fro2
        Ur, sr, Vr, _ = isvd(op, k, philox_omega(k, 0, 40, k + 2), iterations=1)
        res_r = np.sum((M - Ur @ np.diag(sr) @ Vr.T) ** 2)
        assert res_r >= np.sum(s_all[k:] ** 2) - 1e-12 * fro2


def test_error_decays_with_iterations():
    """Theorem 4: the median residual gap over 10 seeds is non-increasing
    in iterations in {1, 2, 4, 8} on low-rank-plus-noise matrices."""
    rng = np.random.default_rng(6)
    gaps = {q: [] for q in (1, 2, 4, 8)}
    for seed in range(10):
        U0, _ = np.linalg.qr(rng.standard_normal((120, 30)))
        V0, _ = np.linalg.qr(rng.standard_normal((80, 30)))
        M = U0 @ np.diag(np.logspace(0, -1.5, 30)) @ V0.T + 1e-3 * rng.standard_normal((120, 80))
        _, _, _, s_all = exact_svd(M, 10)
        opt = np.sqrt(np.sum(s_all[10:] ** 2))
        for q in gaps:
            U, s, V, _ = isvd(DenseOperator(M), 10, philox_omega(seed, 0, 80, 12), iterations=q)
            gaps[q].append(np.linalg.norm(M - U @ np.diag(s) @ V.T) - opt)
    med = [np.median(gaps[q]) for q in (1, 2, 4, 8)]
    assert all(med[i + 1] <= med[i] + 1e-12 for i in range(3)), med
    assert med[-1] < 0.1 * med[0]


def test_sign_rule():
    """Largest-|.| entry of each U column positive; ties -> lowest index."""
    U = np.array([[0.5, -0.7], [-0.5, 0.7], [0.1, 0.1]])
    V = np.array([[1.0, 1.0], [2.0, 2.0]])
    U2, V2 = sign_fix(U, V)
    assert np.array_equal(U2[:, 0], U[:, 0]) and np.array_equal(V2[:, 0], V[:, 0])
    assert np.array_equal(U2[:, 1], -U[:, 1]) and np.array_equal(V2[:, 1], -V[:, 1])


def test_permutation_invariance_ne_and_nc():
    """Relabelling nodes (A' = P A P^T) leaves the singular values unchanged and permutes
    U (and V for NE); Omega' = P Omega for NE, the same Omega for NC (north_star)."""
    g = powerlaw_graph(600, 1500, 2.5, seed=11)
    perm = np.random.default_rng(12).permutation(g.n)
    gp = g.permuted(perm)
    A, Ap = adjacency(g.n, g.row_ptr, g.col_idx), adjacency(gp.n, gp.row_ptr, gp.col_idx)
    om = philox_omega(3, 0, g.n, 20)
    omp = np.empty_like(om)
    omp[perm] = om
    U, s, V, _ = isvd(NEOperator(A, uniform_weights(5), 1 / g.n), 16, om, iterations=2)
    Up, sp_, Vp, _ = isvd(NEOperator(Ap, uniform_weights(5), 1 / g.n), 16, omp, iterations=2)
    assert np.allclose(s, sp_, rtol=1e-12)
    assert np.allclose(Up[perm], U, atol=1e-9) and np.allclose(Vp[perm], V, atol=1e-9)
    X = np.random.default_rng(13).standard_normal((g.n, 8))
    Xp = np.empty_like(X)
    Xp[perm] = X
    om = philox_omega(4, 0, 32, 16)
    U, s, V, _ = isvd(NCOperator(A, X, 3), 8, om, iterations=2)
    Up, sp_, Vp, _ = isvd(NCOperator(Ap, Xp, 3), 8, om, iterations=2)
    assert np.allclose(s, sp_, rtol=1e-12)
    assert np.allclose(Up[perm], U, atol=1e-9) and np.allclose(Vp, V, atol=1e-9)


def test_isvd_rejects_bad_rank():
    """k > min(r, c) is an error."""
    with pytest.raises(ValueError):
        isvd(DenseOperator(np.eye(3)), 4, philox_omega(0, 0, 3, 4), iterations=1)


def test_exact_svd_tall_matches_lapack_svd():
    """exact_svd_tall (Gram route, used for config 4 where l = c) equals the LAPACK SVD of the
    explicit stacked matrix on an NC design matrix of a random graph."""
    from oracle.isvd_oracle import exact_svd_tall, nc_blocks

    rng = np.random.default_rng(21)
    A = _random_connected(300, 500, rng)
    op = NCOperator(A, rng.standard_normal((300, 5)), 3)
    s, V, s_all, Ufun = exact_svd_tall(nc_blocks(op), 8)
    Ue, se, Ve, se_all = exact_svd(op.dense(), 8)
    assert np.allclose(s_all, se_all, rtol=1e-10)
    assert np.allclose(np.abs(V.T @ Ve), np.eye(8), atol=1e-8)
    rows = np.arange(0, 300, 7)
    Ur = Ufun(rows)
    assert np.allclose(np.abs(np.sum(Ur * Ue[rows], axis=0)) / np.linalg.norm(Ur, axis=0) / np.linalg.norm(Ue[rows], axis=0), 1.0, atol=1e-8)


# ---------------------------------------------------------- Eq. 5 embeddings, Eq. 7 W*


def test_embeddings_inner_products_are_the_low_rank_matrix():
    """<L_i, R_j> = U_i^T S V_j -- checked against the product of the factors."""
    from oracle import embeddings

    rng = np.random.default_rng(11)
    U = rng.standard_normal((9, 3))
    V = rng.standard_normal((7, 3))
    s = np.array([3.0, 2.0, 0.5])
    L, R = embeddings(U, s, V)
    want = np.einsum("ik,k,jk->ij", U, s, V)
    assert np.allclose(L @ R.T, want, rtol=0, atol=1e-13)


def test_least_norm_identity_design_matrix_recovers_labels():
    """M = I, k = n: W* = Y exactly (Theorem 1)."""
    from oracle import exact_svd, least_norm

    n = 6
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((n, 2))
    U, s, V, _ = exact_svd(np.eye(n), n)
    W = least_norm(U, s, V, Y)
    assert np.allclose(W, Y, rtol=0, atol=1e-14)


def test_least_norm_equals_lapack_minimum_norm_least_squares():
    """Rank-deficient 12 x 5 M (rank 3), k = 5 >= rank: V S^+ U^T Y is the minimum-norm least-squares
    solution (Theorem 1) -- the same minimiser LAPACK's gelsd (np.linalg.lstsq) returns by a
    different algorithm; a truncated k = 3 gives it too (the cut S^+ drops the zero singular values)."""
    from oracle import exact_svd, least_norm

    rng = np.random.default_rng(5)
    M = rng.standard_normal((12, 3)) @ rng.standard_normal((3, 5))
    Y = rng.standard_normal((12, 4))
    want = np.linalg.lstsq(M, Y, rcond=None)[0]
    for k in (5, 3):
        U, s, V, _ = exact_svd(M, k)
        W = least_norm(U, s, V, Y, shape=M.shape)
        assert np.allclose(W, want, rtol=0, atol=1e-12), k
    # and the minimum norm: any other least-squares solution (add a null-space vector) is longer
    null = np.linalg.svd(M)[2][-1]
    assert np.linalg.norm(want) < np.linalg.norm(want + np.outer(null, np.ones(4)))


def test_least_norm_row_subset_is_the_labelled_problem():
    """Semi-supervised option (i): rows of U and Y restricted to the labelled set equal
    the formula applied to the gathered rows."""
    from oracle import least_norm

    rng = np.random.default_rng(8)
    U = np.linalg.qr(rng.standard_normal((20, 4)))[0]
    V = np.linalg.qr(rng.standard_normal((6, 4)))[0]
    s = np.array([5.0, 3.0, 2.0, 1.0])
    Y = rng.standard_normal((20, 3))
    rows = np.array([1, 4, 5, 11, 19])
    W = least_norm(U, s, V, Y, rows=rows, shape=(20, 6))
    want = V @ np.diag(1 / s) @ U[rows].T @ Y[rows]
    assert np.allclose(W, want, rtol=0, atol=1e-13)


def test_pinv_diag_cuts_numerical_zeros():
    from oracle import pinv_diag

    s = np.array([2.0, 1.0, 1e-20, 0.0])
    assert np.array_equal(pinv_diag(s, 10, 4), [0.5, 1.0, 0.0, 0.0])


def test_spectral_kernel_closed_forms():
    """Eq. 9 discretised: mu = 1, s -> 0 is the identity (x concentrates at 1, on the
    grid); S = 1 stays 1 for any (mu, s); S = (4, 1), mu = 2, s -> 0 gives (16, 1);
    a flat kernel (s -> inf) is the grid mean of S^x."""
    from oracle import spectral_kernel

    s = np.array([3.0, 1.5, 0.2])
    assert np.allclose(spectral_kernel(s, 1.0, 40.0), s, rtol=1e-12)
    assert np.allclose(spectral_kernel(np.ones(3), 0.7, 1.3), 1.0, rtol=1e-14)
    assert np.allclose(spectral_kernel(np.array([4.0, 1.0]), 2.0, 40.0), [16.0, 1.0], rtol=1e-12)
    x = 0.5 + 0.005 * np.arange(301)
    assert np.isclose(spectral_kernel(np.array([2.0]), 1.0, -60.0)[0], np.mean(2.0 ** x), rtol=1e-12)


# ---------------------------------------------------------- label re-use


def test_label_reuse_edgeless_graph_gives_zero_blocks():
    """No edges: A_hat = (D + I)^-1 = I, so B = A_hat - (D + I)^-1 = 0 and the label blocks vanish
    (S:226)."""
    import scipy.sparse as sps

    from oracle import NCOperator

    n = 5
    A = sps.csr_matrix((n, n))
    rng = np.random.default_rng(1)
    X = rng.standard_normal((n, 2))
    Y = np.eye(n)[:, :3]
    op = NCOperator(A, X, 1, Y_train=Y, P=2)
    M = op.dense()
    assert M.shape == (n, 2 * 2 + 3 * 2)
    assert np.array_equal(M[:, 4:], np.zeros((n, 6)))


def test_label_reuse_has_no_self_leak_and_matches_s_a_s():
    """Row i of B Y does not depend on Y_i: B = S A S with S = (D + I)^-1/2 has a zero
    diagonal -- checked by perturbing one label row, and B against S A S built directly."""
    from oracle import NCOperator, label_reuse_adj

    rng = np.random.default_rng(9)
    A = _random_connected(12, 20, rng)
    d = np.asarray(A.sum(axis=1)).ravel()
    S = np.diag(1.0 / np.sqrt(d + 1.0))
    assert np.allclose(label_reuse_adj(A).toarray(), S @ A.toarray() @ S, rtol=0, atol=1e-15)
    X = rng.standard_normal((12, 3))
    Y = np.zeros((12, 4))
    Y[np.arange(12), rng.integers(0, 4, 12)] = 1.0
    Y2 = Y.copy()
    Y2[5] = [7.0, -3.0, 2.0, 9.0]
    M1 = NCOperator(A, X, 0, Y_train=Y, P=1).dense()
    M2 = NCOperator(A, X, 0, Y_train=Y2, P=1).dense()
    assert np.allclose(M1[5, 3:], M2[5, 3:], rtol=0, atol=1e-15)
    assert not np.allclose(M1[:, 3:], M2[:, 3:])  # but the neighbours of node 5 do see it


def test_label_reuse_implicit_equals_explicit():
    """Implicit products of M_LR equal the explicit matrix's (P:328-337 with Eq. 6)."""
    from oracle import NCOperator

    rng = np.random.default_rng(4)
    A = _random_connected(15, 25, rng)
    X = rng.standard_normal((15, 3))
    Y = rng.standard_normal((15, 2))
    op = NCOperator(A, X, 2, Y_train=Y, P=2)
    M = op.dense()
    G = rng.standard_normal((op.shape[1], 5))
    Q = rng.standard_normal((15, 5))
    assert np.allclose(op.matmul(G), M @ G, rtol=0, atol=1e-12)
    assert np.allclose(op.matmul_T(Q), M.T @ Q, rtol=0, atol=1e-12)


# --------------------------------------------- weighted graphs and the A_hat NE basis


def _Aw(n, wedges):
    """Symmetric weighted A from (i, j, w) triples."""
    import scipy.sparse as sps

    r = [i for i, j, _ in wedges] + [j for i, j, _ in wedges]
    c = [j for i, j, _ in wedges] + [i for i, j, _ in wedges]
    v = [w for _, _, w in wedges] * 2
    A = sps.csr_matrix((v, (r, c)), shape=(n, n))
    A.sort_indices()
    return adjacency(n, A.indptr, A.indices, A.data)


def test_weighted_path_hand_values():
    """Path 0-1-2 with A_01 = 2, A_12 = 1 ("A_ij is set to their edge weight").  By hand:
    d = (2, 3, 1) -> T = D^-1 A = [[0, 1, 0], [2/3, 0, 1/3], [0, 1, 0]];
    s = (d+1)^-1/2 = (1/sqrt3, 1/2, 1/sqrt2) -> A_hat = S (A+I) S has
    A_hat_00 = 1/3, A_hat_01 = 2 (1/sqrt3)(1/2) = 1/sqrt3, A_hat_11 = 1/4, A_hat_12 = 1/(2 sqrt2),
    A_hat_22 = 1/2."""
    A = _Aw(3, [(0, 1, 2.0), (1, 2, 1.0)])
    assert np.allclose(transition(A).toarray(), [[0, 1, 0], [2 / 3, 0, 1 / 3], [0, 1, 0]], rtol=0, atol=1e-15)
    Ah = sym_norm_adj(A).toarray()
    want = np.array([[1 / 3, 1 / np.sqrt(3), 0], [1 / np.sqrt(3), 1 / 4, 1 / (2 * np.sqrt(2))],
                     [0, 1 / (2 * np.sqrt(2)), 1 / 2]])
    assert np.allclose(Ah, want, rtol=0, atol=1e-15)


def test_weighted_ne_null_vector_and_unit_weights():
    """Weighted T is still row-stochastic, so M 1 = 0 for sum w = 1, lambda = 1/n; unit
    weights reproduce the unweighted operator exactly."""
    rng = np.random.default_rng(8)
    n = 40
    A0 = _random_connected(n, 30, rng)
    Aw = adjacency(n, A0.indptr, A0.indices, 0.5 + rng.random(A0.nnz))
    Aw = sp_sym(Aw)
    op = NEOperator(Aw, uniform_weights(5), 1.0 / n)
    assert np.abs(op.matmul(np.ones((n, 1)))).max() < 1e-14
    A1 = adjacency(n, A0.indptr, A0.indices, np.ones(A0.nnz))
    G = rng.standard_normal((n, 3))
    assert np.array_equal(NEOperator(A1, uniform_weights(3), 1 / n).matmul(G),
                          NEOperator(A0, uniform_weights(3), 1 / n).matmul(G))


def sp_sym(A):
    """(A + A^T) / 2 as a CSR adjacency with sorted indices (symmetric weights)."""
    import scipy.sparse as sps

    S = sps.csr_matrix((A + A.T) / 2.0)
    S.sort_indices()
    return adjacency(S.shape[0], S.indptr, S.indices, S.data)


@pytest.mark.parametrize("C", [1, 3, 5])
def test_ne_ahat_basis_cycle_spectrum(C):
    """NE over A_hat on the cycle C_n: d = 2, A_hat = (A + I)/3 with eigenvalues
    (1 + 2 cos(2 pi j/n))/3; the j = 0 direction (eigenvalue 1, vector 1) is cancelled by the
    rank-1 term when sum w = 1, lambda = 1/n.  So sigma(M) = {|sum_c w_c ((1 + 2 cos(2 pi j / n))/3)^c|:
    j = 1..n-1} plus 0, and M = M^T."""
    w = uniform_weights(C)
    for n in range(6, 15):
        op = NEOperator(_cycle(n), w, 1.0 / n, basis="Ahat")
        Md = op.dense()
        assert np.allclose(Md, Md.T, rtol=0, atol=1e-15)
        lam = (1 + 2 * np.cos(2 * np.pi * np.arange(1, n) / n)) / 3
        want = np.sort(np.abs([sum(w[c - 1] * x ** c for c in range(1, C + 1)) for x in lam]))[::-1]
        _, _, _, s_all = isvd(op, n - 1, philox_omega(300 + n, 0, n, n), iterations=2)
        assert np.allclose(s_all[: n - 1], want, rtol=0, atol=1e-13)


def test_ne_ahat_basis_complete_graph_is_zero():
    """K_n: A_hat = (J - I + I)/n = J/n, so every power is J/n and sum_c w_c J/n - (1/n) J = 0 when
    sum w = 1 (P:158 with the configs' lambda = 1/n)."""
    for n in range(4, 10):
        op = NEOperator(_complete(n), context_weights(4), 1.0 / n, basis="Ahat")
        assert np.abs(op.dense()).max() < 1e-15


# --------------------------------------------- implicit row gather (option (ii))


def test_row_subset_operator_is_the_submatrix_and_its_svd():
    """M_S = M[S, :] by definition: implicit products equal the explicit rows of dense(M) (both
    families, both directions), and Alg. 1 with l >= rank(M_S) returns the exact SVD of M[S]
     -- checked against LAPACK on the explicit submatrix."""
    from oracle import RowSubsetOperator

    rng = np.random.default_rng(17)
    A = _random_connected(30, 25, rng)
    X = rng.standard_normal((30, 3))
    S = np.sort(rng.choice(30, 11, replace=False))
    for op in (NEOperator(A, uniform_weights(4), 1 / 30), NCOperator(A, X, 2)):
        sub = RowSubsetOperator(op, S)
        Md = op.dense()[S]
        G = rng.standard_normal((op.shape[1], 5))
        H = rng.standard_normal((S.size, 5))
        assert sub.shape == Md.shape
        assert np.allclose(sub.matmul(G), Md @ G, rtol=0, atol=1e-13)
        assert np.allclose(sub.matmul_T(H), Md.T @ H, rtol=0, atol=1e-13)
        r = min(Md.shape)
        _, s, _, _ = isvd(sub, min(5, r), philox_omega(9, 0, Md.shape[1], r), iterations=1)
        assert np.allclose(s, np.linalg.svd(Md, compute_uv=False)[: min(5, r)], rtol=1e-10, atol=1e-13)
