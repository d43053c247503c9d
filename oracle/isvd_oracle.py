"""Plain fp64 oracle: operators of Eq. 3 / Eq. 6 and Alg. 1 + Alg. 2 (left).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Slow and literal on
purpose: products are evaluated at definition level (repeated multiplication,
right to left as the paper's DAG does), never with the Horner
recurrence or any fusion the CUDA path uses.  Library primitives used as single
steps: scipy CSR x dense products, numpy matmul, LAPACK Householder QR
(np.linalg.qr) and LAPACK SVD (np.linalg.svd).

Citations: P:n = /root/reference/PAPER.md line n.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# ---------------------------------------------------------------------------
# Graph matrices (Section 2)
# ---------------------------------------------------------------------------


def adjacency(n: int, row_ptr, col_idx, values=None) -> sp.csr_matrix:
    """A in R^{n x n}: A_ij = edge weight ("A_ij is set to their edge weight"); every
    stored A_ij = 1 when `values` is None (the unweighted configs, reading O12)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    if values is None:
        vals = np.ones(col_idx.size, dtype=np.float64)
    else:
        vals = np.asarray(values, dtype=np.float64)
    return sp.csr_matrix((vals, col_idx, row_ptr), shape=(n, n))


def degrees(A: sp.csr_matrix) -> np.ndarray:
    """D = diag(row sums of A)."""
    return np.asarray(A.sum(axis=1)).ravel()


def transition(A: sp.csr_matrix) -> sp.csr_matrix:
    """T = D^-1 A.  A row with d_i = 0 is left zero (0^-1 := 0)."""
    d = degrees(A)
    inv = np.zeros_like(d)
    nz = d > 0
    inv[nz] = 1.0 / d[nz]
    return sp.csr_matrix(sp.diags(inv) @ A)


def sym_norm_adj(A: sp.csr_matrix) -> sp.csr_matrix:
    """A_hat = (D+I)^-1/2 (A+I) (D+I)^-1/2."""
    n = A.shape[0]
    d = degrees(A)
    s = 1.0 / np.sqrt(d + 1.0)
    S = sp.diags(s)
    return sp.csr_matrix(S @ (A + sp.identity(n, format="csr")) @ S)


# ---------------------------------------------------------------------------
# Context weights (Section 2.1, Fig. 1 code P:252)
# ---------------------------------------------------------------------------


def context_weights(C: int) -> np.ndarray:
    """Normalised triangular weights w_q = (C - q + 1) / (C(C+1)/2), q = 1..C.

    P:91 states P_Q(q|C) prop. to (C-q+1)/C; its closed form does not sum to 1
    for C > 1 (reading O1), so the normalisation of Fig. 1's code
    (``np.array([3, 2, 1]) / 6.0``) is used."""
    if C < 1:
        raise ValueError("C must be >= 1")
    q = np.arange(1, C + 1, dtype=np.float64)
    return (C - q + 1.0) / (C * (C + 1) / 2.0)


def uniform_weights(C: int) -> np.ndarray:
    """w_c = 1/C: walk length ~ U[C] (footnote P:137); the configs' weights."""
    if C < 1:
        raise ValueError("C must be >= 1")
    return np.full(C, 1.0 / C)


# ---------------------------------------------------------------------------
# Implicit design matrices
# ---------------------------------------------------------------------------


class NEOperator:
    """M = sum_c w_c B^c - lambda_ones * 1 1^T + lambda_adj * A   (Eq. 3).

    B = T (row-normalised transition, default) or A_hat (symmetric variant).
    Eq. 3's negative term is -lambda (1 - A) = -lambda 1 1^T + lambda A (reading O2);
    the configs use lambda_ones = 1/n, lambda_adj = 0.
    """

    def __init__(self, A: sp.csr_matrix, weights, lambda_ones: float, lambda_adj: float = 0.0, basis: str = "T"):
        self.A = sp.csr_matrix(A, dtype=np.float64)
        self.n = self.A.shape[0]
        self.w = np.asarray(weights, dtype=np.float64)
        self.lambda_ones = float(lambda_ones)
        self.lambda_adj = float(lambda_adj)
        self.B = transition(self.A) if basis == "T" else sym_norm_adj(self.A)
        self.BT = sp.csr_matrix(self.B.T)  # explicit transpose: no reliance on symmetry
        self.AT = sp.csr_matrix(self.A.T)

    @property
    def shape(self):
        return (self.n, self.n)

    def _apply(self, B, A, G):
        G = np.asarray(G, dtype=np.float64)
        P = G
        acc = np.zeros_like(G)
        for w in self.w:  # B^c G by repeated multiplication (ProductPF P:1001-1005)
            P = B @ P
            acc += w * P
        # rank-1 term through two O(n) products <M2, <M1, G>> (Fig. 1 row1.T @ row1)
        ones = np.ones((self.n, 1))
        acc -= self.lambda_ones * (ones @ (ones.T @ G))
        if self.lambda_adj != 0.0:
            acc += self.lambda_adj * (A @ G)
        return acc

    def matmul(self, G):
        """M . G (the product function u_M; SymbolicPF.dot P:903)."""
        return self._apply(self.B, self.A, G)

    def matmul_T(self, H):
        """M^T . H (SymbolicPF.T().dot)."""
        return self._apply(self.BT, self.AT, H)

    def dense(self) -> np.ndarray:
        """Explicit n x n M (tiny graphs only)."""
        return self.matmul(np.eye(self.n))


def label_reuse_adj(A: sp.csr_matrix) -> sp.csr_matrix:
    """A_hat - (D + I)^-1: the propagation of the label re-use blocks, i.e. A_hat with
    its diagonal zeroed (no label leaks from row i to row i), built as written."""
    d = degrees(A)
    return sp.csr_matrix(sym_norm_adj(A) - sp.diags(1.0 / (d + 1.0)))


class NCOperator:
    """M = [X | A_hat X | A_hat^2 X | ... | A_hat^L X]  in R^{n x d(L+1)}  (Eq. 6),
    optionally with the label re-use blocks:
    M_LR = [M | B Y_train | B^2 Y_train | ... | B^P Y_train],  B = A_hat - (D + I)^-1."""

    def __init__(self, A: sp.csr_matrix, X, L: int, Y_train=None, P: int = 0):
        self.A = sp.csr_matrix(A, dtype=np.float64)
        self.n = self.A.shape[0]
        self.X = np.asarray(X, dtype=np.float64)
        if self.X.shape[0] != self.n:
            raise ValueError("X must have n rows")
        self.d = self.X.shape[1]
        self.L = int(L)
        self.Ahat = sym_norm_adj(self.A)
        self.AhatT = sp.csr_matrix(self.Ahat.T)
        self.P = int(P) if Y_train is not None else 0
        self.Y = None if Y_train is None else np.asarray(Y_train, dtype=np.float64)
        self.y = 0 if self.Y is None else self.Y.shape[1]
        if self.P:
            self.B = label_reuse_adj(self.A)
            self.BT = sp.csr_matrix(self.B.T)

    @property
    def shape(self):
        return (self.n, self.d * (self.L + 1) + self.y * self.P)

    def matmul(self, G):
        """M G = sum_j A_hat^j (X G_j) + sum_p B^p (Y G'_p), G_j = rows [jd, (j+1)d) of G and G'_p
        the following y-row blocks (column concat)."""
        G = np.asarray(G, dtype=np.float64)
        out = np.zeros((self.n, G.shape[1]))
        for j in range(self.L + 1):
            P = self.X @ G[j * self.d : (j + 1) * self.d]
            for _ in range(j):  # A_hat^j applied by j repeated products
                P = self.Ahat @ P
            out += P
        off = self.d * (self.L + 1)
        for p in range(1, self.P + 1):
            P = self.Y @ G[off + (p - 1) * self.y : off + p * self.y]
            for _ in range(p):
                P = self.B @ P
            out += P
        return out

    def matmul_T(self, Q):
        """M^T Q: block j = X^T (A_hat^T)^j Q, then Y^T (B^T)^p Q."""
        Q = np.asarray(Q, dtype=np.float64)
        blocks = []
        for j in range(self.L + 1):
            P = Q
            for _ in range(j):
                P = self.AhatT @ P
            blocks.append(self.X.T @ P)
        for p in range(1, self.P + 1):
            P = Q
            for _ in range(p):
                P = self.BT @ P
            blocks.append(self.Y.T @ P)
        return np.vstack(blocks)

    def dense(self) -> np.ndarray:
        """Explicit M: the blocks A_hat^j X (and B^p Y) stacked side by side."""
        blocks = [self.X]
        P = self.X
        for _ in range(self.L):
            P = self.Ahat @ P
            blocks.append(P)
        P = self.Y
        for _ in range(self.P):
            P = self.B @ P
            blocks.append(P)
        return np.hstack(blocks)


class RowSubsetOperator:
    """M_S = M[S, :] for sorted row ids S (semi-supervised option (ii): "SVD of submatrix
    of M without explicitly computing M nor the submatrix"), by definition of the submatrix:
    M_S G = (M G)[S] and M_S^T H = M^T H_full, H_full = H on the rows S and zero elsewhere."""

    def __init__(self, op, rows):
        self.op = op
        self.rows = np.asarray(rows, dtype=np.int64)

    @property
    def shape(self):
        return (self.rows.size, self.op.shape[1])

    def matmul(self, G):
        return self.op.matmul(G)[self.rows]

    def matmul_T(self, H):
        H = np.asarray(H, dtype=np.float64)
        full = np.zeros((self.op.shape[0], H.shape[1]))
        full[self.rows] = H
        return self.op.matmul_T(full)

    def dense(self):
        return self.op.dense()[self.rows]


class DenseOperator:
    """An explicit matrix behind the same product contract (leaf node)."""

    def __init__(self, M):
        self.M = np.asarray(M, dtype=np.float64)

    @property
    def shape(self):
        return self.M.shape

    def matmul(self, G):
        return self.M @ np.asarray(G, dtype=np.float64)

    def matmul_T(self, H):
        return self.M.T @ np.asarray(H, dtype=np.float64)

    def dense(self):
        return self.M


# ---------------------------------------------------------------------------
# Orthonormalisation (Alg. 2)
# ---------------------------------------------------------------------------


def orthonorm_qr(Y) -> np.ndarray:
    """orthonormHalko (Alg. 2 left): thin Householder QR (LAPACK geqrf),
    returning the unique Q whose R has a positive diagonal."""
    Q, R = np.linalg.qr(np.asarray(Y, dtype=np.float64), mode="reduced")
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return Q * s


def orthonorm_cholesky(Y) -> np.ndarray:
    """orthonormOurs (Alg. 2 right): L = chol(Y^T Y); return Y (L^-1)^T.
    Used only to cross-check orthonorm_qr (same Q in exact arithmetic)."""
    Y = np.asarray(Y, dtype=np.float64)
    Lc = np.linalg.cholesky(Y.T @ Y)
    return np.linalg.solve(Lc, Y.T).T


# ---------------------------------------------------------------------------
# Alg. 1
# ---------------------------------------------------------------------------


def sign_fix(U, V):
    """Sign rule (paper silent): flip each (U_j, V_j) so the largest-|.|
    entry of U_j is positive, ties to the lowest row index."""
    U = np.array(U, dtype=np.float64, copy=True)
    V = np.array(V, dtype=np.float64, copy=True)
    for j in range(U.shape[1]):
        i = int(np.argmax(np.abs(U[:, j])))  # first maximum = lowest index
        if U[i, j] < 0:
            U[:, j] *= -1.0
            V[:, j] *= -1.0
    return U, V


def isvd(op, k: int, omega, iterations: int, orthonorm=orthonorm_qr):
    """iSVD(M, k) of Alg. 1, step by step, in fp64.

    ``omega`` is the c x l starting matrix Q ~ N(0,1)^{c x l} (l = 2k in
    the paper, l = k + p with oversampling p in the configs, reading O6).
    Returns (U[:, :k], s[:k], V[:, :k], s_all) with the sign rule applied."""
    Q = np.asarray(omega, dtype=np.float64)
    r, c = op.shape
    if Q.shape[0] != c:
        raise ValueError("omega must have c rows")
    if not (1 <= k <= min(r, c)) or Q.shape[1] < k:
        raise ValueError("need 1 <= k <= min(r, c) and l >= k")
    for _ in range(iterations):
        Q = orthonorm(op.matmul(Q))  # P:847, (r x l)
        Q = orthonorm(op.matmul_T(Q))  # P:848, (c x l)
    Q = orthonorm(op.matmul(Q))  # P:852, (r x l)
    B = op.matmul_T(Q).T  # P:855, (l x c)
    UB, s, Vt = np.linalg.svd(B, full_matrices=False)
    U = Q @ UB
    Uk, Vk = sign_fix(U[:, :k], Vt[:k].T)
    return Uk, s[:k].copy(), Vk, s.copy()


def exact_svd(M, k: int):
    """SVD_k(M) by definition: LAPACK SVD of the explicit matrix."""
    U, s, Vt = np.linalg.svd(np.asarray(M, dtype=np.float64), full_matrices=False)
    Uk, Vk = sign_fix(U[:, :k], Vt[:k].T)
    return Uk, s[:k].copy(), Vk, s.copy()


def nc_blocks(op: "NCOperator"):
    """The column blocks [X, A_hat X, ..., A_hat^L X] of Eq. 6, each by j repeated
    sparse products, as a list (never concatenated: config 4 is 2.45M x 400)."""
    blocks = [op.X]
    P = op.X
    for _ in range(op.L):
        P = op.Ahat @ P
        blocks.append(P)
    return blocks


def exact_svd_tall(blocks, k: int):
    """Exact SVD_k of a tall M = [B_0 | B_1 | ...] through its c x c Gram:
    M^T M = V S^2 V^T (LAPACK symmetric eigensolver), U = M V S^-1.  Used where M has far more
    rows than columns and l = c makes Alg. 1 exact (config 4, reading O6).  Returns
    (s[:k], V[:, :k], s_all, Ufun) with Ufun(rows) -> U[rows, :k] (sign rule of S:141 is not
    applied: callers compare subspaces)."""
    c = sum(b.shape[1] for b in blocks)
    G = np.empty((c, c))
    offs = np.cumsum([0] + [b.shape[1] for b in blocks])
    for i, bi in enumerate(blocks):
        for j in range(i, len(blocks)):
            gij = bi.T @ blocks[j]
            G[offs[i] : offs[i + 1], offs[j] : offs[j + 1]] = gij
            G[offs[j] : offs[j + 1], offs[i] : offs[i + 1]] = gij.T
    lam, V = np.linalg.eigh(G)
    order = np.argsort(lam)[::-1]
    lam, V = lam[order], V[:, order]
    s_all = np.sqrt(np.maximum(lam, 0.0))

    def Ufun(rows):
        Mr = np.hstack([b[rows] for b in blocks])
        return Mr @ V[:, :k] / s_all[:k]

    return s_all[:k].copy(), V[:, :k].copy(), s_all, Ufun


# ---------------------------------------------------------------------------
# After the SVD: embeddings (Eq. 5) and the least-norm parameters (Eq. 7)
# ---------------------------------------------------------------------------


def embeddings(U, s, V):
    """L = U S^1/2, R = V S^1/2 (Eq. 5): <L_i, R_j> = (U S V^T)_ij."""
    r = np.sqrt(np.asarray(s, dtype=np.float64))
    return np.asarray(U, dtype=np.float64) * r, np.asarray(V, dtype=np.float64) * r


def pinv_diag(s, n_rows: int, n_cols: int):
    """S^+ of Eq. 7: reciprocates the non-zero entries of diag(S).  "Non-zero" is read
    numerically (reading O24): s_i > max(n_rows, n_cols) * eps_fp64 * max(s), LAPACK/numpy's
    default cut for a pseudoinverse."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        return s.copy()
    tol = max(n_rows, n_cols) * np.finfo(np.float64).eps * s.max()
    out = np.zeros_like(s)
    nz = s > tol
    out[nz] = 1.0 / s[nz]
    return out


def least_norm(U, s, V, Y, rows=None, shape=None):
    """W* = M^+ Y ~ V S^+ U^T Y (Eq. 7), multiplied right to left:
    T = U^T Y (k x y), then S^+ T, then V (S^+ T).  ``rows`` (semi-supervised option (i),
    P:209-210) keeps only the labelled rows of U and Y.  ``shape`` = (r, c) of M for the
    numerical-zero cut of S^+ (default: the shapes of U and V)."""
    U = np.asarray(U, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    if rows is not None:
        U = U[rows]
        Y = Y[rows]
    r, c = shape if shape is not None else (U.shape[0], V.shape[0])
    T = U.T @ Y
    T = pinv_diag(s, r, c)[:, None] * T
    return V @ T


def spectral_kernel(s, mu: float, s_bar: float):
    """Gaussian spectral reweighting of Eq. 9 by the discretisation of P:1057-1065:
    E_x[S^x] ~ sum_{x in Omega} S^x softmax_x(-(x - mu)^2 exp(s_bar)), Omega = {0.5, 0.505, ..., 2.0}
    (301 points), s_bar = log(1 / (2 s^2)).  Returns the reweighted diagonal (k-vector)."""
    s = np.asarray(s, dtype=np.float64)
    x = 0.5 + 0.005 * np.arange(301)
    logits = -((x - mu) ** 2) * np.exp(s_bar)
    w = np.exp(logits - logits.max())
    w /= w.sum()
    return np.array([np.sum(si ** x * w) for si in s])
