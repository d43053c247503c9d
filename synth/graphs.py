"""Seeded synthetic graphs standing in for the paper's datasets.

PAPER.md Table 1 (lines 418-439) lists the datasets whose node/edge counts the
configs copy; none of their edges is used or reproduced here.  The recipes are
SURVEY.md section 8(d2); the readings (O5, O12, O16, O17, O19) are listed in
DESIGN.md section "Readings".

All graphs are undirected, unweighted, without self-loops or duplicate edges
(ledger O12/O16), and are returned as a symmetric CSR with sorted rows:
``row_ptr`` int64[n+1], ``col_idx`` int32[2m].
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import streams


@dataclass
class Graph:
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col_idx: np.ndarray  # int32[nnz], nnz = 2m
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def m(self) -> int:
        return self.nnz // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def row_slice(self, r0: int, r1: int) -> "tuple[np.ndarray, np.ndarray]":
        """CSR of rows [r0, r1) with GLOBAL column ids (row partition)."""
        rp = self.row_ptr[r0 : r1 + 1] - self.row_ptr[r0]
        ci = self.col_idx[self.row_ptr[r0] : self.row_ptr[r1]]
        return rp.astype(np.int64), ci

    def permuted(self, perm: np.ndarray) -> "Graph":
        """Relabel node v -> perm[v] (used by permutation-invariance tests)."""
        perm = np.asarray(perm, dtype=np.int64)
        rows = np.repeat(np.arange(self.n, dtype=np.int64), self.degrees())
        return _csr_from_directed(perm[rows], perm[self.col_idx.astype(np.int64)], self.n, self.name + "/perm")


def edge_keys_to_csr(keys: np.ndarray, n: int, name: str = "") -> Graph:
    """Undirected edge keys (u*n + v, u < v) -> symmetric sorted CSR."""
    keys = np.asarray(keys, dtype=np.int64)
    u = keys // n
    v = keys - u * n
    return _csr_from_directed(np.concatenate([u, v]), np.concatenate([v, u]), n, name)


def _csr_from_directed(rows: np.ndarray, cols: np.ndarray, n: int, name: str) -> Graph:
    k = rows.astype(np.int64) * n + cols.astype(np.int64)
    k.sort()
    r = k // n
    c = (k - r * n).astype(np.int32)
    counts = np.bincount(r, minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return Graph(n=n, row_ptr=row_ptr, col_idx=c, name=name)


def edges_to_graph(n: int, edges, name: str = "") -> Graph:
    """Small helper: list of (u, v) undirected pairs -> Graph (dedup, no self loops)."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
    if e.size and (e[:, 0] == e[:, 1]).any():
        raise ValueError("self-loops are not part of the input model (ledger O16)")
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    keys = np.unique(lo * n + hi)
    return edge_keys_to_csr(keys, n, name)


def _sorted_unique(x: np.ndarray) -> np.ndarray:
    """Sorted distinct values (sort + adjacent compare; avoids np.unique's slow paths)."""
    s = np.sort(np.asarray(x, dtype=np.int64))
    if s.size == 0:
        return s
    keep = np.empty(s.size, dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def _in_sorted(sorted_arr: np.ndarray, x: np.ndarray) -> np.ndarray:
    if sorted_arr.size == 0:
        return np.zeros(x.shape, dtype=bool)
    i = np.searchsorted(sorted_arr, x)
    i = np.minimum(i, sorted_arr.size - 1)
    return sorted_arr[i] == x


def _collect_distinct(initial: np.ndarray, draw, need: int, seed: int, label: str) -> np.ndarray:
    """Return `need` distinct candidate keys that are not in `initial`.

    `draw(offset, count)` returns `count` candidate keys of a stream starting at
    draw index `offset`; negative keys are rejections.  Batches are drawn until
    enough distinct new keys exist; when a batch overshoots, the kept subset is
    the `need` keys with the smallest seeded hash (a uniform, deterministic
    choice among the distinct drawn pairs)."""
    acc = _sorted_unique(initial)
    got = []
    offset = 0
    salt = streams.stream_state(seed, label + "/keep")
    while need > 0:
        b = int(need * 1.25) + 4096
        cand = draw(offset, b)
        offset += b
        cand = _sorted_unique(cand[cand >= 0])
        cand = cand[~_in_sorted(acc, cand)]
        if cand.size > need:
            h = streams.mix64(cand.astype(np.uint64) ^ salt)
            sel = np.argpartition(h, need - 1)[:need]
            cand = np.sort(cand[sel])
        got.append(cand)
        need -= cand.size
        if need > 0:
            acc = _sorted_unique(np.concatenate([acc, cand]))
    return np.concatenate(got) if got else np.zeros(0, dtype=np.int64)


class AliasSampler:
    """Walker alias table: draws index i with probability w_i / sum(w) in O(1)."""

    def __init__(self, w: np.ndarray):
        n = w.size
        p = w.astype(np.float64) * (n / w.sum())
        prob = np.ones(n, dtype=np.float64)
        alias = np.arange(n, dtype=np.int64)
        small = [int(i) for i in np.nonzero(p < 1.0)[0]]
        large = [int(i) for i in np.nonzero(p >= 1.0)[0]]
        p = p.tolist()
        while small and large:
            s = small.pop()
            g = large[-1]
            prob[s] = p[s]
            alias[s] = g
            p[g] = (p[g] + p[s]) - 1.0
            if p[g] < 1.0:
                large.pop()
                small.append(g)
        self.prob, self.alias, self.n = prob, alias, n

    def sample(self, raw: np.ndarray) -> np.ndarray:
        """Map raw uint64 draws to indices: high 32 bits pick the column, low 32 bits the coin."""
        hi = (raw >> np.uint64(32)).astype(np.uint64)
        col = ((hi * np.uint64(self.n)) >> np.uint64(32)).astype(np.int64)
        coin = (raw & np.uint64(0xFFFFFFFF)).astype(np.float64) * (2.0 ** -32)
        return np.where(coin < self.prob[col], col, self.alias[col])


def _powerlaw_weights(n: int, m: int, gamma: float) -> "tuple[np.ndarray, float]":
    """Static-model weights w_i = (i + i0)^-alpha, alpha = 1/(gamma-1), with i0
    chosen by bisection so the expected top degree 2m w_0 / sum(w) equals the
    natural cutoff n^alpha."""
    alpha = 1.0 / (gamma - 1.0)
    target = float(n) ** alpha
    idx = np.arange(n, dtype=np.float64)

    def top(i0):
        w = (idx + i0) ** (-alpha)
        return 2.0 * m * w[0] / w.sum()

    lo, hi = 1e-6, float(n)
    for _ in range(64):
        mid = 0.5 * (lo + hi)
        if top(mid) > target:
            lo = mid
        else:
            hi = mid
    i0 = 0.5 * (lo + hi)
    return (idx + i0) ** (-alpha), i0


def powerlaw_graph(n: int, m: int, gamma: float, seed: int, name: str = "powerlaw") -> Graph:
    """Connected power-law graph with exactly m undirected edges."""
    if m < n - 1:
        raise ValueError("need m >= n-1 for a connected graph")
    w, _ = _powerlaw_weights(n, m, gamma)
    alias = AliasSampler(w)
    # step 2: random spanning tree, node pi_t attaches to an earlier node drawn prop. to w
    pi = streams.permutation(seed, "tree-order", n)
    cum_pi = np.cumsum(w[pi])
    t = np.arange(1, n, dtype=np.int64)
    r = streams.uniform(seed, "tree-parent", 0, n - 1) * cum_pi[t - 1]
    pos = np.minimum(np.searchsorted(cum_pi, r, side="right"), t - 1)
    a, b = pi[t], pi[pos]
    tree = np.minimum(a, b) * n + np.maximum(a, b)

    # step 3: fill with i.i.d. endpoint pairs drawn prop. to w (alias table), distinct, not in the tree
    def draw(off, cnt):
        ix = alias.sample(streams.u64(seed, "fill", 2 * off, 2 * cnt))
        u, v = ix[0::2], ix[1::2]
        key = np.minimum(u, v) * n + np.maximum(u, v)
        key[u == v] = -1
        return key

    fill = _collect_distinct(tree, draw, m - (n - 1), seed, "fill")
    keys = np.concatenate([tree, fill])
    # step 4: relabel by a seeded uniform permutation (ids uncorrelated with degree)
    perm = streams.permutation(seed, "relabel", n)
    u = perm[keys // n]
    v = perm[keys % n]
    keys = np.minimum(u, v) * n + np.maximum(u, v)
    return edge_keys_to_csr(keys, n, name)


def sbm_graph(n: int, m: int, blocks: int, ratio: float, seed: int, name: str = "sbm") -> Graph:
    """Stochastic block model with p_in/p_out = ratio and exactly m edges."""
    sizes = np.full(blocks, n // blocks, dtype=np.int64)
    sizes[: n % blocks] += 1
    perm = streams.permutation(seed, "blocks", n)  # block b holds perm[starts[b]:starts[b]+sizes[b]]
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    block_of = np.empty(n, dtype=np.int64)
    for bi in range(blocks):
        block_of[perm[starts[bi] : starts[bi] + sizes[bi]]] = bi
    pairs_in = sizes * (sizes - 1) // 2
    n_in = int(pairs_in.sum())
    n_out = n * (n - 1) // 2 - n_in
    p_intra = ratio * n_in / (ratio * n_in + n_out)
    cum_in = np.cumsum(pairs_in).astype(np.float64)

    def draw(off, cnt):
        u4 = streams.uniform(seed, "sbm", 4 * off, 4 * cnt).reshape(cnt, 4)
        intra = u4[:, 0] < p_intra
        # intra: block prop. to its pair count, then a uniform pair inside it
        bsel = np.minimum(np.searchsorted(cum_in, u4[:, 1] * cum_in[-1], side="right"), blocks - 1)
        sz = sizes[bsel]
        iu = np.minimum((u4[:, 2] * sz).astype(np.int64), sz - 1)
        iv = np.minimum((u4[:, 3] * sz).astype(np.int64), sz - 1)
        ui = perm[starts[bsel] + iu]
        vi = perm[starts[bsel] + iv]
        # inter: uniform node pair, rejected unless in different blocks
        uo = np.minimum((u4[:, 2] * n).astype(np.int64), n - 1)
        vo = np.minimum((u4[:, 3] * n).astype(np.int64), n - 1)
        u = np.where(intra, ui, uo)
        v = np.where(intra, vi, vo)
        key = np.minimum(u, v) * n + np.maximum(u, v)
        bad = (u == v) | (~intra & (block_of[uo] == block_of[vo]))
        key[bad] = -1
        return key

    keys = _collect_distinct(np.zeros(0, dtype=np.int64), draw, m, seed, "sbm")
    return edge_keys_to_csr(keys, n, name)


def uniform_graph(n: int, m: int, seed: int, name: str = "uniform") -> Graph:
    """Uniform G(n, m): m distinct pairs drawn uniformly."""

    def draw(off, cnt):
        uv = streams.uniform(seed, "gnm", 2 * off, 2 * cnt)
        ix = np.minimum((uv * n).astype(np.int64), n - 1)
        u, v = ix[0::2], ix[1::2]
        key = np.minimum(u, v) * n + np.maximum(u, v)
        key[u == v] = -1
        return key

    keys = _collect_distinct(np.zeros(0, dtype=np.int64), draw, m, seed, "gnm")
    return edge_keys_to_csr(keys, n, name)


def make_graph(cfg: dict) -> Graph:
    kind = cfg["graph"]
    if kind == "powerlaw":
        return powerlaw_graph(cfg["n"], cfg["m"], cfg["gamma"], cfg["seed"], cfg["name"])
    if kind == "sbm":
        return sbm_graph(cfg["n"], cfg["m"], cfg["blocks"], cfg["ratio"], cfg["seed"], cfg["name"])
    if kind == "uniform":
        return uniform_graph(cfg["n"], cfg["m"], cfg["seed"], cfg["name"])
    raise ValueError(kind)


def make_features(n: int, d: int, seed: int) -> np.ndarray:
    """X ~ N(0,1) fp32, row-major n x d (config 2 text; ledger O18 for config 4)."""
    return streams.normal_f32(seed, "X", n * d).reshape(n, d)


def connected_components(g: Graph) -> int:
    """Number of connected components (label propagation by min over neighbours)."""
    n = g.n
    lab = np.arange(n, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), g.degrees())
    cols = g.col_idx.astype(np.int64)
    while True:
        nl = lab.copy()
        np.minimum.at(nl, rows, lab[cols])
        nl = nl[nl]  # pointer jumping
        if np.array_equal(nl, lab):
            break
        lab = nl
    return int(np.unique(lab).size)
