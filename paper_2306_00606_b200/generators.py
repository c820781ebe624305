"""Synthetic graph recipes for the BASELINE configs (host side, not timed).

Each recipe returns raw ``(k, 2)`` int64 edge pairs that are then cleaned by
:func:`paper_2306_00606_b200.graph.build_graph` (the device CSR builder), so a
graph is a pure function of its recipe parameters.

* ``rmat_codes`` reproduces the reference R-MAT sampler
  (``efgraph/graph.py:204-246``) bit for bit, vectorised: the reference draws
  ``rng.random((batch, scale))`` in batches and inserts canonical codes into a
  Python ``set`` until ``target`` distinct codes exist (:234-237).  Because
  numpy's PCG64 double stream does not depend on how it is chunked, the
  resulting set is exactly "the first ``target`` distinct non-loop codes of the
  pair stream" (or every distinct code among the first ``cap`` pairs when the
  attempt cap truncates).  We compute that set with numpy instead of a Python
  loop (265 s -> a few seconds at scale 22).
* The other recipes follow SURVEY.md §8(d) (BA, ER G(n,m), Chung-Lu, WS).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "rmat_codes",
    "rmat_edges",
    "er_edges_gnm",
    "ba_edges",
    "chung_lu_edges",
    "ws_edges",
]

_CHUNK_PAIRS = 1 << 19


def _pack_bits(bits: np.ndarray, scale: int) -> np.ndarray:
    """Row bit-matrix (column 0 = most significant) -> int64, i.e. ``bits @ weights``."""
    packed = np.packbits(bits, axis=1, bitorder="big").astype(np.int64)
    out = np.zeros(bits.shape[0], dtype=np.int64)
    for j in range(packed.shape[1]):
        out = (out << 8) | packed[:, j]
    return out >> (8 * packed.shape[1] - scale)


def _pair_codes(r: np.ndarray, a: float, b: float, c: float, scale: int):
    """Canonical codes lo*side+hi for one block of draws (``graph.py:644-651``)."""
    ab = a + b
    u = _pack_bits(r >= ab, scale)
    v = _pack_bits(((r >= a) & (r < ab)) | (r >= ab + c), scale)
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    return lo * np.int64(1 << scale) + hi


def _sorted_unique(x: np.ndarray) -> np.ndarray:
    # np.unique is pathologically slow on this numpy build; sort + mask is not
    s = np.sort(x)
    if s.size == 0:
        return s
    keep = np.empty(s.size, dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def rmat_codes(scale: int, avg_degree: int, probs, seed: int):
    """Distinct undirected edge codes of the reference R-MAT; returns (codes, truncated).

    ``codes`` is sorted ascending (the reference's set order is irrelevant
    because ``build_graph`` canonicalises).  Semantics of ``graph.py:213-246``.
    """
    a, b, c, _ = (float(p) for p in probs)
    side = 1 << scale
    target = (side * avg_degree) // 2
    cap = 20 * target
    rng = np.random.default_rng(seed)
    drawn = 0
    parts = []          # per-chunk codes, stream order
    n_uniq = 0
    while drawn < cap:
        # draw at least what is still missing, plus a margin for duplicates
        want = min(int(1.15 * (target - n_uniq)) + 1024, cap - drawn)
        got = 0
        while got < want:
            k = min(_CHUNK_PAIRS, want - got)
            parts.append(_pair_codes(rng.random((k, scale)), a, b, c, scale))
            got += k
        drawn += want
        uniq = _sorted_unique(np.concatenate(parts))
        n_uniq = uniq.size
        if n_uniq >= target:
            break
    if n_uniq <= target:
        return uniq, n_uniq < target
    # more distinct codes than needed: keep the first `target` in stream order
    stream = np.concatenate(parts)
    perm = np.argsort(stream, kind="stable")
    srt = stream[perm]
    start = np.empty(srt.size, dtype=bool)
    start[0] = True
    np.not_equal(srt[1:], srt[:-1], out=start[1:])
    first = perm[start]                       # first stream index of each distinct code
    cut = np.partition(first, target - 1)[target - 1]
    return _sorted_unique(stream[: cut + 1]), False


def rmat_edges(scale: int, avg_degree: int, probs=(0.57, 0.19, 0.19, 0.05), seed: int = 0):
    """(edges (k,2) int64, truncated) with the reference's edge set."""
    codes, truncated = rmat_codes(scale, avg_degree, probs, seed)
    side = np.int64(1 << scale)
    edges = np.empty((codes.size, 2), dtype=np.int64)
    edges[:, 0] = codes // side
    edges[:, 1] = codes % side
    return edges, truncated


def er_edges_gnm(n: int = 1_000_000, draws: int = 8_080_000, seed: int = 0):
    """ER-1M recipe of SURVEY.md §8(d): uniform endpoint pairs, cleaned by build_graph."""
    return np.random.default_rng(seed).integers(0, n, size=(draws, 2))


def ba_edges(n: int = 2000, m: int = 3, seed: int = 0):
    """Barabasi-Albert via networkx (the BASELINE correctness config)."""
    import networkx as nx

    return np.asarray(list(nx.barabasi_albert_graph(n, m, seed=seed).edges()), dtype=np.int64)


def chung_lu_edges(n: int = 1 << 20, gamma: float = 2.1, max_weight: float = 2e5,
                   mean_degree: float = 16.0, seed: int = 0):
    """Chung-Lu power law: w_i = W((i+i0)/i0)^(-1/(gamma-1)),
    i0 chosen so the mean weight is ``mean_degree``; floor(sum w / 2) endpoint
    pairs drawn proportionally to w."""
    expo = -1.0 / (gamma - 1.0)
    idx = np.arange(n, dtype=np.float64)

    def mean_for(i0):
        return float(np.mean(max_weight * ((idx + i0) / i0) ** expo))

    lo, hi = 1e-3, 1e6
    for _ in range(200):
        mid = np.sqrt(lo * hi)
        if mean_for(mid) > mean_degree:
            hi = mid
        else:
            lo = mid
    i0 = np.sqrt(lo * hi)
    w = max_weight * ((idx + i0) / i0) ** expo
    rng = np.random.default_rng(seed)
    k = int(np.floor(w.sum() / 2))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = np.searchsorted(cdf, rng.random(k), side="right")
    v = np.searchsorted(cdf, rng.random(k), side="right")
    return np.stack([np.minimum(u, n - 1), np.minimum(v, n - 1)], axis=1).astype(np.int64)


def ws_edges(n: int = 4_000_000, k: int = 20, p: float = 0.05, seed: int = 0):
    """Watts-Strogatz: ring lattice (u, u+j mod n), j=1..k/2, each target rewired
    uniformly with probability p."""
    rng = np.random.default_rng(seed)
    half = k // 2
    u = np.repeat(np.arange(n, dtype=np.int64), half)
    v = (u + np.tile(np.arange(1, half + 1, dtype=np.int64), n)) % n
    rewire = rng.random(u.size) < p
    v[rewire] = rng.integers(0, n, size=int(rewire.sum()))
    return np.stack([u, v], axis=1)
