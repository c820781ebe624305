"""Undirected simple graphs in CSR form -- drop-in for ``efgraph.graph``.

Mirrors /root/reference/pkg/src/efgraph/graph.py: the same ``Graph`` fields and
accessors (:34-87), ``RmatParams`` validation (:90-112), ``build_graph``
semantics (:147-190) and ``generate_rmat`` output (:204-246).  The cleaning
(self-loop drop, symmetrise, dedupe, isolated-node drop, dense relabel, sorted
CSR) runs on the GPU (K1, csrc/csr_build.cu) and returns bit-identical arrays.
CSR arrays live in page-locked host memory so the EF call's host->device copy
runs at full PCIe/C2C speed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = [
    "Graph",
    "RmatParams",
    "DEFAULT_RMAT_PROBS",
    "build_graph",
    "generate_rmat",
    "cluster_count",
]

DEFAULT_RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)  # graph.py:29

_MAX_NODES = 2**31  # neighbor ids are int32 (graph.py:31)


class Graph:
    """Immutable undirected simple graph (same attributes as efgraph.graph.Graph).

    n, m; offsets int64[n+1]; neighbors int32[2m], strictly ascending per row;
    orig_ids int64[n] ascending; relabeling dict orig -> dense (built lazily:
    a 2M-entry Python dict is expensive and EF never reads it).
    """

    __slots__ = ("n", "m", "offsets", "neighbors", "orig_ids", "_relabeling")

    def __init__(self, n, m, offsets, neighbors, orig_ids, relabeling=None):
        self.n = int(n)
        self.m = int(m)
        self.offsets = offsets
        self.neighbors = neighbors
        self.orig_ids = orig_ids
        self._relabeling = relabeling

    @property
    def relabeling(self) -> dict:
        if self._relabeling is None:
            self._relabeling = {int(o): i for i, o in enumerate(self.orig_ids.tolist())}
        return self._relabeling

    def __repr__(self):
        return f"Graph(n={self.n}, m={self.m})"

    def _check_id(self, v: int) -> None:
        if not 0 <= v < self.n:
            raise ValueError(f"node id {v} out of range [0, {self.n})")

    def degree(self, v: int) -> int:
        self._check_id(v)
        return int(self.offsets[v + 1] - self.offsets[v])

    def degrees(self) -> np.ndarray:
        """Per-node degree array (int64)."""
        return np.diff(self.offsets)

    def adjacency(self, v: int) -> np.ndarray:
        """Sorted neighbor ids of v (read-only view)."""
        self._check_id(v)
        return self.neighbors[self.offsets[v]: self.offsets[v + 1]]

    def has_edge(self, u: int, v: int) -> bool:
        """Membership by binary search on the lower-degree endpoint (graph.py:72-82)."""
        self._check_id(u)
        self._check_id(v)
        if u == v:
            return False
        if self.degree(u) > self.degree(v):
            u, v = v, u
        adj = self.adjacency(u)
        pos = int(np.searchsorted(adj, v))
        return pos < adj.size and int(adj[pos]) == v

    def avg_degree(self) -> float:
        return 0.0 if self.n == 0 else 2.0 * self.m / self.n


@dataclass(frozen=True)
class RmatParams:
    """Parameters of the recursive-matrix generator (graph.py:90-112)."""

    scale: int
    avg_degree: int
    quadrant_probs: tuple = DEFAULT_RMAT_PROBS
    seed: int = 0

    def __post_init__(self):
        if self.scale < 1:
            raise ValueError("scale must be >= 1")
        if self.avg_degree < 1:
            raise ValueError("avg_degree must be >= 1")
        probs = tuple(float(p) for p in self.quadrant_probs)
        if len(probs) != 4 or any(p < 0 for p in probs):
            raise ValueError("quadrant_probs must be 4 nonnegative reals")
        if abs(sum(probs) - 1.0) > 1e-9:
            raise ValueError(f"quadrant_probs must sum to 1, got {sum(probs)}")


def _empty_graph() -> Graph:
    return Graph(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int64), {})


def build_graph(edges, device: int | None = None) -> Graph:
    """Build the cleaned CSR of raw (u, v) pairs on the GPU (graph.py:147-190).

    Self-loops dropped, symmetrised, deduplicated, isolated nodes removed,
    dense relabel in ascending original-id order.  Degenerate input yields
    the empty graph; more than 2^31-1 nodes raises ValueError.
    """
    arr = np.asarray(edges, dtype=np.int64)
    if arr.size == 0:
        return _empty_graph()
    arr = np.ascontiguousarray(arr.reshape(-1, 2))
    ctx = _native.context(device)
    L = _native.lib()
    n = _native.ctypes.c_int64()
    m = _native.ctypes.c_int64()
    _native.check(L.efg_build_graph(ctx.handle, _native.ptr(arr), arr.shape[0],
                                    _native.ctypes.byref(n), _native.ctypes.byref(m)))
    return _fetch(ctx, n.value, m.value)


def _fetch(ctx, n: int, m: int) -> Graph:
    if n == 0:
        return _empty_graph()
    offsets = _native.pinned_empty(n + 1, np.int64)
    neighbors = _native.pinned_empty(2 * m, np.int32)
    orig_ids = np.empty(n, np.int64)
    _native.check(_native.lib().efg_fetch_graph(ctx.handle, _native.ptr(offsets), _native.ptr(neighbors),
                                                _native.ptr(orig_ids)))
    return Graph(n, m, offsets, neighbors, orig_ids)


def generate_rmat(params: RmatParams, device: int | None = None) -> tuple[Graph, bool]:
    """R-MAT sample identical to the reference's (graph.py:204-246); returns (graph, truncated).

    Sampled on the GPU (csrc/rmat.cu): numpy PCG64's double stream is
    reproduced by 128-bit LCG jump-ahead from np.random.default_rng(seed)'s
    state; the edge set is the first floor(2^N*M/2) distinct non-loop codes of
    the pair stream, cleaned by K1.  Bit-identical CSR (tests compare the
    reference's sha256 fingerprints).
    """
    st = np.random.default_rng(params.seed).bit_generator.state["state"]
    mask = (1 << 64) - 1
    state = np.array([st["state"] & mask, st["state"] >> 64], dtype=np.uint64)
    inc = np.array([st["inc"] & mask, st["inc"] >> 64], dtype=np.uint64)
    probs = np.array([float(p) for p in params.quadrant_probs], dtype=np.float64)
    ctx = _native.context(device)
    C = _native.ctypes
    tr, n, m = C.c_int32(), C.c_int64(), C.c_int64()
    _native.check(_native.lib().efg_rmat_build(ctx.handle, int(params.scale), int(params.avg_degree),
                                               _native.ptr(probs), _native.ptr(state), _native.ptr(inc),
                                               C.byref(tr), C.byref(n), C.byref(m)))
    return _fetch(ctx, n.value, m.value), bool(tr.value)


def cluster_count(g) -> int:
    """Middle-node triplets: sum over nodes of C(deg, 2) (graph.py:249-255)."""
    d = np.diff(np.asarray(g.offsets, dtype=np.int64))
    return int(np.sum(d * (d - 1) // 2))
