"""Expected Force centrality on the GPU -- drop-in for ``efgraph.expected_force``.

Same public surface and semantics as
/root/reference/pkg/src/efgraph/expected_force.py:
``EFResult`` (:54-71), ``FLAG_*`` (:47-49), ``cluster_degree`` (:74-88),
``entropy_from_histogram`` (:91-111), ``ef`` (:114-120), ``write_ef_csv``
(:123-130), ``ef_cluster_centric`` (:138-174), ``ef_vertex_centric`` (:345-418),
plus ``key_nodes`` (device top-k ranking, semantics of analysis.py:101,240).

The per-seed cluster sums run in hand-written sm_100a kernels behind the C ABI
(include/efg.h); there is no CPU fallback.  ``workers`` and ``chunk_size`` are
validated exactly like the reference (ValueError below 1) and otherwise do not
change the result -- the reference guarantees bitwise-identical output for any
value (expected_force.py:141-146), and so do the kernels (fixed-order sums).

Engines (``engine=``): "factorized" (default for cluster_centric) sums clusters
in degree classes with exact triangle corrections; "direct" (default for
vertex_centric, the original formulation) visits every star and chain.  Both
return identical cluster_total/flags and EF within 1e-15 relative of each other.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native

__all__ = [
    "EFResult",
    "FLAG_OK",
    "FLAG_NO_CLUSTERS",
    "FLAG_ZERO_DEGREE_CLUSTERS",
    "cluster_degree",
    "entropy_from_histogram",
    "ef_cluster_centric",
    "ef_vertex_centric",
    "ef",
    "write_ef_csv",
    "key_nodes",
]

FLAG_OK = 0
FLAG_NO_CLUSTERS = 1  # node participates in no cluster (e.g. isolated edge)
FLAG_ZERO_DEGREE_CLUSTERS = 2  # clusters exist but all have degree 0


@dataclass
class EFResult:
    """Per-node Expected Force scores plus diagnostics (expected_force.py:54-71).

    ef: float64 >= 0; cluster_total: int64 mass 2*C(deg,2) + sum(deg_i - 1);
    flags: uint8 FLAG_*; clusters_processed: distinct clusters (cluster_centric)
    or per-node visits (vertex_centric).  ``stats`` (extra): device timings
    and counters of the call.
    """

    ef: np.ndarray
    cluster_total: np.ndarray
    flags: np.ndarray
    clusters_processed: int
    stats: dict | None = field(default=None, repr=False, compare=False)


def cluster_degree(g, i: int, v: int, j: int) -> int:
    """Out-degree of the cluster with middle v and wings i, j (expected_force.py:74-88)."""
    if i == j:
        raise ValueError("cluster wings must be distinct")
    if not (g.has_edge(v, i) and g.has_edge(v, j)):
        raise ValueError(f"({i}, {v}, {j}) is not a middle-node triplet")
    d = g.degree(v) + g.degree(i) + g.degree(j) - 4
    if g.has_edge(i, j):
        d -= 2
    return d


def entropy_from_histogram(h) -> float:
    """Entropy of a cluster-degree histogram {degree: count} (expected_force.py:91-111).

    Degree-0 clusters and the empty histogram carry no mass; natural log.
    """
    items = sorted(h.items())
    total = 0
    for d, c in items:
        if d < 0 or c < 0:
            raise ValueError("histogram keys and counts must be non-negative")
        total += d * c
    if total == 0:
        return 0.0
    w = 0.0
    for d, c in items:
        if d > 0:
            w += c * d * math.log(d)
    return math.log(total) - w / total


def _empty_result() -> EFResult:
    return EFResult(ef=np.zeros(0), cluster_total=np.zeros(0, np.int64), flags=np.zeros(0, np.uint8),
                    clusters_processed=0)


def _engine_code(engine) -> int:
    if isinstance(engine, int):
        return engine
    try:
        return _native.ENGINES[engine or "auto"]
    except KeyError:
        raise ValueError(f"unknown engine {engine!r}; expected one of {sorted(_native.ENGINES)}") from None


def _run(g, mode: int, engine, device, want_tw: bool = False) -> EFResult:
    n = int(g.n)
    if n == 0:
        return _empty_result()
    offsets = np.ascontiguousarray(g.offsets, dtype=np.int64)
    neighbors = np.ascontiguousarray(g.neighbors, dtype=np.int32)
    ctx = _native.context(device)
    out_ef = _native.pinned_empty(n, np.float64)
    out_tot = _native.pinned_empty(n, np.int64)
    out_fl = _native.pinned_empty(n, np.uint8)
    T = np.empty(n, np.int64) if want_tw else None
    W = np.empty(n, np.float64) if want_tw else None
    processed = ctypes.c_int64()
    st = _native.Stats()
    _native.check(_native.lib().efg_expected_force(
        ctx.handle, _native.ptr(offsets), _native.ptr(neighbors), n, mode, _engine_code(engine),
        _native.ptr(out_ef), _native.ptr(out_tot), _native.ptr(out_fl), ctypes.byref(processed),
        _native.ptr(T), _native.ptr(W), ctypes.byref(st)))
    stats = st.as_dict()
    if want_tw:
        stats["T"] = T
        stats["W"] = W
    return EFResult(ef=out_ef, cluster_total=out_tot, flags=out_fl, clusters_processed=int(processed.value),
                    stats=stats)


def ef(g, mode: str = "cluster_centric", workers: int = 1, chunk_size: int = 4096, *,
       engine: str | None = None, device: int | None = None) -> EFResult:
    """Dispatch to one of the two Expected Force formulations (expected_force.py:114-120)."""
    if mode == "cluster_centric":
        return ef_cluster_centric(g, workers=workers, chunk_size=chunk_size, engine=engine, device=device)
    if mode == "vertex_centric":
        return ef_vertex_centric(g, workers=workers, engine=engine, device=device)
    raise ValueError(f"unknown mode {mode!r}; expected cluster_centric or vertex_centric")


def ef_cluster_centric(g, workers: int = 1, chunk_size: int = 4096, *, engine: str | None = None,
                       device: int | None = None) -> EFResult:
    """Expected Force with single-count cluster accounting (expected_force.py:138-174).

    ``clusters_processed`` = number of distinct clusters = sum C(deg, 2).
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    return _run(g, _native.MODE_CLUSTER_CENTRIC, engine, device)


def ef_vertex_centric(g, workers: int = 1, *, engine: str | None = None, device: int | None = None) -> EFResult:
    """Expected Force by independent per-node walks (expected_force.py:345-418).

    ``clusters_processed`` = per-node cluster visits = 3 * sum C(deg, 2).
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return _run(g, _native.MODE_VERTEX_CENTRIC, engine, device)


def write_ef_csv(g, result: EFResult, stream) -> None:
    """``node,ef,cluster_total`` rows, original ids ascending, 9 significant digits
    (expected_force.py:123-130)."""
    import os

    stream.write("node,ef,cluster_total\n")
    orig = np.ascontiguousarray(g.orig_ids, dtype=np.int64)
    efv = np.ascontiguousarray(result.ef, dtype=np.float64)
    tot = np.ascontiguousarray(result.cluster_total, dtype=np.int64)
    n = int(efv.size)
    if n == 0:
        return
    # rows formatted by the C ABI's host formatter (%.9g == Python's format(x, ".9g"))
    buf = np.empty(64 * n, np.uint8)
    length = ctypes.c_int64()
    _native.check(_native.lib().efg_format_ef_csv(
        _native.ptr(orig), _native.ptr(efv), _native.ptr(tot), n, len(os.sched_getaffinity(0)),
        _native.ptr(buf), buf.size, ctypes.byref(length)))
    stream.write(buf[: length.value].tobytes().decode("ascii"))


def key_nodes(result, k: int | None = None, frac: float | None = None, device: int | None = None) -> np.ndarray:
    """Top-ranked seeds by EF (device top-k, K5): the ``k`` (or ceil(frac*n))
    dense ids with the largest EF, ties to the smaller id -- the order of
    ``np.lexsort((ids, -ef))`` (cf. analysis.py:101 and :240)."""
    efv = np.ascontiguousarray(result.ef if hasattr(result, "ef") else result, dtype=np.float64)
    n = efv.size
    if (k is None) == (frac is None):
        raise ValueError("pass exactly one of k or frac")
    if k is None:
        if not 0 < frac <= 1:
            raise ValueError("frac must be in (0, 1]")
        k = math.ceil(frac * n)
    if k < 0:
        raise ValueError("k must be >= 0")
    k = min(int(k), n)
    out = np.empty(k, np.int64)
    if k == 0:
        return out
    ctx = _native.context(device)
    _native.check(_native.lib().efg_topk(ctx.handle, _native.ptr(efv), n, k, _native.ptr(out)))
    return out
