"""numpy restatement of efgraph/graph.py:147-190 `build_graph` (TEST INFRASTRUCTURE ONLY).

Same steps and output arrays as the reference: drop self-loops (:159),
orig_ids = sorted distinct endpoints (:163), dense relabel by searchsorted
(:167-168), dedupe canonical (lo, hi) codes (:169), symmetrise and sort by
(src, dst) (:174-178), offsets by bincount + cumsum (:180-181).  Uses sort-
based dedupe (np.unique is very slow on this numpy build) -- same results.
"""
from __future__ import annotations

import numpy as np


def _uniq(x):
    s = np.sort(x)
    if s.size == 0:
        return s
    keep = np.empty(s.size, bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def build_csr(edges):
    """-> (n, m, offsets int64[n+1], neighbors int32[2m], orig_ids int64[n])."""
    arr = np.asarray(edges, dtype=np.int64)
    if arr.size == 0:
        return 0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int64)
    arr = arr.reshape(-1, 2)
    arr = arr[arr[:, 0] != arr[:, 1]]
    if arr.shape[0] == 0:
        return 0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int64)
    orig = _uniq(arr.ravel())
    n = int(orig.size)
    lo = np.searchsorted(orig, np.minimum(arr[:, 0], arr[:, 1]))
    hi = np.searchsorted(orig, np.maximum(arr[:, 0], arr[:, 1]))
    codes = _uniq(lo * np.int64(n) + hi)
    m = int(codes.size)
    lo = codes // n
    hi = codes % n
    src = np.concatenate([lo, hi])
    dst = np.concatenate([hi, lo])
    key = np.sort(src * np.int64(n) + dst)
    src = key // n
    dst = key % n
    offsets = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=offsets[1:])
    return n, m, offsets, dst.astype(np.int32), orig


def cluster_count(offsets) -> int:
    d = np.diff(np.asarray(offsets, dtype=np.int64))
    return int(np.sum(d * (d - 1) // 2))
