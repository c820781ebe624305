"""Boundary-count brute force (TEST INFRASTRUCTURE ONLY).

Restates the reference's independent oracle pkg/tests/oracles.py:27-61: the
degree of a cluster is the literal number of edges leaving the explicit
3-node set, and EF is -sum p ln p over individual cluster entries with
p = d / total, zero-degree entries skipped; stars are listed twice.
Tiny graphs only (pure Python).
"""
from __future__ import annotations

import math


def adjacency(edges):
    adj = {}
    for u, v in edges:
        u, v = int(u), int(v)
        if u != v:
            adj.setdefault(u, set()).add(v)
            adj.setdefault(v, set()).add(u)
    return adj


def _boundary(adj, members):
    inside = set(members)
    return sum(1 for x in inside for y in adj[x] if y not in inside)


def expected_force(adj):
    """orig id -> EF by explicit enumeration (oracles.py:33-61)."""
    out = {}
    for u in adj:
        entries = []
        nb = sorted(adj[u])
        for a in range(len(nb)):
            for b in range(a + 1, len(nb)):
                d = _boundary(adj, (u, nb[a], nb[b]))
                entries += [d, d]
        for i in nb:
            for k in sorted(adj[i]):
                if k != u:
                    entries.append(_boundary(adj, (u, i, k)))
        total = sum(entries)
        if total == 0:
            out[u] = 0.0
            continue
        h = 0.0
        for d in entries:
            if d > 0:
                p = d / total
                h -= p * math.log(p)
        out[u] = h
    return out


def cluster_count(adj) -> int:
    return sum(len(s) * (len(s) - 1) // 2 for s in adj.values())
