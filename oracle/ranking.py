"""Ranking consumers, CPU restatement (TEST INFRASTRUCTURE ONLY).

Restates the reference's analysis.py so the device ranking kernels
(`efg_ef_bins`, `efg_rank_ascending`) can be checked:
* `ef_bins` follows analysis.py:84-103 (numpy argmin -> lowest id on ties;
  targets lo + i*(hi-lo)/(k-1) in that operation order);
* `rank_ascending` is analysis.py:240, np.argsort(ef, kind="stable");
* `window_starts` is analysis.py:236-239.
Pinned against the reference's own known answers (pkg/tests/test_analysis.py:61-84)
in tests/test_oracle.py.  Never imported by the product.
"""
from __future__ import annotations

import numpy as np


def ef_bins(values, k: int = 10):
    if k < 1:
        raise ValueError("k must be >= 1")
    values = np.asarray(values, dtype=np.float64)
    if np.unique(values).size < k:
        raise ValueError(f"only {np.unique(values).size} distinct EF values; choose k <= that")
    lo = float(values.min())
    hi = float(values.max())
    out = []
    for i in range(k):
        target = lo if k == 1 else lo + i * (hi - lo) / (k - 1)
        rep = int(np.argmin(np.abs(values - target)))
        out.append((target, rep, float(values[rep])))
    return out


def rank_ascending(values):
    return np.argsort(np.asarray(values, dtype=np.float64), kind="stable")


def window_starts(n: int, window: int, scenarios: int):
    if scenarios == 1:
        return [0]
    return [round(i * (n - window) / (scenarios - 1)) for i in range(scenarios)]
