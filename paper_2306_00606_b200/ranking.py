"""Downstream ranking consumers of the EF scores, on the device.

Mirrors the ranking half of the reference's analysis module
(`/root/reference/pkg/src/efgraph/analysis.py`); the SIR experiments that
consume these rankings are out of scope.

* `EFBin`, `ef_bins` -- analysis.py:60-64, :84-103: k targets equally spaced
  over [min EF, max EF], the node nearest each, ties to the lowest id.  Same
  validation and messages (`ValueError` for k < 1 and for fewer than k
  distinct EF values).
* `ef_rank_ascending` -- `np.argsort(ef, kind="stable")` (analysis.py:240).
* `immunization_windows` -- the contiguous rank windows of
  immunization_experiment (analysis.py:214-243): window = ceil(frac*n), starts
  equally spaced, same validation.

All three run in libefg.so (`efg_ef_bins`, `efg_rank_ascending`); there is no
host fallback.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass(frozen=True)
class EFBin:
    target_ef: float
    representative: int  # dense node id
    achieved_ef: float


def _ef_array(ef_result) -> np.ndarray:
    values = ef_result.ef if hasattr(ef_result, "ef") else ef_result
    return np.ascontiguousarray(values, dtype=np.float64)


def ef_bins(ef_result, k: int = 10, device: int | None = None) -> list[EFBin]:
    """k targets equally spaced over [min EF, max EF], nearest node each (analysis.py:84-103).

    Ties go to the lowest node id. Requires at least k distinct EF values.
    """
    if k < 1:
        raise ValueError("k must be >= 1")
    values = _ef_array(ef_result)
    if values.size == 0:
        raise ValueError("only 0 distinct EF values; choose k <= that")
    targets = np.empty(k, np.float64)
    reps = np.empty(k, np.int64)
    ctx = _native.context(device)
    _native.check(_native.lib().efg_ef_bins(ctx.handle, _native.ptr(values), values.size, k,
                                            _native.ptr(targets), _native.ptr(reps)))
    return [EFBin(target_ef=float(t), representative=int(r), achieved_ef=float(values[r]))
            for t, r in zip(targets.tolist(), reps.tolist())]


def ef_rank_ascending(ef_result, device: int | None = None) -> np.ndarray:
    """Dense ids by EF ascending, ties by ascending id: np.argsort(ef, kind="stable")."""
    values = _ef_array(ef_result)
    order = np.empty(values.size, np.int64)
    if values.size:
        ctx = _native.context(device)
        _native.check(_native.lib().efg_rank_ascending(ctx.handle, _native.ptr(values), values.size,
                                                       _native.ptr(order)))
    return order


def immunization_windows(ef_result, frac: float = 0.05, scenarios: int = 10,
                         device: int | None = None) -> list[tuple[int, np.ndarray]]:
    """(window_start, immunized dense ids) per scenario, as analysis.py:230-243 cuts them."""
    if not 0.0 < frac < 1.0:
        raise ValueError("frac must be in (0, 1)")
    if scenarios < 1:
        raise ValueError("scenarios and reps must be >= 1")
    values = _ef_array(ef_result)
    n = values.size
    window = math.ceil(frac * n)
    if window > n - 1:
        raise ValueError(f"window of {window} nodes leaves no index case on {n} nodes")
    order = ef_rank_ascending(values, device=device)
    if scenarios == 1:
        starts = [0]
    else:
        starts = [round(i * (n - window) / (scenarios - 1)) for i in range(scenarios)]
    return [(start, order[start:start + window]) for start in starts]
