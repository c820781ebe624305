"""GPU parity of the ranking consumers (analysis.py:84-103, :214-243) against
oracle/ranking.py and the reference's own known answers
(pkg/tests/test_analysis.py:61-84).  Indices and targets bit-exact."""
import math

import numpy as np
import pytest

import paper_2306_00606_b200 as efg
from oracle import ranking as R

pytestmark = pytest.mark.gpu


def _same(bins, want):
    assert [(b.target_ef, b.representative, b.achieved_ef) for b in bins] == want


def test_ef_bins_reference_known_answers():
    bins = efg.ef_bins(np.arange(10, dtype=float), k=10)
    assert [b.target_ef for b in bins] == list(map(float, range(10)))
    assert [b.representative for b in bins] == list(range(10))
    assert [b.representative for b in efg.ef_bins(np.array([0.0, 10.0]), k=2)] == [0, 1]
    assert efg.ef_bins(np.array([0.0, 10.0, 0.0]), k=2)[0].representative == 0
    values = np.random.default_rng(3).random(50) * 7
    lo, hi = values.min(), values.max()
    for i, b in enumerate(efg.ef_bins(values, k=10)):
        assert b.target_ef == lo + i * (hi - lo) / 9
    with pytest.raises(ValueError, match="distinct"):
        efg.ef_bins(np.array([1.0, 1.0, 2.0]), k=3)
    with pytest.raises(ValueError):
        efg.ef_bins(np.array([1.0, 2.0]), k=0)
    _same(efg.ef_bins(np.array([4.0]), k=1), R.ef_bins([4.0], k=1))


def test_ef_bins_and_rank_on_real_ef(golden):
    for name in ("rmat_14_16_1",):
        efv = golden[name].get("ef")
        for k in (1, 2, 10, 37):
            _same(efg.ef_bins(efv, k=k), R.ef_bins(efv, k=k))
        assert np.array_equal(efg.ef_rank_ascending(efv), R.rank_ascending(efv))
    # many ties, including signed zero, at a size with multiple sort passes
    rng = np.random.default_rng(5)
    vals = rng.integers(0, 50, size=300_001).astype(float) / 7.0
    vals[::97] = -0.0
    assert np.array_equal(efg.ef_rank_ascending(vals), R.rank_ascending(vals))
    _same(efg.ef_bins(vals, k=20), R.ef_bins(vals, k=20))
    res = efg.ef_cluster_centric(efg.generate_rmat(efg.RmatParams(scale=12, avg_degree=8, seed=3))[0])
    _same(efg.ef_bins(res, k=10), R.ef_bins(res.ef, k=10))


def test_immunization_windows():
    rng = np.random.default_rng(1)
    vals = rng.random(1000).round(2)
    order = R.rank_ascending(vals)
    got = efg.immunization_windows(vals, frac=0.05, scenarios=7)
    window = math.ceil(0.05 * 1000)
    starts = R.window_starts(1000, window, 7)
    assert [s for s, _ in got] == starts
    for (s, ids) in got:
        assert np.array_equal(ids, order[s:s + window])
    assert [s for s, _ in efg.immunization_windows(vals, frac=0.5, scenarios=1)] == [0]
    with pytest.raises(ValueError):
        efg.immunization_windows(vals, frac=1.0)
    with pytest.raises(ValueError, match="index case"):
        efg.immunization_windows(np.array([1.0, 2.0]), frac=0.9)
