"""Pin the CPU oracle (oracle/) against the reference's own golden vectors.

The fixtures in tests/golden/ were produced by running the reference package
itself (scripts/make_golden.py).  If the oracle agrees with them, it can check
the GPU path at sizes the reference cannot run.
"""
import math

import numpy as np
import pytest

from conftest import ef_close
from oracle import brute
from oracle import ef as O
from oracle import graph as G


def test_oracle_matches_reference_on_every_golden_case(golden):
    checked = 0
    for name, case in golden.items():
        if case.n == 0:
            continue
        off, nb = case.get("offsets"), case.get("neighbors")
        ef, tot, fl, T, W = O.ef_seeds(off, nb, threads=4)
        assert np.array_equal(tot, case.get("cluster_total")), name
        assert np.array_equal(fl, case.get("flags")), name
        assert ef_close(ef, case.get("ef"), rtol=1e-12, atol=1e-14), name
        # T is exact; EF = ln T - W/T reproduces the oracle's own ef
        live = T > 0
        assert np.all(ef[~live] == 0.0)
        assert ef_close(np.log(T[live].astype(np.float64)) - W[live] / T[live], ef[live], rtol=1e-13, atol=1e-14), name
        assert O.cluster_count(off) == case.meta["cluster_count"]
        checked += 1
    assert checked >= 250


def test_oracle_is_bitwise_on_almost_all_cases(golden):
    # same operation order as _scores_from_histograms; only libm log vs numpy log may differ
    same = total = 0
    for case in golden.values():
        if case.n == 0:
            continue
        ef = O.ef_seeds(case.get("offsets"), case.get("neighbors"), threads=2)[0]
        same += int(np.array_equal(ef, case.get("ef")))
        total += 1
    assert same >= 0.95 * total


def test_graph_restatement_matches_reference_build(golden):
    for name, case in golden.items():
        edges = case.get("edges")
        if edges is None:
            continue
        n, m, off, nb, orig = G.build_csr(edges)
        assert (n, m) == (case.n, case.m), name
        assert np.array_equal(off, case.get("offsets")), name
        assert np.array_equal(nb, case.get("neighbors")), name
        assert np.array_equal(orig, case.get("orig_ids")), name


def test_brute_force_restatement_matches_reference_brute(golden):
    for name, case in golden.items():
        want = case.get("ef_brute")
        if want is None or case.n > 60:
            continue
        bf = brute.expected_force(brute.adjacency(case.get("edges")))
        got = np.array([bf[int(o)] for o in case.get("orig_ids")])
        assert np.allclose(got, want, rtol=0, atol=1e-12), name
        assert brute.cluster_count(brute.adjacency(case.get("edges"))) == case.meta["naive_cluster_count"]


def test_known_answers(golden):
    # closed forms asserted by the reference (test_expected_force.py:69-92, test_acceptance.py:59-72)
    s3 = golden["star3"]
    ef = O.ef_seeds(s3.get("offsets"), s3.get("neighbors"))[0]
    assert ef[0] == pytest.approx(math.log(6), abs=1e-12)
    assert np.allclose(ef[1:], math.log(2), atol=1e-12)
    p4 = golden["path4"]
    ef, tot, fl, T, W = O.ef_seeds(p4.get("offsets"), p4.get("neighbors"))
    assert ef[0] == 0.0 and ef[3] == 0.0 and tot[0] == 1
    assert ef[1] == pytest.approx(math.log(3), abs=1e-12)
    k3 = golden["triangle"]
    ef, tot, fl, _, _ = O.ef_seeds(k3.get("offsets"), k3.get("neighbors"))
    assert np.all(ef == 0.0) and set(fl.tolist()) == {2}
    e = golden["edge"]
    assert O.ef_seeds(e.get("offsets"), e.get("neighbors"))[2].tolist() == [1, 1]


def test_seed_subset_equals_full_run(golden):
    case = golden["rmat_12_8_3"]
    off, nb = case.get("offsets"), case.get("neighbors")
    seeds = np.random.default_rng(0).choice(case.n, 300, replace=False)
    ef, tot, fl, T, W = O.ef_seeds(off, nb, seeds=seeds, threads=3)
    assert np.array_equal(ef, case.get("ef")[seeds]) or ef_close(ef, case.get("ef")[seeds], 1e-14, 0)
    assert np.array_equal(tot, case.get("cluster_total")[seeds])


def test_ranking_oracle_known_answers():
    """oracle/ranking.py against the reference's own ef_bins known answers
    (pkg/tests/test_analysis.py:61-84)."""
    import pytest as _pytest
    from oracle import ranking as R

    bins = R.ef_bins(list(range(10)), k=10)
    assert [b[0] for b in bins] == list(map(float, range(10)))
    assert [b[1] for b in bins] == list(range(10))
    assert [b[1] for b in R.ef_bins([0.0, 10.0], k=2)] == [0, 1]
    assert R.ef_bins([0.0, 10.0, 0.0], k=2)[0][1] == 0
    values = np.random.default_rng(3).random(50) * 7
    lo, hi = values.min(), values.max()
    for i, b in enumerate(R.ef_bins(values, k=10)):
        assert b[0] == lo + i * (hi - lo) / 9
    with _pytest.raises(ValueError, match="distinct"):
        R.ef_bins([1.0, 1.0, 2.0], k=3)
    assert R.rank_ascending([2.0, 1.0, 2.0, 0.5]).tolist() == [3, 1, 0, 2]


def test_threaded_single_seed_walk_equals_per_seed_walk(golden):
    """efo_ef_seed_threads (the hub-fixture generator, scripts/make_hub_fixtures.py)
    gives the per-seed walk's outputs bit for bit: same histogram, same order."""
    checked = 0
    for name, case in sorted(golden.items()):
        off, nb = case.get("offsets"), case.get("neighbors")
        if off is None or case.n < 3:
            continue
        ef, tot, fl, T, W = O.ef_seeds(off, nb)
        deg = np.diff(off)
        for s in {0, int(np.argmax(deg)), case.n - 1}:
            got = O.ef_seed_threads(off, nb, s, threads=3)
            assert got == (ef[s], tot[s], fl[s], T[s], W[s]), (name, s)
            checked += 1
        if checked > 120:
            break
    assert checked > 60
