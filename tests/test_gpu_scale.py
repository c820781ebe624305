"""Larger graphs: GPU vs the CPU oracle on sampled seeds, shard invariance,
and size-independent invariants (mass identity, entropy bound, exact T)."""
import numpy as np
import pytest

import paper_2306_00606_b200 as efg
from paper_2306_00606_b200 import generators as gen
from paper_2306_00606_b200.expected_force import _run
from conftest import ef_close
from oracle import ef as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmat18():
    g, _ = efg.generate_rmat(efg.RmatParams(scale=18, avg_degree=16, seed=7))
    return g


@pytest.fixture(scope="module")
def ws():
    return efg.build_graph(gen.ws_edges(n=200_000, k=20, p=0.05, seed=0))


@pytest.fixture(scope="module")
def chung_lu():
    return efg.build_graph(gen.chung_lu_edges(n=1 << 16, max_weight=2e4, seed=0))


def _check_sample(g, res, k=400, seed=0):
    rng = np.random.default_rng(seed)
    deg = np.diff(g.offsets)
    # uniform sample + the largest hubs
    seeds = np.unique(np.concatenate([rng.choice(g.n, min(k, g.n), replace=False), np.argsort(-deg)[:8]]))
    ef, tot, fl, T, W = O.ef_seeds(g.offsets, g.neighbors, seeds=seeds, threads=8)
    assert np.array_equal(res.cluster_total[seeds], tot)
    assert np.array_equal(res.flags[seeds], fl)
    assert ef_close(res.ef[seeds], ef)
    assert np.array_equal(res.stats["T"][seeds], T)


@pytest.mark.parametrize("engine", ["factorized", "direct"])
def test_rmat18_sampled_seeds_vs_oracle(rmat18, engine):
    res = _run(rmat18, 0, engine, None, want_tw=True)
    _check_sample(rmat18, res)


def test_watts_strogatz_triangle_heavy(ws):
    res = _run(ws, 0, "factorized", None, want_tw=True)
    _check_sample(ws, res, k=2000)


def test_chung_lu_hubs(chung_lu):
    res = _run(chung_lu, 0, "factorized", None, want_tw=True)
    _check_sample(chung_lu, res, k=300)


def test_invariants_full_graph(rmat18):
    r = efg.ef_cluster_centric(rmat18)
    deg = np.diff(rmat18.offsets)
    s1 = np.add.reduceat(deg[rmat18.neighbors], rmat18.offsets[:-1])
    assert np.array_equal(r.cluster_total, deg * (deg - 1) + s1 - deg)      # mass identity
    assert np.all(r.ef >= 0.0)
    live = r.cluster_total >= 1
    assert np.all(r.ef[live] <= np.log(r.cluster_total[live]) + 1e-12)       # entropy bound
    assert r.clusters_processed == efg.cluster_count(rmat18)


@pytest.mark.parametrize("engine", ["factorized", "direct"])
def test_shards_are_bitwise_identical_to_one_pass(rmat18, engine):
    import torch
    from paper_2306_00606_b200 import device as D

    dg = D.DeviceGraph.from_host(rmat18)
    n = rmat18.n
    full = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_range(dg, 0, n, *full, engine=engine)
    for parts in (2, 3, 8):
        b = D.shard_bounds(dg, parts, engine)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        outs = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
        for r in range(parts):
            lo, hi = int(b[r]), int(b[r + 1])
            if hi > lo:
                D.ef_range(dg, lo, hi, outs[0][lo:hi], outs[1][lo:hi], outs[2][lo:hi], engine=engine)
        torch.cuda.synchronize()
        for x, y in zip(full, outs):
            assert torch.equal(x, y)
    # top-k on device equals host lexsort
    efh = full[0].cpu().numpy()
    assert np.array_equal(D.topk(full[0], 500), np.lexsort((np.arange(n), -efh))[:500])
