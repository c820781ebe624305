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


@pytest.fixture(scope="module")
def dense_core():
    # a 1100-clique inside a sparse random graph: clique members have more than
    # 1024 higher-ranked neighbours, so the triangle listing takes Adj+(v) in parts
    rng = np.random.default_rng(3)
    k = 1100
    iu = np.triu_indices(k, 1)
    clique = np.stack(iu, 1).astype(np.int64)
    extra = rng.integers(0, 30000, size=(200000, 2))
    return efg.build_graph(np.concatenate([clique, extra]))


def test_dense_core_listing_parts(dense_core):
    g = dense_core
    res_f = _run(g, 0, "factorized", None, want_tw=True)
    res_d = _run(g, 0, "direct", None, want_tw=True)
    assert np.array_equal(res_f.stats["T"], res_d.stats["T"])
    assert np.array_equal(res_f.cluster_total, res_d.cluster_total)
    assert ef_close(res_f.ef, res_d.ef)
    rng = np.random.default_rng(1)
    seeds = np.unique(np.concatenate([rng.choice(np.arange(1100, g.n), 300, replace=False), [0, 1, 2]]))
    seeds = seeds[np.diff(g.offsets)[seeds] < 1200]  # keep the oracle cheap: at most a few clique members
    ef, tot, fl, T, W = O.ef_seeds(g.offsets, g.neighbors, seeds=seeds, threads=8)
    assert np.array_equal(res_f.stats["T"][seeds], T)
    assert ef_close(res_f.ef[seeds], ef)


@pytest.mark.parametrize("graph", ["rmat18", "dense_core"])
def test_listing_hash_map_matches_bitmap(graph, request, monkeypatch):
    # Adj+(v) parts whose labels reach past the bitmap (lim > 65536: graphs with
    # that many nodes of degree > 256) take the hash form of the listing scan;
    # EFG_MID_BM_LIMIT=0 forces it on every part: the fixed-point sums are
    # exact, so the results are bitwise those of the bitmap scan
    g = request.getfixturevalue(graph)
    base = _run(g, 0, "factorized", None, want_tw=True)
    monkeypatch.setenv("EFG_MID_BM_LIMIT", "0")
    hashed = _run(g, 0, "factorized", None, want_tw=True)
    assert np.array_equal(base.stats["T"], hashed.stats["T"])
    assert np.array_equal(base.stats["W"], hashed.stats["W"])
    assert np.array_equal(base.ef, hashed.ef) and np.array_equal(base.cluster_total, hashed.cluster_total)


def test_dense_core_shards_bitwise(dense_core):
    # whole-graph passes list triangles, shards run the per-seed path: both sum
    # the same exact fixed-point values, so the results are bitwise identical
    import torch
    from paper_2306_00606_b200 import device as D

    dg = D.DeviceGraph.from_host(dense_core)
    n = dense_core.n
    full = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_range(dg, 0, n, *full)
    b = D.shard_bounds(dg, 3, "factorized")
    outs = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    for r in range(3):
        lo, hi = int(b[r]), int(b[r + 1])
        if hi > lo:
            D.ef_range(dg, lo, hi, outs[0][lo:hi], outs[1][lo:hi], outs[2][lo:hi])
    torch.cuda.synchronize()
    for x, y in zip(full, outs):
        assert torch.equal(x, y)


@pytest.mark.parametrize("nparts", [1, 3, 8])
def test_distributed_parts_bitwise(rmat18, nparts):
    # parts of a whole-graph pass summed as the all-reduce would, then finished:
    # bitwise equal to the single-GPU pass
    import torch
    from paper_2306_00606_b200 import device as D

    dg = D.DeviceGraph.from_host(rmat18)
    n = rmat18.n
    full = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_range(dg, 0, n, *full)
    words = torch.zeros(D.DIST_WORDS * n, dtype=torch.int64, device="cuda")
    ws = torch.zeros(n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(words)
    s = torch.empty_like(ws)
    for p in range(nparts):
        D.ef_partial(dg, p, nparts, w, s)
        words += w
        ws += s
    out = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_finish(dg, 0, n, words, ws, *out)
    torch.cuda.synchronize()
    for x, y in zip(full, out):
        assert torch.equal(x, y)


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_row_partitioned_parts_bitwise(rmat18, nparts):
    # the row-partitioned distributed pass emulated on one GPU: every part's
    # rows phase writes its node range's Adj+ rows into one shared buffer (the
    # union is what the broadcast exchange assembles on every rank), then each
    # part lists its units; words summed as the all-reduce would: bitwise equal
    # to the single-GPU pass
    import torch
    from paper_2306_00606_b200 import device as D

    dg = D.DeviceGraph.from_host(rmat18)
    n = rmat18.n
    full = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_range(dg, 0, n, *full)
    bounds = D.part_bounds(dg, nparts)
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) >= 0)
    adjp = torch.empty(dg.neighbors.numel(), dtype=torch.int32, device="cuda")
    dplus = torch.empty(n, dtype=torch.int32, device="cuda")
    words = [torch.empty(D.DIST_WORDS * n, dtype=torch.int64, device="cuda") for _ in range(nparts)]
    wss = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nparts)]
    for p in range(nparts):
        D.ef_partial_rows(dg, p, nparts, bounds, adjp, dplus, words[p], wss[p])
    for p in range(nparts):
        D.ef_partial_tables(dg, p, nparts, bounds, words[p], wss[p])
    for p in range(nparts):
        D.ef_partial_list(dg, p, nparts, bounds, adjp, dplus, words[p], wss[p])
    tot_w = torch.stack(words).sum(0)
    tot_s = torch.stack(wss).sum(0)
    out = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_finish(dg, 0, n, tot_w, tot_s, *out)
    torch.cuda.synchronize()
    for x, y in zip(full, out):
        assert torch.equal(x, y)


def test_algorithm1_cross_checks_every_seed(rmat18):
    # three independent decompositions (degree classes + listing, per-seed
    # walks, the paper's middle-triplet scatter) agree on every seed
    a = _run(rmat18, 0, "factorized", None, want_tw=True)
    b = _run(rmat18, 0, "alg1", None, want_tw=True)
    assert np.array_equal(a.stats["T"], b.stats["T"])
    assert np.array_equal(a.cluster_total, b.cluster_total)
    assert np.array_equal(a.flags, b.flags)
    assert ef_close(a.ef, b.ef)  # the parity bar; alg1's W is an fp64 atomic sum (order varies)


def test_star_beyond_listing_bound():
    # a star with more than 10^6 leaves: maximum degree above the listing's
    # fixed-point bound, so the whole-graph pass takes the per-seed triangle
    # path; closed forms: centre EF = ln(k(k-1)), leaf EF = ln(k-1)
    k = 1_000_001
    edges = np.stack([np.zeros(k, np.int64), np.arange(1, k + 1, dtype=np.int64)], 1)
    g = efg.build_graph(edges)
    r = efg.ef_cluster_centric(g)
    deg = np.diff(g.offsets)
    centre = int(np.argmax(deg))
    assert deg[centre] == k
    assert ef_close(np.array([r.ef[centre]]), np.array([np.log(k * (k - 1.0))]))
    leaves = np.flatnonzero(deg == 1)
    assert np.all(np.abs(r.ef[leaves] - np.log(k - 1.0)) <= 1e-9 * np.log(k - 1.0) + 1e-12)
    assert np.array_equal(r.cluster_total, deg * (deg - 1) + np.add.reduceat(deg[g.neighbors], g.offsets[:-1]) - deg)


@pytest.mark.parametrize("splits,piece_kb", [("none", None), ("40", None), ("15,35,62", None),
                                             ("5,10,20,40,60,80,90", None), ("15,35,62", 64)])
def test_staged_chunks_bitwise(rmat18, splits, piece_kb, monkeypatch):
    # host inputs reach the device in row chunks and the engine takes up each
    # chunk's rows as it lands (class lists selected once, per-chunk runs from
    # k_chunk_counts): any split gives the device-resident result bit for bit,
    # from page-locked and from pageable host arrays
    import torch
    from paper_2306_00606_b200 import device as D
    from paper_2306_00606_b200.graph import Graph

    dg = D.DeviceGraph.from_host(rmat18)
    n = rmat18.n
    full = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    D.ef_range(dg, 0, n, *full)
    want = [x.cpu().numpy() for x in full]
    monkeypatch.setenv("EFG_STAGE_SPLITS", splits)
    if piece_kb:  # pageable staging in 64 KB pieces: ~300 gate / copy / event triples, more than a
        # stream queue holds before the workers open the first gates (enqueue and staging overlap)
        monkeypatch.setenv("EFG_STAGE_PIECE_KB", str(piece_kb))
    pageable = Graph(n, rmat18.m, np.array(rmat18.offsets, copy=True), np.array(rmat18.neighbors, copy=True), None)
    for g in (rmat18, pageable):
        r = efg.ef_cluster_centric(g)
        assert np.array_equal(r.ef, want[0]) and np.array_equal(r.cluster_total, want[1])
        assert np.array_equal(r.flags, want[2])
