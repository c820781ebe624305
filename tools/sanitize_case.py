"""Workload for compute-sanitizer (tools/sanitize.sh): every engine and
triangle path of libefg.so on small graphs -- BA-2000, R-MAT(12, 8, seed 3),
the 1100-clique dense core (Adj+(v) in parts), a hub-heavy Chung-Lu graph
(hub tasks, far-field chain tables), the per-seed shard path, a distributed
part + finish, an isolated edge, and the ranking kernels -- each checked
against the oracle so a silently wrong result also fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_00606_b200 as efg  # noqa: E402
from paper_2306_00606_b200 import generators as gen  # noqa: E402
from paper_2306_00606_b200.expected_force import _run  # noqa: E402
from oracle import ef as O  # noqa: E402


def close(a, b):
    return bool(np.all(np.abs(np.asarray(a) - np.asarray(b)) <= 1e-9 * np.abs(b) + 1e-12))


def check(name, g, engines=("factorized", "direct"), seeds=None):
    """Both engines against the oracle; returns the factorized result."""
    ef, tot, fl, T, W = O.ef_seeds(g.offsets, g.neighbors, seeds=seeds, threads=8)
    idx = np.arange(g.n) if seeds is None else seeds
    out = {}
    for engine in engines:
        r = _run(g, 0, engine, None, want_tw=True)
        assert np.array_equal(r.cluster_total[idx], tot), (name, engine)
        assert np.array_equal(r.stats["T"][idx], T), (name, engine)
        assert close(r.ef[idx], ef), (name, engine)
        out[engine] = r
    print(f"ok {name} n={g.n} m={g.m}", flush=True)
    return out["factorized"]


def main():
    check("ba2000", efg.build_graph(gen.ba_edges(2000, 3, seed=0)))
    g, _ = efg.generate_rmat(efg.RmatParams(scale=12, avg_degree=8, seed=3))
    r = check("rmat_12_8_3", g, engines=("factorized", "direct", "alg1"))
    top = efg.key_nodes(r, frac=0.05)
    assert np.array_equal(top, np.lexsort((np.arange(g.n), -r.ef))[: top.size])
    efg.ef_bins(r, 8)
    efg.ef_rank_ascending(r)
    check("chunglu_2e14", efg.build_graph(gen.chung_lu_edges(n=1 << 14, max_weight=5e3, seed=1)))
    rng = np.random.default_rng(3)
    k = 1100
    clique = np.stack(np.triu_indices(k, 1), 1).astype(np.int64)
    extra = rng.integers(0, 3000, size=(20000, 2))
    dense = efg.build_graph(np.concatenate([clique, extra]))
    seeds = np.unique(np.concatenate([rng.choice(np.arange(k, dense.n), 100, replace=False), [0, 1]]))
    check("dense_core", dense, seeds=seeds)
    check("isolated_edge", efg.build_graph([(0, 1), (2, 3), (3, 4)]))
    # per-seed (shard) path and a distributed part + finish on the device API
    import torch
    from paper_2306_00606_b200 import device as D

    dg = D.DeviceGraph.from_host(g)
    n = g.n
    out = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
    b = D.shard_bounds(dg, 3, "factorized")
    for p in range(3):
        lo, hi = int(b[p]), int(b[p + 1])
        if hi > lo:
            D.ef_range(dg, lo, hi, out[0][lo:hi], out[1][lo:hi], out[2][lo:hi])
    torch.cuda.synchronize()
    assert np.array_equal(out[0].cpu().numpy(), r.ef)
    words = torch.zeros(D.DIST_WORDS * n, dtype=torch.int64, device="cuda")
    ws = torch.zeros(n, dtype=torch.float64, device="cuda")
    w, s = torch.empty_like(words), torch.empty_like(ws)
    for p in range(2):
        D.ef_partial(dg, p, 2, w, s)  # self-contained parts (efg_ef_partial)
        words += w
        ws += s
    D.ef_finish(dg, 0, n, words, ws, *out)
    torch.cuda.synchronize()
    assert np.array_equal(out[0].cpu().numpy(), r.ef)
    # pageable host inputs (staging ring) through the public API
    gp = efg.Graph(g.n, g.m, np.array(g.offsets), np.array(g.neighbors), None)
    assert np.array_equal(efg.ef_cluster_centric(gp).ef, r.ef)
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()
