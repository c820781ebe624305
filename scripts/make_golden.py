"""Generate golden vectors from the REFERENCE package (run in the dev container).

Imports efgraph from /root/reference/pkg/src (read-only, never copied) and its
test helpers' semantics (edge generators restated below), runs the reference's
own build_graph / ef_cluster_centric / ef_vertex_centric / brute-force oracle,
and stores inputs + outputs under tests/golden/.  The GPU box cannot import
the reference: the parity tests compare against these files.

Usage:  python scripts/make_golden.py
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
from efgraph.graph import RmatParams, build_graph, cluster_count, generate_rmat  # noqa: E402
from efgraph.expected_force import ef_cluster_centric, ef_vertex_centric  # noqa: E402
import oracles  # noqa: E402  (the reference's brute-force oracle, pkg/tests/oracles.py)


# edge generators: same definitions as pkg/tests/conftest.py:12-30
def star_edges(leaves, center=0):
    return [(center, center + i) for i in range(1, leaves + 1)]


def path_edges(nodes):
    return [(i, i + 1) for i in range(nodes - 1)]


def cycle_edges(nodes):
    return [(i, (i + 1) % nodes) for i in range(nodes)]


def complete_edges(nodes):
    return [(i, j) for i in range(nodes) for j in range(i + 1, nodes)]


def er_edges(n, p, seed):
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < p
    iu, ju = np.triu_indices(n, 1)
    keep = mask[iu, ju]
    return list(zip(iu[keep].tolist(), ju[keep].tolist()))


def main():
    cases = {}  # name -> (edges or None, graph)
    small = {
        "star3": star_edges(3), "path4": path_edges(4), "triangle": [(0, 1), (1, 2), (0, 2)],
        "cycle5": cycle_edges(5), "k4": complete_edges(4), "star7_path3": star_edges(7) + path_edges(3),
        "edge": [(0, 1)], "k5": complete_edges(5), "star5": star_edges(5), "path10": path_edges(10),
        "k6": complete_edges(6), "cycle9": cycle_edges(9), "path3": path_edges(3),
        "dup_loop": [(0, 1), (1, 0), (2, 2)], "relabel": [(5, 9)], "loop_only": [(3, 3)],
        "isolated_loop": [(0, 1), (7, 7)], "export": [(9, 5), (5, 3), (9, 3), (3, 1)],
    }
    for s in range(5):
        small[f"er40_{s}"] = er_edges(40, 0.1, s)
    for s in range(20):
        small[f"er80_{300 + s}"] = er_edges(80, 0.08, 300 + s)
    for s in range(4):
        small[f"er80_{s}"] = er_edges(80, 0.08, s)
    for s in range(8):
        small[f"er60_{s}"] = er_edges(60, 0.08, s)
    for s in range(3):
        small[f"er200_{100 + s}"] = er_edges(200, 0.05, 100 + s)
    # acceptance c01 mixed set (pkg/tests/test_acceptance.py:31-46)
    i = 0
    got = 0
    while got < 200:
        if i % 2 == 0:
            n = 20 + (i * 7) % 180
            p = 0.03 + 0.004 * (i % 20)
            e = er_edges(n, p, seed=1000 + i)
            g = build_graph(e)
            if g.n:
                small[f"mixed_{i}"] = e
                got += 1
        else:
            params = RmatParams(scale=5 + i % 3, avg_degree=2 + i % 5, seed=2000 + i)
            g, _ = generate_rmat(params)
            if g.n:
                cases[f"mixed_{i}"] = ("rmat", (5 + i % 3, 2 + i % 5, 2000 + i), g)
                got += 1
        i += 1
    for name, e in small.items():
        cases[name] = ("edges", e, build_graph(e))
    for (s, m, seed) in [(8, 4, 5), (8, 4, 77), (9, 6, 5), (10, 8, 1), (12, 8, 3), (14, 16, 1)]:
        g, _ = generate_rmat(RmatParams(scale=s, avg_degree=m, seed=seed))
        cases[f"rmat_{s}_{m}_{seed}"] = ("rmat", (s, m, seed), g)
    import networkx as nx
    ba = np.asarray(list(nx.barabasi_albert_graph(2000, 3, seed=0).edges()), dtype=np.int64)
    cases["ba2000"] = ("edges", ba, build_graph(ba))

    arrays = {}
    index = {}
    for name, (kind, src, g) in cases.items():
        t0 = time.time()
        a = ef_cluster_centric(g)
        t_cc = time.time() - t0
        rec = {"kind": kind, "n": g.n, "m": g.m, "clusters_processed": a.clusters_processed,
               "cluster_count": cluster_count(g), "t_cluster_centric_s": round(t_cc, 3)}
        if kind == "rmat":
            rec["rmat"] = list(src)
        else:
            arrays[f"{name}__edges"] = np.asarray(src, dtype=np.int64).reshape(-1, 2)
        if g.m <= 20000:
            b = ef_vertex_centric(g)
            rec["vertex_clusters_processed"] = b.clusters_processed
            rec["vertex_bitwise_equal"] = bool(np.array_equal(a.ef, b.ef))
        if kind == "edges" and g.n <= 200:
            adj = oracles.adjacency(src)
            bf = oracles.expected_force(adj)
            arrays[f"{name}__ef_brute"] = np.array([bf[int(o)] for o in g.orig_ids], np.float64)
            rec["naive_cluster_count"] = oracles.naive_cluster_count(adj)
        arrays[f"{name}__offsets"] = g.offsets
        arrays[f"{name}__neighbors"] = g.neighbors
        arrays[f"{name}__orig_ids"] = g.orig_ids
        arrays[f"{name}__ef"] = a.ef
        arrays[f"{name}__cluster_total"] = a.cluster_total
        arrays[f"{name}__flags"] = a.flags
        index[name] = rec
        print(name, rec, flush=True)
    np.savez_compressed("tests/golden/reference_ef.npz", **arrays)
    with open("tests/golden/reference_ef.json", "w") as fh:
        json.dump({"generator": "scripts/make_golden.py", "reference": "efgraph 0.1.0 (/root/reference/pkg)",
                   "numpy": np.__version__, "cases": index}, fh, indent=1)


if __name__ == "__main__":
    main()
