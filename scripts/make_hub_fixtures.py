"""Oracle fixtures for the hub seeds of the two hub-heavy BASELINE configs.

The largest seeds are the ones that exercise the hub split, the far-field
chain tables and the bitmap triangle paths, and they are the ones a per-seed
CPU walk cannot finish inside a GPU test.  This script (run once, here, in
the dev container) computes them with the oracle's threaded single-seed walk
(oracle/ef_oracle.c efo_ef_seed_threads: the reference's node_histogram,
expected_force.py:370-391, with exact bitmap membership, and the entropy pass
in the reference's order, :312-327) and writes tests/golden/hub_fixtures.json:

  rmat22   -- generate_rmat(RmatParams(22, 21, seed=0)) (graph.py:204-246, via
              the host restatement generators.rmat_edges + oracle.graph.build_csr,
              sha256 checked against the reference generator's fingerprint):
              the top 40 hubs by degree, plus every 8th hub of the rest of the
              degree > 16384 class and 4 seeds from each smaller class;
  chunglu  -- Chung-Lu gamma=2.1, n=2^20, W=2e5: the top 10
              hubs plus 4 seeds of every degree class.

Per seed: dense id, degree, ef (repr), exact T = sum w*d, W (repr),
cluster_total, flags.  tests/test_gpu_configs.py compares the GPU path with
these on the device-built graphs (same sha256).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ef as O  # noqa: E402
from oracle import graph as OG  # noqa: E402
from paper_2306_00606_b200 import generators as gen  # noqa: E402

RMAT22_SHA256 = "2c4b690446b61f1441357f8f4b08d437b12f7885f3375516d3c984b96c831891"
CLASSES = [(0, 32), (33, 256), (257, 1024), (1025, 4096), (4097, 16384), (16385, 65536), (65537, 1 << 40)]


def fingerprint(n, m, off, nb, orig):
    h = hashlib.sha256()
    h.update(np.int64([n, m]).tobytes())
    for a in (off, nb, orig):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def pick(deg, top, every_hub=0, per_class=4, seed=0):
    n = deg.size
    order = np.lexsort((np.arange(n), -deg))  # degree descending, ties to the lower id
    seeds = list(order[:top])
    if every_hub:
        hubs = order[top:][deg[order[top:]] > 16384]
        seeds += list(hubs[::every_hub])
    rng = np.random.default_rng(seed)
    for lo, hi in CLASSES:
        ids = np.flatnonzero((deg >= lo) & (deg <= hi))
        ids = np.setdiff1d(ids, seeds)
        if ids.size:
            seeds += list(rng.choice(ids, size=min(per_class, ids.size), replace=False))
    return sorted(set(int(s) for s in seeds))


def run(name, n, m, off, nb, orig, seeds, threads):
    deg = np.diff(off)
    rows = []
    t0 = time.time()
    for s in seeds:
        ef, tot, fl, T, W = O.ef_seed_threads(off, nb, s, threads=threads)
        rows.append({"seed": s, "degree": int(deg[s]), "ef": repr(ef), "T": str(T), "W": repr(W),
                     "cluster_total": tot, "flags": fl})
    print(f"{name}: {len(seeds)} seeds in {time.time() - t0:.1f} s", flush=True)
    return {"n": n, "m": m, "dmax": int(deg.max()), "sha256": fingerprint(n, m, off, nb, orig), "seeds": rows}


def main():
    threads = len(os.sched_getaffinity(0))
    out = {"generator": "scripts/make_hub_fixtures.py", "oracle": "oracle/ef_oracle.c efo_ef_seed_threads"}
    e, _ = gen.rmat_edges(22, 21, seed=0)
    n, m, off, nb, orig = OG.build_csr(e)
    del e
    rec = run("rmat22", n, m, off, nb, orig, pick(np.diff(off), 40, every_hub=8), threads)
    assert rec["sha256"] == RMAT22_SHA256, "host R-MAT restatement differs from the reference generator"
    rec["workload"] = "generate_rmat(RmatParams(scale=22, avg_degree=21, seed=0))"
    out["rmat22"] = rec
    del off, nb, orig
    e = gen.chung_lu_edges(n=1 << 20, max_weight=2e5, seed=0)
    n, m, off, nb, orig = OG.build_csr(e)
    rec = run("chunglu", n, m, off, nb, orig, pick(np.diff(off), 10), threads)
    rec["workload"] = "chung_lu_edges(n=2^20, gamma=2.1, max_weight=2e5, seed=0) -> build_graph"
    out["chunglu"] = rec
    path = os.path.join(ROOT, "tests", "golden", "hub_fixtures.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
