"""Fingerprint the reference R-MAT generator's graphs (run HERE, needs /root/reference).

Writes tests/golden/rmat_fingerprints.json: sha256 over (n, m, offsets, neighbors,
orig_ids) exactly as the reference CLI fingerprints a graph (efgraph/cli.py:220-226),
for the params the tests and the bench use.  The GPU box cannot import the
reference; the device generator + device CSR builder are checked against these.
"""
import hashlib, json, sys, time

import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
from efgraph.graph import RmatParams, generate_rmat


def fingerprint(g):
    # same byte stream as efgraph/cli.py:220-226
    h = hashlib.sha256()
    h.update(np.int64([g.n, g.m]).tobytes())
    for arr in (g.offsets, g.neighbors, g.orig_ids):
        h.update(arr.tobytes())
    return h.hexdigest()


if __name__ == "__main__":
    params = [(1, 1, 3), (5, 2, 2000), (8, 4, 11), (9, 6, 5), (10, 8, 1), (12, 8, 3),
              (14, 16, 1), (16, 8, 42)]
    if "--big" in sys.argv:
        params = [(22, 21, 0)]
    out = {}
    for s, m, seed in params:
        t = time.time()
        g, trunc = generate_rmat(RmatParams(scale=s, avg_degree=m, seed=seed))
        out[f"{s},{m},{seed}"] = {"n": g.n, "m": g.m, "truncated": trunc, "sha256": fingerprint(g),
                                  "dmax": int(g.degrees().max()) if g.n else 0,
                                  "gen_seconds": round(time.time() - t, 1)}
        print(out, flush=True)
    name = "rmat_fingerprints_big.json" if "--big" in sys.argv else "rmat_fingerprints.json"
    json.dump(out, open(f"tests/golden/{name}", "w"), indent=1)
