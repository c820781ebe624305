"""Synthetic-graph recipes: the vectorised R-MAT reproduces the reference sampler."""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import graph as G
from paper_2306_00606_b200.generators import rmat_edges


def fingerprint(n, m, off, nb, orig):
    # same byte stream as efgraph/cli.py:220-226
    h = hashlib.sha256()
    h.update(np.int64([n, m]).tobytes())
    for a in (off, nb, orig):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_rmat_matches_reference_golden_graphs(golden):
    done = 0
    for name, case in golden.items():
        if case.meta["kind"] != "rmat" or case.meta["rmat"][0] > 12:
            continue
        s, m, seed = case.meta["rmat"]
        edges, trunc = rmat_edges(s, m, seed=seed)
        n, mm, off, nb, orig = G.build_csr(edges)
        assert (n, mm) == (case.n, case.m), name
        assert np.array_equal(off, case.get("offsets")) and np.array_equal(nb, case.get("neighbors")), name
        assert np.array_equal(orig, case.get("orig_ids")), name
        done += 1
    assert done >= 50


def test_rmat_fingerprints_match_reference():
    fps = json.loads((GOLDEN / "rmat_fingerprints.json").read_text())
    for key, rec in fps.items():
        s, m, seed = map(int, key.split(","))
        if s > 16:
            continue
        edges, trunc = rmat_edges(s, m, seed=seed)
        assert trunc == rec["truncated"], key
        n, mm, off, nb, orig = G.build_csr(edges)
        assert fingerprint(n, mm, off, nb, orig) == rec["sha256"], key


def test_truncation_semantics():
    # all mass on one corner: every draw is a self-loop (reference test_graph.py:150-155)
    edges, trunc = rmat_edges(1, 1, probs=(1.0, 0.0, 0.0, 0.0), seed=0)
    assert trunc and edges.shape == (0, 2)
