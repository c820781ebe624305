"""BASELINE.json configs on the GPU against the CPU oracle.

* ER-1M, WS (n=400K) and Chung-Lu (n=2^16, W=2e4): every seed, exact
  cluster_total/flags/T, EF within 1e-9 relative;
* R-MAT scale 22 (the bench graph, sha256 equal to the reference generator's):
  a uniform seed sample plus hubs of every size class against the oracle, and
  size-independent invariants over all 2.18 M seeds (mass identity, entropy
  bound, sum C(d,2)), and bitwise determinism of the full pass.
Both engines are checked where the oracle finishes in seconds.
"""
import hashlib

import numpy as np
import pytest

import paper_2306_00606_b200 as efg
from paper_2306_00606_b200 import generators as gen
from paper_2306_00606_b200.expected_force import _run
from conftest import ef_close
from oracle import ef as O

pytestmark = pytest.mark.gpu
RMAT22_SHA256 = "2c4b690446b61f1441357f8f4b08d437b12f7885f3375516d3c984b96c831891"


def _full_parity(g, engines=("factorized",), threads=16):
    ef, tot, fl, T, W = O.ef_seeds(g.offsets, g.neighbors, threads=threads)
    for engine in engines:
        r = _run(g, 0, engine, None, want_tw=True)
        assert np.array_equal(r.cluster_total, tot), engine
        assert np.array_equal(r.flags, fl), engine
        assert np.array_equal(r.stats["T"], T), engine
        assert ef_close(r.ef, ef), (engine, float(np.max(np.abs(r.ef - ef) / (np.abs(ef) + 1e-300))))
        assert r.clusters_processed == efg.cluster_count(g)


def test_er_1m_every_seed():
    g = efg.build_graph(gen.er_edges_gnm())
    assert (g.n, g.m) == (1_000_000, 8_079_944)
    _full_parity(g, engines=("factorized", "direct"))


def test_watts_strogatz_every_seed():
    g = efg.build_graph(gen.ws_edges(n=400_000, k=20, p=0.05, seed=0))
    _full_parity(g, engines=("factorized", "direct"))


def test_chung_lu_every_seed():
    g = efg.build_graph(gen.chung_lu_edges(n=1 << 16, max_weight=2e4, seed=0))
    _full_parity(g, engines=("factorized", "direct"))


@pytest.fixture(scope="module")
def rmat22():
    g, trunc = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
    assert not trunc
    return g


def test_rmat22_matches_reference_generator(rmat22):
    g = rmat22
    h = hashlib.sha256()
    h.update(np.int64([g.n, g.m]).tobytes())
    for a in (g.offsets, g.neighbors, g.orig_ids):
        h.update(np.ascontiguousarray(a).tobytes())
    assert (g.n, g.m) == (2_181_017, 44_040_192)
    assert h.hexdigest() == RMAT22_SHA256


def test_rmat22_sampled_seeds_and_invariants(rmat22):
    g = rmat22
    r = _run(g, 0, "factorized", None, want_tw=True)
    deg = np.diff(g.offsets)
    # invariants over all seeds
    s1 = np.add.reduceat(deg[g.neighbors], g.offsets[:-1])
    assert np.array_equal(r.cluster_total, deg * (deg - 1) + s1 - deg)
    assert np.all(r.ef >= 0.0)
    live = r.cluster_total >= 1
    assert np.all(r.ef[live] <= np.log(r.cluster_total[live]) + 1e-12)
    assert r.clusters_processed == 127_263_919_491
    # oracle on a sample: uniform + hubs from every degree class (the largest ones
    # take minutes on the CPU and are covered by the engine cross-check below)
    rng = np.random.default_rng(0)
    order = np.argsort(-deg, kind="stable")
    hubs = np.concatenate([order[40:46], order[300:304], order[2000:2004], order[9000:9004]])
    seeds = np.unique(np.concatenate([rng.choice(g.n, 600, replace=False), hubs]))
    ef, tot, fl, T, W = O.ef_seeds(g.offsets, g.neighbors, seeds=seeds, threads=16)
    assert np.array_equal(r.cluster_total[seeds], tot)
    assert np.array_equal(r.flags[seeds], fl)
    assert np.array_equal(r.stats["T"][seeds], T)
    assert ef_close(r.ef[seeds], ef)
    # determinism of the full pass
    r2 = efg.ef_cluster_centric(g)
    assert np.array_equal(r.ef, r2.ef)


def test_rmat22_engines_agree_on_every_seed(rmat22):
    g = rmat22
    a = _run(g, 0, "factorized", None, want_tw=True)
    b = _run(g, 0, "direct", None, want_tw=True)
    assert np.array_equal(a.stats["T"], b.stats["T"])            # exact integer T, every seed incl. the top hub
    assert np.array_equal(a.cluster_total, b.cluster_total)
    assert ef_close(a.ef, b.ef, rtol=1e-12, atol=1e-13)
