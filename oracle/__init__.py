"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference EF path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference arm may import this package, and only as the checker or the CPU
baseline.  The product package (paper_2306_00606_b200) never imports it.

* ef_oracle.c / ef.py  -- per-seed histogram + entropy, restating
  efgraph/expected_force.py:370-391 and :306-328 (see the C header).
* graph.py             -- numpy restatement of efgraph/graph.py:147-190
  (build_graph) and :249-255 (cluster_count).
* brute.py             -- the reference's independent boundary-count oracle
  (pkg/tests/oracles.py:27-61), restated for tiny graphs.

Pinned in tests/test_oracle.py against golden vectors produced by the
reference package itself (scripts/make_golden.py -> tests/golden/).
"""
