"""The reference's OWN EF test files, unchanged, run against the GPU backend
(INTEGRATION.md section 3).

A child pytest collects baseline/_ref/efgraph_tests/ (the reference's
pkg/tests, installed by scripts/install_reference.sh next to the unmodified
package) with the ref_gpu_backend plugin, which rebinds efgraph's EF entry
points (and, in the second run, build_graph) to this repo's sm_100a path.

  * test_expected_force.py (pkg/tests/test_expected_force.py:29-179): known
    answers, oracle equivalence, determinism, invariants, counts;
  * test_acceptance.py c01-c03 (pkg/tests/test_acceptance.py:31-83): 200 mixed
    graphs cluster vs vertex mode < 1e-9, closed forms at 1e-12, counts;
  * test_graph.py TestBuildGraph / TestQueries / TestClusterCount / TestRmat
    (:56-160) with K1 as build_graph and the device sampler as generate_rmat;
  * test_cli.py TestEf / TestBench (:47-84, :185-202): the reference CLI,
    whose `compute_ef` then resolves to the GPU engine.

The child's report must list the reference's test ids as passed, and the
plugin's call counts prove the GPU functions were the ones called.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "efgraph_tests")


def _run_child(tmp_path, targets, rebind_graph=False, kexpr=None):
    if not os.path.isdir(REF_TESTS):
        pytest.fail("baseline/_ref/efgraph_tests missing: run scripts/install_reference.sh before shipping")
    report = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    env["EFG_BACKEND_REPORT"] = str(report)
    env["EFG_REBIND_GRAPH"] = "1" if rebind_graph else "0"
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_gpu_backend", "-p", "no:cacheprovider", "-rA", "-q",
           "--rootdir", REF_TESTS, "-c", os.devnull]
    if kexpr:
        cmd += ["-k", kexpr]
    cmd += [os.path.join(REF_TESTS, t) for t in targets]
    p = subprocess.run(cmd, env=env, cwd=REF_TESTS, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    print(out[-6000:])
    assert p.returncode == 0, out[-4000:]
    calls = json.loads(report.read_text())
    passed = [ln.split()[1] for ln in out.splitlines() if ln.startswith("PASSED ")]
    return calls, passed, out


def test_reference_expected_force_suite_on_gpu(tmp_path):
    calls, passed, out = _run_child(tmp_path, ["test_expected_force.py"])
    assert len(passed) >= 20, out[-2000:]
    assert any("TestKnownAnswers" in t or "TestClosedForms" in t or "star" in t for t in passed)
    assert calls.get("ef_cluster_centric", 0) > 50 and calls.get("ef_vertex_centric", 0) > 5, calls


def test_reference_acceptance_c01_c03_on_gpu(tmp_path):
    calls, passed, out = _run_child(tmp_path, ["test_acceptance.py"], kexpr="c01 or c02 or c03")
    ids = " ".join(passed)
    for c in ("test_c01", "test_c02", "test_c03"):
        assert c in ids, out[-2000:]
    assert calls.get("ef_cluster_centric", 0) >= 200 and calls.get("ef_vertex_centric", 0) >= 200, calls


def test_reference_graph_builder_suite_with_k1(tmp_path):
    calls, passed, out = _run_child(tmp_path, ["test_graph.py"], rebind_graph=True,
                                    kexpr="TestBuildGraph or TestClusterCount or TestRmat or TestQueries")
    assert len(passed) >= 5, out[-2000:]
    assert calls.get("build_graph", 0) >= 5, calls


def test_reference_cli_ef_and_bench_on_gpu(tmp_path):
    calls, passed, out = _run_child(tmp_path, ["test_cli.py"], kexpr="TestEf or TestBench")
    ids = " ".join(passed)
    assert "test_star_scores" in ids and "test_modes_and_workers_agree_bytewise" in ids, out[-2000:]
    assert "test_small_sweep" in ids, out[-2000:]
    assert calls.get("ef", 0) >= 5, calls
