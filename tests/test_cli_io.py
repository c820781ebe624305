"""Host-side CLI and edge-list I/O (no GPU): parser semantics of
efgraph/graph.py:115-144 (reference tests test_graph.py:19-53), manifest on
failure and usage errors through the `--backend gpu` hook into the
reference CLI (test_cli.py), and the C-ABI CSV row formatter against the
reference's f-string rows (expected_force.py:123-130)."""
import io
import json

import numpy as np
import pytest

from paper_2306_00606_b200.cli import main
from paper_2306_00606_b200.expected_force import EFResult, write_ef_csv
from paper_2306_00606_b200.graph import Graph
from paper_2306_00606_b200.io import load_edge_list, write_edge_list


class TestLoadEdgeList:
    def test_plain_pairs(self):
        assert load_edge_list(io.StringIO("0 1\n1 2\n")).tolist() == [[0, 1], [1, 2]]

    def test_comments_and_extra_tokens(self):
        assert load_edge_list(io.StringIO("# c\n3 4 0.5\n")).tolist() == [[3, 4]]

    def test_percent_comment_and_blank_lines(self):
        assert load_edge_list(io.StringIO("% hdr\n\n5 6\n")).tolist() == [[5, 6]]

    def test_malformed_token_reports_line(self):
        with pytest.raises(ValueError, match="line 1"):
            load_edge_list(io.StringIO("a b\n"))

    def test_malformed_on_later_line(self):
        with pytest.raises(ValueError, match="line 3"):
            load_edge_list(io.StringIO("0 1\n# ok\n2 x\n"))

    def test_single_token_line(self):
        with pytest.raises(ValueError, match="line 2"):
            load_edge_list(io.StringIO("0 1\n7\n"))

    def test_negative_id_rejected(self):
        with pytest.raises(ValueError, match="negative"):
            load_edge_list(io.StringIO("0 -2\n"))

    def test_empty_input(self):
        assert load_edge_list(io.StringIO("")).shape == (0, 2)

    def test_duplicates_kept_in_order(self):
        assert load_edge_list(io.StringIO("1 0\n1 0\n0 0\n")).tolist() == [[1, 0], [1, 0], [0, 0]]

    def test_no_trailing_newline_and_large(self):
        rng = np.random.default_rng(0)
        e = rng.integers(0, 10**9, size=(5000, 2))
        text = "\n".join(f"{a} {b}" for a, b in e)
        assert np.array_equal(load_edge_list(io.StringIO(text)), e)


def test_write_edge_list_round_trip(golden):
    case = golden["export"]
    g = Graph(case.n, case.m, case.get("offsets"), case.get("neighbors"), case.get("orig_ids"))
    buf = io.StringIO()
    write_edge_list(g, buf)
    pairs = [tuple(map(int, ln.split())) for ln in buf.getvalue().strip().splitlines()]
    assert pairs == sorted(pairs) and all(u < v for u, v in pairs)
    assert sorted(pairs) == sorted({tuple(sorted(p)) for p in case.get("edges").tolist()})


def _reference_cli_available():
    try:
        import importlib
        import os
        import sys

        p = os.environ.get("EFGRAPH_PATH")
        if p and p not in sys.path:
            sys.path.insert(0, p)
        importlib.import_module("efgraph.cli")
        return True
    except ImportError:
        return False


needs_ref = pytest.mark.skipif(not _reference_cli_available(), reason="reference efgraph not installed "
                               "(scripts/install_reference.sh)")


def test_write_ef_csv_matches_reference_rows():
    rng = np.random.default_rng(0)
    n = 200_000
    ef = rng.random(n) * 25
    ef[::7] = 0.0
    ef[::11] = 1e-5 * rng.random(ef[::11].size)
    ef[::13] = 1e-12 * rng.random(ef[::13].size)
    ef[:6] = [1e16, 123456789.5, 0.1, np.nextafter(0, 1), 2.5e-310, 99999999.95]
    orig = np.arange(n, dtype=np.int64) * 3 + 10**12
    tot = rng.integers(0, 2**62, n)
    g = Graph(n, 0, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), orig)
    r = EFResult(ef=ef, cluster_total=tot, flags=np.zeros(n, np.uint8), clusters_processed=0)
    buf = io.StringIO()
    write_ef_csv(g, r, buf)
    # the reference's writer, expected_force.py:127-130
    want = "node,ef,cluster_total\n" + "".join(f"{int(o)},{e:.9g},{int(t)}\n" for o, e, t in zip(orig, ef, tot))
    assert buf.getvalue() == want


@needs_ref
def test_usage_errors():
    assert main(["generate", "--scale", "4", "--avg-degree", "2"]) == 2
    assert main(["generate", "--scale", "4", "--avg-degree", "2", "--probs", "1,2", "--output", "x"]) == 2
    assert main([]) == 2


@needs_ref
def test_backend_flag_errors():
    assert main(["--backend", "tpu", "ef"]) == 2


@needs_ref
def test_unreadable_input_writes_error_manifest(tmp_path):
    out = tmp_path / "ef.csv"
    assert main(["ef", "--input", str(tmp_path / "missing.txt"), "--output", str(out)]) == 1
    manifest = json.loads((tmp_path / "ef.csv.manifest.json").read_text())
    assert manifest["status"] == "error" and "missing.txt" in manifest["error"]
