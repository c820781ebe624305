"""Host-side CLI and edge-list I/O (no GPU): parser semantics of
efgraph/graph.py:115-144 (reference tests test_graph.py:19-53), manifest on
failure and usage errors (test_cli.py)."""
import io
import json

import numpy as np
import pytest

from paper_2306_00606_b200.cli import main
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


def test_usage_errors():
    assert main(["generate", "--scale", "4", "--avg-degree", "2"]) == 2
    assert main(["generate", "--scale", "4", "--avg-degree", "2", "--probs", "1,2", "--output", "x"]) == 2
    assert main([]) == 2


def test_unreadable_input_writes_error_manifest(tmp_path):
    out = tmp_path / "ef.csv"
    assert main(["ef", "--input", str(tmp_path / "missing.txt"), "--output", str(out)]) == 1
    manifest = json.loads((tmp_path / "ef.csv.manifest.json").read_text())
    assert manifest["status"] == "error" and "missing.txt" in manifest["error"]
