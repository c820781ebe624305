"""CLI end to end on the GPU: the reference CLI with `--backend gpu` bound
(paper_2306_00606_b200/cli.py; reference test_cli.py TestGenerate/TestEf/
TestBench), the added `topk`, and GPU-vs-CPU backend output values."""
import hashlib
import json
import math

import pytest

from paper_2306_00606_b200.cli import main

pytestmark = pytest.mark.gpu


def _run(*argv):
    return main([str(a) for a in argv])


def test_generate_matches_reference_target(tmp_path):
    out = tmp_path / "g.txt"
    assert _run("generate", "--scale", 10, "--avg-degree", 8, "--seed", 1, "--output", out) == 0
    assert len(out.read_text().strip().splitlines()) == (2**10 * 8) // 2
    m = json.loads((tmp_path / "g.txt.manifest.json").read_text())
    assert m["status"] == "ok" and m["graph"]["edges"] == 4096 and m["truncated"] is False
    b = tmp_path / "b.txt"
    assert _run("generate", "--scale", 10, "--avg-degree", 8, "--seed", 1, "--output", b) == 0
    assert hashlib.sha256(out.read_bytes()).digest() == hashlib.sha256(b.read_bytes()).digest()


def test_ef_star_and_manifest(tmp_path):
    inp = tmp_path / "star.txt"
    inp.write_text("0 1\n0 2\n0 3\n")
    out = tmp_path / "ef.csv"
    assert _run("ef", "--input", inp, "--mode", "cluster", "--output", out) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "node,ef,cluster_total"
    node, score, total = lines[1].split(",")
    assert (node, total) == ("0", "6") and float(score) == pytest.approx(math.log(6), abs=1e-8)
    m = json.loads((tmp_path / "ef.csv.manifest.json").read_text())
    assert m["clusters_processed"] == 3 and m["time_to_solution_ms"] > 0 and m["clusters_per_ms"] > 0


def test_modes_and_workers_agree(tmp_path):
    inp = tmp_path / "g.txt"
    assert _run("generate", "--scale", 8, "--avg-degree", 6, "--seed", 4, "--output", inp) == 0
    outs = []
    for tag, mode, workers in (("a", "cluster", 1), ("b", "cluster", 8), ("c", "vertex", 1)):
        out = tmp_path / f"{tag}.csv"
        assert _run("ef", "--input", inp, "--mode", mode, "--workers", workers, "--output", out) == 0
        outs.append(out.read_bytes())
    assert outs[0] == outs[1] == outs[2]


def test_bench_and_topk(tmp_path):
    out = tmp_path / "bench.csv"
    assert _run("bench", "--scale", 9, "--degrees", "2,4", "--modes", "cluster,vertex", "--repeats", 1,
                "--output", out) == 0
    rows = out.read_text().strip().splitlines()
    assert rows[0] == "mode,scale,avg_degree,workers,time_ms,clusters_per_ms" and len(rows) == 5
    inp = tmp_path / "g.txt"
    assert _run("generate", "--scale", 9, "--avg-degree", 6, "--seed", 2, "--output", inp) == 0
    top = tmp_path / "top.csv"
    assert _run("topk", "--input", inp, "--frac", 0.05, "--output", top) == 0
    assert top.read_text().splitlines()[0] == "rank,node,ef"


def test_gpu_backend_values_match_reference_backend(tmp_path):
    inp = tmp_path / "g.txt"
    assert _run("generate", "--scale", 9, "--avg-degree", 8, "--seed", 3, "--output", inp) == 0
    outs = {}
    for be in ("gpu", "cpu"):
        out = tmp_path / f"{be}.csv"
        assert main(["--backend", be, "ef", "--input", str(inp), "--output", str(out)]) == 0
        rows = [ln.split(",") for ln in out.read_text().strip().splitlines()[1:]]
        outs[be] = rows
        m = json.loads((tmp_path / f"{be}.csv.manifest.json").read_text())
        assert m["status"] == "ok" and m["graph"]["sha256"]
    assert [r[0] for r in outs["gpu"]] == [r[0] for r in outs["cpu"]]
    assert [r[2] for r in outs["gpu"]] == [r[2] for r in outs["cpu"]]        # cluster_total exact
    for a, b in zip(outs["gpu"], outs["cpu"]):                                # %.9g values (ties may round apart)
        assert float(a[1]) == pytest.approx(float(b[1]), rel=2e-9, abs=1e-12)
