"""bench.py host-side contract (no GPU): the torchrun-free `--gpus N` path
re-executes itself under torch.distributed.run with the driver's launch line,
and the reference arm's sampling helpers draw BASELINE.md 3's samples."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gpus_flag_self_launches_torchrun(monkeypatch):
    seen = {}

    def fake_execv(path, argv):
        seen["path"], seen["argv"] = path, argv
        raise SystemExit(0)

    monkeypatch.setattr(os, "execv", fake_execv)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    with pytest.raises(SystemExit):
        bench.main()
    argv = seen["argv"]
    assert argv[0] == sys.executable and argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--nnodes=1" in argv
    assert argv[argv.index("--master-addr") + 1] == "127.0.0.1"
    assert argv[-4:] == ["--gpus", "4", "--steps", "3"] and argv[-5].endswith("bench.py")


def test_reference_samples_follow_baseline_md():
    rng_draw = bench.uniform_sample(10_000, 2000, 0)
    assert rng_draw.size == 2000 and np.all(np.diff(rng_draw) > 0)
    assert np.array_equal(rng_draw, np.sort(np.random.default_rng(0).choice(10_000, 2000, replace=False)))
    assert [b[2] for b in bench.BUCKETS] == [200, 100, 20, 2]


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "efgraph")),
                    reason="reference not installed (scripts/install_reference.sh)")
def test_reference_arm_runs_the_unmodified_reference_on_ba2000(capsys, monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--config", "ba2000", "--steps", "1",
                                      "--warmup", "0"])
    bench.main()
    import json

    line = json.loads([ln for ln in capsys.readouterr().out.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert "efgraph" in line["cpu_baseline"]["reference"]
