"""bench.py contract smoke on the GPU box: the default single-rank line and a
torchrun-free `--gpus 2` run (bench.py re-executes itself under
torch.distributed.run; on a 1-GPU box the two ranks share the device and use
gloo host collectives) on a small config, checking the JSON keys the driver
reads."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def _check_line(d, n_gpus):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "e2e", "roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == n_gpus and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


def test_bench_single_rank_ba2000():
    d = _bench("--config", "ba2000", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1")
    _check_line(d, 1)


def test_bench_two_ranks_without_torchrun():
    env_keys = [k for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK") if k in os.environ]
    assert not env_keys  # the self-launch path is the one under test
    d = _bench("--gpus", "2", "--config", "er1m", "--steps", "3", "--warmup", "3", "--e2e-steps", "1")
    _check_line(d, 2)
    assert "2 parts" in d["config"]["parallelism"]
