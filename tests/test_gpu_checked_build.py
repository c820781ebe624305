"""Device bounds checks (the compute-sanitizer stand-in: the tool is closed on
the B200 pool, profiles/r02_compute_sanitizer_closed.txt).

libefg_checked.so is libefg.so compiled with -DEFG_BOUNDS_CHECK: the risky
device indices -- F/G/PT table gathers, shared-map positions, bitmap words,
row ranges, Adj+ writes -- are checked in the kernels; a failed check is
recorded and clamped (no out-of-bounds access happens) and the call returns
status 2.  tools/sanitize_case.py drives every engine and triangle path on
small graphs (BA-2000, R-MAT 12/8, a hub-heavy Chung-Lu graph, an
1100-clique dense core, an isolated edge, shards, a distributed part +
finish, pageable staging, ranking) and compares each against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2306_00606_b200", "libefg_checked.so")


def test_bounds_checked_build_runs_every_path_clean():
    if not os.path.exists(CHECKED):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2306_00606_b200"), "checked"], check=True)
    env = dict(os.environ, EFG_LIB=CHECKED)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "bounds check failed" not in out
    assert "sanitize workload ok" in out
