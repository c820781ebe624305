import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
REF_INSTALL = ROOT / "baseline" / "_ref"  # the unmodified reference (scripts/install_reference.sh)
if (REF_INSTALL / "efgraph").is_dir():
    os.environ.setdefault("EFGRAPH_PATH", str(REF_INSTALL))  # the CLI hooks into the reference's CLI


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libefg.so")


class GoldenCase:
    """One reference-generated fixture (scripts/make_golden.py)."""

    def __init__(self, name, meta, z):
        self.name = name
        self.meta = meta
        self._z = z

    def get(self, key):
        k = f"{self.name}__{key}"
        return self._z[k] if k in self._z.files else None

    @property
    def n(self):
        return self.meta["n"]

    @property
    def m(self):
        return self.meta["m"]


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN / "reference_ef.json").read_text())["cases"]
    z = np.load(GOLDEN / "reference_ef.npz")
    return {name: GoldenCase(name, rec, z) for name, rec in meta.items()}


def ef_close(got, want, rtol=1e-9, atol=1e-12):
    """Parity bar of BASELINE.json: |got - want| <= 1e-9 |want| + 1e-12 (fp64)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return got.shape == want.shape and bool(np.all(np.abs(got - want) <= rtol * np.abs(want) + atol))


# edge generators: same definitions as the reference's pkg/tests/conftest.py:12-30
def star_edges(leaves, center=0):
    return [(center, center + i) for i in range(1, leaves + 1)]


def path_edges(nodes):
    return [(i, i + 1) for i in range(nodes - 1)]


def cycle_edges(nodes):
    return [(i, (i + 1) % nodes) for i in range(nodes)]


def complete_edges(nodes):
    return [(i, j) for i in range(nodes) for j in range(i + 1, nodes)]


def er_edges(n, p, seed):
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < p
    iu, ju = np.triu_indices(n, 1)
    keep = mask[iu, ju]
    return list(zip(iu[keep].tolist(), ju[keep].tolist()))
