"""Edge-list text I/O with the reference's format and error contract.

Mirrors efgraph/graph.py:115-144 (`load_edge_list`) and :258-269
(`write_edge_list`).  A vectorised fast path handles clean files (two or more
non-negative integer tokens per line, comments and blank lines allowed); any
irregularity falls back to the reference's line-by-line parser so that error
messages name the same line numbers.
"""
from __future__ import annotations

import io
import re

import numpy as np

__all__ = ["load_edge_list", "write_edge_list"]

_CLEAN = re.compile(rb"\A(?:[ \t]*(?:[#%][^\n]*)?\n|[ \t]*\d+[ \t]+\d+(?:[ \t]+[^\n]*)?[ \t]*\n)*\Z")
_PAIRS = re.compile(rb"\A(?:[ \t]*\n|[ \t]*\d+[ \t]+\d+[ \t]*\n)*\Z")


def _slow(lines) -> np.ndarray:
    us, vs = [], []
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line[0] in "#%":
            continue
        tokens = line.split()
        if len(tokens) < 2:
            raise ValueError(f"line {lineno}: expected at least 2 tokens, got {len(tokens)}")
        try:
            u = int(tokens[0])
            v = int(tokens[1])
        except ValueError:
            raise ValueError(f"line {lineno}: non-integer node id in {tokens[:2]}") from None
        if u < 0 or v < 0:
            raise ValueError(f"line {lineno}: negative node id in ({u}, {v})")
        us.append(u)
        vs.append(v)
    out = np.empty((len(us), 2), dtype=np.int64)
    out[:, 0] = us
    out[:, 1] = vs
    return out


def load_edge_list(stream) -> np.ndarray:
    """Parse a whitespace-separated edge list into a (k, 2) int64 array (graph.py:115-144).

    '#'/'%' lines are comments, blank lines skipped, extra tokens ignored,
    duplicates and self-loops kept in input order.  ValueError names the line.
    """
    text = stream.read()
    data = text.encode() if isinstance(text, str) else bytes(text)
    if data and not data.endswith(b"\n"):
        data += b"\n"
    if _PAIRS.match(data):  # exactly two ids per line: one C-level split
        return np.array(data.split(), dtype=np.int64).reshape(-1, 2)
    if _CLEAN.match(data):
        rows = [ln.split()[:2] for ln in data.splitlines() if ln.strip() and ln.lstrip()[:1] not in (b"#", b"%")]
        if not rows:
            return np.zeros((0, 2), dtype=np.int64)
        flat = np.array([t for r in rows for t in r], dtype=np.int64)
        return flat.reshape(-1, 2)
    return _slow(io.StringIO(data.decode(errors="replace")))


def write_edge_list(g, stream) -> None:
    """One undirected edge per line in original ids, smaller first, sorted (graph.py:258-269)."""
    deg = np.diff(np.asarray(g.offsets, dtype=np.int64))
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    dst = np.asarray(g.neighbors, dtype=np.int64)
    keep = dst > src
    orig = np.asarray(g.orig_ids, dtype=np.int64)
    u = orig[src[keep]].tolist()
    v = orig[dst[keep]].tolist()
    stream.write("".join(f"{a} {b}\n" for a, b in zip(u, v)))
