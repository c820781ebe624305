"""ctypes front end of ef_oracle.c (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libeforacle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        lib.efo_ef_seeds.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int64, ctypes.c_int,
                                     p, p, p, p, p]
        lib.efo_ef_seeds.restype = ctypes.c_int
        lib.efo_ef_seed_threads.argtypes = [ctypes.c_int64, p, p, ctypes.c_int64, ctypes.c_int, p, p, p, p, p]
        lib.efo_ef_seed_threads.restype = ctypes.c_int
        lib.efo_cluster_count.argtypes = [ctypes.c_int64, p]
        lib.efo_cluster_count.restype = ctypes.c_int64
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def ef_seeds(offsets, neighbors, seeds=None, threads: int = 1):
    """Per-seed (ef, cluster_total, flags, T, W) for `seeds` (None = every node).

    T is the exact integer sum of w*d and W the fp64 sum of w*d*ln d, both in
    the reference's accumulation order (expected_force.py:312-324)."""
    lib = _load()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    neighbors = np.ascontiguousarray(neighbors, dtype=np.int32)
    n = offsets.size - 1
    if seeds is not None:
        seeds = np.ascontiguousarray(seeds, dtype=np.int64)
        k = seeds.size
    else:
        k = n
    ef = np.zeros(k, np.float64)
    tot = np.zeros(k, np.int64)
    flags = np.zeros(k, np.uint8)
    T = np.zeros(k, np.int64)
    W = np.zeros(k, np.float64)
    rc = lib.efo_ef_seeds(n, _ptr(offsets), _ptr(neighbors), _ptr(seeds), k, int(threads),
                          _ptr(ef), _ptr(tot), _ptr(flags), _ptr(T), _ptr(W))
    if rc != 0:
        raise RuntimeError(f"efo_ef_seeds failed rc={rc}")
    return ef, tot, flags, T, W


def ef_seed_threads(offsets, neighbors, seed: int, threads: int = 8):
    """One seed's (ef, cluster_total, flags, T, W) with its cluster walk split
    over `threads` (exact bitmap membership; same histogram as ef_seeds)."""
    lib = _load()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    neighbors = np.ascontiguousarray(neighbors, dtype=np.int32)
    ef = np.zeros(1, np.float64)
    tot = np.zeros(1, np.int64)
    flags = np.zeros(1, np.uint8)
    T = np.zeros(1, np.int64)
    W = np.zeros(1, np.float64)
    rc = lib.efo_ef_seed_threads(offsets.size - 1, _ptr(offsets), _ptr(neighbors), int(seed), int(threads),
                                 _ptr(ef), _ptr(tot), _ptr(flags), _ptr(T), _ptr(W))
    if rc != 0:
        raise RuntimeError(f"efo_ef_seed_threads failed rc={rc}")
    return float(ef[0]), int(tot[0]), int(flags[0]), int(T[0]), float(W[0])


def cluster_count(offsets) -> int:
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    return int(_load().efo_cluster_count(offsets.size - 1, _ptr(offsets)))
