"""ctypes binding of libefg.so (the C ABI declared in include/efg.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every compute entry point raises.  Status codes map to
exceptions: 1 -> ValueError (the reference's argument errors), 2/3 ->
EFGDeviceError (an OSError, so the reference CLI's "ValueError/OSError ->
manifest status:error" contract still holds, cli.py:76-85), 4 -> MemoryError.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EFG_LIB") or os.path.join(_HERE, "libefg.so")  # EFG_LIB: A/B builds

MODE_CLUSTER_CENTRIC = 0
MODE_VERTEX_CENTRIC = 1
ENGINE_AUTO = 0
ENGINE_FACTORIZED = 1
ENGINE_DIRECT = 2
ENGINE_ALG1 = 3
ENGINES = {"auto": ENGINE_AUTO, "factorized": ENGINE_FACTORIZED, "direct": ENGINE_DIRECT, "alg1": ENGINE_ALG1}

# every symbol include/efg.h declares (checked by tests/test_native.py)
EXPORTED = (
    "efg_abi_version", "efg_last_error", "efg_create", "efg_destroy", "efg_set_stream",
    "efg_synchronize", "efg_build_graph", "efg_fetch_graph", "efg_graph_device",
    "efg_expected_force", "efg_expected_force_device", "efg_shard_bounds", "efg_part_bounds", "efg_ef_partial", "efg_ef_partial_rows", "efg_ef_partial_tables",
    "efg_ef_partial_list",
    "efg_ef_finish",
    "efg_topk",
    "efg_topk_device", "efg_rank_ascending", "efg_ef_bins", "efg_host_alloc", "efg_host_free", "efg_profile_enable", "efg_profile_reset",
    "efg_profile_report", "efg_profile_timeline", "efg_rmat_build", "efg_format_ef_csv",
)


class EFGDeviceError(OSError):
    """A CUDA / NCCL failure inside libefg (status 2 or 3)."""


class Stats(ctypes.Structure):
    _fields_ = [
        ("ms_device", ctypes.c_double),
        ("ms_prepare", ctypes.c_double),
        ("ms_enumerate", ctypes.c_double),
        ("ms_h2d", ctypes.c_double),
        ("ms_d2h", ctypes.c_double),
        ("clusters_processed", ctypes.c_int64),
        ("cluster_visits", ctypes.c_int64),
        ("terms", ctypes.c_int64),
        ("bytes_alg", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("engine", ctypes.c_int32),
        ("dmax", ctypes.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()


def build(verbose: bool = False) -> str:
    """Compile libefg.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True, stdout=out)
    return LIB_PATH


def lib():
    """Load libefg.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make -C {_HERE}` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        p, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        P = ctypes.POINTER
        sig = {
            "efg_abi_version": ([], ctypes.c_int),
            "efg_last_error": ([], ctypes.c_char_p),
            "efg_create": ([ctypes.c_int, P(p)], ctypes.c_int),
            "efg_destroy": ([p], ctypes.c_int),
            "efg_set_stream": ([p, p], ctypes.c_int),
            "efg_synchronize": ([p], ctypes.c_int),
            "efg_build_graph": ([p, p, i64, P(i64), P(i64)], ctypes.c_int),
            "efg_fetch_graph": ([p, p, p, p], ctypes.c_int),
            "efg_graph_device": ([p, P(p), P(p), P(i64), P(i64)], ctypes.c_int),
            "efg_expected_force": ([p, p, p, i64, i32, i32, p, p, p, P(i64), p, p, P(Stats)], ctypes.c_int),
            "efg_expected_force_device": ([p, p, p, i64, i64, i64, i32, p, p, p, p, p, P(Stats)], ctypes.c_int),
            "efg_shard_bounds": ([p, p, p, i64, i32, i32, p], ctypes.c_int),
            "efg_part_bounds": ([p, p, p, i64, i32, p], ctypes.c_int),
            "efg_ef_partial": ([p, p, p, i64, i32, i32, p, p, P(Stats)], ctypes.c_int),
            "efg_ef_partial_rows": ([p, p, p, i64, i32, i32, p, p, p, p, p, P(Stats)], ctypes.c_int),
            "efg_ef_partial_tables": ([p, p, p, i64, i32, i32, p, p, p, P(Stats)], ctypes.c_int),
            "efg_ef_partial_list": ([p, p, p, i64, i32, i32, p, p, p, p, p, P(Stats)], ctypes.c_int),
            "efg_ef_finish": ([p, p, p, i64, i64, i64, p, p, p, p, p, p, p], ctypes.c_int),
            "efg_topk": ([p, p, i64, i64, p], ctypes.c_int),
            "efg_topk_device": ([p, p, i64, i64, p], ctypes.c_int),
            "efg_rank_ascending": ([p, p, i64, p], ctypes.c_int),
            "efg_ef_bins": ([p, p, i64, i64, p, p], ctypes.c_int),
            "efg_host_alloc": ([i64, P(p)], ctypes.c_int),
            "efg_host_free": ([p], ctypes.c_int),
            "efg_profile_enable": ([p, i32], ctypes.c_int),
            "efg_profile_reset": ([p], ctypes.c_int),
            "efg_profile_report": ([p, ctypes.c_char_p, i64], ctypes.c_int),
            "efg_profile_timeline": ([p, ctypes.c_char_p, i64], ctypes.c_int),
            "efg_rmat_build": ([p, i32, i64, p, p, p, P(i32), P(i64), P(i64)], ctypes.c_int),
            "efg_format_ef_csv": ([p, p, p, i64, i32, p, i64, P(i64)], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().efg_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 4:
        raise MemoryError(msg)
    raise EFGDeviceError(msg)


def ptr(a) -> ctypes.c_void_p:
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class Context:
    """One libefg context (device + stream + device scratch)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        check(lib().efg_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        self._fin = weakref.finalize(self, lib().efg_destroy, h)

    def close(self):
        self._fin()

    def profile(self, on: bool = True) -> None:
        check(lib().efg_profile_enable(self.handle, int(on)))

    def profile_reset(self) -> None:
        check(lib().efg_profile_reset(self.handle))

    def profile_report(self) -> dict:
        import json

        buf = ctypes.create_string_buffer(1 << 16)
        check(lib().efg_profile_report(self.handle, buf, len(buf)))
        return {k: {"ms": v[0], "launches": int(v[1])} for k, v in json.loads(buf.value.decode()).items()}

    def profile_timeline(self) -> list:
        """[(name, start_ms, ms)] of the last profiled call, in issue order."""
        import json

        buf = ctypes.create_string_buffer(1 << 20)
        check(lib().efg_profile_timeline(self.handle, buf, len(buf)))
        return [tuple(x) for x in json.loads(buf.value.decode())]


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()
_default_device = int(os.environ.get("EFG_DEVICE", "0"))


def set_device(device: int) -> None:
    global _default_device
    _default_device = int(device)


def context(device: int | None = None) -> Context:
    dev = _default_device if device is None else int(device)
    with _ctx_lock:
        c = _contexts.get(dev)
        if c is None:
            c = _contexts[dev] = Context(dev)
        return c


# Recycled page-locked blocks: cudaHostAlloc costs ~1 ms per 10 MB, so the
# blocks behind released arrays are kept (per size, bounded) and reused.
_pool: dict[int, list[int]] = {}
_pool_bytes = 0
_POOL_LIMIT = 8 << 30
_pool_lock = threading.Lock()


def _release(addr: int, nbytes: int) -> None:
    global _pool_bytes
    with _pool_lock:
        if _pool_bytes + nbytes <= _POOL_LIMIT:
            _pool.setdefault(nbytes, []).append(addr)
            _pool_bytes += nbytes
            return
    lib().efg_host_free(ctypes.c_void_p(addr))


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array backed by page-locked host memory (block recycled when the array dies)."""
    global _pool_bytes
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    nbytes = max(64, (count * dtype.itemsize + 63) & ~63)
    addr = None
    with _pool_lock:
        free = _pool.get(nbytes)
        if free:
            addr = free.pop()
            _pool_bytes -= nbytes
    if addr is None:
        raw = ctypes.c_void_p()
        check(lib().efg_host_alloc(nbytes, ctypes.byref(raw)))
        addr = raw.value
    buf = (ctypes.c_char * nbytes).from_address(addr)
    arr = np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
    weakref.finalize(buf, _release, addr, nbytes)
    return arr
