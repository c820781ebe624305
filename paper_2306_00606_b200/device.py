"""Device-resident entry points (graph already in HBM) over torch CUDA tensors.

torch is used only as plumbing here (device allocation, streams, the
distributed process group); the compute is libefg.so.  These are the calls
bench.py times for the in-HBM `value` and that the multi-GPU path shards.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .expected_force import _engine_code


def _dptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class DeviceGraph:
    """A CSR resident on one GPU (torch int64 offsets [n+1], int32 neighbors [2m])."""

    def __init__(self, offsets, neighbors, n: int, orig_ids=None):
        self.offsets = offsets
        self.neighbors = neighbors
        self.n = int(n)
        self.m = int(neighbors.numel() // 2)
        self.orig_ids = orig_ids

    @classmethod
    def from_host(cls, g, device=None, non_blocking=False):
        import torch

        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        off = torch.from_numpy(np.ascontiguousarray(g.offsets, dtype=np.int64)).to(dev, non_blocking=non_blocking)
        nb = torch.from_numpy(np.ascontiguousarray(g.neighbors, dtype=np.int32)).to(dev, non_blocking=non_blocking)
        return cls(off, nb, g.n, getattr(g, "orig_ids", None))


def _ctx_for(t):
    return _native.context(t.device.index if t.device.index is not None else 0)


# torch reports its default (legacy) stream as handle 0; the C ABI reads NULL
# as "use the library's own stream", so name the legacy stream explicitly.
_CUDA_STREAM_LEGACY = 0x1


def _bind_stream(ctx, stream) -> None:
    h = stream.cuda_stream or _CUDA_STREAM_LEGACY
    _native.check(_native.lib().efg_set_stream(ctx.handle, ctypes.c_void_p(h)))


def ef_range(dg: DeviceGraph, lo: int, hi: int, out_ef, out_total, out_flags, engine="factorized",
             T=None, W=None, stats: bool = False, stream=None):
    """EF of seeds [lo, hi) into device tensors (index = seed - lo).  Returns a
    stats dict when ``stats`` (synchronising), else runs async on the context's
    stream (set to torch's current stream so torch ordering holds)."""
    import torch

    ctx = _ctx_for(dg.offsets)
    L = _native.lib()
    s = torch.cuda.current_stream(dg.offsets.device) if stream is None else stream
    _bind_stream(ctx, s)
    st = _native.Stats() if stats else None
    _native.check(L.efg_expected_force_device(
        ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n, int(lo), int(hi), _engine_code(engine),
        _dptr(out_ef), _dptr(out_total), _dptr(out_flags), _dptr(T), _dptr(W),
        ctypes.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


DIST_WORDS = 9  # EFG_DIST_WORDS: uint64 words per node of a distributed pass


def part_bounds(dg: DeviceGraph, nparts: int) -> np.ndarray:
    """Contiguous node ranges of the distributed pass, balanced by row work
    (efg_part_bounds; identical on every rank: it depends only on the degrees)."""
    import torch

    ctx = _ctx_for(dg.offsets)
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    out = np.zeros(nparts + 1, np.int64)
    _native.check(_native.lib().efg_part_bounds(ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n,
                                                int(nparts), _native.ptr(out)))
    return out


def ef_partial(dg: DeviceGraph, part: int, nparts: int, words, ws, stats: bool = False):
    """One self-contained part of a distributed whole-graph pass (efg_ef_partial):
    integer words int64[DIST_WORDS * n] and stars terms f64[n] of part `part`
    of `nparts`; sum both over all parts, then ef_finish."""
    import torch

    ctx = _ctx_for(dg.offsets)
    L = _native.lib()
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    st = _native.Stats() if stats else None
    _native.check(L.efg_ef_partial(ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n, int(part), int(nparts),
                                   _dptr(words), _dptr(ws), ctypes.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


def ef_partial_rows(dg: DeviceGraph, part: int, nparts: int, bounds, adjp, dplus, words, ws, stats: bool = False):
    """The rows phase of a row-partitioned part (efg_ef_partial_rows): the part's
    neighbour degrees and S1/S2 (into words), its label-sorted Adj+ rows into
    adjp (int32[2m], slot space) and |Adj+| into dplus (int32[n])."""
    import torch

    ctx = _ctx_for(dg.offsets)
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    st = _native.Stats() if stats else None
    _native.check(_native.lib().efg_ef_partial_rows(
        ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n, int(part), int(nparts), _native.ptr(b),
        _dptr(adjp), _dptr(dplus), _dptr(words), _dptr(ws), ctypes.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


def ef_partial_tables(dg: DeviceGraph, part: int, nparts: int, bounds, words, ws, stats: bool = False):
    """The tables phase of a row-partitioned part (efg_ef_partial_tables): the
    part's histograms, chain tables and pushes into words / ws (after its rows
    phase on the same context; runs while the Adj+ row exchange is in flight)."""
    import torch

    ctx = _ctx_for(dg.offsets)
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    st = _native.Stats() if stats else None
    _native.check(_native.lib().efg_ef_partial_tables(
        ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n, int(part), int(nparts), _native.ptr(b),
        _dptr(words), _dptr(ws), ctypes.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


def ef_partial_list(dg: DeviceGraph, part: int, nparts: int, bounds, adjp, dplus, words, ws, stats: bool = False):
    """The listing phase of a row-partitioned part (efg_ef_partial_list) on the
    exchanged adjp / dplus; adds the part's triangle words into words."""
    import torch

    ctx = _ctx_for(dg.offsets)
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    st = _native.Stats() if stats else None
    _native.check(_native.lib().efg_ef_partial_list(
        ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n, int(part), int(nparts), _native.ptr(b),
        _dptr(adjp), _dptr(dplus), _dptr(words), _dptr(ws), ctypes.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


def ef_finish(dg: DeviceGraph, lo: int, hi: int, words, ws, out_ef, out_total, out_flags, T=None, W=None):
    """Outputs of seeds [lo, hi) from the summed words of all parts (efg_ef_finish)."""
    import torch

    ctx = _ctx_for(dg.offsets)
    L = _native.lib()
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    _native.check(L.efg_ef_finish(ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n, int(lo), int(hi),
                                  _dptr(words), _dptr(ws), _dptr(out_ef), _dptr(out_total), _dptr(out_flags),
                                  _dptr(T), _dptr(W)))


def shard_bounds(dg: DeviceGraph, parts: int, engine="factorized") -> np.ndarray:
    """K2: contiguous seed shards of balanced engine work (identical on every rank)."""
    import torch

    ctx = _ctx_for(dg.offsets)
    L = _native.lib()
    _bind_stream(ctx, torch.cuda.current_stream(dg.offsets.device))
    out = np.zeros(parts + 1, np.int64)
    _native.check(L.efg_shard_bounds(ctx.handle, _dptr(dg.offsets), _dptr(dg.neighbors), dg.n,
                                     _engine_code(engine), int(parts), _native.ptr(out)))
    return out


def topk(ef_tensor, k: int) -> np.ndarray:
    """K5 on a device EF tensor -> host int64 ids (np.lexsort((ids, -ef))[:k])."""
    import torch

    ctx = _ctx_for(ef_tensor)
    L = _native.lib()
    _bind_stream(ctx, torch.cuda.current_stream(ef_tensor.device))
    k = min(int(k), ef_tensor.numel())
    out = np.empty(k, np.int64)
    if k:
        _native.check(L.efg_topk_device(ctx.handle, _dptr(ef_tensor), ef_tensor.numel(), k, _native.ptr(out)))
    return out
