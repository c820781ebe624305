"""Multi-GPU Expected Force.

Two schemes, both one process per GPU (torch.distributed, NCCL over NVLink on
B200 boxes) with the full CSR replicated in every rank's HBM:

* ``ef_distributed`` (whole-graph passes, the default of bench.py): rank p
  prepares the rows of its node range only (neighbour degrees, S1/S2, the
  label-sorted Adj+ rows, chain tables and pushes: efg_ef_partial_rows), the
  ranks exchange their Adj+ rows (one broadcast per part), rank p lists the
  triangles of its share of work units (efg_ef_partial_list), and ONE
  all-reduce sums the per-node integer words and stars terms; every rank then
  finishes all seeds locally (efg_ef_finish).  Integer sums and disjoint
  supports make the result bitwise identical to the single-GPU pass for any
  world size.
* ``ef_sharded`` (seed shards; the direct engine and explicit seed ranges):
  K2 cuts the seed range into contiguous shards of equal engine work
  (`shard_bounds`, the same bounds on every rank because they depend only on
  the graph); each rank runs the EF kernels on its shard; the per-seed
  outputs (ef f64, cluster_total i64, flags u8 = 17 B/seed) are exchanged
  with ONE all-gather of a packed, padded byte buffer.  Seeds have a single
  owner and their sums run in a fixed order, so the result is bitwise
  identical for any world size.

There is no reference counterpart (the reference is single-process threads,
expected_force.py:163-167); SURVEY.md §8(e) specifies this path.
"""
from __future__ import annotations

import numpy as np

RECORD_BYTES = 17  # f64 ef + i64 cluster_total + u8 flags


def _all_reduce_sum(t, group, async_op=False):
    """All-reduce (sum) of a device tensor: NCCL in place (asynchronous on
    request: the work handle is returned); under gloo (CPU tests, or ranks
    sharing one GPU) through a host copy, synchronously."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl" or t.device.type == "cpu":
        return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group,
                               async_op=async_op and dist.get_backend(group) == "nccl")
    h = t.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    t.copy_(h)
    return None


def ef_cluster_centric_distributed(g, group=None, T=None, W=None):
    """Public multi-GPU entry point: host ``Graph`` in, ``EFResult`` out on every
    rank (the ef_cluster_centric contract, expected_force.py:138-174, run as
    one process per GPU).  Each rank copies the CSR from its host arrays to
    its own GPU (the graph is replicated), runs its part of
    the whole-graph pass, joins the one all-reduce, finishes every seed and
    copies the outputs back."""
    import torch

    from . import device as D
    from .expected_force import EFResult, _empty_result
    from .graph import cluster_count

    if g.n == 0:
        return _empty_result()
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = D.DeviceGraph.from_host(g, device=dev.index, non_blocking=True)
    ef, tot, fl = ef_distributed(dg, group=group, T=T, W=W)
    return EFResult(ef=ef.cpu().numpy(), cluster_total=tot.cpu().numpy(), flags=fl.cpu().numpy(),
                    clusters_processed=cluster_count(g))


def exchange_rows(adjp, dplus, slot_bounds, node_bounds, group=None, async_op=False):
    """Every part's slot range of adjp and node range of dplus to every rank:
    one broadcast per part, rooted at the part's rank, in place (NCCL over
    NVLink; under gloo through host memory).  With async_op (NCCL) the
    broadcasts are queued on NCCL's stream and their work handles returned:
    the caller overlaps them with the tables phase and waits before listing."""
    import torch.distributed as dist

    world = len(node_bounds) - 1
    nccl = dist.get_backend(group) == "nccl"
    works = []
    for p in range(world):
        for buf, lo, hi in ((adjp, slot_bounds[p], slot_bounds[p + 1]), (dplus, node_bounds[p], node_bounds[p + 1])):
            lo, hi = int(lo), int(hi)
            if hi <= lo:
                continue
            view = buf[lo:hi]
            if nccl or view.device.type == "cpu":
                w = dist.broadcast(view, src=p, group=group, async_op=async_op and nccl)
                if w is not None:
                    works.append(w)
            else:
                h = view.cpu()
                dist.broadcast(h, src=p, group=group)
                view.copy_(h)
    return works


def ef_distributed(dg, group=None, rows=None, tables=None, listing=None, finish=None, T=None, W=None):
    """EF of every seed of DeviceGraph `dg`, the whole-graph pass split over
    the ranks of `group`; returns (ef, cluster_total, flags) on every rank.

    Rank p prepares only its node range's rows (efg_ef_partial_rows: neighbour
    degrees, S1/S2, label-sorted Adj+ rows), the ranks exchange the Adj+ rows
    (one broadcast per part, exchange_rows, asynchronous under NCCL) while
    rank p builds its rows' chain tables and pushes (efg_ef_partial_tables),
    rank p lists the triangles of its work units (efg_ef_partial_list), ONE
    all-reduce sums the integer words and stars terms, and every rank
    finishes all seeds (efg_ef_finish).  `rows(dg, part, nparts, bounds, adjp,
    dplus, words, ws)` / `tables(dg, part, nparts, bounds, words, ws)` /
    `listing(...)` / `finish(dg, words, ws, ef, tot, fl)` default to the GPU
    library; tests substitute CPU stand-ins under gloo."""
    import torch
    import torch.distributed as dist

    from . import device as D

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = dg.offsets.device
    n = dg.n
    bounds = D.part_bounds(dg, world) if rows is None else np.linspace(0, n, world + 1).astype(np.int64)
    words = torch.empty(D.DIST_WORDS * n, dtype=torch.int64, device=dev)
    ws = torch.empty(n, dtype=torch.float64, device=dev)
    adjp = torch.empty(max(1, dg.neighbors.numel()), dtype=torch.int32, device=dev)
    dplus = torch.empty(max(1, n), dtype=torch.int32, device=dev)
    (rows or D.ef_partial_rows)(dg, rank, world, bounds, adjp, dplus, words, ws)
    works = []
    if world > 1:
        slot_bounds = dg.offsets[torch.as_tensor(bounds, device=dev)].cpu().numpy()
        works = exchange_rows(adjp, dplus, slot_bounds, bounds, group, async_op=True)
    if tables is not None:
        tables(dg, rank, world, bounds, words, ws)
    elif rows is None:
        D.ef_partial_tables(dg, rank, world, bounds, words, ws)
    for w in works:  # the listing reads every part's rows
        w.wait()
    # integer words: exact in any order; stars terms: one nonzero per node.  The
    # chain / S1 / S2 words and the stars terms are final after the tables
    # phase: their all-reduce runs while the listing does; the triangle words
    # [3n, 7n) follow it
    early = []
    if world > 1:
        early = [_all_reduce_sum(words[: 3 * n], group, async_op=True),
                 _all_reduce_sum(words[7 * n:], group, async_op=True),
                 _all_reduce_sum(ws, group, async_op=True)]
    (listing or D.ef_partial_list)(dg, rank, world, bounds, adjp, dplus, words, ws)
    if world > 1:
        _all_reduce_sum(words[3 * n: 7 * n], group)
        for w in early:
            if w is not None:
                w.wait()
    ef = torch.empty(n, dtype=torch.float64, device=dev)
    tot = torch.empty(n, dtype=torch.int64, device=dev)
    fl = torch.empty(n, dtype=torch.uint8, device=dev)
    if finish is None:
        D.ef_finish(dg, 0, n, words, ws, ef, tot, fl, T=T, W=W)
    else:
        finish(dg, words, ws, ef, tot, fl)
    return ef, tot, fl


def row_bytes(pad_to: int) -> int:
    """Bytes of one rank's packed record block: ef f64 | total i64 | flags u8 (8-aligned)."""
    return 16 * pad_to + ((pad_to + 7) & ~7)


def pack_shard(ef, total, flags, pad_to: int):
    """Pack one shard's outputs into a uint8 tensor [row_bytes(pad_to)] (ef | total | flags)."""
    import torch

    L = ef.numel()
    buf = torch.zeros(row_bytes(pad_to), dtype=torch.uint8, device=ef.device)
    buf[: 8 * L] = ef.view(torch.uint8)
    buf[8 * pad_to: 8 * pad_to + 8 * L] = total.view(torch.uint8)
    buf[16 * pad_to: 16 * pad_to + L] = flags.view(torch.uint8)
    return buf


def unpack_all(gathered, bounds, pad_to: int):
    """gathered: uint8 tensor [world * pad_to * 17] -> (ef, total, flags) over all seeds."""
    import torch

    world = len(bounds) - 1
    parts = gathered.view(world, row_bytes(pad_to))
    efs, tots, fls = [], [], []
    for r in range(world):
        L = int(bounds[r + 1] - bounds[r])
        row = parts[r]
        efs.append(row[: 8 * L].view(torch.float64))
        tots.append(row[8 * pad_to: 8 * pad_to + 8 * L].view(torch.int64))
        fls.append(row[16 * pad_to: 16 * pad_to + L])
    return torch.cat(efs), torch.cat(tots), torch.cat(fls)


def ef_sharded(dg, engine="factorized", group=None, compute=None, bounds=None):
    """Expected Force of every seed of DeviceGraph `dg`, computed across the
    ranks of `group`; returns device tensors (ef, cluster_total, flags) on
    every rank.  `compute(dg, lo, hi, ef, total, flags)` defaults to the GPU
    engine (device.ef_range); tests substitute a CPU stand-in under gloo."""
    import torch
    import torch.distributed as dist

    from . import device as D

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if bounds is None:
        bounds = D.shard_bounds(dg, world, engine) if world > 1 else np.array([0, dg.n], np.int64)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    pad_to = int(max(1, np.max(np.diff(bounds))))
    dev = dg.offsets.device
    ef = torch.empty(hi - lo, dtype=torch.float64, device=dev)
    tot = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    fl = torch.empty(hi - lo, dtype=torch.uint8, device=dev)
    if hi > lo:
        if compute is None:
            D.ef_range(dg, lo, hi, ef, tot, fl, engine=engine)
        else:
            compute(dg, lo, hi, ef, tot, fl)
    if world == 1:
        return ef, tot, fl
    mine = pack_shard(ef, tot, fl, pad_to)
    if dist.get_backend(group) == "nccl":
        gathered = torch.empty(world * mine.numel(), dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(gathered, mine, group=group)  # one NCCL all-gather over NVLink
    else:  # gloo (CPU tests, ranks sharing one GPU): list form through host memory
        mine_h = mine.cpu()
        parts = [torch.empty_like(mine_h) for _ in range(world)]
        dist.all_gather(parts, mine_h, group=group)
        gathered = torch.cat(parts).to(dev)
    return unpack_all(gathered, bounds, pad_to)
