"""N>1 paths on CPU (gloo, world 2 and 3):

* ef_sharded: the ranks shard the seeds, compute their shard (CPU oracle
  standing in for the GPU engine), exchange with the packed all-gather, and
  must reproduce the single-pass result bitwise;
* ef_distributed: row-partitioned parts write their node range's Adj+ rows,
  exchange_rows (one broadcast per part) must assemble every row on every
  rank, and the one all-reduce of the integer words must be exact."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ef as O
from paper_2306_00606_b200 import distributed as Dist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class HostGraph:
    def __init__(self, offsets, neighbors):
        self.offsets = torch.from_numpy(np.asarray(offsets, np.int64))
        self.neighbors = torch.from_numpy(np.asarray(neighbors, np.int32))
        self.n = self.offsets.numel() - 1


def _oracle_compute(dg, lo, hi, ef, tot, fl):
    e, t, f, _, _ = O.ef_seeds(dg.offsets.numpy(), dg.neighbors.numpy(), seeds=np.arange(lo, hi), threads=1)
    ef.copy_(torch.from_numpy(e))
    tot.copy_(torch.from_numpy(t))
    fl.copy_(torch.from_numpy(f))


def _worker(rank, world, port, offsets, neighbors, bounds, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dg = HostGraph(offsets, neighbors)
        ef, tot, fl = Dist.ef_sharded(dg, compute=_oracle_compute, bounds=bounds)
        np.savez(f"{out_path}.{rank}.npz", ef=ef.numpy(), tot=tot.numpy(), fl=fl.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_matches_single_pass(golden, tmp_path, world):
    case = golden["rmat_12_8_3"]
    off, nb = case.get("offsets"), case.get("neighbors")
    n = case.n
    # uneven contiguous shards (the packed buffer is padded to the largest)
    cuts = np.linspace(0, n, world + 1).astype(np.int64)
    cuts[1] = max(1, cuts[1] // 3)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, off, nb, cuts, str(tmp_path / "out")))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    want_ef, want_tot, want_fl, _, _ = O.ef_seeds(off, nb, threads=2)
    for r in range(world):
        z = np.load(tmp_path / f"out.{r}.npz")
        assert np.array_equal(z["ef"], want_ef)
        assert np.array_equal(z["tot"], want_tot)
        assert np.array_equal(z["fl"], want_fl)


def test_pack_unpack_roundtrip():
    bounds = np.array([0, 3, 3, 7], np.int64)
    pad = 4
    parts = []
    for r in range(3):
        L = int(bounds[r + 1] - bounds[r])
        ef = torch.arange(L, dtype=torch.float64) + 10 * r
        tot = torch.arange(L, dtype=torch.int64) * 7 + r
        fl = torch.full((L,), r, dtype=torch.uint8)
        parts.append(Dist.pack_shard(ef, tot, fl, pad))
    ef, tot, fl = Dist.unpack_all(torch.cat(parts), bounds, pad)
    assert ef.tolist() == [0, 1, 2, 20, 21, 22, 23]
    assert tot.tolist() == [0, 7, 14, 2, 9, 16, 23]
    assert fl.tolist() == [0, 0, 0, 2, 2, 2, 2]


# --- ef_distributed: row-partitioned parts, row exchange, one all-reduce ----
def _expected_rows(dg):
    m2 = dg.neighbors.numel()
    adjp = (np.arange(m2, dtype=np.int64) * 7 + 3) % (2**31 - 1)
    dplus = np.arange(dg.n, dtype=np.int64) * 3 + 1
    return adjp.astype(np.int32), dplus.astype(np.int32)


def _split_rows(T, W):
    """Stand-in for efg_ef_partial_rows: part p writes its node range's rows
    (a known pattern) into adjp / dplus, an arbitrary (seeded) integer split of
    every node's T into word 0 (negative pieces exercise wrap-free int64 sums)
    and W of its node range (disjoint supports)."""
    def rows(dg, part, nparts, bounds, adjp, dplus, words, ws):
        n = dg.n
        lo, hi = int(bounds[part]), int(bounds[part + 1])
        ea, ed = _expected_rows(dg)
        so, se = int(dg.offsets[lo]), int(dg.offsets[hi])
        adjp[so:se] = torch.from_numpy(ea[so:se])
        dplus[lo:hi] = torch.from_numpy(ed[lo:hi])
        rng = np.random.default_rng(1234)  # same draws on every rank
        pieces = rng.integers(-2**40, 2**40, size=(nparts, n))
        pieces[-1] = T - pieces[:-1].sum(axis=0)
        w = np.zeros(words.numel(), np.int64)
        w[:n] = pieces[part]
        words.copy_(torch.from_numpy(w))
        s = np.where((np.arange(n) >= lo) & (np.arange(n) < hi), W, 0.0)
        ws.copy_(torch.from_numpy(s))
    return rows


def _check_listing(dg, part, nparts, bounds, adjp, dplus, words, ws):
    """Stand-in for efg_ef_partial_list: the exchanged rows must be complete."""
    ea, ed = _expected_rows(dg)
    assert np.array_equal(adjp.numpy(), ea), "Adj+ row exchange incomplete"
    assert np.array_equal(dplus.numpy(), ed), "|Adj+| exchange incomplete"


def _finish(dg, words, ws, ef, tot, fl):
    n = dg.n
    T = words[:n].numpy()
    W = ws.numpy()
    e = np.where(T > 0, np.log(np.maximum(T, 1)) - W / np.maximum(T, 1), 0.0)
    ef.copy_(torch.from_numpy(e))
    tot.copy_(torch.from_numpy(T))
    fl.zero_()


def _dist_worker(rank, world, port, offsets, neighbors, T, W, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dg = HostGraph(offsets, neighbors)
        ef, tot, fl = Dist.ef_distributed(dg, rows=_split_rows(T, W), listing=_check_listing, finish=_finish)
        np.savez(f"{out_path}.{rank}.npz", ef=ef.numpy(), tot=tot.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_allreduce_is_exact(golden, tmp_path, world):
    case = golden["rmat_12_8_3"]
    off, nb = case.get("offsets"), case.get("neighbors")
    _, _, _, T, W = O.ef_seeds(off, nb, threads=2)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, off, nb, T, W, str(tmp_path / "d")))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    want = np.where(T > 0, np.log(np.maximum(T, 1)) - W / np.maximum(T, 1), 0.0)
    for r in range(world):
        z = np.load(tmp_path / f"d.{r}.npz")
        assert np.array_equal(z["tot"], T)
        assert np.array_equal(z["ef"], want)
