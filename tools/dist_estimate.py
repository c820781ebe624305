"""Per-rank device time of the distributed whole-graph pass, emulated on one
GPU (R-MAT22).  Each part of N runs alone, as one rank of an N-GPU job would:
its rows phase (efg_ef_partial_rows: its node range's neighbour degrees,
S1/S2, Adj+ rows, chain tables, pushes), then -- after every part's rows are in
the shared buffers, which is what the broadcast exchange assembles on each
rank -- its listing phase (efg_ef_partial_list), and the finish.  The two
collectives are not run (one GPU): they are estimated from their bytes at the
measured NVLink figures of B200_PROFILING.md (peer copy 770 GB/s per
direction; 8-rank all-reduce bus bandwidth 725 GB/s).

Usage: python tools/dist_estimate.py [N ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2306_00606_b200 as efg  # noqa: E402
from paper_2306_00606_b200 import device as D  # noqa: E402

g, _ = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
dg = D.DeviceGraph.from_host(g)
n, m2 = g.n, 2 * g.m
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]


def timed(fn):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def single():
    D.ef_range(dg, 0, n, *out)


single()
t1 = min(timed(single) for _ in range(3))
res = {"single_gpu_ms": t1, "parts": {}}
print(f"single-GPU pass {t1:.2f} ms")
PROFILE = "--profile" in sys.argv
for N in [int(x) for x in sys.argv[1:] if x.isdigit()] or [2, 4, 8]:
    bounds = D.part_bounds(dg, N)
    adjp = torch.empty(m2, dtype=torch.int32, device="cuda")
    dplus = torch.empty(n, dtype=torch.int32, device="cuda")
    words = [torch.empty(D.DIST_WORDS * n, dtype=torch.int64, device="cuda") for _ in range(N)]
    wss = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(N)]
    for p in range(N):  # warm-up (and the shared rows every listing part reads)
        D.ef_partial_rows(dg, p, N, bounds, adjp, dplus, words[p], wss[p])
    rows = [min(timed(lambda p=p: D.ef_partial_rows(dg, p, N, bounds, adjp, dplus, words[p], wss[p]))
                for _ in range(3)) for p in range(N)]
    tabs, lst = [], []
    for p in range(N):
        t, u = [], []
        for _ in range(3):
            D.ef_partial_rows(dg, p, N, bounds, adjp, dplus, words[p], wss[p])  # re-clear the part's words
            t.append(timed(lambda p=p: D.ef_partial_tables(dg, p, N, bounds, words[p], wss[p])))
            u.append(timed(lambda p=p: D.ef_partial_list(dg, p, N, bounds, adjp, dplus, words[p], wss[p])))
        tabs.append(min(t))
        lst.append(min(u))
    tw = torch.stack(words).sum(0)
    ts = torch.stack(wss).sum(0)
    fin = min(timed(lambda: D.ef_finish(dg, 0, n, tw, ts, *out)) for _ in range(3))
    full = torch.empty(n, dtype=torch.float64, device="cuda")
    D.ef_range(dg, 0, n, full, torch.empty(n, dtype=torch.int64, device="cuda"),
               torch.empty(n, dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(full, out[0]), "distributed parts differ from the single pass"
    # collectives: rows exchange (each rank receives the other parts' slot ranges + dplus)
    # and the all-reduce of 9n words + n stars terms (ring: 2 (N-1)/N of the bytes)
    xch_bytes = (N - 1) / N * (4 * m2 + 4 * n)
    ar_bytes = 2 * (N - 1) / N * (8 * (D.DIST_WORDS + 1) * n)
    xch_ms = xch_bytes / 770e9 * 1e3
    ar_ms = ar_bytes / 725e9 * 1e3
    # the exchange overlaps the tables phase (asynchronous broadcasts) and the
    # all-reduce of the chain / S1 / S2 words and stars terms the listing; only
    # the triangle words' all-reduce (4 of the 10 per-node words) follows it:
    # per rank rows + max(tables, exchange) + max(listing, early reduce) + late reduce + finish
    ar_early, ar_late = ar_ms * 6 / 10, ar_ms * 4 / 10
    per = [r + max(t, xch_ms) + max(l, ar_early) for r, t, l in zip(rows, tabs, lst)]
    total = max(per) + fin + ar_late
    ideal = t1 / N
    res["parts"][N] = {"rows_ms": rows, "tables_ms": tabs, "list_ms": lst, "finish_ms": fin, "exchange_ms_est": xch_ms,
                       "allreduce_ms_est": ar_ms, "per_rank_ms": total, "ideal_ms": ideal,
                       "ratio_to_ideal": total / ideal, "bitwise_equal": True,
                       "bounds": [int(x) for x in bounds]}
    print(f"N={N}: rows max {max(rows):.2f} ms, tables max {max(tabs):.2f} ms, list max {max(lst):.2f} ms, max part {max(per):.2f} ms "
          f"(min {min(per):.2f}), finish {fin:.2f}, exchange ~{xch_ms:.2f}, all-reduce ~{ar_ms:.2f} "
          f"-> per rank {total:.2f} ms vs ideal {ideal:.2f} ({total / ideal:.2f}x)")
    if PROFILE:  # live per-kernel times of the slowest rows part and part 0's listing
        from paper_2306_00606_b200 import _native
        ctx = _native.context(0)
        pm = int(np.argmax(rows))
        for name, fn in (("rows", lambda: D.ef_partial_rows(dg, pm, N, bounds, adjp, dplus, words[pm], wss[pm])),
                         ("tables", lambda: D.ef_partial_tables(dg, pm, N, bounds, words[pm], wss[pm])),
                         ("list", lambda: D.ef_partial_list(dg, 0, N, bounds, adjp, dplus, words[0], wss[0]))):
            ctx.profile_reset()
            ctx.profile(True)
            fn()
            torch.cuda.synchronize()
            ctx.profile(False)
            rep = ctx.profile_report()
            tot = sum(v["ms"] for v in rep.values())
            print(f"  N={N} {name}: {tot:.2f} ms in kernels; " + ", ".join(
                f"{k}={v['ms']:.3f}" for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])[:12]))
print(json.dumps(res))
