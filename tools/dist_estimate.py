"""Per-part device time of the distributed whole-graph pass on one GPU
(R-MAT22): each part of N runs alone, as one rank of an N-GPU job would
(without the all-reduce).  Usage: python tools/dist_estimate.py [N ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2306_00606_b200 as efg  # noqa: E402
from paper_2306_00606_b200 import device as D  # noqa: E402

g, _ = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
dg = D.DeviceGraph.from_host(g)
n = g.n
words = torch.empty(D.DIST_WORDS * n, dtype=torch.int64, device="cuda")
ws = torch.empty(n, dtype=torch.float64, device="cuda")
out = [torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for N in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
    for _ in range(2):
        D.ef_partial(dg, 0, N, words, ws)
    parts = [min(timed(lambda p=p: D.ef_partial(dg, p, N, words, ws)) for _ in range(3)) for p in range(N)]
    fin = min(timed(lambda: D.ef_finish(dg, 0, n, words, ws, *out)) for _ in range(3))
    print(f"N={N}: part ms max {max(parts):.2f} min {min(parts):.2f}, finish {fin:.2f} ms "
          f"-> per-rank {max(parts) + fin:.2f} ms + all-reduce of {D.DIST_WORDS * 8 * n / 1e6 + 8 * n / 1e6:.0f} MB")
