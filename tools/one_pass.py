"""One device-resident EF pass over R-MAT22 (profiling target: ncu -k <kernel> python tools/one_pass.py)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2306_00606_b200 as efg  # noqa: E402
from paper_2306_00606_b200 import device as D  # noqa: E402

g, _ = efg.generate_rmat(efg.RmatParams(scale=int(sys.argv[1]) if len(sys.argv) > 1 else 22, avg_degree=21, seed=0))
dg = D.DeviceGraph.from_host(g)
out = [torch.empty(g.n, dtype=t, device="cuda") for t in (torch.float64, torch.int64, torch.uint8)]
for _ in range(2):
    D.ef_range(dg, 0, g.n, *out)
torch.cuda.synchronize()
print("ok", g.n, g.m)
