"""Timeline of one end-to-end call (host CSR -> EF -> host) on R-MAT22: every
launch and copy with its start relative to the call's first record, plus idle
gaps on the compute stream (profiling adds an event pair per launch)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2306_00606_b200 as efg  # noqa: E402
from paper_2306_00606_b200 import _native  # noqa: E402

g, _ = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
keep = efg.ef_cluster_centric(g)
keep = (keep, efg.ef_cluster_centric(g))
ctx = _native.context(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(2):
    flush.fill_(1)
    torch.cuda.synchronize()
    ctx.profile_reset()
    ctx.profile(True)
    t0 = time.perf_counter()
    r = efg.ef_cluster_centric(g)
    t1 = time.perf_counter()
    ctx.profile(False)
    tl = ctx.profile_timeline()
    print(f"call {it}: wall {1e3 * (t1 - t0):.2f} ms, stats device {r.stats['ms_device']:.2f} prepare {r.stats['ms_prepare']:.2f}")
end = 0.0
for name, st, ms in tl:
    gap = st - end if not name.startswith(("h2d", "d2h")) else 0.0
    flag = f"  <-- gap {gap:.3f}" if gap > 0.05 else ""
    print(f"{st:8.3f} {ms:8.3f}  {name}{flag}")
    if not name.startswith(("h2d",)):
        end = max(end, st + ms)
