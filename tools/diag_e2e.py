import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2306_00606_b200 as efg
from paper_2306_00606_b200 import device as D, generators as gen
g = efg.build_graph(gen.rmat_edges(22, 21, seed=0)[0])
dg = D.DeviceGraph.from_host(g)
n = g.n
out = [torch.empty(n, dtype=t, device='cuda') for t in (torch.float64, torch.int64, torch.uint8)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for it in range(3):
    flush.fill_(1); torch.cuda.synchronize()
    st = D.ef_range(dg, 0, n, *out, stats=True)
    print('device-path stats', round(st['ms_device'],2), round(st['ms_prepare'],2), round(st['ms_enumerate'],2))
    flush.fill_(1); torch.cuda.synchronize()
    t0=time.perf_counter(); r = efg.ef_cluster_centric(g); t1=time.perf_counter()
    print('e2e', round((t1-t0)*1e3,2), 'dev', round(r.stats['ms_device'],2), round(r.stats['ms_prepare'],2), round(r.stats['ms_enumerate'],2), round(r.stats['ms_h2d'],2))
    flush.fill_(1); torch.cuda.synchronize()
    ev0=torch.cuda.Event(enable_timing=True); ev1=torch.cuda.Event(enable_timing=True)
    ev0.record(); D.ef_range(dg, 0, n, *out); ev1.record(); torch.cuda.synchronize()
    print('device-path events', round(ev0.elapsed_time(ev1),2))
