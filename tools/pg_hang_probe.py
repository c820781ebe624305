import faulthandler, sys, time, os
faulthandler.enable()
sys.path.insert(0, ".")
import numpy as np
import paper_2306_00606_b200 as efg
from paper_2306_00606_b200.graph import Graph
g, _ = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
gp = Graph(g.n, g.m, np.array(g.offsets, copy=True), np.array(g.neighbors, copy=True), None)
for i in range(6):
    t0 = time.perf_counter(); r = efg.ef_cluster_centric(gp); print(i, "pageable ok", round((time.perf_counter()-t0)*1e3, 2), flush=True)
