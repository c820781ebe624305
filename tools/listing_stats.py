"""Listing-work statistics of a config graph (host numpy; graph cached under /tmp): rows per middle class,
useful scan span per row, steps under the per-row unroll rule, and a step-cost model (tools, r02)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import bench
import os
t = time.time()
cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
cache = f"/tmp/hg_{cfg}.npz"
if os.path.exists(cache):
    z = np.load(cache); n, m, off, nbr = int(z["n"]), int(z["m"]), z["off"], z["nbr"]
else:
    n, m, off, nbr, _ = bench.host_graph(cfg)
    np.savez(cache, n=n, m=m, off=off, nbr=nbr)
print("graph", n, m, time.time() - t, flush=True)
deg = np.diff(off).astype(np.int64)
# label: rank in (degree desc, id asc)?  above(dj,j,dv,v) = dj>dv or (dj==dv and j>v): higher degree / higher id ranks above
order = np.lexsort((-np.arange(n), -deg))  # label 0 = top
label = np.empty(n, np.int64); label[order] = np.arange(n)
src = np.repeat(np.arange(n), deg)
lab_s, lab_d = label[src], label[nbr]
plus = lab_d < lab_s  # nbr ranks above src: entry of Adj+(src)
ps, pd = src[plus], lab_d[plus]
dplus = np.bincount(ps, minlength=n)
key = ps.astype(np.int64) * n + pd
key.sort()
pstart = np.concatenate([[0], np.cumsum(dplus)])
# pairs (v middle, u row): u in Adj(v), u below v  -> u = src with v = nbr in Adj+(u)
U_ = src[plus]; V_ = nbr[plus]
span = np.searchsorted(key, U_.astype(np.int64) * n + label[V_]) - pstart[U_]
pu = dplus[U_]
dv = deg[V_]
print("rows", U_.size, "sum span", span.sum(), "sum pu", pu.sum(), flush=True)
for name, sel in [("big dv>256", dv > 256), ("small 32<dv<=256", (dv > 32) & (dv <= 256)), ("warp dv<=32", dv <= 32)]:
    sp = span[sel]; p = pu[sel]
    lim = np.minimum(p, np.maximum(sp + 1, 1))  # entries read before the stop
    Uw = np.where(np.minimum(p, sp + 1) <= 32, 1, np.where(np.minimum(p, sp + 1) <= 64, 2, 4))
    steps = np.ceil(np.minimum(p, sp + 1) / (32 * Uw))
    slots = steps * 32 * Uw
    print(f"{name}: rows {sel.sum():,} span {sp.sum():,} mean {sp.mean():.1f} rows span0 {(sp==0).sum():,} "
          f"<=32 {(sp<=32).sum():,} <=128 {(sp<=128).sum():,}  steps {steps.sum():,.0f} slots {slots.sum():,.0f} "
          f"lane-eff {sp.sum()/max(slots.sum(),1):.3f}")
    h = np.histogram(sp, bins=[0, 1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 1 << 30])
    print("   span hist", list(zip(h[1][:-1].tolist(), h[0].tolist())))
sel = dv > 256
p = pu[sel]; sp = span[sel]
lim_cap = np.minimum(p, label[V_][sel])
print("big rows: pu<=16", (lim_cap <= 16).sum(), "pu<=32", (lim_cap <= 32).sum(), "pu<=8", (lim_cap <= 8).sum(), "total", sel.sum())
sel = (dv > 32) & (dv <= 256)
p = pu[sel]
lim_cap = np.minimum(p, label[V_][sel])
print("small rows: pu<=16", (lim_cap <= 16).sum(), "pu<=32", (lim_cap <= 32).sum(), "pu<=8", (lim_cap <= 8).sum(), "total", sel.sum())
cU = {1: 45.0, 2: 75.0, 4: 135.0}
sel = dv > 256
p = pu[sel]; sp = span[sel]; lab_v = label[V_][sel]; lab_u = label[U_][sel]
need = np.minimum(p, sp + 1)
def cost(U):
    return np.ceil(need / (32 * U)) * cU[U]
c1, c2, c4 = cost(1), cost(2), cost(4)
cap = np.minimum(p, lab_v)
cur = np.where(cap <= 32, c1, np.where(cap <= 64, c2, c4))
best = np.minimum(np.minimum(c1, c2), c4)
print("current", cur.sum() / 1e9, "G  oracle-U", best.sum() / 1e9, "G  all-U4", c4.sum() / 1e9, " all-U2", c2.sum()/1e9, " all-U1", c1.sum()/1e9)
# estimate span by uniform-label fraction
est = p * (lab_v / np.maximum(lab_u, 1))
for f in (1.0, 2.0, 4.0):
    e = np.minimum(cap, est * f)
    u = np.where(e <= 32, c1, np.where(e <= 64, c2, c4))
    print("est x", f, u.sum() / 1e9)
