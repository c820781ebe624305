"""Benchmark: Expected Force of every seed of the R-MAT scale-22 graph (44M edges).

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  N>1 is launched by torchrun (one process per GPU, NCCL).

A "step" is one full-graph EF pass (every seed: ef, cluster_total, flags) over
the device-resident CSR of BASELINE.json's configs[2] graph (R-MAT scale 22,
avg degree 21, seed 0: n=2,181,017, m=44,040,192; edge set bit-identical to
the reference generator, verified by sha256 fingerprint).  N>1: each rank
runs one part of the whole-graph pass (its nodes' chain tables and pushes,
its share of the triangle-listing work units) and one NCCL all-reduce sums
the per-node integer words; every rank then finishes all seeds (direct
engine: seeds sharded by balanced work prefix, K2, and one all-gather).
Per-step work is the whole graph for any N ("strong" scaling of a fixed job).

value       = seeds/s over the timed steps (inputs resident in HBM), max over ranks
e2e         = seeds/s through the public API ef_cluster_centric(g) from pinned
              host arrays: H2D of the CSR + compute + D2H of ef/cluster_total/flags
roofline    = the dominant kernel (live CUDA-event timing of each kernel in a
              profiled step) against measured HBM bandwidth (MEASURED_PEAKS.json)
cpu_baseline= the C oracle port (oracle/, the reference's per-seed algorithm)
              on a stratified seed sample, work-extrapolated to the full graph
--impl reference: the same CPU port with every host thread = the reference arm.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRICS = {
    "rmat22": "EF seeds/sec, full-graph Expected Force (R-MAT scale-22, 44M edges)",
    "er1m": "EF seeds/sec, full-graph Expected Force (Erdos-Renyi n=1M, avg degree 16)",
    "ws4m": "EF seeds/sec, full-graph Expected Force (Watts-Strogatz n=4M, k=20, p=0.05)",
    "chunglu": "EF seeds/sec, full-graph Expected Force (Chung-Lu gamma=2.1, n=2^20)",
    "ba2000": "EF seeds/sec, full-graph Expected Force (Barabasi-Albert n=2000, m=3)",
}

CONFIGS = {
    # name: (description, builder kwargs)
    "rmat22": "R-MAT scale-22 avg-degree 21 seed 0 (reference generate_rmat), ~44M undirected edges",
    "er1m": "Erdos-Renyi G(n,m) n=1M avg degree 16 (SURVEY 8(d) recipe)",
    "ws4m": "Watts-Strogatz n=4M k=20 p=0.05 (SURVEY 8(d) recipe)",
    "chunglu": "Chung-Lu gamma=2.1 n=2^20 W=2e5 (SURVEY 8(d) recipe)",
    "ba2000": "Barabasi-Albert n=2000 m=3 seed 0",
}
RMAT22_SHA256 = "2c4b690446b61f1441357f8f4b08d437b12f7885f3375516d3c984b96c831891"  # reference fingerprint


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def raw_edges(config):
    from paper_2306_00606_b200 import generators as gen

    if config == "rmat22":
        e, _ = gen.rmat_edges(22, 21, seed=0)
        return e
    if config == "er1m":
        return gen.er_edges_gnm()
    if config == "ws4m":
        return gen.ws_edges()
    if config == "chunglu":
        return gen.chung_lu_edges()
    if config == "ba2000":
        return gen.ba_edges()
    raise ValueError(config)


def fingerprint(g):
    h = hashlib.sha256()
    h.update(np.int64([g.n, g.m]).tobytes())
    for a in (g.offsets, g.neighbors, g.orig_ids):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def kernel_bytes_model(offsets, neighbors):
    """Algorithmic bytes per launch of the triangle-listing kernels.

    A whole-graph pass lists each triangle at its middle vertex v
    (csrc/ef_factor.cu k_mid_big for dv > 256, k_mid_small for 32 < dv <= 256,
    k_mid_warp for dv <= 32):
    every lower-ranked neighbour u of v is a row, and the label-sorted Adj+(u)
    is read up to v itself (pos_u(v) + 1 labels of 4 B).  Per examined slot of
    v's row 8 B (neighbour id + degree), per kept row 12 B (|Adj+(u)|, start),
    per entry of Adj+(v) 8 B (label + node id), per seed 40 B.  The hit
    gathers (12 B per triangle) are not counted: a lower bound.  Computed on
    the GPU with torch (one sort of the oriented edges)."""
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    off = torch.as_tensor(np.asarray(offsets, dtype=np.int64), device=dev)
    nb = torch.as_tensor(np.asarray(neighbors, dtype=np.int64), device=dev)
    n = off.numel() - 1
    deg = off[1:] - off[:-1]
    src = torch.repeat_interleave(torch.arange(n, device=dev), deg)
    dn, ds = deg[nb], deg[src]
    up = (dn > ds) | ((dn == ds) & (nb > src))                 # nb ranks above src: nb in Adj+(src)
    # rank label: position in descending (degree, id) order
    order = torch.argsort(deg * (n + 1) + torch.arange(n, device=dev), descending=True)
    label = torch.empty(n, dtype=torch.int64, device=dev)
    label[order] = torch.arange(n, device=dev)
    u, v = src[up], nb[up]
    pu = torch.bincount(u, minlength=n)
    key = u * n + label[v]
    srt = torch.argsort(key)
    start = torch.cumsum(pu, 0) - pu
    pos = torch.empty_like(srt)
    pos[srt] = torch.arange(srt.numel(), device=dev) - start[u[srt]]
    keep = pu[u] >= 2
    probes_v = torch.zeros(n, dtype=torch.int64, device=dev).index_add_(0, v[keep], pos[keep] + 1)
    rows_v = torch.bincount(v[keep], minlength=n)
    pv = torch.bincount(u, minlength=n)  # |Adj+| per node
    out = {}
    for name, lo, hi in (("k_mid_big", 256, 1 << 40), ("k_mid_small", 32, 256), ("k_mid_warp", -1, 32)):
        msk = (deg > lo) & (deg <= hi)
        probes = int(probes_v[msk].sum())
        rows = int(rows_v[msk].sum())
        slots = int(deg[msk].sum())
        seeds = int(msk.sum())
        ent = int(pv[msk].sum())
        out[name] = {"probes": probes, "rows": rows, "slots": slots, "seeds": seeds,
                     "bytes": 4 * probes + 8 * slots + 12 * rows + 8 * ent + 40 * seeds}
    return out


def algorithmic_bytes_per_seed(offsets, neighbors):
    """B(v) = 16 + 8 dv + sum_{i in Adj v} (16 + 8 di) + 17 (int64 offsets,
    int32 ids and degrees, f64+i64+u8 outputs)."""
    deg = np.diff(offsets)
    s1 = np.add.reduceat(deg[neighbors], offsets[:-1]) if neighbors.size else np.zeros_like(deg)
    return 16 + 8 * deg + 16 * deg + 8 * s1 + 17


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def stratified_sample(offsets, neighbors, rng_seed=0, budget=3.0e9):
    """Seeds for the CPU timing: 200/100/20/2 per degree bucket (<=32, 33-1024,
    1025-16384, >16384) within a total work budget, and the
    per-bucket work totals for the ratio extrapolation."""
    deg = np.diff(offsets)
    s1 = np.add.reduceat(deg[neighbors], offsets[:-1])
    work = deg * (deg - 1) // 2 + s1            # per-seed visits of the reference walk
    rng = np.random.default_rng(rng_seed)
    buckets = [(0, 32, 200), (33, 1024, 100), (1025, 16384, 20), (16385, 1 << 62, 2)]
    picks = []
    for lo, hi, k in buckets:
        ids = np.flatnonzero((deg >= lo) & (deg <= hi))
        if ids.size == 0:
            continue
        sel = rng.choice(ids, size=min(k, ids.size), replace=False)
        sel = sel[np.argsort(work[sel])]
        # keep within budget: drop the heaviest picks of the bucket if needed
        while sel.size > 1 and work[sel].sum() > budget / len(buckets):
            sel = sel[:-1]
        picks.append((ids, sel))
    return work, picks


def cpu_port_rate(offsets, neighbors, threads, rng_seed=0, budget=3.0e9):
    """Time the oracle port on the stratified sample; extrapolate the full-graph
    time by per-bucket work ratio.  Returns (seconds_full_graph_est, sample_desc, sample_seconds)."""
    from oracle import ef as O

    work, picks = stratified_sample(offsets, neighbors, rng_seed, budget)
    est = 0.0
    total_sample_s = 0.0
    desc = []
    for ids, sel in picks:
        t0 = time.perf_counter()
        O.ef_seeds(offsets, neighbors, seeds=sel, threads=threads)
        dt = time.perf_counter() - t0
        total_sample_s += dt
        w_sel = float(work[sel].sum())
        est += dt * float(work[ids].sum()) / max(w_sel, 1.0)
        desc.append(f"{sel.size}/{ids.size}")
    return est, "stratified seeds per degree bucket " + ",".join(desc), total_sample_s


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (oracle port,
    every host thread) on the same workload; rank 0 only."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import graph as OG

    t0 = time.perf_counter()
    edges = raw_edges(args.config)
    n, m, offsets, neighbors, orig = OG.build_csr(edges)
    setup_s = time.perf_counter() - t0
    threads = len(os.sched_getaffinity(0))
    times, est = [], None
    # per-step sample work scaled so the whole K+W run stays within a few
    # minutes; the default 20+3 steps measured 11.1 s of sampled CPU work each
    # on a 16-thread host (4.8 min run; one hub seed of degree > 16384 is the
    # floor of every step)
    budget = 3.0e9 * min(1.0, 3.0 / max(1, args.warmup + args.steps))
    for step in range(args.warmup + args.steps):
        t_est, sample, sample_s = cpu_port_rate(offsets, neighbors, threads, rng_seed=step, budget=budget)
        if step >= args.warmup:
            times.append(t_est)
            est = (sample, sample_s)
    t_full = float(np.median(times))
    value = n / t_full
    line = {
        "metric": METRICS[args.config],
        "value": value, "unit": "seeds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+int64", "data": "synthetic", "impl": "reference",
        "config": {"workload": CONFIGS[args.config], "n": n, "m": m, "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "seeds/s", "cores": threads, "kind": "port",
                         "sample": f"{est[0]}; {est[1]:.1f} s of sampled CPU work per step, extrapolated by work ratio"},
        "e2e": {"value": value, "unit": "seeds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup_s,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmat22", choices=sorted(CONFIGS))
    ap.add_argument("--engine", default="factorized", choices=["factorized", "direct"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2306_00606_b200 as efg
    from paper_2306_00606_b200 import _native
    from paper_2306_00606_b200 import device as D
    from paper_2306_00606_b200.distributed import ef_distributed, ef_sharded

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    _native.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    # ---- graph: rank 0 builds (host generator + device K1), broadcast to the others
    t0 = time.perf_counter()
    if rank == 0:
        if args.config == "rmat22":  # device sampler, bit-identical to the reference generator
            g, _ = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
        else:
            g = efg.build_graph(raw_edges(args.config))
        meta = [g.n, g.m]
    else:
        meta = [0, 0]
    if world > 1:
        mt = torch.tensor(meta, dtype=torch.int64, device=dev)
        dist.broadcast(mt, 0)
        meta = mt.tolist()
    n, m = int(meta[0]), int(meta[1])
    if rank == 0:
        dg = D.DeviceGraph.from_host(g, device=local)
    else:
        dg = D.DeviceGraph(torch.empty(n + 1, dtype=torch.int64, device=dev),
                           torch.empty(2 * m, dtype=torch.int32, device=dev), n)
    if world > 1:
        dist.broadcast(dg.offsets, 0)
        dist.broadcast(dg.neighbors, 0)
        if rank != 0:
            # host copy for the e2e leg (pinned)
            off_h = _native.pinned_empty(n + 1, np.int64)
            nb_h = _native.pinned_empty(2 * m, np.int32)
            off_h[:] = dg.offsets.cpu().numpy()
            nb_h[:] = dg.neighbors.cpu().numpy()
            from paper_2306_00606_b200.graph import Graph
            g = Graph(n, m, off_h, nb_h, None)
    setup_s = time.perf_counter() - t0
    sha_ok = None
    if rank == 0 and args.config == "rmat22":
        sha_ok = fingerprint(g) == RMAT22_SHA256

    # ---- shards (graph-level plan, identical on all ranks)
    bounds = D.shard_bounds(dg, world, args.engine) if world > 1 else np.array([0, n], np.int64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        if world > 1 and args.engine == "factorized":
            return ef_distributed(dg)  # parts of the whole-graph pass + one all-reduce of integer words
        return ef_sharded(dg, engine=args.engine, bounds=bounds)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps, CUDA events on the stream
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
            out = step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n / (ms_per_step / 1e3)

    # ---- profiled step: live per-kernel event timing + launch count
    ctx = _native.context(local)
    ctx.profile_reset()
    ctx.profile(True)
    torch.cuda.synchronize()
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    pe = torch.empty(hi - lo, dtype=torch.float64, device=dev)
    pt = torch.empty(hi - lo, dtype=torch.int64, device=dev)
    pf = torch.empty(hi - lo, dtype=torch.uint8, device=dev)
    st = D.ef_range(dg, lo, hi, pe, pt, pf, engine=args.engine, stats=True)
    ctx.profile(False)
    kernels = ctx.profile_report()

    # ---- end to end through the public API from pinned host buffers
    e2e = None
    if world == 1:
        efg.ef_cluster_centric(g, engine=args.engine)
        times = []
        for _ in range(args.e2e_steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = efg.ef_cluster_centric(g, engine=args.engine)
            times.append(time.perf_counter() - t0)
        t_e2e = float(np.median(times))
        e2e = {"value": n / t_e2e, "unit": "seeds/s", "h2d_bytes_per_step": int(r.stats["h2d_bytes"]),
               "d2h_bytes_per_step": int(r.stats["d2h_bytes"]), "ms_per_step": t_e2e * 1e3,
               "ms_h2d": r.stats["ms_h2d"], "ms_d2h": r.stats["ms_d2h"], "ms_device_events": r.stats["ms_device"],
               "ms_prepare": r.stats["ms_prepare"], "ms_enumerate": r.stats["ms_enumerate"],
               "ms_wall_all": [round(t * 1e3, 2) for t in times]}
        # parity spot check of the timed output against the e2e output
        assert np.array_equal(out[0].cpu().numpy(), r.ef)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (live CUDA-event duration of the profiled step)
    peak, peak_kind = measured_peaks()
    dom = max(kernels.items(), key=lambda kv: kv[1]["ms"]) if kernels else (None, {"ms": 0.0, "launches": 1})
    offs, nbrs = np.asarray(g.offsets), np.asarray(g.neighbors)
    b_alg = int(algorithmic_bytes_per_seed(offs, nbrs).sum())
    model = kernel_bytes_model(offs, nbrs) if args.engine == "factorized" else {}
    dom_ms = dom[1]["ms"] / max(dom[1]["launches"], 1)
    dom_base = dom[0].split("<")[0].strip("() ")  # live names carry template arguments (k_mid_block<false>)
    dom_bytes = model.get(dom_base, {}).get("bytes")
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(dom[0], tj.get(dom_base))
        except (OSError, ValueError):
            traffic = None
    roofline = {
        "bound": "hbm", "kernel": dom[0], "unit": "GB/s", "peak": peak, "peak_kind": peak_kind,
        "achieved": dom_bytes / (dom_ms / 1e3) / 1e9 if dom_bytes else None,
        "frac": dom_bytes / (dom_ms / 1e3) / 1e9 / peak if dom_bytes else None,
        "traffic": traffic, "kernel_ms": dom_ms, "kernel_bytes_alg": dom_bytes,
        "kernel_share_of_step": dom[1]["ms"] / sum(v["ms"] for v in kernels.values()) if kernels else None,
        "pass_achieved": b_alg / (ms_per_step / 1e3) / 1e9,
        "pass_frac": b_alg / (ms_per_step / 1e3) / 1e9 / peak,
        "bytes_alg_pass": b_alg,
        "note": "achieved = kernel_bytes_alg (listing model: 4 B/label read + 8 B/slot + 12 B/row + 8 B/Adj+(v) "
                "entry + 40 B/seed, DESIGN.md) / live event time; "
                "pass_* = SURVEY 8(d) B_alg of the whole graph / step time; traffic = ncu dram bytes per launch "
                "(profiles/dram_traffic.json)",
    }
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = len(os.sched_getaffinity(0))
        t_full, sample, sample_s = cpu_port_rate(np.asarray(g.offsets), np.asarray(g.neighbors), threads)
        cpu = {"value": n / t_full, "unit": "seeds/s", "cores": threads, "kind": "port",
               "sample": f"{sample}; {sample_s:.1f} s of CPU work, extrapolated by work ratio to {t_full:.0f} s"}
    line = {
        "metric": METRICS[args.config],
        "value": value, "unit": "seeds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+int64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config], "n": n, "m": m, "engine": args.engine,
                   "parallelism": (f"whole-graph pass in {world} parts + 1 all-reduce" if world > 1 and args.engine == "factorized"
                                   else f"seed-sharded x{world}"),
                   "l2": "flushed between timed steps (256 MB write)",
                   "graph_sha256_matches_reference": sha_ok},
        "e2e": e2e,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "gpu_launches": int(st["launches"]) * args.steps,
        "kernels_ms": {k: round(v["ms"], 4) for k, v in sorted(kernels.items(), key=lambda kv: -kv[1]["ms"])},
        "listing_model": model,
        "clocks": clocks.summary(),
        "setup_s": setup_s,
        "stats": {k: v for k, v in st.items() if k not in ("T", "W")},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
