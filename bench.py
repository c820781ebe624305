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

`--gpus N` without a torchrun environment re-executes itself under
torch.distributed.run (N local ranks, 127.0.0.1).  Ranks that outnumber the
visible GPUs share them and use gloo host collectives (a smoke mode only).

value        = seeds/s over the timed steps (inputs resident in HBM), max over ranks
e2e          = seeds/s through the public API (ef_cluster_centric(g); N > 1:
               distributed.ef_cluster_centric_distributed) from the repo Graph's
               pinned host arrays: H2D of the CSR + compute + D2H of
               ef/cluster_total/flags; e2e_pageable: the same from ordinary
               numpy arrays (what the reference's Graph holds)
roofline     = the dominant kernel (live CUDA-event timing of each kernel in a
               profiled step) against measured HBM bandwidth (MEASURED_PEAKS.json)
cpu_baseline = the UNMODIFIED reference (baseline/_ref): its per-middle loop
               _chunk_histograms on a uniform draw of 2,000 middles, all host
               threads (BASELINE.md 3 "per-seed rate"); --cpu-port adds the C
               port of the reference walk (oracle/) as an extra line
--impl reference: the unmodified reference on the host cores = the reference arm.
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
SAMPLED = ("rmat22", "chunglu")  # full reference runs take hours: timed on seed samples
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
    return fingerprint_arrays(g.n, g.m, g.offsets, g.neighbors, g.orig_ids)


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
        if os.environ.get("EFG_BENCH_CLOCKS") == "off":  # diagnostics only
            return self
        fields = os.environ.get("EFG_BENCH_CLOCK_FIELDS", self.FIELDS)
        period = os.environ.get("EFG_BENCH_CLOCK_MS", "200")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", period], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_live(self, timeout=3.0):
        """Block until nvidia-smi has reported once (its start-up takes ~0.1-0.3 s)."""
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)
        self.mark = len(self.lines)

    def ensure_sample(self, step, timeout=3.0):
        """A timed region shorter than the 200 ms sampling period may see no sample: keep
        running the same step (untimed, the numbers are already taken) until one arrives."""
        import torch

        t0 = time.perf_counter()
        while self.proc and len(self.lines) <= getattr(self, "mark", 0) and time.perf_counter() - t0 < timeout:
            step()
            torch.cuda.synchronize()

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
        for ln in self.lines[getattr(self, "mark", 0):] or self.lines:  # the samples of the timed steps
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


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
BUCKETS = [(0, 32, 200), (33, 1024, 100), (1025, 16384, 20), (16385, 1 << 62, 2)]


def host_graph(config):
    """(n, m, offsets, neighbors, orig_ids) of the config graph built on the HOST
    (generators.py restatements + oracle.graph.build_csr, the numpy restatement
    of build_graph pinned bit-exact by tests) -- the reference arm's input, so
    that no kernel of ours touches the reference's path."""
    from oracle import graph as OG

    return OG.build_csr(raw_edges(config))


def load_reference():
    """The UNMODIFIED reference package from baseline/_ref (scripts/install_reference.sh)."""
    if not os.path.isdir(os.path.join(REF_DIR, "efgraph")):
        raise RuntimeError("baseline/_ref is missing: run scripts/install_reference.sh")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import efgraph
    import efgraph.expected_force as RE
    import efgraph.graph as RG

    return efgraph, RE, RG


class RefGraph:
    """The reference's Graph over given CSR arrays, plus what its EF driver
    precomputes once per call (expected_force.py:155-157): deg, key span and
    the undirected edge codes (timed: the one-off setup)."""

    def __init__(self, n, m, offsets, neighbors, orig_ids):
        _, RE, RG = load_reference()
        self.RE = RE
        self.g = RG.Graph(n=n, m=m, offsets=offsets, neighbors=neighbors, orig_ids=orig_ids, relabeling={})
        t0 = time.perf_counter()
        self.deg = self.g.degrees()
        self.span = RE._key_span(self.deg)
        self.codes = RE._und_edge_codes(self.g)
        self.setup_s = time.perf_counter() - t0

    def middles(self, seeds, threads):
        """The reference's per-middle loop `_chunk_histograms(g, deg, codes, span,
        v, v + 1)` (expected_force.py:222) over the sampled middles, mapped on a
        ThreadPoolExecutor of `threads` workers exactly as ef_cluster_centric
        maps its chunks (:160-167).  Returns wall seconds."""
        from concurrent.futures import ThreadPoolExecutor

        RE, g = self.RE, self.g
        work = lambda v: RE._chunk_histograms(g, self.deg, self.codes, self.span, int(v), int(v) + 1)  # noqa: E731
        t0 = time.perf_counter()
        if threads == 1:
            for v in seeds:
                work(v)
        else:
            with ThreadPoolExecutor(max_workers=threads) as pool:
                list(pool.map(work, seeds))
        return time.perf_counter() - t0

    def full(self, threads):
        """The reference's full-graph ef_cluster_centric(g, workers=threads)."""
        t0 = time.perf_counter()
        r = self.RE.ef_cluster_centric(self.g, workers=threads)
        return time.perf_counter() - t0, r


def uniform_sample(n, size, rng_seed):
    rng = np.random.default_rng(rng_seed)
    return np.sort(rng.choice(n, size=min(size, n), replace=False))


def ref_uniform_rate(rg, threads, size=2000, rng_seed=0):
    """Per-seed rate of the reference's per-middle loop on a uniform sample
    (2,000 seeds of default_rng(0) in the run of record)."""
    seeds = uniform_sample(rg.g.n, size, rng_seed)
    dt = rg.middles(seeds, threads)
    return seeds.size / dt, dt, seeds.size


def ref_stratified(rg, threads, rng_seed=0):
    """Work-weighted extrapolation of the reference's per-middle loop over the
    whole graph: 200/100/20/2 uniformly drawn middles per degree bucket
    (BASELINE.md 3), the whole draw timed (no heavy seed dropped); full time =
    sum over buckets of (bucket pairs / sampled pairs) x sampled seconds."""
    deg = np.asarray(rg.deg)
    c2 = deg * (deg - 1) // 2
    rng = np.random.default_rng(rng_seed)
    est, parts = 0.0, []
    for lo, hi, k in BUCKETS:
        ids = np.flatnonzero((deg >= lo) & (deg <= hi))
        if ids.size == 0:
            continue
        sel = rng.choice(ids, size=min(k, ids.size), replace=False)
        dt = rg.middles(np.sort(sel), threads)
        est += dt * float(c2[ids].sum()) / max(float(c2[sel].sum()), 1.0)
        parts.append({"bucket": f"{lo}-{hi if hi < 1 << 40 else 'max'}", "sampled": int(sel.size),
                      "of": int(ids.size), "seconds": round(dt, 3), "pairs": int(c2[sel].sum())})
    return est, parts


def cpu_port_rate(offsets, neighbors, threads, rng_seed=0):
    """The C port of the reference's per-seed walk (oracle/ef_oracle.c, vertex
    formulation: 3x the visits of the cluster-centric loop) on the stratified
    draw (all drawn seeds timed, none dropped; single-seed scheduling so every
    thread has work); extrapolated by per-bucket work ratio.  An extra,
    labelled figure beside the reference's own."""
    from oracle import ef as O

    deg = np.diff(offsets)
    s1 = np.add.reduceat(deg[neighbors], offsets[:-1])
    work = deg * (deg - 1) // 2 + s1
    rng = np.random.default_rng(rng_seed)
    est, total_s, desc = 0.0, 0.0, []
    for lo, hi, k in BUCKETS:
        ids = np.flatnonzero((deg >= lo) & (deg <= hi))
        if ids.size == 0:
            continue
        sel = rng.choice(ids, size=min(k, ids.size), replace=False)
        t0 = time.perf_counter()
        if sel.size < threads and deg[sel].max() > 16384:  # a few hubs: split each hub's walk over the threads
            for s in sel:
                O.ef_seed_threads(offsets, neighbors, int(s), threads=threads)
        else:
            O.ef_seeds(offsets, neighbors, seeds=sel, threads=threads)
        dt = time.perf_counter() - t0
        total_s += dt
        est += dt * float(work[ids].sum()) / max(float(work[sel].sum()), 1.0)
        desc.append(f"{sel.size}/{ids.size}")
    return est, "stratified seeds per degree bucket " + ",".join(desc), total_s


def run_reference(args):
    """--impl reference: the UNMODIFIED reference (baseline/_ref) on the host
    cores, rank 0 only.  Sampled configs (R-MAT22, Chung-Lu): each step times
    the reference's per-middle loop on a fresh uniform draw of middles (the
    per-seed rate of BASELINE.md 3); full-graph configs (BA, ER-1M, WS-4M):
    each step is one ef_cluster_centric(g, workers=cores)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    try:
        load_reference()
    except Exception as exc:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"{type(exc).__name__}: {exc}"}), flush=True)
        return
    t0 = time.perf_counter()
    n, m, offsets, neighbors, orig = host_graph(args.config)
    sha = fingerprint_arrays(n, m, offsets, neighbors, orig)
    rg = RefGraph(n, m, offsets, neighbors, orig)
    setup_s = time.perf_counter() - t0
    threads = len(os.sched_getaffinity(0))
    sampled = args.config in SAMPLED
    times = []
    for step in range(args.warmup + args.steps):
        if sampled:  # every step times BASELINE.md 3's draw (default_rng(0)): bounded, comparable steps
            rate, dt, k = ref_uniform_rate(rg, threads, size=args.ref_sample, rng_seed=0)
            ms = 1e3 * n / rate
        else:
            dt, _ = rg.full(threads)
            ms = dt * 1e3
        if step >= args.warmup:
            times.append(ms)
    ms_step = float(np.median(times))
    value = n / (ms_step / 1e3)
    if sampled:
        sample = (f"uniform draw of {args.ref_sample} middles (default_rng(0), BASELINE.md 3) timed every step, reference "
                  f"_chunk_histograms(g, deg, codes, span, v, v+1) on a {threads}-worker ThreadPoolExecutor; "
                  f"per-seed rate (ms_per_step = n / rate: the uniform extrapolation, which misses the hubs and so "
                  f"overstates the reference's full-graph speed); merge/entropy pass not included")
    else:
        sample = f"full graph: reference ef_cluster_centric(g, workers={threads})"
    line = {
        "metric": METRICS[args.config],
        "value": value, "unit": "seeds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+int64", "data": "synthetic", "impl": "reference",
        "config": {"workload": CONFIGS[args.config], "n": n, "m": m, "parallelism": f"{threads} host threads",
                   "graph_sha256": sha},
        "cpu_baseline": {"value": value, "unit": "seeds/s", "cores": threads, "kind": "reference",
                         "sample": sample, "reference": "efgraph 0.1.0 (baseline/_ref, unmodified)"},
        "e2e": {"value": value, "unit": "seeds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup_s, "ref_setup_s": rg.setup_s,
        "cpu": {"os_cpu_count": os.cpu_count(), "affinity": threads},
    }
    if args.ref_stratified and sampled:
        est, parts = ref_stratified(rg, threads)
        line["stratified_extrapolation"] = {"seconds_full_graph": est, "seeds_per_s": n / est, "buckets": parts,
                                            "label": "extrapolated (work-weighted by C(d,2) per bucket)"}
    print(json.dumps(line), flush=True)


def fingerprint_arrays(n, m, offsets, neighbors, orig_ids):
    h = hashlib.sha256()
    h.update(np.int64([n, m]).tobytes())
    for a in (offsets, neighbors, orig_ids):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def self_launch(args):
    """`--gpus N` (N > 1) outside torchrun: re-exec this script under
    torch.distributed.run with N local ranks on 127.0.0.1 (the driver's own
    launch line), so a plain `python bench.py --gpus N` measures N ranks."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


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
    ap.add_argument("--cpu-port", action="store_true", help="also time the C port of the reference walk (extra line)")
    ap.add_argument("--ref-sample", type=int, default=2000, help="middles per reference-arm step (sampled configs)")
    ap.add_argument("--ref-stratified", action="store_true",
                    help="reference arm: add the stratified 200/100/20/2 extrapolation (hub seeds: minutes)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2306_00606_b200 as efg
    from paper_2306_00606_b200 import _native
    from paper_2306_00606_b200 import device as D
    from paper_2306_00606_b200.distributed import ef_cluster_centric_distributed, ef_distributed, ef_sharded

    rank, world, local = env_rank()
    ndev = torch.cuda.device_count()
    local_dev = local % max(ndev, 1)
    torch.cuda.set_device(local_dev)
    _native.set_device(local_dev)
    backend = "nccl" if world <= ndev else "gloo"  # ranks sharing a GPU (smoke runs): host collectives
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")           # communicator ranks/devices in the log
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_dev))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local_dev)

    # ---- graph: rank 0 builds (device R-MAT sampler / K1), broadcast to the others
    t0 = time.perf_counter()
    if rank == 0:
        if args.config == "rmat22":  # device sampler, bit-identical to the reference generator
            g, _ = efg.generate_rmat(efg.RmatParams(scale=22, avg_degree=21, seed=0))
        else:
            g = efg.build_graph(raw_edges(args.config))
        meta = [g.n, g.m]
    else:
        meta = [0, 0]

    def bcast(t):
        if backend == "nccl":
            dist.broadcast(t, 0)
        else:
            h = t.cpu()
            dist.broadcast(h, 0)
            t.copy_(h)

    if world > 1:
        mt = torch.tensor(meta, dtype=torch.int64, device=dev)
        bcast(mt)
        meta = mt.tolist()
    n, m = int(meta[0]), int(meta[1])
    if rank == 0:
        dg = D.DeviceGraph.from_host(g, device=local_dev)
    else:
        dg = D.DeviceGraph(torch.empty(n + 1, dtype=torch.int64, device=dev),
                           torch.empty(2 * m, dtype=torch.int32, device=dev), n)
    if world > 1:
        bcast(dg.offsets)
        bcast(dg.neighbors)
        if rank != 0:  # host copy for the e2e leg (pinned)
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

    # ---- the step: N = 1 one whole-graph pass; N > 1 the distributed pass
    # (factorized: parts + one all-reduce) or seed shards + one all-gather
    bounds = D.shard_bounds(dg, world, args.engine) if world > 1 else np.array([0, n], np.int64)
    distributed = world > 1 and args.engine == "factorized"
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        if distributed:
            return ef_distributed(dg)
        return ef_sharded(dg, engine=args.engine, bounds=bounds)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX)
            t = h
        return float(t.item())

    # ---- timed region: K steps, L2 flushed between steps, CUDA events on the stream
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    import gc

    gc.collect()
    gc.disable()  # no collector pause inside a timed step (the step's host syncs would stretch it)
    with ClockSampler(local_dev) as clocks:
        clocks.wait_live()
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
        clocks.ensure_sample(step)
    gc.enable()
    step_ms = [a.elapsed_time(b) for a, b in ev]  # this rank's per-step device times (diagnostic)
    ms = max_over_ranks(float(sum(step_ms)))
    ms_per_step = ms / args.steps
    value = n / (ms_per_step / 1e3)

    # ---- profiled step: the same step with live per-kernel event timing + launch count
    ctx = _native.context(local_dev)
    ctx.profile_reset()
    ctx.profile(True)
    torch.cuda.synchronize()
    if distributed:  # this rank's rows phase, the row exchange, its listing phase (the timed step's kernels)
        from paper_2306_00606_b200.distributed import exchange_rows
        words = torch.empty(D.DIST_WORDS * n, dtype=torch.int64, device=dev)
        ws = torch.empty(n, dtype=torch.float64, device=dev)
        adjp = torch.empty(2 * m, dtype=torch.int32, device=dev)
        dplus = torch.empty(n, dtype=torch.int32, device=dev)
        pb = D.part_bounds(dg, world)
        st = D.ef_partial_rows(dg, rank, world, pb, adjp, dplus, words, ws, stats=True)
        exchange_rows(adjp, dplus, dg.offsets[torch.as_tensor(pb, device=dev)].cpu().numpy(), pb)
        st2 = D.ef_partial_tables(dg, rank, world, pb, words, ws, stats=True)
        st3 = D.ef_partial_list(dg, rank, world, pb, adjp, dplus, words, ws, stats=True)
        st["launches"] += st2["launches"] + st3["launches"]
    else:
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        pe = torch.empty(hi - lo, dtype=torch.float64, device=dev)
        pt = torch.empty(hi - lo, dtype=torch.int64, device=dev)
        pf = torch.empty(hi - lo, dtype=torch.uint8, device=dev)
        st = D.ef_range(dg, lo, hi, pe, pt, pf, engine=args.engine, stats=True)
    ctx.profile(False)
    kernels = ctx.profile_report()
    if distributed:  # the finish kernels of the step (head + k_list_out, k_epilogue), outside the parts' stats calls
        n_launch_finish = 9
    else:
        n_launch_finish = 0

    # ---- end to end through the public API: host CSR -> device -> EF -> host
    def e2e_run(graph):
        if world == 1:
            return efg.ef_cluster_centric(graph, engine=args.engine)
        return ef_cluster_centric_distributed(graph)

    def e2e_time(graph, steps):
        # warm-up as the timed loop runs: the previous result is alive during the
        # next call, so two sets of recycled page-locked output blocks circulate
        keep = e2e_run(graph)
        keep = (keep, e2e_run(graph))
        del keep
        times = []
        for _ in range(steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            r = e2e_run(graph)
            times.append(max_over_ranks(time.perf_counter() - t0))
        return float(np.median(times)), times, r

    t_e2e, times, r = e2e_time(g, args.e2e_steps)
    h2d = (n + 1) * 8 + 2 * m * 4
    e2e = {"value": n / t_e2e, "unit": "seeds/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 17 * n,
           "ms_per_step": t_e2e * 1e3, "host_buffers": "pinned (repo Graph arrays)",
           "ms_wall_all": [round(t * 1e3, 2) for t in times]}
    if world == 1 and r.stats:
        e2e.update({"ms_h2d": r.stats["ms_h2d"], "ms_d2h": r.stats["ms_d2h"], "ms_device_events": r.stats["ms_device"],
                    "ms_prepare": r.stats["ms_prepare"], "ms_enumerate": r.stats["ms_enumerate"]})
    assert np.array_equal(out[0].cpu().numpy(), r.ef)  # the timed output equals the public API's
    # a drop-in caller's arrays: the reference Graph holds ordinary (pageable) numpy arrays
    from paper_2306_00606_b200.graph import Graph
    gp = Graph(n, m, np.array(g.offsets, copy=True), np.array(g.neighbors, copy=True), None)
    t_pg, times_pg, r_pg = e2e_time(gp, args.e2e_steps)
    assert np.array_equal(r_pg.ef, r.ef)
    e2e_pageable = {"value": n / t_pg, "unit": "seeds/s", "ms_per_step": t_pg * 1e3,
                    "host_buffers": "pageable numpy arrays (the reference Graph's)",
                    "ms_wall_all": [round(t * 1e3, 2) for t in times_pg]}
    if world == 1 and r_pg.stats:
        e2e_pageable.update({"ms_h2d": r_pg.stats["ms_h2d"], "ms_device_events": r_pg.stats["ms_device"]})

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
    dom_base = dom[0].split("<")[0].strip("() ")  # live names carry template arguments (k_mid_big<false>)
    dom_bytes = model.get(dom_base, {}).get("bytes")
    if dom_bytes and distributed:
        dom_bytes = dom_bytes / world  # this rank's part of the listing work units (approximately 1/N)
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
        "alg_saving_vs_naive_bytes": b_alg / (ms_per_step / 1e3) / 1e9 / peak,
        "naive_bytes_pass": b_alg,
        "note": "achieved = kernel_bytes_alg (listing model: 4 B/label read + 8 B/slot + 12 B/row + 8 B/Adj+(v) "
                "entry + 40 B/seed, DESIGN.md) / live event time; alg_saving_vs_naive_bytes = SURVEY 8(d) "
                "naive-enumeration bytes of the whole graph / step time / peak (NOT a roofline fraction: the "
                "factorised pass never moves those bytes); traffic = ncu dram bytes per launch "
                "(profiles/dram_traffic.json)",
    }
    cpu = cpu_port = None
    if not args.no_cpu_baseline and world == 1:
        threads = len(os.sched_getaffinity(0))
        try:
            rg = RefGraph(n, m, offs, nbrs, np.asarray(g.orig_ids))
            if args.config in SAMPLED:  # the reference arm's statistic: BASELINE.md 3's fixed uniform draw
                runs = [ref_uniform_rate(rg, threads, size=args.ref_sample, rng_seed=0) for _ in range(3)]
                rate = float(np.median([d[0] for d in runs]))
                dt, k = sum(d[1] for d in runs), runs[0][2]
                sample = (f"uniform draw of {k} middles (default_rng(0), BASELINE.md 3), median of 3 timings; "
                          f"reference _chunk_histograms(g, deg, codes, span, v, v+1) (expected_force.py:222) on a "
                          f"{threads}-worker thread pool, {dt:.1f} s in all; a per-seed rate -- it misses the hubs, "
                          f"so it overstates the reference's full-graph speed (stratified extrapolation: "
                          f"profiles/r02_bench_ref_*_strat*)")
            else:  # full graph in ~10-30 s here: the reference's own ef_cluster_centric
                dt, _ = rg.full(threads)
                rate = n / dt
                sample = f"full graph: reference ef_cluster_centric(g, workers={threads}), {dt:.1f} s"
            cpu = {"value": rate, "unit": "seeds/s", "cores": threads, "kind": "reference", "sample": sample,
                   "reference": "efgraph 0.1.0 (baseline/_ref, unmodified)", "ref_setup_s": rg.setup_s}
            del rg
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unavailable": f"{type(exc).__name__}: {exc}"}
        if args.cpu_port:
            t_full, sample, sample_s = cpu_port_rate(offs, nbrs, threads)
            cpu_port = {"value": n / t_full, "unit": "seeds/s", "cores": threads, "kind": "port",
                        "sample": f"{sample}; {sample_s:.1f} s of CPU work, extrapolated by work ratio to "
                                  f"{t_full:.0f} s"}
    line = {
        "metric": METRICS[args.config],
        "value": value, "unit": "seeds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "step_ms": [round(x, 3) for x in step_ms], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+int64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config], "n": n, "m": m, "engine": args.engine,
                   "parallelism": (f"whole-graph pass in {world} parts: rows per part, Adj+ row exchange "
                                   f"({world} broadcasts), listing per part, 1 all-reduce ({backend})" if distributed
                                   else f"seed-sharded x{world}"),
                   "l2": "flushed between timed steps (256 MB write)",
                   "graph_sha256_matches_reference": sha_ok},
        "e2e": e2e,
        "e2e_pageable": e2e_pageable,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "cpu_port": cpu_port,
        "gpu_launches": (int(st["launches"]) + n_launch_finish) * args.steps,
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
