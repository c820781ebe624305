"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*) into
per-kernel totals for the LAST full EF pass of the run (the profiled step), and
write profiles/dram_traffic.json (dram bytes per launch of each kernel)."""
import collections
import csv
import json
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("efg::<unnamed>::", "").replace("void ", "")
    return name.strip()


path = sys.argv[1]
out_json = sys.argv[2] if len(sys.argv) > 2 else None
rows = [r for r in csv.reader(open(path)) if len(r) >= 15 and r[0] != "ID"]
launch = collections.OrderedDict()
for r in rows:
    key = int(r[0])
    d = launch.setdefault(key, {"name": r[4], "stream": r[6], "grid": r[8], "block": r[7]})
    d[r[12]] = float(r[14].replace(",", ""))
items = list(launch.values())
# the profiled EF pass = from the last k_deg launch up to the first k_topk/end
starts = [i for i, d in enumerate(items) if short(d["name"]) == "k_deg"]
seg = items[starts[-1]:] if starts else items
tot = collections.OrderedDict()
for d in seg:
    k = short(d["name"])
    t = tot.setdefault(k, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    t["launches"] += 1
    t["ms"] += d.get("gpu__time_duration.sum", 0) / 1e6
    t["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
all_ms = sum(t["ms"] for t in tot.values())
print(f"{'kernel':45s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'dram GB':>8s} {'GB/s':>8s}")
for k, t in sorted(tot.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k[:45]:45s} {t['launches']:8d} {t['ms']:9.3f} {t['ms']/all_ms*100:5.1f}% {t['dram_bytes']/1e9:8.3f} "
          f"{t['dram_bytes']/max(t['ms'],1e-9)/1e6:8.1f}")
print(f"total {all_ms:.3f} ms over {sum(t['launches'] for t in tot.values())} launches (serialised, cold cache)")
if out_json:
    # live-profile names of the templated launches (csrc/ef_factor.cu)
    alias = {"k_tri_seed<128, 512, 1>": "k_tri_seed_256", "k_tri_seed<256, 1024, 1>": "k_tri_seed_1024",
             "k_tri_seed<512, 4096, 0>": "k_tri_seed_4096"}
    out = {}
    for k, t in tot.items():
        out[k] = t["dram_bytes"] / t["launches"]
        if k in alias:
            out[alias[k]] = out[k]
        base = k.split("<")[0]
        if base != k and base not in out:
            out[base] = out[k]
    json.dump(out, open(out_json, "w"), indent=1)
