"""Summarise an ncu --page source --print-source sass CSV: opcode mix and hottest SASS lines of one kernel."""
import collections
import csv
import sys

path, pat = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if cur is not None:
        cur["rows"].append(r)
for b in blocks:
    if pat not in b["name"]:
        continue
    hdr, data = b["rows"][0], b["rows"][1:]
    iS, iI, iW, iA = (hdr.index(k) for k in ("Source", "Instructions Executed", "Warp Stall Sampling (All Samples)", "Address"))
    f = lambda x: float(x or 0)
    tot = sum(f(r[iI]) for r in data)
    totw = sum(f(r[iW]) for r in data) or 1
    print(b["name"][:90], "warp-instr %.3e" % tot, "sass lines", len(data))
    ops = collections.Counter()
    for r in data:
        ops[r[iS].split()[0] if r[iS] else "?"] += f(r[iI])
    print([(k, round(v / tot * 100, 1)) for k, v in ops.most_common(20)])
    top = sorted(range(len(data)), key=lambda k: -f(data[k][iW]))[:ntop]
    for k in sorted(top):
        r = data[k]
        print(f"{r[iA]} {f(r[iI])/tot*100:5.2f}%i {f(r[iW])/totw*100:5.2f}%s  {r[iS][:90]}")
    break
