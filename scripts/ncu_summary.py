"""Key per-kernel metrics from an ncu report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
idi = hdr.index("ID")
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Branch Efficiency"]
cur = None
for r in rows[1:]:
    if r[mi] in want:
        key = (r[idi], r[ki])
        if key != cur:
            print("==", r[idi], r[ki][:100])
            cur = key
        print(f"    {r[mi]:38s} {r[vi]} {r[ui]}")
