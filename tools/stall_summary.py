"""Aggregate warp-stall reasons (all samples) of the kernel in an ncu report, plus the
occupancy / issue figures from the details page.

    python tools/stall_summary.py <report.ncu-rep>
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = {}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    for i in cols:
        try:
            agg[hdr[i]] = agg.get(hdr[i], 0.0) + float(r[i] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1.0
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in
                          sorted(agg.items(), key=lambda x: -x[1])[:8]))
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
want = ("Duration", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size",
        "Waves Per SM", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler")
for r in csv.reader(io.StringIO(det)):
    if len(r) > 14 and r[12] in want:
        print(f"  {r[12]}: {r[14]} {r[13]}")
