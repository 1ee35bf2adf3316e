#!/usr/bin/env python
"""Per-opcode executed-instruction mix of the search kernel from an ncu
report (source page, SASS), normalised per warp-point.  Usage:
  ncu_mix.py report.ncu-rep points_per_launch"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, pts = sys.argv[1], float(sys.argv[2]) / 32
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
agg, samp = collections.Counter(), collections.Counter()
tot = stot = 0
for r in data:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
    if not m:
        continue
    n, w = int(r[iE] or 0), int(r[iW] or 0)
    agg[m.group(2)] += n
    samp[m.group(2)] += w
    tot += n
    stot += w
print(f"warp-instructions per warp-point: {tot / pts:.1f}  (stall samples {stot})")
fp64 = sum(agg[k] for k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "I2F", "F2F", "FRND")) / pts
print(f"FP64-pipe class instructions per warp-point: {fp64:.1f}")
for op, n in agg.most_common(24):
    print(f"  {op:10s} {n / pts:7.2f}  {100 * n / tot:5.1f}%  stall samples {samp[op]}")
