#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)
into per-kernel totals and shares.  Usage: ncu_summary.py launches.csv [title]"""
import collections
import csv
import io
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path, title=""):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.defaultdict(lambda: [0, 0.0, ""])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:70]
        ms = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        a = agg[short]
        a[0] += 1
        a[1] += ms
        a[2] = f'grid {r["Grid Size"]} block {r["Block Size"]}'
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"# {title}", "# per-kernel device time (ncu, --clock-control none; cold-cache serialised — compare shares)"]
    for k, (n, ms, geo) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{ms:11.3f} ms  {100 * ms / tot:5.1f}%  n={n:3d}  avg {ms / n:9.3f} ms  {k}  [{geo}]")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
