#!/usr/bin/env python
"""FAST_CM range-certificate coverage per bench workload: for each kernel, the
fraction of (configuration, binade of N) cells over the workload's N range
where pass 1 runs without per-point range checks, and where the MWP-CWP case
is proven (rpg_plan_cert_counts).  Usage: cert_report.py [c2|c3|c6 ...]"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_00142_b200 import search as S  # noqa: E402


def main(names):
    out = {}
    for name in names:
        wl = bench.Workload(name)
        k_lo, k_hi = 6, 16  # N = 64..65536: binades 6..16
        rows = {}
        for k in wl.kernels:
            with S.Plan(wl.specs[k], wl.hw, wl.space, S.SearchOptions(arith="fastcm")) as plan:
                c = plan.cert_counts()
            cells = len(wl.space) * (k_hi - k_lo + 1)
            rows[k] = {m: round(sum(c[m][k_lo:k_hi + 1]) / cells, 4) for m in c}
        tot = {m: round(sum(r[m] for r in rows.values()) / len(rows), 4) for m in ("free", "cwp", "mwp", "both")}
        out[name] = {"mean": tot, "kernels": rows}
        print(name, "mean coverage", json.dumps(tot))
    return out


if __name__ == "__main__":
    res = main(sys.argv[1:] or ["c2", "c3", "c6"])
    print(json.dumps(res))
