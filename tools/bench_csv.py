#!/usr/bin/env python
"""Sample-CSV throughput: format and parse a synthetic
C4-shaped sample set (10^6 rows: D1, bx, by, bz, 5 metrics) with the native
data kit (rpg_samples_format / rpg_samples_parse), all host threads vs one
thread; checks the round trip is exact.  One JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1906_00142_b200 import samples as SM  # noqa: E402


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    X, ys, var = bench.c4_data(m, 0.01)
    names = sorted(ys)
    s = SM.SampleSet(names, (np.arange(m, dtype=np.int64) + 64)[:, None],  # distinct points
                     np.column_stack([X[:, 1:].astype(np.int64), np.ones((m, 1), np.int64)]),
                     np.column_stack([ys[k] for k in names]), SM.Provenance("synthetic", 1906, 0.01))
    out = {"rows": m, "threads": os.cpu_count()}
    for label, thr in (("all", 0), ("one", 1)):
        t0 = time.perf_counter()
        text = SM.format_samples(s, n_threads=thr)
        t1 = time.perf_counter()
        back = SM.parse_samples(text, n_threads=thr)
        t2 = time.perf_counter()
        out[f"format_s_{label}"] = t1 - t0
        out[f"parse_s_{label}"] = t2 - t1
    out["bytes"] = len(text)
    out["parse_rows_per_s_all"] = m / out["parse_s_all"]
    out["round_trip_exact"] = bool(np.array_equal(back.values, s.values) and np.array_equal(back.data, s.data)
                                   and np.array_equal(back.configs, s.configs))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
