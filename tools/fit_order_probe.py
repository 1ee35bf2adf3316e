#!/usr/bin/env python
"""Which of data or process state makes a C4 fit's sample passes slow?  Fits
the given metrics in the given order (RPG_FIT_TRACE=1 prints the per-step
anatomy).  Usage: python tools/fit_order_probe.py METRIC [METRIC ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_00142_b200 import fit as G  # noqa: E402

X, ys, variables = bench.c4_data(bench.C4_SAMPLES, 0.01)
for name in sys.argv[1:]:
    print("==", name, file=sys.stderr, flush=True)
    n = None
    if ":" in name:  # METRIC:M fits the first M samples
        name, n = name.split(":")[0], int(name.split(":")[1])
    try:
        G.fit_rational(X[:n], ys[name][:n], variables, [2, 2, 2], [1, 1, 1])
    except (G.DegenerateFit, G.SvdFailure) as e:
        print("failed", e, file=sys.stderr)
