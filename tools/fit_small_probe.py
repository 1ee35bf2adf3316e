#!/usr/bin/env python
"""Small C4-shaped fits (sanitizer runs): the 5 metrics of the synthetic
GEMM kernel on M noisy samples, default bounds."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_00142_b200 import fit as G  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
X, ys, variables = bench.c4_data(m, 0.01)
for name in sorted(ys):
    try:
        f, rep = G.fit_rational(X, ys[name], variables, [2, 2, 2], [1, 1, 1])
        print(name, rep.safeguard, [float(c).hex() for c in f.den.coeffs][:2])
    except (G.DegenerateFit, G.SvdFailure) as e:
        print(name, "failed", e)
