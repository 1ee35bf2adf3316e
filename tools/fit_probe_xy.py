#!/usr/bin/env python
"""Probe: the acceptance target restricted to (x, y) (bounds (2,2)/(1,1),
nd = 4) and to (x, y, z) (nd = 8), 20000 samples with 1 % noise: the GPU
fit's safeguard stages against O3's, as unit-vector distances."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import o3_fit as O3  # noqa: E402
from paper_1906_00142_b200 import fit as G  # noqa: E402
from tests.test_gpu_fit import target  # noqa: E402


def unit(v):
    v = np.asarray(v, dtype=float)
    n = np.linalg.norm(v)
    v = v / n if n > 0 else v
    i = int(np.argmax(np.abs(v)))
    return v * np.sign(v[i]) if v[i] != 0 else v


rng = np.random.default_rng(5150)
P = rng.uniform(1.0, 4.0, (20000, 3))
H = rng.uniform(1.0, 4.0, (50, 3))
e = rng.uniform(-0.01, 0.01, len(P))
for name, cols, bounds in (("xyz", [0, 1, 2], ([2, 2, 2], [1, 1, 1])), ("xy", [0, 1], ([2, 2], [1, 1]))):
    noisy = target(P, cols) * (1 + e)
    tg, to = {}, {}
    f, rep = G.fit_rational(P[:, cols], noisy, ["x", "y", "z"][:len(cols)], *bounds, trace=tg)
    fo, ro = O3.fit_rational(P[:, cols], noisy, ["x", "y", "z"][:len(cols)], *bounds, trace=to)
    g, o = O3.eval_ratfunc(f, H[:, cols]), O3.eval_ratfunc(fo, H[:, cols])
    sg, so = tg.get("stages", []), to.get("stages", [])
    dist = [float(np.linalg.norm(unit(a) - unit(b))) for a, b in zip(sg, so)]
    print(json.dumps({"case": name, "safeguard": [rep.safeguard, ro.safeguard], "stages": [len(sg), len(so)],
                      "stop": [tg.get("stop"), to.get("stop")], "stage_dist": dist,
                      "qmin": [tg.get("round_qmin"), to.get("round_qmin")],
                      "maxrel": float(np.max(np.abs(g - o) / np.abs(o)))}))
