#!/usr/bin/env python
"""Bit-level A/B of two librpgpu.so builds on the C4 fit (every metric's
fitted coefficients and every safeguard stage vector, as hex).

Usage: python tools/fit_ab_bits.py OLD.so [NEW.so] [--samples M]
  (NEW defaults to the in-tree library).  Prints one JSON line:
  {"identical": bool, "diffs": [...]}.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_1906_00142_b200 import abi as A
A.load_library(sys.argv[2])
import bench
from paper_1906_00142_b200 import fit as G
out = {}
for noise in (0.0, 0.01):
    X, ys, variables = bench.c4_data(int(sys.argv[3]), noise)
    for name in sorted(ys):
        tr = {}
        try:
            f, rep = G.fit_rational(X, ys[name], variables, [2, 2, 2], [1, 1, 1], trace=tr)
            res = [float(c).hex() for c in list(f.num.coeffs) + list(f.den.coeffs)] + [rep.safeguard]
        except (G.DegenerateFit, G.SvdFailure) as e:
            res = [type(e).__name__, str(e)]
        out[f"{name}@{noise}"] = {"result": res,
                                  "stages": [[float(v).hex() for v in st] for st in tr.get("stages", [])]}
print(json.dumps(out))
"""


def run(lib, m):
    p = subprocess.run([sys.executable, "-c", _CHILD, ROOT, lib, str(m)], capture_output=True, text=True,
                       timeout=1200)
    if p.returncode:
        raise SystemExit(p.stderr[-3000:])
    return json.loads(p.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("old")
    ap.add_argument("new", nargs="?", default=os.path.join(ROOT, "paper_1906_00142_b200", "librpgpu.so"))
    ap.add_argument("--samples", type=int, default=1_000_000)
    a = ap.parse_args()
    o, n = run(a.old, a.samples), run(a.new, a.samples)
    diffs = [k for k in sorted(set(o) | set(n)) if o.get(k) != n.get(k)]
    first = {}
    for k in diffs:  # the first safeguard stage whose vector differs (None: only the result)
        so, sn = o.get(k, {}).get("stages", []), n.get(k, {}).get("stages", [])
        first[k] = next((i for i in range(max(len(so), len(sn)))
                         if i >= len(so) or i >= len(sn) or so[i] != sn[i]), None)
    print(json.dumps({"identical": not diffs, "diffs": diffs, "first_stage": first, "n_fits": len(o)}))


if __name__ == "__main__":
    main()
