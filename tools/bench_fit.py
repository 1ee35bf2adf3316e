#!/usr/bin/env python
"""C4 fit benchmark: rational least-squares fits from 10^6
synthetic profiled samples per metric, variables (D1, bx, by), default
bounds num (2,2,2) / den (1,1,1) -> 10^6 x 35 sample matrices, 5 metrics of
the synthetic GEMM kernel, clean and 1 % noise.  GPU = librpgpu.so's K3
(rpg_fit_rational, host buffers in the timed region); CPU = oracle O3
(numpy/LAPACK, all host cores) on the same arrays.  One JSON line.

Usage: python tools/bench_fit.py [--samples 1000000] [--noise 0.01] [--cpu]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=1_000_000)
    ap.add_argument("--noise", type=float, default=0.0)
    ap.add_argument("--cpu", action="store_true", help="also time oracle O3 (slow)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-warmup", action="store_true", help="skip the small warm-up fit (profiling)")
    args = ap.parse_args()
    from paper_1906_00142_b200 import fit as G
    from paper_1906_00142_b200 import formats as F
    from oracle import o3_fit as O3

    rng = np.random.default_rng(1906)
    m = args.samples
    D = rng.integers(64, 65537, m).astype(float)
    cfg = np.array(F.integer_configs(), dtype=float)[rng.integers(0, 7262, m)][:, :2]
    X = np.ascontiguousarray(np.column_stack([D, cfg]))
    spec = F.load_kernel_spec(os.path.join(ROOT, "data", "polybench", "gemm.kernel.json"))
    ys = {}
    for name in F.REQUIRED_METRICS:
        y = O3.eval_ratfunc(spec.ground_truth[name], X)
        if args.noise > 0:
            y = y * (1 + rng.uniform(-args.noise, args.noise, m))
        ys[name] = np.ascontiguousarray(y)
    nb, db = [2, 2, 2], [1, 1, 1]
    # warm-up (context, module load)
    if not args.no_warmup:
        try:
            G.fit_rational(X[:4096], ys[F.METRIC_COMP][:4096], spec.variables, nb, db)
        except (G.DegenerateFit, G.SvdFailure):
            pass
    times, safeguards = [], {}
    for _ in range(args.reps):
        t0 = time.perf_counter()
        for name, y in ys.items():
            try:
                _, rep = G.fit_rational(X, y, spec.variables, nb, db)
                safeguards[name] = rep.safeguard
            except (G.DegenerateFit, G.SvdFailure) as e:
                safeguards[name] = f"failed: {e}"
        times.append(time.perf_counter() - t0)
    gpu_s = min(times)
    # the fit_all_metrics path: every metric at once (rpg_fit_rational_multi)
    times_multi = []
    names = list(ys)
    for _ in range(args.reps):
        t0 = time.perf_counter()
        res = G.fit_rational_multi(X, [ys[k] for k in names], spec.variables, [(nb, db)] * len(names))
        times_multi.append(time.perf_counter() - t0)
    multi = {k: (r[1].safeguard if not isinstance(r, Exception) else f"failed: {r}") for k, r in zip(names, res)}
    n = 35
    flops = len(ys) * (2 * m * n * n - 2 * n ** 3 / 3 + 3 * m * n)  # BASELINE.md C4 formula
    line = {"metric": "C4 rational fit time (5 metrics)", "samples_per_metric": m, "columns": n,
            "noise_rel": args.noise, "gpu_seconds": gpu_s, "gpu_samples_per_s": len(ys) * m / gpu_s,
            "qr_flops": flops, "gpu_tflops_qr_equiv": flops / gpu_s / 1e12,
            "safeguard": safeguards, "api": "rpg_fit_rational (host buffers, incl. H2D), one metric after another",
            "multi_seconds": min(times_multi), "multi_samples_per_s": len(ys) * m / min(times_multi),
            "multi_outcomes_equal": multi == safeguards,
            "multi_api": "rpg_fit_rational_multi (X uploaded once, 5 concurrent fits)"}
    if args.cpu:
        t0 = time.perf_counter()
        for name, y in ys.items():
            try:
                O3.fit_rational(X, y, spec.variables, nb, db)
            except O3.DegenerateFit:
                pass
        cpu_s = time.perf_counter() - t0
        line.update({"cpu_seconds": cpu_s, "cpu_kind": "O3 numpy/LAPACK",
                     "cpu_threads": len(os.sched_getaffinity(0))})
    print(json.dumps(line))


if __name__ == "__main__":
    main()
