#!/usr/bin/env python
"""Small searches for compute-sanitizer (racecheck / synccheck / memcheck):
every search kernel family — the configuration-major FAST_CM kernel (two
tuples per thread and one), the specialized FAST / EXACT kernels, the
ahead-of-time generic kernels, the Ec-dump evaluate kernel — on the C2 gemm
model and on the zoo's flat tie landscape (every config in the tie group:
the pass-2 overflow path and the shared-memory key reductions), plus one
C5-shape (3-D space) search.  Exits non-zero if any result differs from
oracle O1, so a sanitizer run is also a parity run.

Usage: compute-sanitizer --tool racecheck python tools/sanitize_search.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import o1  # noqa: E402
from paper_1906_00142_b200 import abi as A  # noqa: E402
from paper_1906_00142_b200 import formats as F  # noqa: E402
from paper_1906_00142_b200 import search as S  # noqa: E402
from tests import zoo  # noqa: E402


def check(name, spec, hw, space, data, **kw):
    opts = S.SearchOptions(**kw)
    want = o1.search_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), opts.struct(),
                           A.config_array(space), data, 4)
    with S.Plan(spec, hw, space, opts) as plan:
        got = plan.search_batch(data)
        if kw.get("arith") != "fastcm":
            plan.evaluate(data[:2])
    same = np.array_equal(got.view(np.uint8), want.view(np.uint8))
    print(f"{name:40s} {'ok' if same else 'MISMATCH'}", flush=True)
    return same


def main():
    hw = zoo.b200_hw()
    gemm = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))
    space2 = F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 1021, dtype=np.int64).reshape(-1, 1)[:48]
    ok = True
    ok &= check("gemm fastcm (pair)", gemm, hw, space2, data, arith="fastcm")
    # one full J = 3 wave on 148 SMs (96-tuple groups) + a J = 2 remainder,
    # certified bodies (range certificate)
    big = np.arange(64, 64 + 148 * 96 + 100, dtype=np.int64).reshape(-1, 1)
    ok &= check("gemm fastcm (J=3 wave + J=2 rest)", gemm, hw, space2[::5], big, arith="fastcm")
    for k in ("c6_stencil", "c6_reduce"):  # all three proven-case bodies, infeasible configs, ties
        c6 = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "stressed", f"{k}.models.json")))
        ok &= check(f"{k} fastcm", c6, F.load_profile(os.path.join(ROOT, "data", "b200.profile")), space2, data,
                    arith="fastcm")
    ok &= check("gemm fast specialized", gemm, hw, space2, data[:16], arith="fast")
    ok &= check("gemm exact specialized", gemm, hw, space2, data[:8], arith="exact")
    ok &= check("gemm fast generic", gemm, hw, space2, data[:8], arith="fast", kernel="generic")
    flat = zoo.const_spec(25, 0, 0, 0, 1)
    pow2 = F.enumerate_configs()
    d1 = np.array([[64], [128], [1000]], dtype=np.int64)
    for arith in ("fastcm", "fast", "exact"):
        ok &= check(f"flat ties {arith}", flat, zoo.sample_hw(), pow2, d1, arith=arith, rep_mode="ceil")
    ok &= check("flat ties generic", flat, zoo.sample_hw(), pow2, d1, arith="exact", kernel="generic")
    c5 = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "stress", "stencil3d_nm.models.json")))
    space3 = F.integer_configs(1024, dims=3)[::17]
    ok &= check("c5 fast (3-D space)", c5, hw, space3, np.array([[64, 64], [4000, 9000]], dtype=np.int64),
                arith="fast")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
