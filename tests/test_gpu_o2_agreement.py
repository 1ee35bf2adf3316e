"""Chosen-config agreement with the reference's own semantics — the exact
rational program the reference's search_optimal interprets (oracle O2,
interp.hpp:44-121 over perfmodel.hpp:648-834, 10^40 floor-division
lowering) — on sampled tuples ("O2 subset"): the GPU winner's
exact program value lies inside O2's tie group (best + best * 1e-12,
pipeline.hpp:660-661), and equals O2's argmin whenever that group is a
single configuration."""
import os

import numpy as np
import pytest

from oracle import o2_exact as o2
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _agree(spec, hw, space, ns, arith):
    with S.Plan(spec, hw, space, S.SearchOptions(arith=arith)) as plan:
        win = plan.search_batch(np.array(ns, dtype=np.int64).reshape(-1, 1))
    for t, n in enumerate(ns):
        vals, feas, ties = o2.search(spec, hw, [n], space)
        g = int(win["cfg_idx"][t])
        if not feas:
            assert g < 0
            continue
        best = vals[feas[0]]
        assert g >= 0 and vals[g] >= 0
        assert vals[g] <= best + best * o2.rat(1e-12), (n, space[g], float(vals[g]), float(best))
        if ties == 1:
            assert g == feas[0], (n, space[g], space[feas[0]])


@pytest.mark.parametrize("arith", ["exact", "fast", "fastcm"])
def test_c1_stencil2d_paper_subset(arith):
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "sample_device.profile"))
    _agree(spec, hw, F.enumerate_configs(), [1024, 2048, 4096, 8192], arith)


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
@pytest.mark.parametrize("arith", ["exact", "fast", "fastcm"])
def test_c2_models_sampled(kernel, arith):
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", f"{kernel}.models.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    space = F.integer_configs(1024, dims=2)[::25]
    _agree(spec, hw, space, [64, 4097, 65536], arith)
