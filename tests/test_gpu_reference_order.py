"""The benchmark's arithmetic modes against the reference's operation order.

FAST_CM (the C2/C3 bench default) and FAST are bit-exact against their own
O1 twins (test_gpu_fastcm.py, test_gpu_configs.py); this file pins them to
the reference's order of operations — oracle O1 EXACT, the mul-by-mul
restatement of eval_poly / mwpcwp_cycles (polyfit.hpp:96-130,
perfmodel.hpp:298-395) and of search_optimal's ranking (pipeline.hpp:
575-680) — under the north star's rule (tests/agree.py): 100 % of the
chosen configurations equal, or inside the EXACT minimum's 1e-9 window;
best Ec within 1e-9; occupancy, block count and case tag bit-exact wherever
the winners agree.  Sizes: the whole C2 bench step (65,473 N x 7,262
configs x 3 kernels = 1.426e9 points), all 27 C3 kernels on a strided N
sample, C1 at every N."""
import os

import numpy as np
import pytest

from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

from .agree import assert_agrees_with_exact, exact_winners

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = ("2dconv", "fdtd2d_step1", "fdtd2d_step2", "fdtd2d_step3", "2mm1", "3mm1", "bicg1", "bicg2",
         "gemm", "3dconv", "atax1", "atax2", "gesummv", "syrk", "mvt1", "mvt2", "syr2k",
         "corr", "corr_mean", "corr_reduce", "corr_std", "covar", "covar_mean", "covar_reduce",
         "gramschmidt1", "gramschmidt2", "gramschmidt3")


def _models(name, sub="polybench"):
    return F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", sub, f"{name}.models.json")))


def _b200():
    return F.load_profile(os.path.join(ROOT, "data", "b200.profile"))


def _gpu(spec, hw, space, data, arith, **kw):
    with S.Plan(spec, hw, space, S.SearchOptions(arith=arith, **kw)) as plan:
        return plan.search_batch(data)


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
def test_c2_full_step_fastcm_vs_exact(kernel):
    """The bench's whole C2 step for one kernel (475,464,926 points) in the
    headline arithmetic, every tuple under the north-star rule."""
    spec, hw, space = _models(kernel), _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, dtype=np.int64).reshape(-1, 1)
    exact = exact_winners(spec, hw, space, data)
    got = _gpu(spec, hw, space, data, "fastcm")
    assert_agrees_with_exact(got, spec, hw, space, data, exact=exact)
    fast = _gpu(spec, hw, space, data, "fast")
    assert_agrees_with_exact(fast, spec, hw, space, data, exact=exact)


@pytest.mark.parametrize("kernel", SUITE)
def test_c3_suite_fastcm_vs_exact(kernel):
    spec, hw, space = _models(kernel), _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 97, dtype=np.int64).reshape(-1, 1)
    exact = exact_winners(spec, hw, space, data)
    for arith in ("fastcm", "fast"):
        assert_agrees_with_exact(_gpu(spec, hw, space, data, arith), spec, hw, space, data, exact=exact)


def test_c1_every_n_fastcm_vs_exact():
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "sample_device.profile"))
    space = F.integer_configs(1024, dims=2)
    data = np.arange(1024, 8193, dtype=np.int64).reshape(-1, 1)
    assert_agrees_with_exact(_gpu(spec, hw, space, data, "fastcm"), spec, hw, space, data)
