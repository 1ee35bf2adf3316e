"""Parity at BASELINE.json's configuration sizes (the bench workloads are
parity-test cases too): GPU winners through the C ABI against oracle O1.

* C1 (configs[0]): 2DCONV — the reference's stencil2d ground truth on its
  sample device, and the fitted 2DCONV model on the B200 profile — best
  (bx, by) over all 7,262 integer configs for EVERY N = 1024..8192
  (52,061,278 points per model), plus the paper-style subset N in
  {1024, 2048, 4096, 8192} x enumerate_configs();
* C2 (configs[1], the bench workload): all 65,473 N x 7,262 configs x 3
  kernels = 1.426e9 points, 100 % winner agreement (bit-exact records) in
  the benchmark's FAST mode against O1's FAST twin, and a strided sample in
  EXACT mode against O1 EXACT;
* C3 (configs[2]): all 27 suite kernels on a strided N sample;
* C5 (configs[4]): the 5-variable stress model over the 3-D space on a
  sample of the (N, M) grid.
The O1 legs use every host core of the GPU box."""
import os

import numpy as np
import pytest

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = ("2dconv", "fdtd2d_step1", "fdtd2d_step2", "fdtd2d_step3", "2mm1", "3mm1", "bicg1", "bicg2",
         "gemm", "3dconv", "atax1", "atax2", "gesummv", "syrk", "mvt1", "mvt2", "syr2k",
         "corr", "corr_mean", "corr_reduce", "corr_std", "covar", "covar_mean", "covar_reduce",
         "gramschmidt1", "gramschmidt2", "gramschmidt3")


def _threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _models(name, sub="polybench"):
    return F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", sub, f"{name}.models.json")))


def _b200():
    return F.load_profile(os.path.join(ROOT, "data", "b200.profile"))


def _check(spec, hw, space, data, arith):
    arith_c = A.RPG_ARITH_FAST if arith == "fast" else A.RPG_ARITH_EXACT
    want = o1.search_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw),
                           A.options_struct(arith=arith_c), A.config_array(space), data, _threads())
    with S.Plan(spec, hw, space, S.SearchOptions(arith=arith)) as plan:
        got = plan.search_batch(data)
    mism = np.nonzero((got.view(np.uint8).reshape(len(got), -1) !=
                       want.view(np.uint8).reshape(len(want), -1)).any(axis=1))[0]
    assert len(mism) == 0, (len(mism), data[mism[:3]].tolist(), got[mism[:3]], want[mism[:3]])
    return got


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_c1_stencil2d_every_n(arith):
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "sample_device.profile"))
    data = np.arange(1024, 8193, dtype=np.int64).reshape(-1, 1)
    _check(spec, hw, F.integer_configs(1024, dims=2), data, arith)


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_c1_fitted_2dconv_every_n(arith):
    data = np.arange(1024, 8193, dtype=np.int64).reshape(-1, 1)
    _check(_models("2dconv"), _b200(), F.integer_configs(1024, dims=2), data, arith)


def test_c1_paper_subset():
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "sample_device.profile"))
    data = np.array([[1024], [2048], [4096], [8192]], dtype=np.int64)
    got = _check(spec, hw, F.enumerate_configs(), data, "exact")
    space = F.enumerate_configs()
    # SURVEY.md 8c sanity fact: all 51 configs feasible, winner 1024 x 1.
    assert (got["n_feasible"] == 51).all()
    assert all(space[i][:2] == (1024, 1) for i in got["cfg_idx"])


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
def test_c2_full_workload_fast_bit_exact(kernel):
    """The benchmark's whole step for one kernel: 475,464,926 points."""
    data = np.arange(64, 65537, dtype=np.int64).reshape(-1, 1)
    _check(_models(kernel), _b200(), F.integer_configs(1024, dims=2), data, "fast")


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
def test_c2_sampled_exact(kernel):
    data = np.arange(64, 65537, 37, dtype=np.int64).reshape(-1, 1)
    _check(_models(kernel), _b200(), F.integer_configs(1024, dims=2), data, "exact")


@pytest.mark.parametrize("kernel", SUITE)
def test_c3_suite_sampled(kernel):
    data = np.arange(64, 65537, 331, dtype=np.int64).reshape(-1, 1)
    space = F.integer_configs(1024, dims=2)
    _check(_models(kernel), _b200(), space, data, "fast")
    _check(_models(kernel), _b200(), space, data[::4], "exact")


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_c5_stress_sampled(arith):
    v = np.unique(np.linspace(64, 65536, 182).round().astype(np.int64))
    nn, mm = np.meshgrid(v, v, indexing="ij")
    grid = np.stack([nn.ravel(), mm.ravel()], axis=1)
    data = np.ascontiguousarray(grid[:: 33124 // 24][:24])
    _check(_models("stencil3d_nm", "stress"), _b200(), F.integer_configs(1024, dims=3), data, arith)


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
def test_c2_fast_agrees_with_reference_order(kernel):
    """The benchmark's FAST arithmetic against the reference's operation
    order (O1 EXACT) at the north star's tolerance: the FAST winner equals
    the EXACT winner, or its EXACT cycle estimate is within 1e-9 (relative)
    of the EXACT minimum (ties within the tolerance count as agreement)."""
    spec, hw = _models(kernel), _b200()
    space = F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 7, dtype=np.int64).reshape(-1, 1)
    pk = A.PackedModel(spec, drop_zero_terms=False)
    sp = A.config_array(space)
    exact = o1.search_batch(pk, A.profile_struct(hw), A.options_struct(arith=A.RPG_ARITH_EXACT), sp, data,
                            _threads())
    with S.Plan(spec, hw, space, S.SearchOptions(arith="fast")) as plan:
        fast = plan.search_batch(data)
    diff = np.nonzero(fast["cfg_idx"] != exact["cfg_idx"])[0]
    if len(diff):
        ec, _, _ = o1.evaluate_batch(pk, A.profile_struct(hw), A.options_struct(arith=A.RPG_ARITH_EXACT), sp,
                                     np.ascontiguousarray(data[diff]), _threads())
        for j, t in enumerate(diff):
            row = ec[j]
            best = row[row >= 0].min()
            assert row[fast["cfg_idx"][t]] <= best * (1 + 1e-9), (int(data[t, 0]), best)
    rel = np.abs(fast["best_ec"] - exact["best_ec"]) / np.maximum(1.0, np.abs(exact["best_ec"]))
    assert rel.max() <= 1e-9
