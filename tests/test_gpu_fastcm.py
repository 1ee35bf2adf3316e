"""RPG_ARITH_FAST_CM — the configuration-major search (rpg_kernels.cuh
search_body_cm, rpg_jit.cu build_cm): per-configuration collapse of the
block-dimension part, Horner in N per point.  Winner records must be
byte-identical to oracle O1's FAST_CM twin (fast_cm_poly) on the C2/C3
models over the full 7,262-config space, on random and division-edge models,
and across awkward batch shapes (tuple counts that are not multiples of 32,
a single tuple, fewer configurations than warps per CTA).  Plans that the
mode cannot serve fail loudly."""
import os

import numpy as np
import pytest

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

from .agree import assert_agrees_with_exact
from .test_gpu_configs import SUITE, _b200, _models, _threads
from .test_gpu_fuzz import _case, _edge_case

pytestmark = pytest.mark.gpu


def _o1(spec, hw, space, data, rep="real", regs=0.0, shared=0.0):
    opts = S.SearchOptions(arith="fastcm", rep_mode=rep, regs_per_thread=regs,
                           shared_words_per_block=shared)
    return o1.search_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), opts.struct(),
                           A.config_array(space), data, _threads())


def _gpu(spec, hw, space, data, rep="real", regs=0.0, shared=0.0):
    opts = S.SearchOptions(arith="fastcm", rep_mode=rep, regs_per_thread=regs,
                           shared_words_per_block=shared)
    with S.Plan(spec, hw, space, opts) as plan:
        return plan.search_batch(data)


def _same(got, want, data):
    g = got.view(np.uint8).reshape(len(got), -1)
    w = want.view(np.uint8).reshape(len(want), -1)
    bad = np.nonzero((g != w).any(axis=1))[0]
    assert len(bad) == 0, (len(bad), data[bad[:3]].tolist(), got[bad[:3]], want[bad[:3]])


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
def test_c2_models_full_space(kernel):
    spec, hw, space = _models(kernel), _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 61, dtype=np.int64).reshape(-1, 1)   # 1,074 N (not a multiple of 32)
    _same(_gpu(spec, hw, space, data), _o1(spec, hw, space, data), data)


def test_suite_models_sample():
    hw, space = _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 4093, dtype=np.int64).reshape(-1, 1)
    for k in SUITE:
        spec = _models(k)
        _same(_gpu(spec, hw, space, data), _o1(spec, hw, space, data), data)


@pytest.mark.parametrize("seed", [s for s in range(24) if s % 3 and s % 4])
def test_random_models(seed):
    spec, hw, space, data, rep = _case(seed)
    _same(_gpu(spec, hw, space, data, rep, 24.0), _o1(spec, hw, space, data, rep, 24.0), data)


@pytest.mark.parametrize("seed", range(12))
def test_division_edges(seed):
    spec, hw, space, data, rep = _edge_case(seed)
    _same(_gpu(spec, hw, space, data, rep, 24.0), _o1(spec, hw, space, data, rep, 24.0), data)


@pytest.mark.parametrize("n_tuples,n_space", [(1, 7262), (33, 7262), (5, 1), (40, 3), (64, 129)])
def test_batch_shapes(n_tuples, n_space):
    spec, hw = _models("gemm"), _b200()
    full = F.integer_configs(1024, dims=2)
    rng = np.random.default_rng(n_tuples * 1000 + n_space)
    space = [full[i] for i in np.sort(rng.choice(len(full), n_space, replace=False))]
    data = rng.integers(1, 70000, size=(n_tuples, 1)).astype(np.int64)
    _same(_gpu(spec, hw, space, data), _o1(spec, hw, space, data), data)


def test_agrees_with_exact_mode():
    """FAST_CM and EXACT differ only in rounding: the north star's rule
    (tests/agree.py) on a strided gemm sample; the full C2 step is in
    test_gpu_reference_order.py."""
    spec, hw, space = _models("gemm"), _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 257, dtype=np.int64).reshape(-1, 1)
    assert_agrees_with_exact(_gpu(spec, hw, space, data), spec, hw, space, data)


def test_unsupported_plans_fail_loudly():
    hw = _b200()
    space = F.integer_configs(1024, dims=2)
    with pytest.raises(ValueError, match="specialized"):
        S.Plan(_models("gemm"), hw, space, S.SearchOptions(arith="fastcm", kernel="generic"))
    c5 = F.models_to_metric_spec(F.read_models(os.path.join(os.path.dirname(__file__), "..", "data",
                                                            "stress", "stencil3d_nm.models.json")))
    with pytest.raises(ValueError, match="one data parameter"):
        S.Plan(c5, hw, F.integer_configs(1024, dims=3), S.SearchOptions(arith="fastcm"))
    with S.Plan(_models("gemm"), hw, space, S.SearchOptions(arith="fastcm")) as plan:
        with pytest.raises(ValueError, match="fast_cm"):
            plan.search_batch_subsets(np.array([[1024]], dtype=np.int64), [0, 1], [0])


def _o1_eval(spec, hw, space, data, rep="real", regs=0.0, shared=0.0):
    opts = S.SearchOptions(arith="fastcm", rep_mode=rep, regs_per_thread=regs,
                           shared_words_per_block=shared)
    return o1.evaluate_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), opts.struct(),
                             A.config_array(space), data, _threads())


def _eval_same(spec, hw, space, data, rep="real", regs=0.0):
    opts = S.SearchOptions(arith="fastcm", rep_mode=rep, regs_per_thread=regs)
    with S.Plan(spec, hw, space, opts) as plan:
        ec, tag, wocc = plan.evaluate(data)
        win = plan.search_batch(data)
    oec, otag, owocc = _o1_eval(spec, hw, space, data, rep, regs)
    assert np.array_equal(ec.view(np.int64), oec.view(np.int64)), np.argwhere(ec.view(np.int64) != oec.view(np.int64))[:5]
    assert np.array_equal(tag, otag) and np.array_equal(wocc, owocc)
    # The full ranking from the table heads with the search's winner.
    for t in range(min(len(data), 6)):
        res = S.ranking_from_table(A.config_array(space), ec[t], tag[t], wocc[t], hw.W_max, 1e-12)
        if win["cfg_idx"][t] >= 0:
            assert res.ranking[0].config == tuple(int(v) for v in A.config_array(space)[win["cfg_idx"][t]])
            assert res.ties == win["ties"][t]


@pytest.mark.parametrize("kernel", ["2dconv", "gemm", "atax1"])
def test_evaluate_table_c2_models(kernel):
    """rpg_evaluate in the headline arithmetic (the Ec dump): every point
    bit-identical to O1's FAST_CM twin; the ranking of the table heads with
    the search's winner."""
    spec, hw, space = _models(kernel), _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 2731, dtype=np.int64).reshape(-1, 1)  # 24 N (not a multiple of the tile)
    _eval_same(spec, hw, space, data)


@pytest.mark.parametrize("seed", [s for s in range(24) if s % 3 and s % 4])
def test_evaluate_random_models(seed):
    spec, hw, space, data, rep = _case(seed)
    _eval_same(spec, hw, space, data, rep, 24.0)


@pytest.mark.parametrize("seed", range(12))
def test_evaluate_division_edges(seed):
    spec, hw, space, data, rep = _edge_case(seed)
    _eval_same(spec, hw, space, data, rep, 24.0)


def test_search_optimal_single_tuple_fastcm():
    """search_optimal (one tuple, full ranking) in the headline arithmetic."""
    spec, hw, space = _models("gemm"), _b200(), F.integer_configs(1024, dims=2)
    res = S.search_optimal(spec, [4096], hw, space, S.SearchOptions(arith="fastcm"))
    with S.Plan(spec, hw, space, S.SearchOptions(arith="fastcm")) as plan:
        w = plan.search_batch(np.array([[4096]], dtype=np.int64))[0]
    assert res.ranking[0].config == tuple(int(v) for v in A.config_array(space)[w["cfg_idx"]])
    assert len(res.ranking) == w["n_feasible"] and res.evaluated == len(space)


def test_c2_bench_workload_full():
    """The benchmark's default C2 workload in its default mode: all 65,473 N
    x 7,262 configs x 3 kernels (1.426e9 points), every winner record
    byte-identical to O1's FAST_CM twin (all host cores)."""
    hw, space = _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, dtype=np.int64).reshape(-1, 1)
    for k in ("2dconv", "gemm", "atax1"):
        spec = _models(k)
        _same(_gpu(spec, hw, space, data), _o1(spec, hw, space, data), data)


def test_search_batch_out_buffer():
    """search_batch(out=...) fills a caller-provided (e.g. pinned) array with
    the same records it would return, and rejects a mismatched one."""
    spec, hw, space = _models("gemm"), _b200(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 5000, 37, dtype=np.int64).reshape(-1, 1)
    with S.Plan(spec, hw, space, S.SearchOptions(arith="fastcm")) as plan:
        want = plan.search_batch(data)
        out = np.empty(len(data), dtype=A.WINNER_DTYPE)
        got = plan.search_batch(data, out=out)
        assert got is out and np.array_equal(out.view(np.uint8), want.view(np.uint8))
        with pytest.raises(ValueError):
            plan.search_batch(data, out=np.empty(len(data) - 1, dtype=A.WINNER_DTYPE))
