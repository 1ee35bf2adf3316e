"""C6, the non-degenerate landscape (data/stressed/make_c6.py): 22.5 % of
the points infeasible (registers), every winner inside a multi-member exact
tie group (T-symmetric metrics), all three MWP-CWP cases present.  The GPU
search over the whole C6 step (65,473 N x 7,262 configs x 3 kernels) in the
headline arithmetic (FAST_CM) and in FAST against oracle O1 EXACT under the
north-star rule (tests/agree.py), bit-exact against O1's FAST_CM twin and in
EXACT on a strided N sample."""
import os

import numpy as np
import pytest

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

from .agree import assert_agrees_with_exact, exact_winners, threads

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ("c6_stencil", "c6_kloop", "c6_reduce")


def _spec(k):
    return F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "stressed", f"{k}.models.json")))


def _hw():
    return F.load_profile(os.path.join(ROOT, "data", "b200.profile"))


def _gpu(spec, hw, space, data, arith):
    with S.Plan(spec, hw, space, S.SearchOptions(arith=arith)) as plan:
        return plan.search_batch(data)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c6_full_step_vs_exact(kernel):
    spec, hw, space = _spec(kernel), _hw(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, dtype=np.int64).reshape(-1, 1)
    exact = exact_winners(spec, hw, space, data)
    # the landscape is what it claims: infeasible points, multi-member ties
    assert (exact["n_feasible"] < len(space)).all()
    assert (exact["ties"] >= 2).mean() > 0.99
    for arith in ("fastcm", "fast"):
        got = _gpu(spec, hw, space, data, arith)
        assert_agrees_with_exact(got, spec, hw, space, data, exact=exact)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c6_bit_exact_vs_o1_twins(kernel):
    spec, hw, space = _spec(kernel), _hw(), F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 61, dtype=np.int64).reshape(-1, 1)
    pk, hws, cfg = A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), A.config_array(space)
    for arith in ("fastcm", "exact"):
        opts = S.SearchOptions(arith=arith)
        want = o1.search_batch(pk, hws, opts.struct(), cfg, data, threads())
        got = _gpu(spec, hw, space, data, arith)
        assert got.tobytes() == want.tobytes(), arith


def test_c6_covers_every_case():
    """All three MWP-CWP cases and infeasible points occur (Ec dump in the
    headline arithmetic, bit-exact vs O1's FAST_CM twin)."""
    hw, space = _hw(), F.integer_configs(1024, dims=2)
    data = np.array([64, 200, 1000, 3000, 10000, 30000, 65536], dtype=np.int64).reshape(-1, 1)
    seen = set()
    for k in KERNELS:
        spec = _spec(k)
        opts = S.SearchOptions(arith="fastcm")
        with S.Plan(spec, hw, space, opts) as plan:
            ec, tag, wocc = plan.evaluate(data)
        oec, otag, owocc = o1.evaluate_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw),
                                             opts.struct(), A.config_array(space), data, threads())
        assert np.array_equal(ec.view(np.int64), oec.view(np.int64))
        assert np.array_equal(tag, otag) and np.array_equal(wocc, owocc)
        assert (ec < 0).any()
        seen |= set(np.unique(tag[ec >= 0]).tolist())
    assert {A.RPG_CASE_BOTH_SATURATED, A.RPG_CASE_CWP_BOUND, A.RPG_CASE_MWP_BOUND} <= seen
