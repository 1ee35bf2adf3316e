"""GPU parity: the CUDA evaluator (through the C ABI) against oracle O1.

Bar (BASELINE.json north_star): occupancy, block counts, case tags and the
chosen configuration bit-exact; Ec bit-exact in EXACT mode (O1 restates the
reference's operation order with -ffp-contract=off, the kernel compiles with
-fmad=false), and bit-exact against O1's FAST twin in FAST mode.  FAST vs the
reference's order is checked at the north star's tolerance: Ec within 1e-9
relative, winners equal or inside O1's tie group.
"""
import numpy as np
import pytest

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

from . import zoo

pytestmark = pytest.mark.gpu

CASES = zoo.cases(small=True)
IDS = [c.name for c in CASES]


def _opts(c, arith, kernel="specialized"):
    return S.SearchOptions(regs_per_thread=c.regs_fallback,
                           shared_words_per_block=c.shared_fallback,
                           rep_mode=c.rep_mode, arith=arith, kernel=kernel)


def _oracle(c, arith, what):
    pk = A.PackedModel(c.spec, drop_zero_terms=False)
    opts = _opts(c, arith).struct()
    hw = A.profile_struct(c.hw)
    space = A.config_array(c.space)
    if what == "evaluate":
        return o1.evaluate_batch(pk, hw, opts, space, c.data, 8)
    return o1.search_batch(pk, hw, opts, space, c.data, 8)


@pytest.mark.parametrize("kernel", ["specialized", "generic"])
@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_evaluate_bit_exact(case, arith, kernel):
    with S.Plan(case.spec, case.hw, case.space, _opts(case, arith, kernel)) as plan:
        ec, tag, wocc = plan.evaluate(case.data)
    oec, otag, owocc = _oracle(case, arith, "evaluate")
    assert np.array_equal(ec.view(np.int64), oec.view(np.int64)) or np.array_equal(ec, oec), (
        np.argwhere(ec != oec)[:5], ec[ec != oec][:5], oec[ec != oec][:5])
    assert np.array_equal(tag, otag)
    assert np.array_equal(wocc, owocc)


@pytest.mark.parametrize("kernel", ["specialized", "generic"])
@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_search_winners_bit_exact(case, arith, kernel):
    with S.Plan(case.spec, case.hw, case.space, _opts(case, arith, kernel)) as plan:
        got = plan.search_batch(case.data)
    want = _oracle(case, arith, "search")
    for f in ("cfg_idx", "ties", "n_feasible", "b_active", "w_active", "w_occ", "case_tag"):
        assert np.array_equal(got[f], want[f]), (f, got[f], want[f])
    assert np.array_equal(got["ec"], want["ec"])
    assert np.array_equal(got["best_ec"], want["best_ec"])


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_fast_mode_within_tolerance_of_reference_order(case):
    """FAST (collapse + DFMA) vs the reference's operation order (O1 EXACT):
    Ec within 1e-9 relative wherever both are feasible; winner equal or a
    member of the exact tie group at 1e-9."""
    with S.Plan(case.spec, case.hw, case.space, _opts(case, "fast")) as plan:
        ec, tag, wocc = plan.evaluate(case.data)
        win = plan.search_batch(case.data)
    oec, otag, owocc = _oracle(case, "exact", "evaluate")
    both = (ec >= 0) & (oec >= 0)
    rel = np.abs(ec[both] - oec[both]) / np.maximum(1.0, np.abs(oec[both]))
    assert rel.max(initial=0.0) <= 1e-9
    for t in range(len(case.data)):
        idx = int(win["cfg_idx"][t])
        row = oec[t]
        feas = row >= 0
        if idx < 0:
            assert not feas.any() or (feas & ~(ec[t] >= 0)).any()
            continue
        best = row[feas].min()
        assert row[idx] >= 0 and row[idx] <= best * (1 + 1e-9) + 1e-300


@pytest.mark.parametrize("case", CASES[:10], ids=IDS[:10])
def test_single_tuple_ranking_matches_oracle(case):
    """search_optimal drop-in: full ranking order, ties, counts."""
    for t in range(min(3, len(case.data))):
        data = case.data[t]
        try:
            res = S.search_optimal(case.spec, list(data), case.hw, case.space, _opts(case, "exact"))
        except S.NoFeasibleConfig:
            res = None
        pk = A.PackedModel(case.spec, drop_zero_terms=False)
        w, order = o1.search_one(pk, A.profile_struct(case.hw), _opts(case, "exact").struct(),
                                 A.config_array(case.space), data)
        if w.n_feasible == 0:
            assert res is None
            continue
        assert res.ties == w.ties
        assert res.evaluated == len(case.space)
        assert len(res.ranking) == w.n_feasible
        got = [r.config for r in res.ranking]
        want = [tuple(int(v) for v in case.space[i]) for i in order]
        assert got == want


def test_errors_mirror_reference():
    spec = zoo.stencil_spec()
    with pytest.raises(ValueError, match="configuration space is empty"):
        S.search_optimal(spec, [64], zoo.sample_hw(), [])
    spec2 = zoo.random_spec(np.random.default_rng(1), ["D2", "bx", "by"])
    with S.Plan(spec2, zoo.sample_hw(), F.enumerate_configs()) as plan:
        with pytest.raises(F.PipelineError, match="D2"):
            plan.search_batch(np.array([[64]], dtype=np.int64))


def test_no_feasible_config_flag():
    # Every config infeasible: registers starve every block.
    spec = zoo.const_spec(10, 1, 1, 0, 4, R=1e9)
    with S.Plan(spec, zoo.sample_hw(), F.enumerate_configs()) as plan:
        w = plan.search_batch(np.array([[64], [128]], dtype=np.int64))
    assert (w["cfg_idx"] == -1).all() and (w["n_feasible"] == 0).all()
    with pytest.raises(S.NoFeasibleConfig):
        S.search_optimal(spec, [64], zoo.sample_hw(), F.enumerate_configs())


@pytest.mark.parametrize("kernel", ["specialized", "generic"])
def test_large_space_3d(kernel):
    """The full 30,343-config 3-D space (C5 shape)."""
    rng = np.random.default_rng(7)
    spec = zoo.random_spec(rng, ["D1", "D2", "bx", "by", "bz"], sparsity=0.5)
    space = F.integer_configs(dims=3)
    data = rng.integers(16, 2049, size=(6, 2))
    c = zoo.Case("big3d", spec, zoo.b200_hw(), space, data)
    with S.Plan(spec, c.hw, space, _opts(c, "exact", kernel)) as plan:
        got = plan.search_batch(data)
    want = _oracle(c, "exact", "search")
    assert np.array_equal(got, want)


@pytest.mark.parametrize("tol", [0.0, 1e-12])
@pytest.mark.parametrize("arith,kernel", [("exact", "specialized"), ("fast", "specialized"),
                                          ("exact", "generic"), ("fast", "generic"), ("fastcm", "specialized")])
def test_infinite_cycle_estimates_and_empty_tie_group(tol, arith, kernel):
    """Every feasible Ec is +inf (an overflowing metric).  With tol = 0 the
    tie bound is inf + inf*0 = NaN, the tie group is empty and the ranking's
    head is the lowest (Ec, lex) config with ties = 0 (O1, and the
    reference's sort); with tol > 0 the group is every config.  Records
    bit-identical to O1 either way."""
    from .zoo import b200_hw, const_spec
    hw, space = b200_hw(), F.enumerate_configs()
    data = np.array([[100], [2000]], dtype=np.int64)
    for comp, unc, coal, syn, tb in [(1e308, 1, 1, 1, 1), (1, 1e308, 1e308, 1, 1), (1, 1, 1, 1, 1e308)]:
        spec = const_spec(comp, unc, coal, syn, tb)
        opts = S.SearchOptions(arith=arith, kernel=kernel, tie_rel_tol=tol)
        want = o1.search_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), opts.struct(),
                               A.config_array(space), data, 2)
        with S.Plan(spec, hw, space, opts) as plan:
            got = plan.search_batch(data)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (got, want)
