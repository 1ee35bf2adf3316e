"""Randomized GPU-vs-O1 parity: many random models, profiles, spaces and data
tuples, with metric magnitudes spread over many decades (so the division
fast paths, the quotient-based near-zero test and the IEEE fall-back all get
exercised), signed coefficients (negative metrics, infeasible points),
tiny/huge denominators, both repetition modes, both arithmetic modes and
both kernels.  Evaluate tables and winner records must be bit-identical."""
import numpy as np
import pytest

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import search as S

from . import zoo

pytestmark = pytest.mark.gpu

N_CASES = 24


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    variables = ["D1", "bx", "by"] if seed % 3 else ["D1", "D2", "bx", "by", "bz"]
    spec = zoo.random_spec(rng, variables, positive=bool(seed % 2), sparsity=0.3)
    # Spread magnitudes: scale every metric's numerator and denominator by
    # random powers of ten (the quotient's magnitude moves by their ratio).
    for name, f in spec.models.items():
        pn = 10.0 ** rng.integers(-6, 7)
        pd = 10.0 ** rng.integers(-4, 5)
        f.num.coeffs = [c * pn for c in f.num.coeffs]
        f.den.coeffs = [c * pd for c in f.den.coeffs]
        if seed % 5 == 0 and name == F.METRIC_SYNCH:
            f.den.coeffs = [c * 1e-13 for c in f.den.coeffs]   # near-singular denominators
    if seed % 4 == 0:  # register / shared models instead of constants
        del spec.constants[F.METRIC_REGS]
        spec.models[F.METRIC_REGS] = F.make_ratfunc(variables, [0] * (len(variables) - 2) + [1, 1],
                                                    [16.0, 0.01, 0.02, 0.0001], [0] * len(variables), [1.0])
    hw = zoo.random_hw(rng)
    dims = 3 if "bz" in variables else 2
    full = F.integer_configs(1024, dims=dims)
    idx = np.sort(rng.choice(len(full), size=min(len(full), int(rng.integers(40, 900))), replace=False))
    space = [full[i] for i in idx]
    d = len(variables) - dims
    data = rng.integers(1, 70000, size=(int(rng.integers(3, 12)), d)).astype(np.int64)
    rep = "ceil" if seed % 3 == 2 else "real"
    return spec, hw, space, data, rep


def _opts(arith, kernel, rep):
    return S.SearchOptions(arith=arith, kernel=kernel, rep_mode=rep, regs_per_thread=24.0,
                           shared_words_per_block=0.0)


@pytest.mark.parametrize("kernel", ["specialized", "generic"])
@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_bit_exact(seed, arith, kernel):
    spec, hw, space, data, rep = _case(seed)
    opts = _opts(arith, kernel, rep)
    pk = A.PackedModel(spec, drop_zero_terms=False)
    args = (pk, A.profile_struct(hw), opts.struct(), A.config_array(space), data)
    oec, otag, owocc = o1.evaluate_batch(*args, 4)
    owin = o1.search_batch(*args, 4)
    with S.Plan(spec, hw, space, opts) as plan:
        ec, tag, wocc = plan.evaluate(data)
        win = plan.search_batch(data)
    assert np.array_equal(ec.view(np.int64), oec.view(np.int64)), np.argwhere(ec.view(np.int64) != oec.view(np.int64))[:5]
    assert np.array_equal(tag, otag)
    assert np.array_equal(wocc, owocc)
    assert np.array_equal(win.view(np.uint8), owin.view(np.uint8)), (win, owin)


def _edge_case(seed):
    """Metric magnitudes around the specialized kernel's quotient range
    tests (rpg_device.cuh ratio_fast / FastDiv): numerators near 2^-969 and
    2^-928 (tiny dividend, tiny quotient), denominators near 2^-39, quotients
    near 2^38, plus plain ones — each metric picks one regime at random."""
    rng = np.random.default_rng(5000 + seed)
    variables = ["D1", "bx", "by"]
    spec = zoo.random_spec(rng, variables, positive=True, sparsity=0.3)
    regimes = [(-969, 0), (-928, 0), (-931, -39), (0, -39), (0, -41), (38, 0), (36, -3), (0, 0)]
    for f in spec.models.values():
        en, ed = regimes[int(rng.integers(len(regimes)))]
        en += int(rng.integers(-3, 4))
        ed += int(rng.integers(-3, 4))
        f.num.coeffs = [c * 2.0 ** en for c in f.num.coeffs]
        f.den.coeffs = [c * 2.0 ** ed for c in f.den.coeffs]
    hw = zoo.random_hw(rng)
    full = F.integer_configs(1024, dims=2)
    idx = np.sort(rng.choice(len(full), size=int(rng.integers(200, 900)), replace=False))
    data = rng.integers(1, 70000, size=(int(rng.integers(3, 9)), 1)).astype(np.int64)
    return spec, hw, [full[i] for i in idx], data, "real"


@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("seed", range(12))
def test_fuzz_division_edges_bit_exact(seed, arith):
    spec, hw, space, data, rep = _edge_case(seed)
    opts = _opts(arith, "specialized", rep)
    pk = A.PackedModel(spec, drop_zero_terms=False)
    args = (pk, A.profile_struct(hw), opts.struct(), A.config_array(space), data)
    oec, otag, owocc = o1.evaluate_batch(*args, 4)
    owin = o1.search_batch(*args, 4)
    with S.Plan(spec, hw, space, opts) as plan:
        ec, tag, wocc = plan.evaluate(data)
        win = plan.search_batch(data)
    assert np.array_equal(ec.view(np.int64), oec.view(np.int64))
    assert np.array_equal(tag, otag)
    assert np.array_equal(wocc, owocc)
    assert np.array_equal(win.view(np.uint8), owin.view(np.uint8)), (win, owin)
