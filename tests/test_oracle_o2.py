"""Pins O2 (exact-rational program semantics) to the reference's exact KATs
and measures O1 (FP64) against it — the reference's own
"program mirrors the closed form within 1e-9" criterion (CPU only)."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import o1, o2_exact as o2
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F

from . import zoo


@pytest.mark.parametrize("name,hw,m,total", [
    ("cwp_bound", zoo.oracle_hw(), (18, 1, 1, 0, 4), 1640),
    ("both_saturated", zoo.oracle_hw(B_max=2, departure_del_coal_cycles=50), (23, 0, 2, 3, 2), 1050),
    ("mwp_bound", zoo.oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=75, mem_bandwidth_GBps=4),
     (98, 0, 2, 0, 16), 3500),
    ("raw_latency_pin", zoo.oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=30,
                                      departure_del_uncoal_cycles=30, mem_bandwidth_GBps=4),
     (98, 1, 1, 0, 16), 3500),
])
def test_program_reproduces_hand_oracles_exactly(name, hw, m, total):
    # test_perfmodel.cpp:440-497
    assert o2.program_value(zoo.const_spec(*m), hw, [64], (32, 1, 1)) == Fraction(total)


def test_singular_denominator_sentinel():
    # test_perfmodel.cpp:544-556
    spec = zoo.stencil_spec()
    spec.models[F.METRIC_COAL] = F.make_ratfunc(["D1", "bx", "by"], [0, 0, 0], [9], [0, 1, 0], [-32, 1])
    assert o2.program_value(spec, zoo.sample_hw(), [64], (32, 2, 1)) == -1
    assert o2.program_value(spec, zoo.sample_hw(), [64], (16, 2, 1)) != -1


def test_occupancy_guards():
    spec = zoo.stencil_spec()
    assert o2.program_value(spec, zoo.sample_hw(), [64], (64, 32, 1)) == -1   # T > T_max
    assert o2.program_value(zoo.const_spec(10, 1, 1, 0, 4), zoo.oracle_hw(B_max=1), [64], (8, 1, 1)) == -1


@pytest.mark.parametrize("case", [c for c in zoo.cases() if c.name in (
    "stencil_truth_pow2", "stencil_truth_ceil", "random3_0", "random3_3", "regs_shared_models",
    "data_after_blocks", "oracle_both", "singular_coal")], ids=lambda c: c.name)
def test_o1_within_1e9_of_exact_program(case):
    """O1 (FP64 direct order, program feasibility) vs O2 (exact program):
    identical feasibility and Ec within 1e-9 relative (test_perfmodel.cpp:
    499-542, test_pipeline.cpp:303-346) on a sample of each case."""
    pk = A.PackedModel(case.spec, drop_zero_terms=False)
    opts = A.options_struct(rep_mode=A.RPG_REP_CEIL if case.rep_mode == "ceil" else A.RPG_REP_REAL)
    data = case.data[:2]
    space = case.space[:: max(1, len(case.space) // 40)]
    ec, _, _ = o1.evaluate_batch(pk, A.profile_struct(case.hw), opts, A.config_array(space), data)
    for t in range(len(data)):
        for j, c in enumerate(space):
            exact = o2.program_value(case.spec, case.hw, list(data[t]), c, case.rep_mode)
            got = ec[t, j]
            if exact == -1:
                assert got == -1.0, (t, c)
            elif exact < 0:
                assert got < 0
            else:
                assert got >= 0
                assert abs(got - float(exact)) <= 1e-9 * max(1.0, abs(float(exact))), (t, c, got, float(exact))


def test_exact_winner_agreement_sample():
    """The FP64 winner (O1) lies in the exact tie group widened to 1e-9 for
    sampled tuples of the stencil and a random dense model."""
    for case in [c for c in zoo.cases() if c.name in ("stencil_truth_pow2", "random3_0")]:
        pk = A.PackedModel(case.spec, drop_zero_terms=False)
        for t in range(2):
            w, order = o1.search_one(pk, A.profile_struct(case.hw), A.options_struct(),
                                     A.config_array(case.space), case.data[t])
            vals, feas, ties = o2.search(case.spec, case.hw, list(case.data[t]), case.space)
            best = vals[feas[0]]
            assert vals[w.cfg_idx] <= best * (1 + Fraction(1, 10 ** 9))
