"""GPU parity of the bare-program path (`ratprog search --rp`, SURVEY.md 8
f1): programs the reference's emitter writes (oracle O4 restatement) and the
reference's own IR test programs, evaluated by the NVRTC-generated sm_100a
kernels through the C ABI and compared with O4:

* per-point values bit-identical to the C lowering's doubles (O4.evaluate_c);
* winners, best Ec, tie counts and feasible counts identical to
  search_optimal's rules applied to those doubles;
* against the exact-rational interpreter (what the reference ranks): every
  value within 1e-9 relative (pipeline.hpp:271-274) and the winner's exact
  value inside the exact tie window of the exact best;
* the interpreter's errors (zero divisor, step limit, unassigned read,
  falling off the end) and make_binding_plan's PipelineErrors.
"""
import os

import numpy as np
import pytest

from oracle import o4_program as O4
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import program as P
from paper_1906_00142_b200 import search as S

from . import zoo
from .test_program import EARLY, FLOOR_DIV, LOOP_FOREVER, PLATEAU, REMAINDER, WHILE

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAX_CFG = 160


def _cases():
    out = []
    for case in zoo.cases():
        space = case.space[:: max(1, len(case.space) // MAX_CFG)][:MAX_CFG]
        out.append((case, space, case.data[:2]))
    return out


CASES = _cases()


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[c[0].name for c in CASES])
def test_emitted_program_values_and_winners_match_c_lowering(idx):
    case, space, data = CASES[idx]
    prog = O4.generate_rp(case.spec, case.hw, case.rep_mode)
    opts = S.SearchOptions(regs_per_thread=case.regs_fallback,
                           shared_words_per_block=case.shared_fallback)
    with S.Plan(P.serialize(prog), case.hw, space, opts) as plan:
        ec, tag, wocc = plan.evaluate(data)
        win = plan.search_batch(data)
    for t in range(len(data)):
        row = [int(x) for x in data[t]]
        want = [O4.evaluate_c(prog, O4.bindings_for(prog, row, case.hw, c)) for c in space]
        np.testing.assert_array_equal(ec[t], np.array(want), err_msg=case.name)
        assert (tag[t] == 3).all()
        occ = [O4.occupancy_warps(case.hw, case.regs_fallback, case.shared_fallback,
                                  c[0] * c[1] * c[2]) for c in space]
        np.testing.assert_array_equal(wocc[t], np.array(occ))
        feas = [i for i, v in enumerate(want) if v >= 0]
        w = win[t]
        assert w["n_feasible"] == len(feas)
        if not feas:
            assert w["cfg_idx"] == -1
            continue
        vals, order, ties, _ = O4.search(prog, row, case.hw, space, case.regs_fallback,
                                         case.shared_fallback)
        assert w["cfg_idx"] == order[0], case.name
        assert w["ec"] == vals[order[0]] and w["best_ec"] == min(vals[i] for i in feas)
        assert w["ties"] == ties
        assert w["w_occ"] == occ[order[0]]


@pytest.mark.parametrize("idx", range(0, len(CASES), 3), ids=[c[0].name for c in CASES][::3])
def test_emitted_program_against_exact_interpreter(idx):
    case, space, data = CASES[idx]
    space = space[:48]
    prog = O4.generate_rp(case.spec, case.hw, case.rep_mode)
    row = [int(x) for x in data[0]]
    opts = S.SearchOptions(regs_per_thread=case.regs_fallback,
                           shared_words_per_block=case.shared_fallback)
    with S.Plan(prog, case.hw, space, opts) as plan:
        ec, _, _ = plan.evaluate(np.array([row], dtype=np.int64))
        win = plan.search_batch(np.array([row], dtype=np.int64))[0]
    exact = [O4.evaluate_exact(prog, O4.bindings_for(prog, row, case.hw, c)) for c in space]
    for g, x in zip(ec[0], exact):
        if x == -1:
            assert g == -1.0
        else:
            assert abs(g - float(x)) <= 1e-9 * max(1.0, abs(float(x)))
    feas = [i for i, v in enumerate(exact) if v >= 0]
    if feas:
        best = min(exact[i] for i in feas)
        # the GPU winner is in the reference's (exact) tie window, up to the
        # lowering's rounding
        assert float(exact[win["cfg_idx"]]) <= float(best) * (1 + 1e-9) + 1e-9


def _plan(text, space=((32, 1, 1), (64, 2, 1), (128, 1, 1)), step_limit=1_000_000):
    return S.Plan(text, zoo.sample_hw(), list(space), S.SearchOptions(), step_limit=step_limit)


def test_reference_ir_programs_on_the_gpu():
    """test_ir_core.cpp's programs with A/B bound to data parameters."""
    fd = FLOOR_DIV.replace("A", "D1").replace("B", "D2")
    with _plan(fd) as plan:
        ec, _, _ = plan.evaluate(np.array([[7, 2], [-7, 2], [8, 2], [-9, 4]], dtype=np.int64))
        assert ec[:, 0].tolist() == [3, -4, 4, -3] and (ec == ec[:, :1]).all()
    rem = REMAINDER.replace("A", "D1").replace("B", "D2")
    data = np.array([[a, b] for a in range(-6, 7) for b in (1, 2, 3, -2)], dtype=np.int64)
    with _plan(rem) as plan:
        ec, _, _ = plan.evaluate(data)
        assert ec[:, 1].tolist() == [float(a % abs(b)) for a, b in data]
    with _plan(WHILE.replace("X", "D1")) as plan:
        ec, _, _ = plan.evaluate(np.array([[10], [0], [1000]], dtype=np.int64))
        assert ec[:, 2].tolist() == [10, 0, 1000]
    with _plan(PLATEAU.replace("A", "D1")) as plan:
        ec, _, _ = plan.evaluate(np.array([[16], [20], [23], [40]], dtype=np.int64))
        assert ec[:, 0].tolist() == [32, 40, 46, 200]
    # block dimensions as inputs: Y = bx * by - D1 (feasible iff >= 0)
    with _plan("inputs: bx by D1\noutput: Y\n0: mul t bx by\n1: sub Y t D1\n2: halt_return Y\n") as plan:
        r = plan.search_batch(np.array([[40], [100]], dtype=np.int64))
        # 32 - D1 < 0 is infeasible; (64,2,1) and (128,1,1) tie at 128 - D1 with
        # equal occupancy: lex order picks (64,2,1)
        assert r["cfg_idx"].tolist() == [1, 1] and r["ec"].tolist() == [88, 28]
        assert r["ties"].tolist() == [2, 2] and r["n_feasible"].tolist() == [2, 2]


def test_interpreter_errors_surface_from_the_gpu():
    fd = FLOOR_DIV.replace("A", "D1").replace("B", "D2")
    with _plan(fd) as plan:
        with pytest.raises(P.DivisionByZero, match=r"floor_div: zero divisor \[tuple 1"):
            plan.search_batch(np.array([[1, 2], [1, 0], [3, 0]], dtype=np.int64))
        # the plan stays usable after an error
        assert plan.evaluate(np.array([[9, 2]], dtype=np.int64))[0][0, 0] == 4
    with _plan(LOOP_FOREVER.replace("X", "D1"), step_limit=1000) as plan:
        with pytest.raises(P.StepLimitExceeded, match="step limit of 1000"):
            plan.evaluate(np.array([[1]], dtype=np.int64))
    with _plan(EARLY.replace("X", "D1")) as plan:
        ec, _, _ = plan.evaluate(np.array([[-2]], dtype=np.int64))
        assert (ec == -4).all()
        with pytest.raises(P.MissingBinding, match="'T'"):
            plan.evaluate(np.array([[-2], [2]], dtype=np.int64))
    with _plan("inputs: D1\noutput: Y\n0: assign Y D1\n") as plan:
        with pytest.raises(P.EvalError, match="fell off the end"):
            plan.search_batch(np.array([[1]], dtype=np.int64))
    with _plan("inputs: D1\noutput: Y\n0: ceil_div Y 1 0\n1: halt_return Y\n") as plan:
        with pytest.raises(P.DivisionByZero, match="ceil_div"):
            plan.evaluate(np.array([[1]], dtype=np.int64))


def test_binding_errors():
    with _plan("inputs: D2\noutput: Y\n0: assign Y D2\n1: halt_return Y\n") as plan:
        with pytest.raises(F.PipelineError, match="'D2' has no value: 1 data parameter"):
            plan.search_batch(np.array([[1]], dtype=np.int64))
        assert plan.search_batch(np.array([[1, 5]], dtype=np.int64))["ec"][0] == 5
    with pytest.raises(F.PipelineError, match="neither a block dimension"):
        _plan("inputs: foo\noutput: Y\n0: assign Y foo\n1: halt_return Y\n")


def test_search_optimal_ranking_for_a_program():
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    prog = O4.generate_rp(spec, hw)
    space = F.enumerate_configs()
    res = S.search_optimal(prog, [1024], hw, space, S.SearchOptions())
    vals, order, ties, wocc = O4.search(prog, [1024], hw, space)
    assert [r.config for r in res.ranking] == [tuple(space[i]) for i in order]
    assert [r.estimated_cycles for r in res.ranking] == [vals[i] for i in order]
    assert res.ties == ties and res.evaluated == len(space)
    assert all(r.case_tag == "-" for r in res.ranking)
