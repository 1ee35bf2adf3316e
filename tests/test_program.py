"""Bare rational programs on the CPU: the `.rp` parser, oracle O4 (the
program emitters, the exact interpreter and the C lowering) pinned against
the reference's own IR tests (test_ir_core.cpp) and against O2, the lowering
for the C ABI, and NVRTC compilation of the generated program kernels."""
import ctypes as C
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import o2_exact as O2
from oracle import o4_program as O4
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import program as P

from . import zoo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# test_ir_core.cpp:44-53
DIAMOND = ("# pick a value depending on the comparison\n"
           "inputs: A B\n"
           "output: Y\n"
           "0: cmp_lt c A B\n"
           "1: branch_if c -> 2 4\n"
           "2: mul Y A B\n"
           "3: jump -> 5\n"
           "4: sub Y A B\n"
           "5: halt_return Y\n")
FLOOR_DIV = "inputs: A B\noutput: Y\n0: floor_div Y A B\n1: halt_return Y\n"
REMAINDER = ("inputs: A B\noutput: Y\n0: euclid_quot Q A B\n1: mul QB Q B\n"
             "2: sub Y A QB\n3: halt_return Y\n")
LOOP_FOREVER = "inputs: X\noutput: Y\n0: assign Y X\n1: jump -> 1\n2: halt_return Y\n"
EARLY = ("inputs: X\noutput: Y\n0: cmp_lt c X 0\n1: branch_if c -> 2 3\n2: assign T X\n"
         "3: add Y T X\n4: halt_return Y\n")
WHILE = ("inputs: X\noutput: I\n0: assign I 0\n1: cmp_lt c I X\n2: branch_if c -> 3 5\n"
         "3: add I I 1\n4: jump -> 1\n5: halt_return I\n")
PLATEAU = "inputs: A\noutput: Y\n0: floor_div f A 8\n1: mul Y f A\n2: halt_return Y\n"

EVALS = [("exact", O4.evaluate_exact), ("c", O4.evaluate_c)]


def b2(a, b):
    return {"A": a, "B": b}


# ---------------------------------------------------------------------------
# Parser (ir_text.hpp; test_ir_core.cpp:288-336)

@pytest.mark.parametrize("text,needle", [
    ("inputs: A\noutput: Y\n0: frobnicate Y A A\n1: halt_return Y\n", "unknown opcode 'frobnicate'"),
    ("inputs: A\noutput: Y\n5: assign Y A\n", "out of order"),
    ("inputs: A\noutput: Y\n0: assign Y 1/0\n", "zero denominator"),
    ("inputs: A\noutput: Y\n0: assign Y 2.5\n", "decimal"),
    ("inputs: A\n0: assign Y A\n", "output:"),
    ("output: Y\n", "inputs:"),
    ("inputs: A\noutput: Y\n0: add Y A\n", "expects 3 argument(s)"),
    ("inputs: A\noutput: Y\n0: jump 3\n", "0 argument(s)"),
])
def test_parse_errors_name_the_cause(text, needle):
    with pytest.raises(P.ParseError) as e:
        P.parse(text)
    assert needle in str(e.value)


def test_parse_error_location():
    with pytest.raises(P.ParseError) as e:
        P.parse("inputs: A\noutput: Y\n0: assign Y 1/0\n")
    assert e.value.line == 3 and e.value.column >= 11


def test_parse_skips_comments_and_blank_lines():
    p = P.parse("# leading comment\n\ninputs: A B\n# middle comment\noutput: Y\n"
                "0: mul Y A B  # trailing comment\n1: halt_return Y\n")
    assert O4.evaluate_exact(p, b2(6, 7)) == 42


def test_serialize_parse_round_trip_and_rational_literals():
    for text in (DIAMOND, FLOOR_DIV, REMAINDER, WHILE):
        p = P.parse(text)
        q = P.parse(P.serialize(p))
        assert q == p and P.serialize(q) == P.serialize(p)
    b = O4.Builder()
    b.input("X")
    b.output("Y")
    b.mul("Y", O4.var("X"), O4.lit(Fraction(-7, 3)))
    b.halt_return("Y")
    p = b.finish()
    text = P.serialize(p)
    assert "-7/3" in text and P.parse(text) == p


# ---------------------------------------------------------------------------
# Interpreters (test_ir_core.cpp:156-205, 246-262, 338-349, 351-363, 419-444)

@pytest.mark.parametrize("name,ev", EVALS)
def test_integer_part_operations(name, ev):
    p = P.parse(FLOOR_DIV)
    assert ev(p, b2(7, 2)) == 3 and ev(p, b2(-7, 2)) == -4 and ev(p, b2(8, 2)) == 4
    r = P.parse(REMAINDER)
    assert ev(r, b2(7, 2)) == 1 and ev(r, b2(-7, 2)) == 1 and ev(r, b2(7, -2)) == 1
    for a in range(-6, 7):
        for bb in range(1, 4):
            v = ev(r, b2(a, bb))
            assert v == int(v) and v == a % bb


@pytest.mark.parametrize("name,ev", EVALS)
def test_branches_loops_and_min(name, ev):
    p = P.parse(DIAMOND)
    assert ev(p, b2(3, 5)) == 15 and ev(p, b2(5, 3)) == 2 and ev(p, b2(4, 4)) == 0
    assert ev(P.parse(WHILE), {"X": 10}) == 10
    b = O4.Builder()
    b.input("A")
    b.input("B")
    b.output("Y")
    b.emit_min("Y", O4.var("A"), O4.var("B"))
    b.halt_return("Y")
    m = b.finish()
    assert ev(m, b2(3, 5)) == 3 and ev(m, b2(5, 3)) == 3 and ev(m, b2(4, 4)) == 4
    pl = P.parse(PLATEAU)
    assert [ev(pl, {"A": a}) for a in (16, 20, 23, 40)] == [32, 40, 46, 200]


@pytest.mark.parametrize("name,ev", EVALS)
def test_interpreter_errors(name, ev):
    p = P.parse(FLOOR_DIV)
    with pytest.raises(P.MissingBinding):
        ev(p, {"A": 1})
    with pytest.raises(P.DivisionByZero, match="floor_div: zero divisor"):
        ev(p, b2(1, 0))
    with pytest.raises(P.StepLimitExceeded, match="step limit of 1000"):
        ev(P.parse(LOOP_FOREVER), {"X": 1}, 1000)
    early = P.parse(EARLY)
    assert ev(early, {"X": -2}) == -4
    with pytest.raises(P.MissingBinding, match="'T'"):
        ev(early, {"X": 2})
    fell = P.parse("inputs: X\noutput: Y\n0: assign Y X\n")
    with pytest.raises(P.EvalError, match="fell off the end"):
        ev(fell, {"X": 1})
    with pytest.raises(ValueError):
        ev(fell, {"X": 1}, 0)


def test_specialize_bakes_inputs():
    p = P.parse(DIAMOND)
    q = O4.specialize(p, {"B": Fraction(5)})
    assert q.inputs == ["A"]
    assert O4.evaluate_exact(q, {"A": 3}) == O4.evaluate_exact(p, b2(3, 5))
    assert O4.evaluate_exact(q, {"A": 9}) == O4.evaluate_exact(p, b2(9, 5))
    assert P.parse(P.serialize(q)) == q
    with pytest.raises(ValueError):
        O4.specialize(p, {"nope": Fraction(1)})


def test_c_lowering_int64_path_and_double_path():
    p = P.parse(FLOOR_DIV)
    # integral operands below 9e15: exact int64 quotient with floor correction
    assert O4.evaluate_c(p, b2(-9_000_000_000_000_001 + 2, 3)) == (-9_000_000_000_000_001 + 2) // 3
    # non-integral operand: floor of the rounded double quotient
    assert O4.evaluate_c(p, {"A": Fraction(7, 2), "B": 2}) == 1.0
    ceil = P.parse("inputs: A B\noutput: Y\n0: ceil_div Y A B\n1: halt_return Y\n")
    for a, b in [(7, 2), (-7, 2), (7, -2), (-7, -2), (6, 3)]:
        assert O4.evaluate_c(ceil, b2(a, b)) == O4.evaluate_exact(ceil, b2(a, b)) == -((-a) // b)


# ---------------------------------------------------------------------------
# Emitters, pinned against O2 (which the reference's KATs pin)

def test_occupancy_program_matches_direct_occupancy():
    hw = zoo.sample_hw()
    p = O4.generate_occupancy_rp(hw)
    assert p.inputs == ["R", "Z", "T"]
    for R in (0, 16, 32, 63.5):
        for Z in (0, 100, 5000):
            for T in (0, 1, 31, 32, 96, 256, 1024, 1025):
                w = O4.evaluate_exact(p, {"R": Fraction(R), "Z": Fraction(Z), "T": T})
                assert w == O4.occupancy_warps(hw, R, Z, T), (R, Z, T)


@pytest.mark.parametrize("rep_mode", ["real", "ceil"])
def test_emitted_program_exact_value_equals_o2(rep_mode):
    rng = np.random.default_rng(7)
    n = 0
    for case in zoo.cases():
        prog = O4.generate_rp(case.spec, case.hw, rep_mode)
        assert sorted(prog.inputs) == sorted(case.spec.variables)
        assert P.parse(P.serialize(prog)) == prog
        for t in rng.choice(len(case.data), size=min(2, len(case.data)), replace=False):
            data = [int(x) for x in case.data[t]]
            for c in rng.choice(len(case.space), size=min(4, len(case.space)), replace=False):
                cfg = tuple(case.space[c])
                got = O4.evaluate_exact(prog, O4.bindings_for(prog, data, case.hw, cfg))
                assert got == O2.program_value(case.spec, case.hw, data, cfg, rep_mode), \
                    (case.name, data, cfg)
                n += 1
    assert n > 100


def test_c_lowering_within_reference_tolerance_of_exact():
    """pipeline.hpp:271-274: the C lowering agrees with the interpreter
    within 1e-9 relative away from branch boundaries."""
    rng = np.random.default_rng(11)
    worst = 0.0
    for case in zoo.cases()[:12]:
        prog = O4.generate_rp(case.spec, case.hw, case.rep_mode)
        data = [int(x) for x in case.data[0]]
        for c in rng.choice(len(case.space), size=min(6, len(case.space)), replace=False):
            b = O4.bindings_for(prog, data, case.hw, tuple(case.space[c]))
            ex = O4.evaluate_exact(prog, b)
            cv = O4.evaluate_c(prog, b)
            if ex == -1:  # the infeasible sentinel is exact
                assert cv == -1.0
                continue
            worst = max(worst, abs(cv - float(ex)) / max(1.0, abs(float(ex))))
    assert worst < 1e-9


# ---------------------------------------------------------------------------
# Lowering for the C ABI

def test_lowering_binds_inputs_like_make_binding_plan():
    hw = zoo.sample_hw()
    prog = P.parse("inputs: bx D2 mem_latency_cycles by bz D1\noutput: Y\n"
                   "0: add Y bx 1/3\n1: halt_return Y\n")
    low = P.LoweredProgram(prog, hw)
    s = low.struct
    kinds = [s.input_kind[i] for i in range(s.n_inputs)]
    assert kinds == [A.RPG_VAR_BX, 1, P.RPG_INPUT_FIXED, A.RPG_VAR_BY, A.RPG_VAR_BZ, 0]
    assert s.input_fixed[2] == hw.mem_latency_cycles
    assert low.max_data_index() == 1
    assert s.literals[0] == 1 / 3  # to_double of 1/3, correctly rounded
    with pytest.raises(F.PipelineError, match="has no value: 1 data parameter"):
        low.check_binding(1)
    low.check_binding(2)
    with pytest.raises(F.PipelineError, match="neither a block dimension"):
        P.LoweredProgram(P.parse("inputs: foo\noutput: Y\n0: assign Y foo\n1: halt_return Y\n"), hw)
    d0 = P.LoweredProgram(P.parse("inputs: D0\noutput: Y\n0: assign Y D0\n1: halt_return Y\n"), hw)
    with pytest.raises(F.PipelineError, match="'D0' has no value"):
        d0.check_binding(3)


def _emit(prog: P.Program, hw, compile_: bool):
    lib = A.load_library()
    low = P.LoweredProgram(prog, hw)
    hws = A.profile_struct(hw)
    opts = A.options_struct()
    buf = C.create_string_buffer(1 << 23)
    err = C.create_string_buffer(4096)
    cubin = C.c_int64(0)
    n = lib.rpg_emit_program_cuda_source(C.cast(C.pointer(low.struct), C.c_void_p),
                                         C.byref(hws), C.byref(opts), int(compile_), buf,
                                         len(buf), C.byref(cubin), err, len(err))
    assert n > 0, err.value
    return buf.value.decode(), cubin.value


def test_program_kernel_source_compiles_for_sm100a():
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    src, cubin = _emit(O4.generate_rp(spec, hw), hw, True)
    assert "rpg_jit_search" in src and "rp_floor_div" in src and cubin > 10000
    assert "bool a" not in src  # every read of the emitted program is definitely assigned


def test_maybe_unassigned_reads_get_runtime_guards():
    hw = zoo.sample_hw()
    src, _ = _emit(P.parse(EARLY.replace("X", "D1")), hw, False)
    guarded = [l for l in src.splitlines() if l.strip().startswith("bool a")]
    assert len(guarded) == 1  # only T
    src, _ = _emit(P.parse(WHILE.replace("X", "D1")), hw, False)
    assert "bool a" not in src


def test_program_plan_rejects_malformed_programs_before_the_device():
    lib = A.load_library()
    hw = zoo.sample_hw()
    low = P.LoweredProgram(P.parse(FLOOR_DIV.replace("A", "D1").replace("B", "D2")), hw)
    hws = A.profile_struct(hw)
    space = A.config_array(F.enumerate_configs())
    err = C.create_string_buffer(256)
    h = C.c_void_p()
    opts = A.options_struct()
    prog_p = C.cast(C.pointer(low.struct), C.c_void_p)
    rc = lib.rpg_program_plan_create(prog_p, C.byref(hws), None, 0, C.byref(opts), 0,
                                     C.byref(h), err, 256)
    assert rc == A.RPG_E_INVALID and b"configuration space is empty" in err.value
    low.struct.step_limit = 0
    rc = lib.rpg_program_plan_create(prog_p, C.byref(hws), A.ptr(space, A.rpg_config),
                                     len(space), C.byref(opts), 0, C.byref(h), err, 256)
    assert rc == A.RPG_E_INVALID and b"step_limit" in err.value
    low.struct.step_limit = 100
    low._body[0].b = 7  # slot out of range
    rc = lib.rpg_program_plan_create(prog_p, C.byref(hws), A.ptr(space, A.rpg_config),
                                     len(space), C.byref(opts), 0, C.byref(h), err, 256)
    assert rc == A.RPG_E_INVALID and b"operand" in err.value
