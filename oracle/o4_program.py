"""ORACLE O4 — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench cpu legs).

Bare rational programs (the `ratprog search --rp` path):

* ``Builder`` / ``specialize`` — ir_builder.hpp:17-153 (labels, fresh names,
  emit_min, partial evaluation);
* ``emit_occupancy_rp`` / ``emit_mwpcwp_rp`` / ``generate_rp`` — the
  program emitters (perfmodel.hpp:491-834, pipeline.hpp:233-260), so tests
  can feed the GPU the same programs `ratprog gen-rp` writes; pinned against
  O2 (exact program semantics, itself pinned by the reference's KATs);
* ``evaluate_exact`` — ir::evaluate (interp.hpp:44-121) on ``Fraction``s;
* ``evaluate_c`` — the reference's C lowering (pipeline.hpp:263-433): IEEE
  doubles, rp_floor_div's int64 path, literals ``to_double``; where the exact
  interpreter throws (zero divisor, step limit, falling off the end, reading
  an unassigned variable) it raises the same exception;
* ``search`` — pipe::search_optimal for a program (pipeline.hpp:575-680)
  with the occupancy context from the options (:648-650).

The program data classes and exception types are the product's
(paper_1906_00142_b200.program: plain containers); every semantic rule here
is restated independently of the CUDA path.
"""
from __future__ import annotations

import math
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200.program import (DivisionByZero, EvalError, Instr, MissingBinding,
                                           Operand, Program, StepLimitExceeded)

DEFAULT_STEP_LIMIT = 1_000_000  # interp.hpp:31


def var(name: str) -> Operand:
    return Operand(var=name)


def lit(v) -> Operand:
    return Operand(lit=Fraction(v))


class Builder:
    """ir::ProgramBuilder (ir_builder.hpp:17-118)."""

    def __init__(self):
        self.p = Program()
        self.labels: List[Optional[int]] = []
        self.pending: List[int] = []
        self.counter = 0

    def input(self, name):
        self.p.inputs.append(name)

    def output(self, name):
        self.p.output = name

    def make_label(self) -> int:
        self.labels.append(None)
        return len(self.labels) - 1

    def place(self, label: int):
        if self.labels[label] is not None:
            raise RuntimeError("label placed twice")
        self.labels[label] = len(self.p.body)

    def _emit(self, op, t, ops):
        self.p.body.append(Instr(op, t, list(ops)))

    def assign(self, t, a): self._emit("assign", t, [a])
    def neg(self, t, a): self._emit("neg", t, [a])
    def add(self, t, a, b): self._emit("add", t, [a, b])
    def sub(self, t, a, b): self._emit("sub", t, [a, b])
    def mul(self, t, a, b): self._emit("mul", t, [a, b])
    def euclid_quot(self, t, a, b): self._emit("euclid_quot", t, [a, b])
    def euclid_rem(self, t, a, b): self._emit("euclid_rem", t, [a, b])
    def floor_div(self, t, a, b): self._emit("floor_div", t, [a, b])
    def ceil_div(self, t, a, b): self._emit("ceil_div", t, [a, b])
    def cmp_eq(self, t, a, b): self._emit("cmp_eq", t, [a, b])
    def cmp_lt(self, t, a, b): self._emit("cmp_lt", t, [a, b])

    def branch_if(self, cond: str, if_true: int, if_false: int):
        self.pending.append(len(self.p.body))
        self.p.body.append(Instr("branch_if", "", [var(cond)], [if_true, if_false]))

    def jump(self, to: int):
        self.pending.append(len(self.p.body))
        self.p.body.append(Instr("jump", "", [], [to]))

    def halt_return(self, name: str):
        self.p.body.append(Instr("halt_return", "", [var(name)]))

    def emit_min(self, t: str, a: Operand, b: Operand):
        c = self.fresh("min_c")
        self.assign(t, a)
        self.cmp_lt(c, b, a)
        use_b, done = self.make_label(), self.make_label()
        self.branch_if(c, use_b, done)
        self.place(use_b)
        self.assign(t, b)
        self.place(done)

    def fresh(self, prefix: str) -> str:
        s = f"{prefix}_{self.counter}"
        self.counter += 1
        return s

    def finish(self) -> Program:
        for at in self.pending:
            ins = self.p.body[at]
            resolved = []
            for t in ins.jump_targets:
                if self.labels[t] is None:
                    raise RuntimeError("unplaced label used")
                resolved.append(self.labels[t])
            ins.jump_targets = resolved
        self.pending = []
        return self.p


def specialize(p: Program, fixed: Dict[str, Fraction]) -> Program:
    """ir::specialize (ir_builder.hpp:123-151)."""
    for name in fixed:
        if name not in p.inputs:
            raise ValueError(f"specialize: '{name}' is not an input of the program")
    out = Program(output=p.output)
    shift = 0
    for name in p.inputs:
        if name in fixed:
            out.body.append(Instr("assign", name, [lit(fixed[name])]))
            shift += 1
        else:
            out.inputs.append(name)
    for ins in p.body:
        out.body.append(Instr(ins.op, ins.target, list(ins.operands),
                              [t + shift for t in ins.jump_targets]))
    return out


def profile_bindings(hw: F.DeviceProfile) -> Dict[str, Fraction]:
    """perf::profile_bindings (perfmodel.hpp:212-231): exact values."""
    return {k: Fraction(getattr(hw, k)) for k in F.PROFILE_KEYS}


def bake_hardware(p: Program, hw: F.DeviceProfile) -> Program:
    """pipeline.hpp:233-247 (re-validation not restated)."""
    allb = profile_bindings(hw)
    return specialize(p, {k: v for k, v in allb.items() if k in p.inputs})


# ---------------------------------------------------------------------------
# Emitters (perfmodel.hpp:491-834).

def _emit_div(b: Builder, target: str, num: Operand, den: Operand, S: int):
    scale = Fraction(10) ** S
    t, q = b.fresh("dscaled"), b.fresh("dquot")
    b.mul(t, num, lit(scale))
    b.floor_div(q, var(t), den)
    b.mul(target, var(q), lit(1 / scale))


def _emit_ratfunc(b: Builder, target: str, f: F.RationalFunction, variables, infeasible, S):
    def poly(p: F.Polynomial, acc: str):
        b.assign(acc, lit(0))
        for mono, c in zip(p.basis, p.coeffs):
            if c == 0.0:
                continue
            term = b.fresh("term")
            b.assign(term, lit(Fraction(c)))
            for v, e in zip(variables, mono):
                for _ in range(e):
                    b.mul(term, var(term), var(v))
            b.add(acc, var(acc), var(term))
    pnum, pden = b.fresh("fnum"), b.fresh("fden")
    poly(f.num, pnum)
    poly(f.den, pden)
    dz = b.fresh("fdenzero")
    b.cmp_eq(dz, var(pden), lit(0))
    ok = b.make_label()
    b.branch_if(dz, infeasible, ok)
    b.place(ok)
    _emit_div(b, target, var(pnum), var(pden), S)


def _emit_occupancy_core(b: Builder, R: Operand, Z: Operand, t_var: str, fail: int):
    c_big = b.fresh("t_over_max")
    b.cmp_lt(c_big, var("T_max"), var(t_var))
    ok1 = b.make_label()
    b.branch_if(c_big, fail, ok1)
    b.place(ok1)
    c_small = b.fresh("t_under_one")
    b.cmp_lt(c_small, var(t_var), lit(1))
    ok2 = b.make_label()
    b.branch_if(c_small, fail, ok2)
    b.place(ok2)
    wpb = b.fresh("warps_per_block")
    b.ceil_div(wpb, var(t_var), lit(32))
    blocks = b.fresh("blocks")
    b.assign(blocks, var("B_max"))
    lim_w = b.fresh("limit_warps")
    b.floor_div(lim_w, var("W_max"), var(wpb))
    b.emit_min(blocks, var(blocks), var(lim_w))
    r_zero = b.fresh("regs_zero")
    b.cmp_eq(r_zero, R, lit(0))
    skip_r, do_r = b.make_label(), b.make_label()
    b.branch_if(r_zero, skip_r, do_r)
    b.place(do_r)
    rt = b.fresh("regs_per_block")
    b.mul(rt, R, var(t_var))
    lim_r = b.fresh("limit_regs")
    b.floor_div(lim_r, var("R_max"), var(rt))
    b.emit_min(blocks, var(blocks), var(lim_r))
    b.place(skip_r)
    z_zero = b.fresh("shared_zero")
    b.cmp_eq(z_zero, Z, lit(0))
    skip_z, do_z = b.make_label(), b.make_label()
    b.branch_if(z_zero, skip_z, do_z)
    b.place(do_z)
    lim_z = b.fresh("limit_shared")
    b.floor_div(lim_z, var("Z_max"), Z)
    b.emit_min(blocks, var(blocks), var(lim_z))
    b.place(skip_z)
    b_zero = b.fresh("blocks_under_one")
    b.cmp_lt(b_zero, var(blocks), lit(1))
    b_ok = b.make_label()
    b.branch_if(b_zero, fail, b_ok)
    b.place(b_ok)
    bt = b.fresh("threads_resident")
    b.mul(bt, var(blocks), var(t_var))
    warps = b.fresh("warps")
    b.floor_div(warps, var(bt), lit(32))
    b.emit_min(warps, var(warps), var("W_max"))
    return blocks, warps


def emit_occupancy_rp() -> Program:
    """perfmodel.hpp:620-640."""
    b = Builder()
    for n in ("R_max", "Z_max", "T_max", "B_max", "W_max", "R", "Z", "T"):
        b.input(n)
    b.output("W_active")
    fail, done = b.make_label(), b.make_label()
    _, warps = _emit_occupancy_core(b, var("R"), var("Z"), "T", fail)
    b.assign("W_active", var(warps))
    b.jump(done)
    b.place(fail)
    b.assign("W_active", lit(0))
    b.place(done)
    b.halt_return("W_active")
    return b.finish()


def emit_mwpcwp_rp(spec: F.MetricSpec, rep_mode: str = "real", scale_pow10: int = 40) -> Program:
    """perfmodel.hpp:646-834."""
    F.check_metric_spec(spec)
    S = scale_pow10
    b = Builder()
    for v in spec.variables:
        b.input(v)
    for k in F.PROFILE_KEYS:
        b.input(k)
    b.output("total_cycles")
    infeasible, done = b.make_label(), b.make_label()
    has_bz = "bz" in spec.variables
    b.mul("T", var("bx"), var("by"))
    if has_bz:
        b.mul("T", var("T"), var("bz"))
    for v in spec.variables:
        if v not in ("bx", "by", "bz"):
            b.assign(b.fresh("param_anchor"), var(v))

    def metric_value(name):
        target = b.fresh("m_" + name)
        if name in spec.constants:
            b.assign(target, lit(Fraction(spec.constants[name])))
        else:
            _emit_ratfunc(b, target, spec.models[name], spec.variables, infeasible, S)
        return target

    regs = metric_value(F.METRIC_REGS)
    shared = metric_value(F.METRIC_SHARED)
    comp = metric_value(F.METRIC_COMP)
    uncoal = metric_value(F.METRIC_UNCOAL)
    coal = metric_value(F.METRIC_COAL)
    synch = metric_value(F.METRIC_SYNCH)
    total_blocks = metric_value(F.METRIC_TOTAL_BLOCKS)
    mem = b.fresh("m_mem_insts")
    b.add(mem, var(uncoal), var(coal))

    blocks, warps = _emit_occupancy_core(b, var(regs), var(shared), "T", infeasible)
    n_zero = b.fresh("warps_under_one")
    b.cmp_lt(n_zero, var(warps), lit(1))
    n_ok = b.make_label()
    b.branch_if(n_zero, infeasible, n_ok)
    b.place(n_ok)

    b.assign("mem_l_coal", var("mem_latency_cycles"))
    b.sub("txn_extra", var("uncoal_per_mw"), lit(1))
    b.mul("txn_cost", var("txn_extra"), var("departure_del_uncoal_cycles"))
    b.add("mem_l_uncoal", var("mem_latency_cycles"), var("txn_cost"))
    b.add("insts_issued", var(comp), var(mem))
    b.mul("comp_cycles", var("issue_cycles"), var("insts_issued"))
    b.mul("rep_den", var(blocks), var("num_SM"))
    if rep_mode == "ceil":
        b.ceil_div("rep", var(total_blocks), var("rep_den"))
    else:
        _emit_div(b, "rep", var(total_blocks), var("rep_den"), S)

    mem_zero = b.fresh("mem_zero")
    b.cmp_eq(mem_zero, var(mem), lit(0))
    compute_only, with_mem = b.make_label(), b.make_label()
    b.branch_if(mem_zero, compute_only, with_mem)

    b.place(compute_only)
    b.mul("pre0", var("comp_cycles"), var("rep"))
    b.sub("nm1_0", var(warps), lit(1))
    b.mul("sc0", var("departure_del_coal_cycles"), var("nm1_0"))
    b.mul("sc0", var("sc0"), var(synch))
    b.mul("sc0", var("sc0"), var(blocks))
    b.mul("sc0", var("sc0"), var("rep"))
    b.add("total_cycles", var("pre0"), var("sc0"))
    b.jump(done)

    b.place(with_mem)
    _emit_div(b, "r_uncoal", var(uncoal), var(mem), S)
    b.sub("r_coal", lit(1), var("r_uncoal"))
    b.mul("wl_u", var("r_uncoal"), var("mem_l_uncoal"))
    b.mul("wl_c", var("r_coal"), var("mem_l_coal"))
    b.add("weighted_mem_l", var("wl_u"), var("wl_c"))
    b.mul("dd_u", var("r_uncoal"), var("departure_del_uncoal_cycles"))
    b.mul("dd_u", var("dd_u"), var("uncoal_per_mw"))
    b.mul("dd_c", var("r_coal"), var("departure_del_coal_cycles"))
    b.add("departure_delay", var("dd_u"), var("dd_c"))
    b.mul("mc_u", var(uncoal), var("mem_l_uncoal"))
    b.mul("mc_c", var(coal), var("mem_l_coal"))
    b.add("mem_cycles", var("mc_u"), var("mc_c"))
    _emit_div(b, "mwp_no_bw", var("weighted_mem_l"), var("departure_delay"), S)
    b.mul("bw_num", var("freq_GHz"), var("load_bytes_per_warp"))
    _emit_div(b, "bw_per_warp", var("bw_num"), var("mem_latency_cycles"), S)
    b.mul("bw_all_sm", var("bw_per_warp"), var("num_SM"))
    _emit_div(b, "mwp_peak_bw", var("mem_bandwidth_GBps"), var("bw_all_sm"), S)
    b.emit_min("mwp", var("mwp_no_bw"), var("mwp_peak_bw"))
    b.emit_min("mwp", var("mwp"), var(warps))

    comp_zero = b.fresh("comp_zero")
    b.cmp_eq(comp_zero, var("comp_cycles"), lit(0))
    cwp_sat, cwp_div, cwp_done = b.make_label(), b.make_label(), b.make_label()
    b.branch_if(comp_zero, cwp_sat, cwp_div)
    b.place(cwp_sat)
    b.assign("cwp", var(warps))
    b.jump(cwp_done)
    b.place(cwp_div)
    b.add("busy_cycles", var("mem_cycles"), var("comp_cycles"))
    _emit_div(b, "cwp_full", var("busy_cycles"), var("comp_cycles"), S)
    b.emit_min("cwp", var("cwp_full"), var(warps))
    b.place(cwp_done)

    _emit_div(b, "comp_per_mem", var("comp_cycles"), var(mem), S)
    b.sub("mwp_m1", var("mwp"), lit(1))

    eq1, eq2 = b.fresh("mwp_is_n"), b.fresh("cwp_is_n")
    check2, elif_case = b.make_label(), b.make_label()
    case_both, case_cwp, case_mwp, have_pre = (b.make_label(), b.make_label(),
                                               b.make_label(), b.make_label())
    b.cmp_eq(eq1, var("mwp"), var(warps))
    b.branch_if(eq1, check2, elif_case)
    b.place(check2)
    b.cmp_eq(eq2, var("cwp"), var(warps))
    b.branch_if(eq2, case_both, elif_case)

    b.place(elif_case)
    lt1, lt2 = b.fresh("cwp_lt_mwp"), b.fresh("mem_lt_comp")
    second_test = b.make_label()
    b.cmp_lt(lt1, var("cwp"), var("mwp"))
    b.branch_if(lt1, second_test, case_cwp)
    b.place(second_test)
    b.cmp_lt(lt2, var("mem_cycles"), var("comp_cycles"))
    b.branch_if(lt2, case_cwp, case_mwp)

    b.place(case_both)
    b.add("pre_b", var("mem_cycles"), var("comp_cycles"))
    b.mul("ovl_b", var("comp_per_mem"), var("mwp_m1"))
    b.add("pre_b", var("pre_b"), var("ovl_b"))
    b.mul("pre", var("pre_b"), var("rep"))
    b.jump(have_pre)

    b.place(case_cwp)
    b.mul("mem_n", var("mem_cycles"), var(warps))
    _emit_div(b, "mem_span", var("mem_n"), var("mwp"), S)
    b.mul("ovl_c", var("comp_per_mem"), var("mwp_m1"))
    b.add("pre_c", var("mem_span"), var("ovl_c"))
    b.mul("pre", var("pre_c"), var("rep"))
    b.jump(have_pre)

    b.place(case_mwp)
    b.mul("comp_n", var("comp_cycles"), var(warps))
    b.add("pre_m", var("mem_latency_cycles"), var("comp_n"))
    b.mul("pre", var("pre_m"), var("rep"))
    b.place(have_pre)

    b.mul("synch_cost", var("departure_delay"), var("mwp_m1"))
    b.mul("synch_cost", var("synch_cost"), var(synch))
    b.mul("synch_cost", var("synch_cost"), var(blocks))
    b.mul("synch_cost", var("synch_cost"), var("rep"))
    b.add("total_cycles", var("pre"), var("synch_cost"))
    b.jump(done)

    b.place(infeasible)
    b.assign("total_cycles", lit(-1))
    b.place(done)
    b.halt_return("total_cycles")
    return b.finish()


def generate_rp(spec: F.MetricSpec, hw: F.DeviceProfile, rep_mode: str = "real",
                scale_pow10: int = 40) -> Program:
    """pipe::generate_rp (pipeline.hpp:251-255)."""
    return bake_hardware(emit_mwpcwp_rp(spec, rep_mode, scale_pow10), hw)


def generate_occupancy_rp(hw: F.DeviceProfile) -> Program:
    """pipeline.hpp:258-260."""
    return bake_hardware(emit_occupancy_rp(), hw)


# ---------------------------------------------------------------------------
# Interpreters.

def _floor_q(a: Fraction, b: Fraction) -> Fraction:
    q = a / b
    return Fraction(q.numerator // q.denominator)


def _ceil_q(a: Fraction, b: Fraction) -> Fraction:
    q = a / b
    return Fraction(-((-q.numerator) // q.denominator))


_ZERO_MSG = {"floor_div": "floor_div: zero divisor", "ceil_div": "ceil_div: zero divisor",
             "euclid_quot": "euclid_quot: zero divisor", "euclid_rem": "euclid_rem: zero divisor"}


def _run(p: Program, env, step_limit, ops):
    if step_limit < 1:
        raise ValueError("step_limit must be >= 1")
    for name in p.inputs:
        if name not in env:
            raise MissingBinding(f"no value bound for variable '{name}'")
    env = dict(env)

    def val(o):
        if not o.is_var():
            return ops["lit"](o.lit)
        if o.var not in env:
            raise MissingBinding(f"no value bound for variable '{o.var}'")
        return env[o.var]

    pc = steps = 0
    n = len(p.body)
    while True:
        if pc >= n:
            raise EvalError("control fell off the end of the program")
        steps += 1
        if steps > step_limit:
            raise StepLimitExceeded(f"step limit of {step_limit} instructions exceeded "
                                    "(possible non-termination)")
        ins = p.body[pc]
        op = ins.op
        if op == "branch_if":
            pc = ins.jump_targets[0 if val(ins.operands[0]) != 0 else 1]
            continue
        if op == "jump":
            pc = ins.jump_targets[0]
            continue
        if op == "halt_return":
            return val(ins.operands[0])
        a = val(ins.operands[0])
        if op == "assign":
            r = a
        elif op == "neg":
            r = ops["neg"](a)
        else:
            b = val(ins.operands[1])
            if op in _ZERO_MSG:
                if b == 0:
                    raise DivisionByZero(_ZERO_MSG[op])
                r = ops[op](a, b)
            elif op == "cmp_eq":
                r = ops["one"] if a == b else ops["zero"]
            elif op == "cmp_lt":
                r = ops["one"] if a < b else ops["zero"]
            else:
                r = ops[op](a, b)
        env[ins.target] = r
        pc += 1


_EXACT_OPS = {
    "lit": lambda r: r, "neg": lambda a: -a, "one": Fraction(1), "zero": Fraction(0),
    "add": lambda a, b: a + b, "sub": lambda a, b: a - b, "mul": lambda a, b: a * b,
    "floor_div": _floor_q, "ceil_div": _ceil_q,
    "euclid_quot": lambda a, b: _floor_q(a, b) if b > 0 else _ceil_q(a, b),
    "euclid_rem": lambda a, b: a - (_floor_q(a, b) if b > 0 else _ceil_q(a, b)) * b,
}


def evaluate_exact(p: Program, bindings: Dict[str, Fraction],
                   step_limit: int = DEFAULT_STEP_LIMIT) -> Fraction:
    """ir::evaluate (interp.hpp:44-121); rational.hpp:41-62 for the
    integer-part operations."""
    return _run(p, {k: Fraction(v) for k, v in bindings.items()}, step_limit, _EXACT_OPS)


def _c_floor_div(a: float, b: float) -> float:
    """rp_floor_div (pipeline.hpp:326-336)."""
    if a == math.floor(a) and b == math.floor(b) and abs(a) < 9.0e15 and abs(b) < 9.0e15:
        ia, ib = int(a), int(b)
        q = abs(ia) // abs(ib)
        if (ia < 0) != (ib < 0):
            q = -q  # C truncation toward zero
        if ia % ib != 0 and (ia < 0) != (ib < 0):  # C: ia % ib != 0 <=> not divisible
            q -= 1
        return float(q)
    q = a / b
    return q if not math.isfinite(q) else float(math.floor(q))


def _c_ceil_div(a: float, b: float) -> float:
    return -_c_floor_div(-a, b)


def _c_euclid_quot(a: float, b: float) -> float:
    return _c_floor_div(a, b) if b >= 0.0 else _c_ceil_div(a, b)


_C_OPS = {
    "lit": lambda r: float(r),  # to_double: correctly rounded
    "neg": lambda a: -a, "one": 1.0, "zero": 0.0,
    "add": lambda a, b: a + b, "sub": lambda a, b: a - b, "mul": lambda a, b: a * b,
    "floor_div": _c_floor_div, "ceil_div": _c_ceil_div, "euclid_quot": _c_euclid_quot,
    "euclid_rem": lambda a, b: a - b * _c_euclid_quot(a, b),
}


def evaluate_c(p: Program, bindings: Dict[str, float],
               step_limit: int = DEFAULT_STEP_LIMIT) -> float:
    """The C lowering's double semantics (pipeline.hpp:263-433) with the
    interpreter's error conditions."""
    return _run(p, {k: float(v) for k, v in bindings.items()}, step_limit, _C_OPS)


# ---------------------------------------------------------------------------
# Search.

def bindings_for(p: Program, data: Sequence[int], hw: F.DeviceProfile,
                 cfg: Tuple[int, int, int]) -> Dict[str, Fraction]:
    """make_binding_plan + bindings_for (pipeline.hpp:482-532)."""
    hwv = profile_bindings(hw)
    out = {}
    for name in p.inputs:
        if name == "bx":
            out[name] = Fraction(cfg[0])
        elif name == "by":
            out[name] = Fraction(cfg[1])
        elif name == "bz":
            out[name] = Fraction(cfg[2])
        elif name in hwv:
            out[name] = hwv[name]
        elif len(name) >= 2 and name[0] == "D" and name[1:].isdigit():
            k = int(name[1:])
            if k < 1 or k > len(data):
                raise F.PipelineError(f"program input '{name}' has no value: {len(data)} "
                                      "data parameter(s) were given")
            out[name] = Fraction(int(data[k - 1]))
        else:
            raise F.PipelineError(f"program input '{name}' is neither a block dimension, "
                                  "a data parameter, nor a device profile field")
    return out


def active_blocks(hw: F.DeviceProfile, R: float, Z: float, T: int) -> int:
    """perfmodel.hpp:240-252."""
    if T < 1 or T > hw.T_max:
        return 0
    b = min(hw.B_max, hw.W_max // ((T + 31) // 32))
    if R > 0:
        b = min(b, int(math.floor(float(hw.R_max) / (R * T))))
    if Z > 0:
        b = min(b, int(math.floor(float(hw.Z_max) / Z)))
    return 0 if b < 1 else b


def occupancy_warps(hw: F.DeviceProfile, R: float, Z: float, T: int) -> int:
    b = active_blocks(hw, R, Z, T)
    return 0 if b <= 0 else min(b * T // 32, hw.W_max)


def search(p: Program, data: Sequence[int], hw: F.DeviceProfile,
           space: Sequence[Tuple[int, int, int]], regs: float = 0.0, shared: float = 0.0,
           tie_rel_tol: float = 1e-12, exact: bool = False,
           step_limit: int = DEFAULT_STEP_LIMIT):
    """pipe::search_optimal for a bare program (pipeline.hpp:575-680).
    exact=True: the reference's exact-rational ranking; exact=False: the
    same rules on the C lowering's doubles (what the GPU computes).
    Returns (values per config, ranking order, ties, occupancy warps)."""
    if not space:
        raise ValueError("search_optimal: configuration space is empty")
    vals = []
    for c in space:
        b = bindings_for(p, data, hw, c)
        vals.append(evaluate_exact(p, b, step_limit) if exact else evaluate_c(p, b, step_limit))
    feas = [i for i, v in enumerate(vals) if v >= 0]
    if not feas:
        raise RuntimeError("no configuration in the search space can launch on this device")
    wocc = [occupancy_warps(hw, regs, shared, c[0] * c[1] * c[2]) for c in space]
    feas.sort(key=lambda i: (vals[i], tuple(space[i])))
    best = vals[feas[0]]
    tol = Fraction(tie_rel_tol) if exact else tie_rel_tol
    bound = best + best * tol
    ties = 0
    while ties < len(feas) and vals[feas[ties]] <= bound:
        ties += 1
    head = sorted(feas[:ties], key=lambda i: -wocc[i])
    return vals, head + feas[ties:], ties, wocc
