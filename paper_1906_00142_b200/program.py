"""Bare rational programs (`ratprog search --rp`, ratprog_cli.cpp:305-307).

Parses the reference's line-oriented `.rp` format (ir_text.hpp:1-242: same
grammar, checks and ``ParseError`` line/column messages) and lowers a
program for the GPU evaluator: variables become slots, literals become the
nearest doubles (the reference's C lowering, pipeline.hpp:276-433, prints
``to_double`` of each rational), and every program input is bound the way
``make_binding_plan`` binds it (pipeline.hpp:482-516): block dimensions and
data parameters per point, device-profile fields fixed at plan creation.
"""
from __future__ import annotations

import ctypes as C
import re
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi as A
from . import formats as F

OPCODES = ("assign", "neg", "add", "sub", "mul", "euclid_quot", "euclid_rem",
           "floor_div", "ceil_div", "cmp_eq", "cmp_lt", "branch_if", "jump",
           "halt_return")  # ir.hpp:19-34 order
OP = {name: i for i, name in enumerate(OPCODES)}


class EvalError(RuntimeError):
    """ir::EvalError (interp.hpp:19-28)."""


class StepLimitExceeded(EvalError):
    """ir::StepLimitExceeded (interp.hpp:21-25)."""


class MissingBinding(EvalError):
    """ir::MissingBinding (interp.hpp:26-29)."""


class DivisionByZero(ArithmeticError):
    """ratprog::DivisionByZero (rational.hpp:43-60)."""


class ParseError(ValueError):
    """ir::ParseError (ir_text.hpp:27-35)."""

    def __init__(self, line: int, column: int, why: str):
        super().__init__(f"line {line}, column {column}: {why}")
        self.line, self.column = line, column


@dataclass
class Operand:
    var: Optional[str] = None
    lit: Optional[Fraction] = None

    def is_var(self) -> bool:
        return self.var is not None


@dataclass
class Instr:
    op: str
    target: str = ""
    operands: List[Operand] = field(default_factory=list)
    jump_targets: List[int] = field(default_factory=list)


@dataclass
class Program:
    inputs: List[str] = field(default_factory=list)
    output: str = ""
    body: List[Instr] = field(default_factory=list)


_IDENT = re.compile(r"^[A-Za-z_][A-Za-z0-9_]*$")


def _parse_rational(text: str) -> Fraction:
    """rational.hpp:109-148: 'n', 'n/d' (optional leading '-')."""
    m = re.fullmatch(r"(-?)(\d+)(?:/(\d+))?", text)
    if not m:
        raise ValueError(f"bad rational literal '{text}'")
    num = int(m.group(2))
    den = int(m.group(3)) if m.group(3) is not None else 1
    if den == 0:
        raise ValueError(f"bad rational literal '{text}': zero denominator")
    v = Fraction(num, den)
    return -v if m.group(1) else v


def _tokens(line: str) -> List[Tuple[str, int]]:
    out, i = [], 0
    while i < len(line):
        if line[i] == "#":
            break
        if line[i] in " \t\r":
            i += 1
            continue
        j = i
        while j < len(line) and line[j] not in " \t\r#":
            j += 1
        out.append((line[i:j], i + 1))
        i = j
    return out


def parse(text: str) -> Program:
    """ir::parse (ir_text.hpp:99-240)."""
    p = Program()
    saw_inputs = saw_output = False
    line_no = 0
    for raw in text.split("\n"):
        line_no += 1
        toks = _tokens(raw)
        if not toks:
            continue
        if not saw_inputs:
            if toks[0][0] != "inputs:":
                raise ParseError(line_no, toks[0][1], "expected 'inputs:' header")
            for t, col in toks[1:]:
                if not _IDENT.match(t):
                    raise ParseError(line_no, col, f"bad input name '{t}'")
                p.inputs.append(t)
            saw_inputs = True
            continue
        if not saw_output:
            if toks[0][0] != "output:" or len(toks) != 2 or not _IDENT.match(toks[1][0]):
                raise ParseError(line_no, toks[0][1], "expected 'output: <variable>' header")
            p.output = toks[1][0]
            saw_output = True
            continue
        head, col0 = toks[0]
        if not head or head[-1] != ":":
            raise ParseError(line_no, col0, "expected '<index>:'")
        idx_text = head[:-1]
        if not idx_text.isdigit():
            raise ParseError(line_no, col0, f"expected instruction index, got '{idx_text}'")
        if int(idx_text) != len(p.body):
            raise ParseError(line_no, col0, f"instruction index {int(idx_text)} out of order; "
                                            f"expected {len(p.body)}")
        if len(toks) < 2:
            raise ParseError(line_no, col0, "missing opcode")
        opname, opcol = toks[1]
        if opname not in OP:
            raise ParseError(line_no, opcol, f"unknown opcode '{opname}'")
        args, targets, in_t = [], [], False
        for t, col in toks[2:]:
            if t == "->":
                if in_t:
                    raise ParseError(line_no, col, "duplicate '->'")
                in_t = True
            else:
                (targets if in_t else args).append((t, col))
        if opname in ("assign", "neg"):
            want_a, want_t, has_tv = 2, 0, True
        elif opname == "branch_if":
            want_a, want_t, has_tv = 1, 2, False
        elif opname == "jump":
            want_a, want_t, has_tv = 0, 1, False
        elif opname == "halt_return":
            want_a, want_t, has_tv = 1, 0, False
        else:
            want_a, want_t, has_tv = 3, 0, True
        if len(args) != want_a:
            raise ParseError(line_no, opcol, f"{opname} expects {want_a} argument(s), got {len(args)}")
        if len(targets) != want_t:
            raise ParseError(line_no, opcol,
                             f"{opname} expects {want_t} jump target(s), got {len(targets)}")
        ins = Instr(opname)
        a = 0
        if has_tv:
            if not _IDENT.match(args[0][0]):
                raise ParseError(line_no, args[0][1], f"bad target variable '{args[0][0]}'")
            ins.target = args[0][0]
            a = 1
        for t, col in args[a:]:
            if _IDENT.match(t):
                ins.operands.append(Operand(var=t))
            elif "." in t:
                raise ParseError(line_no, col, "decimal literals are not part of the format; use num/den")
            else:
                try:
                    ins.operands.append(Operand(lit=_parse_rational(t)))
                except ValueError as e:
                    raise ParseError(line_no, col, str(e)) from None
        for t, col in targets:
            if not t.isdigit():
                raise ParseError(line_no, col, f"expected instruction index, got '{t}'")
            ins.jump_targets.append(int(t))
        p.body.append(ins)
    if not saw_inputs:
        raise ParseError(line_no + 1, 1, "missing 'inputs:' header")
    if not saw_output:
        raise ParseError(line_no + 1, 1, "missing 'output:' header")
    if not p.body:
        raise ParseError(line_no + 1, 1, "empty program body")
    return p


def serialize(p: Program) -> str:
    """ir::serialize (ir_text.hpp:77-97)."""
    def lit(r: Fraction) -> str:
        return str(r.numerator) if r.denominator == 1 else f"{r.numerator}/{r.denominator}"
    out = ["inputs:" + "".join(" " + i for i in p.inputs), f"output: {p.output}"]
    for i, ins in enumerate(p.body):
        s = f"{i}: {ins.op}"
        if ins.target:
            s += " " + ins.target
        for o in ins.operands:
            s += " " + (o.var if o.is_var() else lit(o.lit))
        if ins.jump_targets:
            s += " ->" + "".join(f" {t}" for t in ins.jump_targets)
        out.append(s)
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------------------
# Lowering for the C ABI (include/rpg.h rpg_program)

RPG_INPUT_FIXED = -100
MAX_DATA = 64  # rpg_device.cuh kMaxData


class rpg_instr(C.Structure):
    _fields_ = [("op", C.c_int32), ("target", C.c_int32), ("a", C.c_int32), ("b", C.c_int32),
                ("t0", C.c_int32), ("t1", C.c_int32)]


class rpg_program(C.Structure):
    _fields_ = [("n_instr", C.c_int32), ("n_slots", C.c_int32), ("n_literals", C.c_int32),
                ("output_slot", C.c_int32), ("body", C.POINTER(rpg_instr)),
                ("literals", C.POINTER(C.c_double)), ("n_inputs", C.c_int32),
                ("reserved", C.c_int32), ("input_slot", C.POINTER(C.c_int32)),
                ("input_kind", C.POINTER(C.c_int32)), ("input_fixed", C.POINTER(C.c_double)),
                ("step_limit", C.c_int64)]


def _profile_value(hw: F.DeviceProfile, key: str) -> float:
    # rational_from_double of the field (exact), as a double
    return float(getattr(hw, key))


class LoweredProgram:
    """rpg_program + the buffers it points into.  Binds inputs exactly as
    make_binding_plan (pipeline.hpp:482-516); unknown inputs raise
    PipelineError with the reference's message."""

    def __init__(self, p: Program, hw: F.DeviceProfile, step_limit: int = 1_000_000):
        slots: Dict[str, int] = {}

        def slot(name: str) -> int:
            if name not in slots:
                slots[name] = len(slots)
            return slots[name]

        for name in p.inputs:
            slot(name)
        lits: List[float] = []
        lit_index: Dict[Fraction, int] = {}

        def operand(o: Operand) -> int:
            if o.is_var():
                return slot(o.var)
            if o.lit not in lit_index:
                lit_index[o.lit] = len(lits)
                lits.append(float(o.lit))  # correctly rounded to_double
            return -1 - lit_index[o.lit]

        body = (rpg_instr * len(p.body))()
        for i, ins in enumerate(p.body):
            r = body[i]
            r.op = OP[ins.op]
            r.target = slot(ins.target) if ins.target else -1
            ops = [operand(o) for o in ins.operands]
            r.a = ops[0] if len(ops) > 0 else 0
            r.b = ops[1] if len(ops) > 1 else 0
            r.t0 = ins.jump_targets[0] if len(ins.jump_targets) > 0 else 0
            r.t1 = ins.jump_targets[1] if len(ins.jump_targets) > 1 else 0
        out_slot = slot(p.output)
        kinds, fixed = [], []
        self.unbindable: List[Tuple[str, int]] = []
        for name in p.inputs:
            if name == "bx":
                kinds.append(A.RPG_VAR_BX)
                fixed.append(0.0)
            elif name == "by":
                kinds.append(A.RPG_VAR_BY)
                fixed.append(0.0)
            elif name == "bz":
                kinds.append(A.RPG_VAR_BZ)
                fixed.append(0.0)
            elif name in F.PROFILE_KEYS:
                kinds.append(RPG_INPUT_FIXED)
                fixed.append(_profile_value(hw, name))
            elif len(name) >= 2 and name[0] == "D" and name[1:].isdigit():
                k = int(name[1:])
                if k < 1 or k > MAX_DATA:
                    # bound to no data parameter: fails at search time with
                    # make_binding_plan's message (needs the tuple width)
                    self.unbindable.append((name, k))
                    k = 1
                kinds.append(k - 1)
                fixed.append(0.0)
            else:
                raise F.PipelineError(f"program input '{name}' is neither a block dimension, "
                                      "a data parameter, nor a device profile field")
        self.program = p
        self.slots = slots
        self._body = body
        self._lits = np.ascontiguousarray(lits if lits else [0.0], dtype=np.float64)
        self._islot = np.ascontiguousarray([slots[n] for n in p.inputs] or [0], dtype=np.int32)
        self._ikind = np.ascontiguousarray(kinds or [0], dtype=np.int32)
        self._ifixed = np.ascontiguousarray(fixed or [0.0], dtype=np.float64)
        self.struct = rpg_program(len(p.body), len(slots), len(lits), out_slot,
                                  C.cast(body, C.POINTER(rpg_instr)),
                                  A.ptr(self._lits, C.c_double), len(p.inputs), 0,
                                  A.ptr(self._islot, C.c_int32), A.ptr(self._ikind, C.c_int32),
                                  A.ptr(self._ifixed, C.c_double), step_limit)

    def max_data_index(self) -> int:
        return max([k for k in self._ikind.tolist() if k >= 0], default=-1)

    def check_binding(self, n_data: int) -> None:
        """make_binding_plan's data-parameter check (pipeline.hpp:498-506)."""
        for name in self.program.inputs:
            if len(name) >= 2 and name[0] == "D" and name[1:].isdigit():
                k = int(name[1:])
                if k < 1 or k > n_data:
                    raise F.PipelineError(f"program input '{name}' has no value: {n_data} "
                                          "data parameter(s) were given")
        for name, k in self.unbindable:
            raise ValueError(f"program input '{name}': data parameters beyond D{MAX_DATA} "
                             "are not supported")

    def slot_name(self, slot: int) -> str:
        for name, s in self.slots.items():
            if s == slot:
                return name
        return f"slot {slot}"

    def raise_eval_error(self, msg: str) -> None:
        """Maps an RPG_E_EVAL message to the interpreter's exception type."""
        m = re.match(r"no value bound for variable slot (\d+)(.*)$", msg)
        if m:
            raise MissingBinding(f"no value bound for variable '{self.slot_name(int(m.group(1)))}'"
                                 f"{m.group(2)}")
        if "zero divisor" in msg:
            raise DivisionByZero(msg)
        if msg.startswith("step limit"):
            raise StepLimitExceeded(msg)
        raise EvalError(msg)
