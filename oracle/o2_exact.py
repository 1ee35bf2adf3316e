"""ORACLE O2 — TEST INFRASTRUCTURE ONLY.

Exact-rational restatement of what the reference's shipped search actually
ranks: ``ir::evaluate`` (interp.hpp:44-121, Boost cpp_rational) running the
program ``emit_mwpcwp_rp`` emits (perfmodel.hpp:648-834) with the hardware
baked in (pipeline.hpp:233-247).  Instead of building the IR, this module
executes the emitted instruction sequence directly on Python ``Fraction``s:

* every literal is the exact binary64 value (rational_from_double,
  rational.hpp:90-104);
* every division the emitter lowers goes through ``emit_div``
  (perfmodel.hpp:501-509): q = floor(a * 10^40 / b) * 10^-40;
* a metric denominator that is exactly zero, T > T_max, T < 1, blocks < 1 or
  warps < 1 yield the sentinel -1 (perfmodel.hpp:533-536, 553-563, 598-603,
  699-703, 829-831);
* the search ranks by exact values: sort by (Ec, lex), tie bound
  best + best * rational(tol) (pipeline.hpp:654-669).

Far too slow for bulk sweeps (that is the point of the GPU path); used on
sampled tuples to measure how often the FP64 evaluator's winner differs from
the exact-rational one (they can differ only inside the 1e-12
tie window or at a case boundary).
"""
from __future__ import annotations

from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

from paper_1906_00142_b200 import formats as F

SCALE = Fraction(10) ** 40


def rat(x: float) -> Fraction:
    return Fraction(x)  # exact for every finite binary64


def floor_div(a: Fraction, b: Fraction) -> Fraction:
    if b == 0:
        raise ZeroDivisionError("floor_div: zero divisor")
    return Fraction((a / b).numerator // (a / b).denominator)


def ceil_div(a: Fraction, b: Fraction) -> Fraction:
    q = a / b
    return Fraction(-((-q.numerator) // q.denominator))


def emit_div(a: Fraction, b: Fraction) -> Fraction:
    """perfmodel.hpp:501-509."""
    return floor_div(a * SCALE, b) / SCALE


def _poly_value(p: F.Polynomial, x: Dict[str, Fraction]) -> Fraction:
    acc = Fraction(0)
    for mono, c in zip(p.basis, p.coeffs):
        if c == 0.0:
            continue  # emit_ratfunc skips zero coefficients (perfmodel.hpp:521)
        term = rat(c)
        for v, e in zip(p.variables, mono):
            for _ in range(e):
                term = term * x[v]
        acc = acc + term
    return acc


class Infeasible(Exception):
    pass


def program_value(spec: F.MetricSpec, hw: F.DeviceProfile, data: Sequence[int],
                  cfg: Tuple[int, int, int], rep_mode: str = "real") -> Fraction:
    """Exact output of the emitted cycle program at one point (-1 sentinel)."""
    try:
        return _program(spec, hw, data, cfg, rep_mode)
    except Infeasible:
        return Fraction(-1)


def _program(spec, hw, data, cfg, rep_mode):
    bx, by, bz = (Fraction(v) for v in cfg)
    x: Dict[str, Fraction] = {"bx": bx, "by": by, "bz": bz}
    for v in spec.variables:
        if v not in ("bx", "by", "bz"):
            x[v] = Fraction(int(data[int(v[1:]) - 1]))
    T = bx * by
    if "bz" in spec.variables:
        T = T * bz

    def metric(name):
        if name in spec.constants:
            return rat(spec.constants[name])
        f = spec.models[name]
        pnum = _poly_value(f.num, x)
        pden = _poly_value(f.den, x)
        if pden == 0:
            raise Infeasible()
        return emit_div(pnum, pden)

    regs = metric(F.METRIC_REGS)
    shared = metric(F.METRIC_SHARED)
    comp = metric(F.METRIC_COMP)
    uncoal = metric(F.METRIC_UNCOAL)
    coal = metric(F.METRIC_COAL)
    synch = metric(F.METRIC_SYNCH)
    tb = metric(F.METRIC_TOTAL_BLOCKS)
    mem = uncoal + coal

    # emit_occupancy_core (perfmodel.hpp:545-614)
    if hw.T_max < T or T < 1:
        raise Infeasible()
    wpb = ceil_div(T, Fraction(32))
    blocks = Fraction(hw.B_max)
    blocks = min(blocks, floor_div(Fraction(hw.W_max), wpb))
    if regs != 0:
        blocks = min(blocks, floor_div(Fraction(hw.R_max), regs * T))
    if shared != 0:
        blocks = min(blocks, floor_div(Fraction(hw.Z_max), shared))
    if blocks < 1:
        raise Infeasible()
    warps = min(floor_div(blocks * T, Fraction(32)), Fraction(hw.W_max))
    if warps < 1:
        raise Infeasible()

    mem_l_coal = rat(hw.mem_latency_cycles)
    mem_l_uncoal = rat(hw.mem_latency_cycles) + (Fraction(hw.uncoal_per_mw) - 1) * rat(hw.departure_del_uncoal_cycles)
    comp_cycles = rat(hw.issue_cycles) * (comp + mem)
    rep_den = blocks * hw.num_SM
    rep = ceil_div(tb, rep_den) if rep_mode == "ceil" else emit_div(tb, rep_den)

    if mem == 0:
        pre0 = comp_cycles * rep
        sc0 = rat(hw.departure_del_coal_cycles) * (warps - 1) * synch * blocks * rep
        return pre0 + sc0

    r_uncoal = emit_div(uncoal, mem)
    r_coal = 1 - r_uncoal
    weighted = r_uncoal * mem_l_uncoal + r_coal * mem_l_coal
    dd = r_uncoal * rat(hw.departure_del_uncoal_cycles) * hw.uncoal_per_mw + r_coal * rat(hw.departure_del_coal_cycles)
    mem_cycles = uncoal * mem_l_uncoal + coal * mem_l_coal
    mwp_no_bw = emit_div(weighted, dd)
    bw_per_warp = emit_div(rat(hw.freq_GHz) * hw.load_bytes_per_warp, rat(hw.mem_latency_cycles))
    mwp_peak_bw = emit_div(rat(hw.mem_bandwidth_GBps), bw_per_warp * hw.num_SM)
    mwp = min(mwp_no_bw, mwp_peak_bw)
    mwp = min(mwp, warps)
    if comp_cycles == 0:
        cwp = warps
    else:
        cwp = min(emit_div(mem_cycles + comp_cycles, comp_cycles), warps)
    comp_per_mem = emit_div(comp_cycles, mem)
    mwp_m1 = mwp - 1
    if mwp == warps and cwp == warps:
        pre = (mem_cycles + comp_cycles + comp_per_mem * mwp_m1) * rep
    elif not (cwp < mwp) or (mem_cycles < comp_cycles):
        pre = (emit_div(mem_cycles * warps, mwp) + comp_per_mem * mwp_m1) * rep
    else:
        pre = (mem_l_coal + comp_cycles * warps) * rep
    synch_cost = dd * mwp_m1 * synch * blocks * rep
    return pre + synch_cost


def search(spec: F.MetricSpec, hw: F.DeviceProfile, data: Sequence[int],
           space: Sequence[Tuple[int, int, int]], rep_mode: str = "real",
           tie_rel_tol: float = 1e-12):
    """Exact cycles per config, ranking order of feasible configs and tie
    count (pipeline.hpp:584-679; occupancy for the tie-break is supplied by
    the caller's direct-path values when needed)."""
    vals = [program_value(spec, hw, data, c, rep_mode) for c in space]
    feas = [i for i, v in enumerate(vals) if v >= 0]
    feas.sort(key=lambda i: (vals[i], tuple(space[i])))
    if not feas:
        return vals, [], 0
    best = vals[feas[0]]
    bound = best + best * rat(tie_rel_tol)
    ties = 0
    while ties < len(feas) and vals[feas[ties]] <= bound:
        ties += 1
    return vals, feas, ties
