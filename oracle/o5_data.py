"""ORACLE O5 — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench cpu legs).

CPU restatements of the hot path's callers:

* ``MT19937_64`` / ``uniform_real`` — std::mt19937_64 (the C++ standard's
  parameters) and rng::uniform_real (rng.hpp:14-21); pinned by the standard's
  10000th-output value and by tests/golden/std_vectors.json;
* ``synthesize`` — data::synthesize (datakit.hpp:164-218) on O1's
  eval_ratfunc (polyfit.hpp:96-130);
* ``sanity_report`` — pipe::sanity_report (pipeline.hpp:770-857) on O1's
  mwpcwp_cycles (the collected side) and O1's search_one over each tuple's
  sampled configurations (the program side).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64: w=64, n=312, m=156, r=31, a=0xB5026F5AA96619E9,
    u=29, d=0x5555555555555555, s=17, b=0x71D67FFFEDA60000, t=37,
    c=0xFFF7EEE000000000, l=43, f=6364136223846793005."""

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            x = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (x ^ (x >> 62)) + i) & MASK64
        self.i = 312

    def _twist(self):
        mt = self.mt
        for k in range(312):
            y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
            v = mt[(k + 156) % 312] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[k] = v
        self.i = 0

    def __call__(self) -> int:
        if self.i >= 312:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


def uniform_real(g: MT19937_64, lo: float, hi: float) -> float:
    c = float(g() >> 11) * 2.0 ** -53
    return lo + (hi - lo) * c


def _poly(p: F.Polynomial, nv: int):
    coef = np.ascontiguousarray(p.coeffs, dtype=np.float64)
    exps = np.ascontiguousarray(np.array(p.basis, dtype=np.uint8).reshape(len(p.basis), nv))
    st = A.rpg_poly(len(coef), 0, A.ptr(coef, C.c_double) if len(coef) else None,
                    exps.ctypes.data_as(C.POINTER(C.c_uint8)) if len(coef) else None)
    return st, (coef, exps)


def eval_ratfunc(f: F.RationalFunction, x: Sequence[float]) -> Optional[float]:
    """O1 eval_ratfunc; None on DenominatorNearZero."""
    lib = o1.lib()
    nv = len(x)
    num, k1 = _poly(f.num, nv)
    den, k2 = _poly(f.den, nv)
    xs = (C.c_double * nv)(*x)
    out = C.c_double(0.0)
    rc = lib.o1_eval_ratfunc(C.byref(num), C.byref(den), nv, xs, C.byref(out))
    return None if rc else out.value


def synthesize(spec: F.SyntheticKernelSpec, data, configs, seed: int):
    """Returns (metric_names, rows [(data tuple, config, [values])], skipped)."""
    names = sorted(spec.ground_truth)
    g = MT19937_64(seed)
    rows, skipped = [], []
    for dp, cfg in zip(data, configs):
        dp = [int(v) for v in dp]
        cfg = tuple(int(v) for v in cfg)
        coords, nxt = [], 0
        for v in spec.variables:
            if v in ("bx", "by", "bz"):
                coords.append(float(cfg["xyz".index(v[1])]))
            else:
                coords.append(float(dp[nxt]))
                nxt += 1
        lab = "(" + ",".join((("D=" if i == 0 else "") + str(p)) for i, p in enumerate(dp)) + \
            f" {cfg[0]}x{cfg[1]}x{cfg[2]})"
        vals, ok = [], True
        for name in names:
            v = eval_ratfunc(spec.ground_truth[name], coords)
            if v is None:
                skipped.append(f"{lab}: metric '{name}' has a singular denominator")
                ok = False
                break
            if v < 0:
                skipped.append(f"{lab}: metric '{name}' is negative ({'%f' % v})")
                ok = False
                break
            vals.append(v)
        if not ok:
            continue
        if spec.noise_rel > 0:
            vals = [v * (1.0 + uniform_real(g, -spec.noise_rel, spec.noise_rel)) for v in vals]
        rows.append((tuple(dp), cfg, vals))
    return names, rows, skipped


def _metrics(vals: Dict[str, float], constants: Dict[str, float]):
    def value(name):
        if name in vals:
            return vals[name]
        if name in constants:
            return constants[name]
        raise F.PipelineError(f"sample provides no metric '{name}' and no constant is "
                              "declared for it")
    R, Z = value(F.METRIC_REGS), value(F.METRIC_SHARED)
    comp, unc, coal = value(F.METRIC_COMP), value(F.METRIC_UNCOAL), value(F.METRIC_COAL)
    syn, tb = value(F.METRIC_SYNCH), value(F.METRIC_TOTAL_BLOCKS)
    return o1.metrics(comp, unc, coal, syn, tb, R=R, Z=Z)


def sanity_report(models: F.MetricModelSet, names: List[str], rows, hw: F.DeviceProfile,
                  rep_mode: str = "real"):
    """pipe::sanity_report over (data, config, values) rows; returns
    (rows [(params, measured_cfg, Ec_i, predicted_cfg, Ec_r, collected)], notes)."""
    hws = A.profile_struct(hw)
    rm = A.RPG_REP_CEIL if rep_mode == "ceil" else A.RPG_REP_REAL
    spec = F.models_to_metric_spec(models)
    pk = A.PackedModel(spec, drop_zero_terms=False)
    opts = A.options_struct(rep_mode=rm)
    groups: Dict[Tuple[int, ...], list] = {}
    for dp, cfg, vals in rows:
        groups.setdefault(tuple(dp), []).append((cfg, dict(zip(names, vals))))
    out, notes = [], []
    for params in sorted(groups):
        members = groups[params]
        best_cfg, best = None, None
        for cfg, vals in members:
            st, bd = o1.mwpcwp_cycles(hws, _metrics(vals, models.constants), cfg, rm)
            if st == 1:  # ZeroOccupancy
                continue
            if st != 0:
                raise F.ModelError("metrics must be non-negative")
            t = bd.total_cycles
            if best is None or t < best or (t == best and cfg < best_cfg):
                best_cfg, best = cfg, t
        label = ",".join(str(p) for p in params)
        if best is None:
            notes.append(f"D=({label}): no sampled configuration is feasible; skipped")
            continue
        space = sorted(cfg for cfg, _ in members)
        w, order = o1.search_one(pk, hws, opts, A.config_array(space), list(params))
        if w.n_feasible == 0:
            notes.append(f"D=({label}): program marks every sampled configuration infeasible; "
                         "skipped")
            continue
        pred = space[w.cfg_idx]
        collected = math.nan
        for cfg, vals in members:
            if cfg == pred:
                st, bd = o1.mwpcwp_cycles(hws, _metrics(vals, models.constants), cfg, rm)
                if st == 0:
                    collected = bd.total_cycles
                break
        out.append((list(params), best_cfg, best, pred, w.ec, collected))
    return out, notes
