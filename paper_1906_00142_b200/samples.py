"""Profiled samples: the reference's data kit (datakit.hpp) for the hot path's
callers — CSV persistence, design points and synthetic measurement.

A ``SampleSet`` is columnar (numpy): ``data`` (n x d int64 data parameters),
``configs`` (n x 3 int64 block dimensions), ``values`` (n x M float64 metric
values, columns in ``metric_names`` order) — the layout the GPU consumes, not
a vector of per-sample maps.

* ``parse_samples`` / ``format_samples`` — datakit.hpp:272-415: the same
  schema, provenance comment, checks and ``CsvError`` messages; reals are
  written shortest-round-trip exactly as ``std::to_chars`` does
  (``format_double``).
* ``synthesize`` — datakit.hpp:164-218: ground-truth rational functions are
  evaluated on the GPU (``rpg_eval_ratfunc_batch``: eval_ratfunc's operation
  order and DenominatorNearZero rule); the noise stream is
  ``std::mt19937_64`` drawn in order for kept points only
  (``rpg_uniform_stream``), so outputs are bit-identical to the reference's.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from decimal import Decimal
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi as A
from . import formats as F


class CsvError(RuntimeError):
    """data::CsvError (datakit.hpp:33-35)."""


@dataclass
class Provenance:
    """data::Provenance (datakit.hpp:40-46)."""
    kind: str = "measured"  # measured | synthetic
    seed: int = 0
    noise_rel: float = 0.0


@dataclass
class SampleSet:
    metric_names: List[str] = field(default_factory=list)
    data: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.int64))
    configs: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int64))
    values: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.float64))
    provenance: Provenance = field(default_factory=Provenance)

    def __len__(self) -> int:
        return int(self.configs.shape[0])

    def dims(self) -> int:
        return int(self.data.shape[1]) if len(self) else 0

    def column(self, name: str) -> np.ndarray:
        return self.values[:, self.metric_names.index(name)]


# ---------------------------------------------------------------------------
# Number formatting

def format_double(v: float) -> str:
    """std::to_chars(double) shortest form (datakit.hpp:225-230): the
    shortest round-trip digits, printed as %f or %e whichever is shorter
    (fixed on a tie)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    t = Decimal(repr(abs(v))).normalize().as_tuple()  # shortest round-trip digits
    digits = "".join(map(str, t.digits))
    exp = t.exponent  # value = digits * 10^exp
    n = len(digits)
    e10 = exp + n - 1
    sci = digits[0] + ("." + digits[1:] if n > 1 else "") + "e" + ("+" if e10 >= 0 else "-") + \
        f"{abs(e10):02d}"
    if exp >= 0:
        fixed = str(int(abs(v)))  # %f of an integral value: its exact digits
    else:
        pos = n + exp
        fixed = (digits[:pos] + "." + digits[pos:]) if pos > 0 else "0." + "0" * (-pos) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def cpp_to_string(v: float) -> str:
    """std::to_string(double): "%f"."""
    return "%f" % v


# ---------------------------------------------------------------------------
# CSV (datakit.hpp:272-415): native, columnar, multi-threaded (rpg_csv.cpp
# behind rpg_samples_parse / rpg_samples_format).

def parse_samples(text, n_threads: int = 0) -> SampleSet:
    """data::parse_samples (datakit.hpp:329-412) — same schema, checks,
    error precedence and CsvError messages — parsed by librpgpu (columnar,
    all host threads by default).  ``text``: str or bytes."""
    lib = A.load_library()
    raw = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib.rpg_samples_parse(raw, len(raw), n_threads, C.byref(h), err, len(err))
    if rc == A.RPG_E_CSV:
        raise CsvError(err.value.decode(errors="replace"))
    A.check(rc, err)
    try:
        n, d, k, kind = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        seed, noise = C.c_uint64(), C.c_double()
        lib.rpg_samples_info(h, C.byref(n), C.byref(d), C.byref(k), C.byref(kind), C.byref(seed),
                             C.byref(noise))
        names = [lib.rpg_samples_metric_name(h, i).decode() for i in range(k.value)]
        data = np.zeros((n.value, d.value), dtype=np.int64)
        cfg = np.zeros((n.value, 3), dtype=np.int64)
        vals = np.zeros((n.value, k.value), dtype=np.float64)
        lib.rpg_samples_copy(h, data.ctypes.data_as(C.c_void_p), cfg.ctypes.data_as(C.c_void_p),
                             vals.ctypes.data_as(C.c_void_p))
    finally:
        lib.rpg_samples_free(h)
    prov = Provenance("synthetic", seed.value, noise.value) if kind.value == 1 else Provenance()
    return SampleSet(names, data, cfg, vals, prov)


def format_samples(s: SampleSet, n_threads: int = 0) -> str:
    """data::format_samples (datakit.hpp:286-326), formatted by librpgpu
    (std::to_chars shortest round-trip reals)."""
    lib = A.load_library()
    n = len(s)
    d = s.dims() if n else int(s.data.shape[1]) if s.data.ndim == 2 else 0
    data = np.ascontiguousarray(s.data, dtype=np.int64).reshape(n, d)
    cfg = np.ascontiguousarray(s.configs, dtype=np.int64).reshape(n, 3)
    vals = np.ascontiguousarray(s.values, dtype=np.float64).reshape(n, len(s.metric_names))
    names = (C.c_char_p * max(1, len(s.metric_names)))(*[m.encode() for m in s.metric_names])
    kind = 1 if s.provenance.kind == "synthetic" else 0
    err = C.create_string_buffer(512)
    args = (data.ctypes.data_as(C.c_void_p), cfg.ctypes.data_as(C.c_void_p),
            vals.ctypes.data_as(C.c_void_p), n, d, names, len(s.metric_names), kind,
            int(s.provenance.seed) % (1 << 64), float(s.provenance.noise_rel), 0)
    # one pass into a buffer sized for the longest possible rows (int64: 20
    # chars + sign; shortest-round-trip double: at most 24 chars)
    cap = 256 + sum(len(m) + 1 for m in s.metric_names) + n * (22 * (d + 3) + 25 * len(s.metric_names) + 1)
    buf = C.create_string_buffer(cap)
    need = lib.rpg_samples_format(*args, buf, cap, err, len(err))
    if need < 0:
        raise CsvError(err.value.decode(errors="replace"))
    if need >= cap:  # cannot happen with the bound above; stay correct anyway
        buf = C.create_string_buffer(need + 1)
        need = lib.rpg_samples_format(*args, buf, need + 1, err, len(err))
    return C.string_at(buf, need).decode("ascii")


def read_samples(path: str) -> SampleSet:
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise CsvError(f"cannot open '{path}'") from None
    try:
        return parse_samples(text)
    except CsvError as e:
        raise CsvError(f"{path}: {e}") from None


def write_samples(s: SampleSet, path: str) -> None:
    text = format_samples(s)
    try:
        with open(path, "wb") as f:
            f.write(text.encode())
    except OSError:
        raise CsvError(f"cannot open '{path}' for writing") from None


# ---------------------------------------------------------------------------
# Design points and synthetic measurement (datakit.hpp:97-218)

def design_points(d_values: Sequence[int], configs: Sequence[Tuple[int, int, int]]):
    """data::design_points (datakit.hpp:99-112): data-major Cartesian
    product; returns (data n x 1, configs n x 3)."""
    if len(d_values) == 0:
        raise ValueError("design_points: no data-parameter values")
    if len(configs) == 0:
        raise ValueError("design_points: no configurations")
    dv = np.asarray(d_values, dtype=np.int64)
    cf = np.asarray(configs, dtype=np.int64).reshape(-1, 3)
    data = np.repeat(dv, len(cf)).reshape(-1, 1)
    return data, np.tile(cf, (len(dv), 1))


def _label(dp, cfg) -> str:
    s = "(" + ",".join((("D=" if i == 0 else "") + str(int(p))) for i, p in enumerate(dp))
    return s + f" {int(cfg[0])}x{int(cfg[1])}x{int(cfg[2])})"


def _poly_struct(p: F.Polynomial, nv: int):
    coef = np.ascontiguousarray(p.coeffs, dtype=np.float64)
    exps = np.ascontiguousarray(np.array(p.basis, dtype=np.uint8).reshape(len(p.basis), nv))
    st = A.rpg_poly(len(coef), 0, A.ptr(coef, C.c_double) if len(coef) else None,
                    exps.ctypes.data_as(C.POINTER(C.c_uint8)) if len(coef) else None)
    return st, (coef, exps)


def eval_ratfunc_batch(f: F.RationalFunction, X: np.ndarray, device: int = 0):
    """poly::eval_ratfunc at every row of X on the GPU: (values, near_zero)."""
    lib = A.load_library()
    X = np.ascontiguousarray(X, dtype=np.float64)
    m, nv = X.shape
    num, keep1 = _poly_struct(f.num, nv)
    den, keep2 = _poly_struct(f.den, nv)
    out = np.empty(m, dtype=np.float64)
    st = np.empty(m, dtype=np.int32)
    err = C.create_string_buffer(512)
    rc = lib.rpg_eval_ratfunc_batch(C.byref(num), C.byref(den), nv, A.ptr(X, C.c_double), m,
                                    device, A.ptr(out, C.c_double), A.ptr(st, C.c_int32),
                                    err, len(err))
    A.check(rc, err)
    return out, st != 0


def uniform_stream(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    """n draws of rng::uniform_real(lo, hi) from std::mt19937_64(seed)."""
    lib = A.load_library()
    out = np.empty(max(n, 0), dtype=np.float64)
    rc = lib.rpg_uniform_stream(C.c_uint64(seed % (1 << 64)), n, lo, hi,
                                A.ptr(out, C.c_double) if n > 0 else None)
    if rc != A.RPG_OK:
        raise ValueError("uniform_stream: bad arguments")
    return out


def synthesize(spec: F.SyntheticKernelSpec, data: np.ndarray, configs: np.ndarray, seed: int,
               skipped: Optional[List[str]] = None, device: int = 0) -> SampleSet:
    """data::synthesize (datakit.hpp:164-218) over the design points
    (data[i], configs[i])."""
    if spec.noise_rel < 0:
        raise ValueError("synthesize: noise_rel must be >= 0")
    if not spec.ground_truth:
        raise ValueError("synthesize: kernel has no metrics")
    data = np.ascontiguousarray(data, dtype=np.int64).reshape(len(configs), -1)
    configs = np.ascontiguousarray(configs, dtype=np.int64).reshape(-1, 3)
    names = sorted(spec.ground_truth)
    n = len(configs)
    # duplicate design points (datakit.hpp:180-183)
    key = np.concatenate([data, configs], axis=1)
    if n:
        _, counts = np.unique(key, axis=0, return_counts=True)
        if (counts > 1).any():
            seen = set()
            for i in range(n):
                k = tuple(key[i])
                if k in seen:
                    raise ValueError("synthesize: duplicate design point " + _label(data[i], configs[i]))
                seen.add(k)
    # coordinates in the kernel's variable order (datakit.hpp:118-142)
    n_data_vars = sum(1 for v in spec.variables if v not in ("bx", "by", "bz"))
    if data.shape[1] < n_data_vars:
        raise ValueError("synthesize: point has fewer data parameters than the kernel")
    if data.shape[1] > n_data_vars:
        raise ValueError("synthesize: point has more data parameters than the kernel")
    cols, nxt = [], 0
    for v in spec.variables:
        if v in ("bx", "by", "bz"):
            cols.append(configs[:, "xyz".index(v[1])].astype(np.float64))
        else:
            cols.append(data[:, nxt].astype(np.float64))
            nxt += 1
    X = np.stack(cols, axis=1) if cols else np.zeros((n, 0))
    vals = np.empty((n, len(names)), dtype=np.float64)
    bad = np.full(n, -1, dtype=np.int64)  # first failing metric (name order)
    why = np.zeros(n, dtype=np.int8)      # 1 singular, 2 negative
    for j, name in enumerate(names):
        v, nz = eval_ratfunc_batch(spec.ground_truth[name], X, device)
        vals[:, j] = v
        fresh = bad < 0
        sing = fresh & nz
        neg = fresh & ~nz & (v < 0)
        bad[sing | neg] = j
        why[sing] = 1
        why[neg] = 2
    keep = bad < 0
    if skipped is not None:
        for i in np.where(~keep)[0]:
            j = int(bad[i])
            lab = _label(data[i], configs[i])
            if why[i] == 1:
                skipped.append(f"{lab}: metric '{names[j]}' has a singular denominator")
            else:
                skipped.append(f"{lab}: metric '{names[j]}' is negative ({cpp_to_string(vals[i, j])})")
    vals = vals[keep]
    if spec.noise_rel > 0 and len(vals):
        u = uniform_stream(seed, vals.size, -spec.noise_rel, spec.noise_rel).reshape(vals.shape)
        vals = vals * (1.0 + u)
    return SampleSet(names, data[keep], configs[keep], vals,
                     Provenance("synthetic", seed % (1 << 64), spec.noise_rel))
