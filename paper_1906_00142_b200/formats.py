"""Host-side data formats of the rational-program evaluator.

Mirrors the reference's data plumbing on the hot path so the GPU path reads
exactly what ``ratprog`` reads (all citations relative to
``/root/reference/proj/include/ratprog``):

* device profiles — ``perf::parse_profile`` / ``load_profile``
  (perfmodel.hpp:87-192), same keys, checks and messages;
* graded-lex monomial bases — ``poly::monomial_basis`` (polyfit.hpp:50-73);
* kernel specs (``ratprog-kernel-v1``, datakit.hpp:491-622) and fitted model
  sets (``ratprog-models-v1``, pipeline.hpp:996-1089);
* ``perf::MetricSpec`` + ``check_metric_spec`` (perfmodel.hpp:401-456);
* ``data::enumerate_configs`` (datakit.hpp:79-94) and the dense integer
  block grids the benchmark sweeps (bx*by[*bz] <= T_max).

Pure host logic: no arithmetic of the evaluator lives here.
"""
from __future__ import annotations

import json
import math
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple


class ProfileError(RuntimeError):
    """perf::ProfileError (perfmodel.hpp:37)."""


class ModelError(RuntimeError):
    """perf::ModelError (perfmodel.hpp:43)."""


class KernelSpecError(RuntimeError):
    """data::KernelSpecError (datakit.hpp:36)."""


class PipelineError(RuntimeError):
    """pipe::PipelineError (pipeline.hpp:41)."""


# ---------------------------------------------------------------------------
# Device profiles (perfmodel.hpp:50-192)

PROFILE_KEYS = (
    "R_max", "Z_max", "T_max", "B_max", "W_max", "num_SM", "freq_GHz",
    "mem_latency_cycles", "departure_del_coal_cycles",
    "departure_del_uncoal_cycles", "mem_bandwidth_GBps", "issue_cycles",
    "load_bytes_per_warp", "uncoal_per_mw",
)
_COUNT_KEYS = ("R_max", "Z_max", "T_max", "B_max", "W_max", "num_SM",
               "load_bytes_per_warp", "uncoal_per_mw")


@dataclass
class DeviceProfile:
    R_max: int = 0
    Z_max: int = 0
    T_max: int = 0
    B_max: int = 0
    W_max: int = 0
    num_SM: int = 0
    freq_GHz: float = 0.0
    mem_latency_cycles: float = 0.0
    departure_del_coal_cycles: float = 0.0
    departure_del_uncoal_cycles: float = 0.0
    mem_bandwidth_GBps: float = 0.0
    issue_cycles: float = 0.0
    load_bytes_per_warp: int = 0
    uncoal_per_mw: int = 0


def parse_profile(text: str) -> DeviceProfile:
    """perf::parse_profile (perfmodel.hpp:111-180)."""
    seen: Dict[str, float] = {}
    for line_no, line in enumerate(text.split("\n"), start=1):
        stripped = line.split("#", 1)[0]
        if stripped.strip(" \t\r") == "":
            continue
        if "=" not in stripped:
            raise ProfileError(f"profile line {line_no}: expected 'key = value'")
        key, value = stripped.split("=", 1)
        key, value = key.strip(" \t\r"), value.strip(" \t\r")
        if key not in PROFILE_KEYS:
            raise ProfileError(f"profile line {line_no}: unknown key '{key}'")
        if key in seen:
            raise ProfileError(f"profile line {line_no}: duplicate key '{key}'")
        try:
            v = _stod(value)
        except ValueError:
            raise ProfileError(
                f"profile line {line_no}: bad numeric value '{value}'") from None
        if not (v > 0):
            raise ProfileError(f"profile line {line_no}: '{key}' must be positive")
        seen[key] = v
    for key in PROFILE_KEYS:
        if key not in seen:
            raise ProfileError(f"profile is missing key '{key}'")
    hw = DeviceProfile()
    for key in PROFILE_KEYS:
        v = seen[key]
        if key in _COUNT_KEYS:
            if not math.isfinite(v) or v != math.floor(v):
                raise ProfileError(f"profile key '{key}' must be an integer")
            setattr(hw, key, int(v))
        else:
            setattr(hw, key, float(v))
    if hw.T_max > 1024:
        raise ProfileError("T_max exceeds 1024, the architectural block limit")
    return hw


_STOD_DEC = re.compile(r"[+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?")
_STOD_HEX = re.compile(r"[+-]?0[xX]([0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)([pP][+-]?\d+)?")
_STOD_SPECIAL = re.compile(r"[+-]?(inf|infinity|nan(\([0-9A-Za-z_]*\))?)", re.IGNORECASE)


def _stod(s: str) -> float:
    """std::stod(s, &used) with used == s.size() (perfmodel.hpp:141-143):
    strtod's grammar — decimal and exponent forms, hexadecimal floats
    (0x1.8p3), inf / infinity / nan[(chars)] in any case — and stod's
    out_of_range on overflow and on underflow of a nonzero literal.  Raises
    ValueError on anything else (no underscores, no surrounding blanks)."""
    if _STOD_SPECIAL.fullmatch(s):
        return float(s.split("(")[0])
    if _STOD_HEX.fullmatch(s):
        sign = -1.0 if s[0] == "-" else 1.0
        body = s.lstrip("+-")
        if not re.search(r"[pP]", body):
            body += "p0"
        try:
            v = sign * float.fromhex(body)
        except OverflowError:
            raise ValueError(s) from None
        digits = re.sub(r"[pP].*$", "", body[2:])
    elif _STOD_DEC.fullmatch(s):
        v = float(s)
        digits = re.sub(r"[eE].*$", "", s)
    else:
        raise ValueError(s)
    if math.isinf(v):
        raise ValueError(s)  # ERANGE: overflow
    if (v == 0.0 or abs(v) < 2.2250738585072014e-308) and re.search(r"[1-9a-fA-F]", digits):
        raise ValueError(s)  # ERANGE: underflow of a nonzero literal
    return v


def load_profile(path: str) -> DeviceProfile:
    """perf::load_profile (perfmodel.hpp:182-192)."""
    try:
        with open(path, "r") as f:
            text = f.read()
    except OSError:
        raise ProfileError(f"cannot open device profile '{path}'") from None
    try:
        return parse_profile(text)
    except ProfileError as e:
        raise ProfileError(f"{path}: {e}") from None


def format_profile(hw: DeviceProfile) -> str:
    """perf::format_profile (perfmodel.hpp:194-208)."""
    out = []
    for key in PROFILE_KEYS:
        v = getattr(hw, key)
        out.append(f"{key} = {_fmt_num(v)}")
    return "\n".join(out) + "\n"


def _fmt_num(v) -> str:
    if isinstance(v, int):
        return str(v)
    return repr(float(v)).rstrip("0").rstrip(".") if float(v).is_integer() else repr(float(v))


# ---------------------------------------------------------------------------
# Polynomials (polyfit.hpp:41-84)

def monomial_basis(bounds: Sequence[int]) -> List[Tuple[int, ...]]:
    """Graded-lex exponent tuples (polyfit.hpp:50-73): ascending total degree,
    ties broken lexicographically with the first variable most significant."""
    for b in bounds:
        if b < 0:
            raise ValueError("negative degree bound")
    tuples: List[Tuple[int, ...]] = [()]
    for b in bounds:
        tuples = [t + (e,) for t in tuples for e in range(b + 1)]
    # Python's sort is stable, like std::stable_sort.
    tuples.sort(key=lambda t: (sum(t), t))
    return tuples


@dataclass
class Polynomial:
    variables: List[str]
    basis: List[Tuple[int, ...]]
    coeffs: List[float]


@dataclass
class RationalFunction:
    num: Polynomial
    den: Polynomial


def make_ratfunc(variables, num_bounds, num_coeffs, den_bounds, den_coeffs,
                 metric: str = "?") -> RationalFunction:
    nb = monomial_basis(num_bounds)
    db = monomial_basis(den_bounds)
    if len(nb) != len(num_coeffs):
        raise KernelSpecError(
            f"metric '{metric}': 'num_coeffs' must have {len(nb)} entries for these bounds")
    if len(db) != len(den_coeffs):
        raise KernelSpecError(
            f"metric '{metric}': 'den_coeffs' must have {len(db)} entries for these bounds")
    return RationalFunction(
        Polynomial(list(variables), nb, [float(c) for c in num_coeffs]),
        Polynomial(list(variables), db, [float(c) for c in den_coeffs]))


# ---------------------------------------------------------------------------
# Metric specs (perfmodel.hpp:401-456)

METRIC_COMP = "comp_insts_per_thread"
METRIC_UNCOAL = "uncoal_mem_insts_per_thread"
METRIC_COAL = "coal_mem_insts_per_thread"
METRIC_SYNCH = "synch_insts_per_block"
METRIC_TOTAL_BLOCKS = "total_blocks"
METRIC_REGS = "regs_per_thread"
METRIC_SHARED = "shared_words_per_block"

REQUIRED_METRICS = (METRIC_COMP, METRIC_UNCOAL, METRIC_COAL, METRIC_SYNCH,
                    METRIC_TOTAL_BLOCKS)
# Slot order of the C ABI (= evaluate_metrics order, perfmodel.hpp:468-476).
METRIC_SLOTS = (METRIC_REGS, METRIC_SHARED, METRIC_COMP, METRIC_UNCOAL,
                METRIC_COAL, METRIC_SYNCH, METRIC_TOTAL_BLOCKS)


@dataclass
class MetricSpec:
    variables: List[str] = field(default_factory=list)
    models: Dict[str, RationalFunction] = field(default_factory=dict)
    constants: Dict[str, float] = field(default_factory=dict)

    def covers(self, name: str) -> bool:
        return name in self.models or name in self.constants


def _is_data_param(v: str) -> bool:
    return len(v) >= 2 and v[0] == "D" and v[1:].isdigit()


def check_metric_spec(spec: MetricSpec) -> None:
    """perf::check_metric_spec (perfmodel.hpp:428-456)."""
    for name in REQUIRED_METRICS:
        if not spec.covers(name):
            raise ModelError(f"metric '{name}' has neither a model nor a constant")
    for name in (METRIC_REGS, METRIC_SHARED):
        if not spec.covers(name):
            raise ModelError(f"metric '{name}' has neither a model nor a constant")
    has_bx = has_by = False
    for v in spec.variables:
        has_bx |= v == "bx"
        has_by |= v == "by"
        if v in PROFILE_KEYS:
            raise ModelError(f"variable '{v}' collides with a hardware field")
        if not _is_data_param(v) and v not in ("bx", "by", "bz"):
            raise ModelError(
                f"variable '{v}' is not a data parameter (D1..Dd) or block dimension")
    if not has_bx or not has_by:
        raise ModelError("metric variables must include bx and by")
    for name, f in spec.models.items():
        if f.num.variables != spec.variables:
            raise ModelError(f"model '{name}' disagrees with the shared variable order")


def data_param_count(spec: MetricSpec) -> int:
    """Highest data-parameter index the spec references (D_k -> k)."""
    d = 0
    for v in spec.variables:
        if _is_data_param(v):
            d = max(d, int(v[1:]))
    return d


# ---------------------------------------------------------------------------
# Kernel specs / model sets (datakit.hpp:491-622, pipeline.hpp:996-1089)

def _ratfunc_from_json(j: dict, variables: List[str], metric: str) -> RationalFunction:
    for key in ("num_bounds", "num_coeffs", "den_bounds", "den_coeffs"):
        if key not in j:
            raise KernelSpecError(f"metric '{metric}' is missing '{key}'")
    for bkey in ("num_bounds", "den_bounds"):
        if len(j[bkey]) != len(variables):
            raise KernelSpecError(
                f"metric '{metric}': '{bkey}' must have one entry per variable")
    return make_ratfunc(variables, j["num_bounds"], j["num_coeffs"],
                        j["den_bounds"], j["den_coeffs"], metric)


def ratfunc_to_json(f: RationalFunction) -> dict:
    def bounds_of(p: Polynomial):
        b = [0] * len(p.variables)
        for mono in p.basis:
            for i, e in enumerate(mono):
                b[i] = max(b[i], e)
        return b
    return {"num_bounds": bounds_of(f.num), "num_coeffs": list(f.num.coeffs),
            "den_bounds": bounds_of(f.den), "den_coeffs": list(f.den.coeffs)}


@dataclass
class SyntheticKernelSpec:
    """data::SyntheticKernelSpec (datakit.hpp:65-72)."""
    name: str = "kernel"
    variables: List[str] = field(default_factory=list)
    ground_truth: Dict[str, RationalFunction] = field(default_factory=dict)
    regs_per_thread: float = 0.0
    shared_words_per_block: float = 0.0
    noise_rel: float = 0.0


def parse_kernel_spec(text: str) -> SyntheticKernelSpec:
    """data::parse_kernel_spec (datakit.hpp:537-584)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise KernelSpecError(f"kernel spec is not valid JSON: {e}") from None
    if j.get("schema") != "ratprog-kernel-v1":
        raise KernelSpecError("kernel spec must declare schema 'ratprog-kernel-v1'")
    spec = SyntheticKernelSpec()
    spec.name = j.get("name", "kernel")
    if "variables" not in j:
        raise KernelSpecError("kernel spec is missing 'variables'")
    spec.variables = list(j["variables"])
    c = j.get("constants", {})
    spec.regs_per_thread = float(c.get(METRIC_REGS, 0.0))
    spec.shared_words_per_block = float(c.get(METRIC_SHARED, 0.0))
    spec.noise_rel = float(j.get("noise_rel", 0.0))
    if spec.noise_rel < 0:
        raise KernelSpecError("noise_rel must be >= 0")
    if not isinstance(j.get("metrics"), dict):
        raise KernelSpecError("kernel spec is missing the 'metrics' object")
    for name in sorted(j["metrics"]):  # std::map iteration order
        spec.ground_truth[name] = _ratfunc_from_json(j["metrics"][name], spec.variables, name)
    for req in REQUIRED_METRICS:
        if req not in spec.ground_truth:
            raise KernelSpecError(f"kernel spec is missing metric '{req}'")
    try:
        check_metric_spec(kernel_to_metric_spec(spec, check=False))
    except ModelError as e:
        raise KernelSpecError(str(e)) from None
    return spec


def load_kernel_spec(path: str) -> SyntheticKernelSpec:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise KernelSpecError(f"cannot open kernel spec '{path}'") from None
    try:
        return parse_kernel_spec(text)
    except KernelSpecError as e:
        raise KernelSpecError(f"{path}: {e}") from None


def format_kernel_spec(spec: SyntheticKernelSpec) -> str:
    j = {"schema": "ratprog-kernel-v1", "name": spec.name,
         "variables": spec.variables,
         "constants": {METRIC_REGS: spec.regs_per_thread,
                       METRIC_SHARED: spec.shared_words_per_block},
         "noise_rel": spec.noise_rel,
         "metrics": {n: ratfunc_to_json(f) for n, f in sorted(spec.ground_truth.items())}}
    return json.dumps(j, indent=2) + "\n"


def kernel_to_metric_spec(spec: SyntheticKernelSpec, check: bool = True) -> MetricSpec:
    """data::to_metric_spec (datakit.hpp:614-622)."""
    m = MetricSpec(list(spec.variables), dict(spec.ground_truth),
                   {METRIC_REGS: spec.regs_per_thread,
                    METRIC_SHARED: spec.shared_words_per_block})
    if check:
        check_metric_spec(m)
    return m


@dataclass
class MetricModelSet:
    """pipe::MetricModelSet (pipeline.hpp:58-68); fit reports kept as dicts."""
    variables: List[str] = field(default_factory=list)
    models: Dict[str, RationalFunction] = field(default_factory=dict)
    reports: Dict[str, dict] = field(default_factory=dict)
    constants: Dict[str, float] = field(default_factory=dict)
    failures: Dict[str, str] = field(default_factory=dict)


def parse_models(text: str) -> MetricModelSet:
    """pipe::parse_models (pipeline.hpp:1020-1069)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise PipelineError(f"models file is not valid JSON: {e}") from None
    if not isinstance(j, dict) or j.get("schema", "") != "ratprog-models-v1":
        raise PipelineError("models file schema must be 'ratprog-models-v1'")
    m = MetricModelSet()
    try:
        m.variables = list(j["variables"])
    except KeyError:
        raise PipelineError("models file is malformed: missing 'variables'") from None
    if not m.variables:
        raise PipelineError("models file declares no variables")
    for name, value in j.get("constants", {}).items():
        m.constants[name] = float(value)
    if not isinstance(j.get("metrics"), dict):
        raise PipelineError("models file is missing the 'metrics' object")
    try:
        for name in sorted(j["metrics"]):
            body = j["metrics"][name]
            m.models[name] = _ratfunc_from_json(body, m.variables, name)
            if "report" in body:
                m.reports[name] = dict(body["report"])
    except KernelSpecError as e:
        raise PipelineError(str(e)) from None
    for name, why in j.get("failures", {}).items():
        m.failures[name] = str(why)
    return m


def read_models(path: str) -> MetricModelSet:
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise PipelineError(f"cannot open '{path}' for reading") from None
    try:
        return parse_models(text)
    except PipelineError as e:
        raise PipelineError(f"{path}: {e}") from None


def format_models(m: MetricModelSet) -> str:
    j = {"schema": "ratprog-models-v1", "variables": m.variables,
         "constants": dict(sorted(m.constants.items())), "metrics": {}}
    for name, f in sorted(m.models.items()):
        body = ratfunc_to_json(f)
        if name in m.reports:
            body["report"] = m.reports[name]
        j["metrics"][name] = body
    j["failures"] = dict(sorted(m.failures.items()))
    return json.dumps(j, indent=2) + "\n"


def models_to_metric_spec(m: MetricModelSet) -> MetricSpec:
    """pipe::to_metric_spec (pipeline.hpp:188-195)."""
    spec = MetricSpec(list(m.variables), dict(m.models), dict(m.constants))
    check_metric_spec(spec)
    return spec


# ---------------------------------------------------------------------------
# Configuration spaces (datakit.hpp:79-94)

def enumerate_configs(max_threads: int = 1024, min_threads: int = 32,
                      dims: int = 2) -> List[Tuple[int, int, int]]:
    """Power-of-two block shapes with thread count in [min, max], lex order."""
    if min_threads < 1 or min_threads > max_threads or max_threads > 1024:
        raise ValueError(
            "enumerate_configs: need 1 <= min_threads <= max_threads <= 1024")
    if dims < 1 or dims > 3:
        raise ValueError("enumerate_configs: dims must be 1, 2 or 3")
    out = []
    bx = 1
    while bx <= 1024:
        by = 1
        while by <= (1024 if dims >= 2 else 1):
            bz = 1
            while bz <= (1024 if dims >= 3 else 1):
                t = bx * by * bz
                if min_threads <= t <= max_threads:
                    out.append((bx, by, bz))
                bz *= 2
            by *= 2
        bx *= 2
    return out


def integer_configs(max_threads: int = 1024, dims: int = 2,
                    min_threads: int = 1) -> List[Tuple[int, int, int]]:
    """Every integer block shape with min <= bx*by[*bz] <= max, lex order —
    the dense config grid of the benchmark sweeps (7,262 shapes for 2-D,
    30,343 for 3-D at max 1024)."""
    out = []
    for bx in range(1, max_threads + 1):
        for by in range(1, (max_threads // bx if dims >= 2 else 1) + 1):
            if dims >= 3:
                for bz in range(1, max_threads // (bx * by) + 1):
                    if bx * by * bz >= min_threads:
                        out.append((bx, by, bz))
            elif bx * by >= min_threads:
                out.append((bx, by, 1))
    return out
