"""pipe::sanity_report batched on the GPU (pipeline.hpp:710-857; SURVEY.md 8
f2): per distinct data tuple of a sample set, the best sampled
configuration under the cycle model fed with the *collected* metrics
(measured_best) against the rational program's argmin over the same sampled
configurations (predicted_best), plus the collected-metric cycles at the
program's pick.

Both sides run on the device in one launch each:

* collected side — ``rpg_mwpcwp_cycles_batch``: perf::mwpcwp_cycles for every
  sample at once (IEEE, the reference's operation order; ZeroOccupancy rows
  are skipped, ModelError propagates as in the reference);
* program side — one metric-spec plan over the union of the sampled
  configurations and ``rpg_search_batch_subsets``: every tuple searched over
  its own sampled configurations (search_optimal's ranking, ties and
  occupancy tie-break on that subset).

The per-group argmin of the collected side and the bookkeeping are host
numpy.  Formatters reproduce format_sanity_{csv,jsonl,text}
(pipeline.hpp:927-993).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import abi as A
from . import formats as F
from . import search as S
from .samples import SampleSet, format_double

Config = Tuple[int, int, int]


@dataclass
class SanityRow:
    data_params: List[int]
    measured_best: Config
    measured_best_cycles: float
    predicted_best: Config
    predicted_best_cycles: float
    collected_cycles: float


@dataclass
class SanityReport:
    param_names: List[str] = field(default_factory=list)
    rows: List[SanityRow] = field(default_factory=list)
    notes: List[str] = field(default_factory=list)


def metrics_from_samples(samples: SampleSet, models: F.MetricModelSet) -> np.ndarray:
    """detail::metrics_from_sample (pipeline.hpp:733-752) for every sample:
    n x 7 in RPG_METRIC_* order; declared constants fill absent columns."""
    n = len(samples)
    out = np.empty((n, len(F.METRIC_SLOTS)), dtype=np.float64)
    for j, name in enumerate(F.METRIC_SLOTS):
        if name in samples.metric_names:
            out[:, j] = samples.column(name)
        elif name in models.constants:
            out[:, j] = models.constants[name]
        else:
            raise F.PipelineError(f"sample provides no metric '{name}' and no constant is "
                                  "declared for it")
    return out


def mwpcwp_cycles_batch(hw: F.DeviceProfile, metrics: np.ndarray, configs: np.ndarray,
                        rep_mode: str = "real", device: int = 0):
    """perf::mwpcwp_cycles per row on the GPU: (total, b, W, tag, status)."""
    lib = A.load_library()
    metrics = np.ascontiguousarray(metrics, dtype=np.float64)
    cfg = A.config_array([tuple(int(v) for v in c) for c in configs]) if len(configs) else \
        np.zeros(0, dtype=[("bx", "<i8"), ("by", "<i8"), ("bz", "<i8")])
    n = len(cfg)
    total = np.empty(n, dtype=np.float64)
    b = np.empty(n, dtype=np.int32)
    w = np.empty(n, dtype=np.int32)
    tag = np.empty(n, dtype=np.uint8)
    st = np.empty(n, dtype=np.int32)
    err = C.create_string_buffer(512)
    hws = A.profile_struct(hw)
    rc = lib.rpg_mwpcwp_cycles_batch(
        C.byref(hws), A.ptr(metrics, C.c_double) if n else None,
        A.ptr(cfg, A.rpg_config) if n else None, n,
        A.RPG_REP_CEIL if rep_mode == "ceil" else A.RPG_REP_REAL, device,
        total.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
        w.ctypes.data_as(C.c_void_p), tag.ctypes.data_as(C.c_void_p),
        st.ctypes.data_as(C.c_void_p), err, len(err))
    A.check(rc, err)
    return total, b, w, tag, st


def mwpcwp_breakdown_batch(hw: F.DeviceProfile, kernel_metrics: np.ndarray, configs: np.ndarray,
                           rep_mode: str = "real", device: int = 0) -> np.ndarray:
    """perf::mwpcwp_cycles per row on the GPU with the full MwpCwpBreakdown
    (rows: KernelMetrics field order, perfmodel.hpp:68-77, mem as given).
    Returns a BREAKDOWN_DTYPE array; `status` 0 ok, 1/4 ZeroOccupancy,
    2/3 ModelError (rpg.h)."""
    lib = A.load_library()
    km = np.ascontiguousarray(kernel_metrics, dtype=np.float64).reshape(-1, 8)
    cfg = A.config_array([tuple(int(v) for v in c) for c in configs]) if len(configs) else \
        np.zeros(0, dtype=[("bx", "<i8"), ("by", "<i8"), ("bz", "<i8")])
    n = len(cfg)
    if len(km) != n:
        raise ValueError("one metrics row per configuration")
    out = np.zeros(n, dtype=A.BREAKDOWN_DTYPE)
    err = C.create_string_buffer(512)
    hws = A.profile_struct(hw)
    rc = lib.rpg_mwpcwp_breakdown_batch(
        C.byref(hws), A.ptr(km, C.c_double) if n else None,
        A.ptr(cfg, A.rpg_config) if n else None, n,
        A.RPG_REP_CEIL if rep_mode == "ceil" else A.RPG_REP_REAL, device,
        out.ctypes.data_as(C.c_void_p), err, len(err))
    A.check(rc, err)
    return out


def _label(params) -> str:
    return ",".join(str(int(p)) for p in params)


def sanity_report(models: F.MetricModelSet, samples: SampleSet, hw: F.DeviceProfile,
                  rep_mode: str = "real", arith: str = "exact", device: int = 0) -> SanityReport:
    """pipe::sanity_report(models, samples, generate_rp(models, hw), hw,
    rep_mode) — the program is the one generated from the models (the CLI's
    `sanity` path, ratprog_cli.cpp:345-366)."""
    if not models.models:
        raise F.PipelineError("sanity report requires at least one fitted model")
    if len(samples) == 0:
        raise F.PipelineError("sanity report requires a non-empty sample set")
    spec = F.models_to_metric_spec(models)
    metrics = metrics_from_samples(samples, models)
    total, _, _, _, status = mwpcwp_cycles_batch(hw, metrics, samples.configs, rep_mode, device)
    if (status >= 2).any():
        # perf::ModelError propagates out of sanity_report (pipeline.hpp:797-806)
        first = int(np.argmax(status >= 2))
        raise F.ModelError("metrics must be non-negative" if status[first] == 2 else
                           "metrics inconsistent: uncoal + coal must equal mem_insts")

    report = SanityReport([f"D{i}" for i in range(1, samples.dims() + 1)])
    # groups: std::map over the data tuple (lexicographic), members in input order
    groups, inverse = np.unique(samples.data, axis=0, return_inverse=True)
    inverse = inverse.reshape(-1)
    order = np.argsort(inverse, kind="stable")
    bounds = np.searchsorted(inverse[order], np.arange(len(groups) + 1))

    # Union space (lex order) and per-sample config index.
    space, cfg_index = np.unique(samples.configs, axis=0, return_inverse=True)
    cfg_index = cfg_index.reshape(-1).astype(np.int32)
    cfg_tuples = [tuple(int(v) for v in c) for c in space]

    measured = []  # (group, member index of the collected argmin)
    for g in range(len(groups)):
        members = order[bounds[g]:bounds[g + 1]]
        best = -1
        for i in members:
            if status[i] != 0:
                continue
            if best < 0 or total[i] < total[best] or (
                    total[i] == total[best] and
                    tuple(samples.configs[i]) < tuple(samples.configs[best])):
                best = int(i)
        if best < 0:
            report.notes.append(f"D=({_label(groups[g])}): no sampled configuration is "
                                "feasible; skipped")
            continue
        measured.append((g, best))
    if not measured:
        return report

    offsets = np.zeros(len(measured) + 1, dtype=np.int64)
    lists = []
    for k, (g, _) in enumerate(measured):
        members = order[bounds[g]:bounds[g + 1]]
        lists.append(cfg_index[members])
        offsets[k + 1] = offsets[k] + len(members)
    flat = np.ascontiguousarray(np.concatenate(lists), dtype=np.int32)
    tuples = np.ascontiguousarray(groups[[g for g, _ in measured]], dtype=np.int64)
    opts = S.SearchOptions(rep_mode=rep_mode, arith=arith, device=device,
                           regs_per_thread=0.0, shared_words_per_block=0.0)
    with S.Plan(spec, hw, cfg_tuples, opts) as plan:
        win = plan.search_batch_subsets(tuples, offsets, flat)

    for k, (g, best) in enumerate(measured):
        w = win[k]
        params = [int(p) for p in groups[g]]
        if w["n_feasible"] == 0:
            report.notes.append(f"D=({_label(params)}): program marks every sampled "
                                "configuration infeasible; skipped")
            continue
        pred = cfg_tuples[int(w["cfg_idx"])]
        collected = math.nan
        members = order[bounds[g]:bounds[g + 1]]
        for i in members:
            if cfg_index[i] == w["cfg_idx"]:
                if status[i] == 0:
                    collected = float(total[i])
                break
        report.rows.append(SanityRow(params, tuple(int(v) for v in samples.configs[best]),
                                     float(total[best]), pred, float(w["ec"]), collected))
    return report


# ---------------------------------------------------------------------------
# Formatters (pipeline.hpp:863-993)

def _config_label(c: Config) -> str:
    return f"{c[0]}x{c[1]}x{c[2]}"


def format_table(header: List[str], rows: List[List[str]]) -> str:
    """detail::format_table (pipeline.hpp:870-893)."""
    width = [len(h) for h in header]
    for row in rows:
        for j, cell in enumerate(row):
            width[j] = max(width[j], len(cell))

    def emit(row):
        parts = []
        for j, cell in enumerate(row):
            parts.append(cell + (" " * (width[j] - len(cell) + 2) if j + 1 < len(row) else ""))
        return "".join(parts) + "\n"

    total = sum(w + (2 if j + 1 < len(width) else 0) for j, w in enumerate(width))
    return emit(header) + "-" * total + "\n" + "".join(emit(r) for r in rows)


def format_sanity_csv(r: SanityReport) -> str:
    out = "".join(p + "," for p in r.param_names)
    out += "ci_bx,ci_by,ci_bz,Ec_i,cr_bx,cr_by,cr_bz,Ec_r,collected_Ec\n"
    for row in r.rows:
        out += "".join(f"{p}," for p in row.data_params)
        m, p = row.measured_best, row.predicted_best
        out += (f"{m[0]},{m[1]},{m[2]},{format_double(row.measured_best_cycles)},"
                f"{p[0]},{p[1]},{p[2]},{format_double(row.predicted_best_cycles)},"
                f"{format_double(row.collected_cycles)}\n")
    return out


def _json_num(v: float):
    return None if not math.isfinite(v) else v


def format_sanity_jsonl(r: SanityReport) -> str:
    out = ""
    for row in r.rows:
        j = {"data_params": row.data_params, "measured_best": list(row.measured_best),
             "Ec_i": _json_num(row.measured_best_cycles),
             "predicted_best": list(row.predicted_best),
             "Ec_r": _json_num(row.predicted_best_cycles),
             "collected_Ec": _json_num(row.collected_cycles)}
        out += json.dumps(j, separators=(",", ":")) + "\n"
    return out


def format_sanity_text(r: SanityReport) -> str:
    header = list(r.param_names) + ["C_i", "Ec_i", "C_r", "Ec_r", "collected Ec"]
    rows = []
    for row in r.rows:
        rows.append([str(p) for p in row.data_params] + [
            _config_label(row.measured_best), format_double(row.measured_best_cycles),
            _config_label(row.predicted_best), format_double(row.predicted_best_cycles),
            format_double(row.collected_cycles)])
    out = format_table(header, rows)
    for note in r.notes:
        out += f"note: {note}\n"
    return out
