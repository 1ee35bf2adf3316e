"""Python mirror of the reference's fit API over librpgpu.so's GPU fit.

``fit_rational`` keeps the shape of ``poly::fit_rational`` (polyfit.hpp:
337-427) — returns (RationalFunction, FitReport) — and ``fit_all_metrics``
that of ``pipe::fit_all_metrics`` (pipeline.hpp:145-184).  All arithmetic
runs in the K3 kernels (rpg_fit.cu); the host only packs arguments.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi as A
from . import formats as F

K_DEFAULT_RANK_TOL = 1e-10
# Largest coefficient vector (numerator + denominator basis) the GPU fit
# handles: its R factor and Jacobi SVD live in one CTA's shared memory
# (rpg_fit.cu kMaxCols).  Three variables at the default bounds need 35.
K_MAX_FIT_COLUMNS = 64


class DegenerateFit(RuntimeError):
    """poly::DegenerateFit (polyfit.hpp:32)."""


class SvdFailure(RuntimeError):
    """poly::SvdFailure (polyfit.hpp:35)."""


class AllMetricsFailed(RuntimeError):
    """pipe::AllMetricsFailed (pipeline.hpp:46)."""


@dataclass
class FitReport:
    """poly::FitReport (polyfit.hpp:86-92) + whether the safeguard ran."""
    residual_norm: float = 0.0
    numerical_rank: int = 0
    singular_values: List[float] = field(default_factory=list)
    truncated: bool = False
    holdout_relative_error: Optional[float] = None
    safeguard: bool = False


def fit_rational(X, y, variables: Sequence[str], num_bounds: Sequence[int],
                 den_bounds: Sequence[int], rank_tol: float = K_DEFAULT_RANK_TOL,
                 device: int = 0, trace: Optional[dict] = None) -> Tuple[F.RationalFunction, FitReport]:
    """poly::fit_rational on the GPU.  ``trace`` (a dict, optional) receives
    the safeguard's stages (rpg_fit_rational_traced): "stages" (raw
    coefficient vectors: unconstrained, first minimizer, reweighted rounds),
    "round_qmin" and "stop" — filled even when the fit then fails."""
    lib = A.load_library()
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    m, nv = X.shape if len(y) else (0, len(variables))
    if len(y) != m:
        raise F.ModelError("fit_rational: points/values size mismatch")
    nb = F.monomial_basis(num_bounds)
    db = F.monomial_basis(den_bounds)
    n = len(nb) + len(db)
    coef = np.zeros(n)
    sig = np.zeros(max(1, min(m, n)))
    rank, trunc, safe = C.c_int32(), C.c_int32(), C.c_int32()
    resid = C.c_double()
    nbnd = (C.c_int32 * nv)(*num_bounds)
    dbnd = (C.c_int32 * nv)(*den_bounds)
    err = C.create_string_buffer(512)
    tr = A.rpg_fit_trace() if trace is not None else None
    rc = lib.rpg_fit_rational_traced(
        A.ptr(X, C.c_double) if m else None, A.ptr(y, C.c_double) if m else None,
        m, nv, nbnd, dbnd, rank_tol, device, A.ptr(coef, C.c_double),
        A.ptr(sig, C.c_double), C.byref(rank), C.byref(trunc),
        C.byref(resid), C.byref(safe), C.byref(tr) if tr is not None else None, err, len(err))
    if tr is not None:
        trace["stages"] = [np.array(tr.stage_coef[i][:n]) for i in range(tr.n_stages)]
        started = tr.n_stages - 1 + (1 if tr.stop_reason in (1, 2) else 0) if tr.n_stages >= 2 else 0
        trace["round_qmin"] = [float(tr.round_qmin[i]) for i in range(started)]
        trace["stop"] = A.FIT_STOP_NAMES.get(tr.stop_reason, str(tr.stop_reason))
    if rc != A.RPG_OK:
        msg = err.value.decode()
        if rc == A.RPG_E_INVALID:
            raise ValueError(msg)
        if rc == A.RPG_E_FIT:
            raise (SvdFailure if msg.startswith("svd") else DegenerateFit)(msg)
        raise A.RpgError(rc, msg)
    f = F.RationalFunction(F.Polynomial(list(variables), nb, list(coef[: len(nb)])),
                           F.Polynomial(list(variables), db, list(coef[len(nb):])))
    rep = FitReport(residual_norm=resid.value, numerical_rank=rank.value,
                    singular_values=list(sig[: min(m, n)]), truncated=bool(trunc.value),
                    safeguard=bool(safe.value))
    return f, rep


def fit_rational_multi(X, ys: Sequence, variables: Sequence[str], bounds: Sequence[Tuple[Sequence[int], Sequence[int]]],
                       rank_tol: float = K_DEFAULT_RANK_TOL, device: int = 0,
                       traces: Optional[List[dict]] = None) -> List[object]:
    """Several fit_rational calls over one sample matrix X, run concurrently
    on the GPU (rpg_fit_rational_multi: X uploaded once, one stream per fit).
    Returns per fit (RationalFunction, FitReport), or the DegenerateFit /
    SvdFailure exception instance for a numerical failure."""
    lib = A.load_library()
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    m, nv = X.shape
    k = len(ys)
    jobs = (A.rpg_fit_job * max(k, 1))()
    keep = []
    shapes = []
    for i, (y, (nb_, db_)) in enumerate(zip(ys, bounds)):
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
        if len(y) != m:
            raise F.ModelError("fit_rational: points/values size mismatch")
        nb, db = F.monomial_basis(nb_), F.monomial_basis(db_)
        n = len(nb) + len(db)
        arrs = dict(y=y, nbnd=np.ascontiguousarray(nb_, dtype=np.int32),
                    dbnd=np.ascontiguousarray(db_, dtype=np.int32), coef=np.zeros(n),
                    sig=np.zeros(max(1, min(m, n))), rank=np.zeros(1, np.int32),
                    trunc=np.zeros(1, np.int32), resid=np.zeros(1), safe=np.zeros(1, np.int32),
                    tr=A.rpg_fit_trace() if traces is not None else None)
        keep.append(arrs)
        shapes.append((nb, db, n))
        J = jobs[i]
        J.y = A.ptr(arrs["y"], C.c_double)
        J.num_bounds = A.ptr(arrs["nbnd"], C.c_int32)
        J.den_bounds = A.ptr(arrs["dbnd"], C.c_int32)
        J.coef_out = A.ptr(arrs["coef"], C.c_double)
        J.sigma_out = A.ptr(arrs["sig"], C.c_double)
        J.rank_out = A.ptr(arrs["rank"], C.c_int32)
        J.truncated_out = A.ptr(arrs["trunc"], C.c_int32)
        J.residual_out = A.ptr(arrs["resid"], C.c_double)
        J.safeguard_out = A.ptr(arrs["safe"], C.c_int32)
        if arrs["tr"] is not None:
            J.trace = C.pointer(arrs["tr"])
    err = C.create_string_buffer(512)
    rc = lib.rpg_fit_rational_multi(A.ptr(X, C.c_double), m, nv, jobs, k, rank_tol, device, err, len(err))
    if rc != A.RPG_OK:
        msg = err.value.decode()
        raise ValueError(msg) if rc == A.RPG_E_INVALID else A.RpgError(rc, msg)
    out: List[object] = []
    for i in range(k):
        J, arrs, (nb, db, n) = jobs[i], keep[i], shapes[i]
        if traces is not None:
            tr = arrs["tr"]
            started = tr.n_stages - 1 + (1 if tr.stop_reason in (1, 2) else 0) if tr.n_stages >= 2 else 0
            traces.append({"stages": [np.array(tr.stage_coef[s_][:n]) for s_ in range(tr.n_stages)],
                           "round_qmin": [float(tr.round_qmin[s_]) for s_ in range(started)],
                           "stop": A.FIT_STOP_NAMES.get(tr.stop_reason, str(tr.stop_reason))})
        if J.status != A.RPG_OK:
            msg = J.message.decode(errors="replace")
            if J.status == A.RPG_E_INVALID:
                raise ValueError(msg)
            if J.status == A.RPG_E_FIT:
                out.append((SvdFailure if msg.startswith("svd") else DegenerateFit)(msg))
                continue
            raise A.RpgError(J.status, msg)
        coef = arrs["coef"]
        f = F.RationalFunction(F.Polynomial(list(variables), nb, list(coef[: len(nb)])),
                               F.Polynomial(list(variables), db, list(coef[len(nb):])))
        rep = FitReport(residual_norm=float(arrs["resid"][0]), numerical_rank=int(arrs["rank"][0]),
                        singular_values=list(arrs["sig"][: min(m, n)]), truncated=bool(arrs["trunc"][0]),
                        safeguard=bool(arrs["safe"][0]))
        out.append((f, rep))
    return out


def default_bounds(n_variables: int) -> Tuple[List[int], List[int]]:
    """pipe::default_bounds (pipeline.hpp:88-93)."""
    return [2] * n_variables, [1] * n_variables


def check_metric_inputs(X, metric_values: Dict[str, np.ndarray], variables: Sequence[str],
                        bounds: Dict[str, Tuple[List[int], List[int]]],
                        constants: Dict[str, float]) -> List[str]:
    """The argument checks of pipe::fit_all_metrics (pipeline.hpp:145-184),
    all done before any fit runs (a sharded caller runs them on every rank, so
    a bad argument raises everywhere before any collective).  Returns the
    metrics in fit order (sorted by name)."""
    if len(X) == 0:
        raise ValueError("fit_all_metrics: sample set is empty")
    order = sorted(metric_values)
    for metric in order:
        if metric in constants:
            raise F.PipelineError(
                f"metric '{metric}' is both a sample column and a declared constant")
        nb, db = bounds.get(metric, default_bounds(len(variables)))
        if len(nb) != len(variables) or len(db) != len(variables):
            raise F.PipelineError(f"degree bounds for metric '{metric}' must have "
                                  f"{len(variables)} entries per side")
        cols = int(np.prod([b + 1 for b in nb])) + int(np.prod([b + 1 for b in db]))
        if cols > K_MAX_FIT_COLUMNS:
            raise ValueError(f"metric '{metric}': {cols} basis columns exceed the GPU fit's "
                             f"limit of {K_MAX_FIT_COLUMNS} (lower its degree bounds)")
    return order


def fit_metrics(X, metric_values: Dict[str, np.ndarray], variables: Sequence[str],
                bounds: Dict[str, Tuple[List[int], List[int]]], metrics: Sequence[str],
                rank_tol: float = K_DEFAULT_RANK_TOL, device: int = 0, fit_fn=None) -> Dict[str, object]:
    """Fits the listed metrics; per metric the outcome is (RationalFunction,
    report dict) or, for a numerical failure (``fit_fn`` raised DegenerateFit
    or SvdFailure), the failure message (str)."""
    out: Dict[str, object] = {}
    if fit_fn is None:
        # the GPU fit: every metric at once (one upload of X, concurrent fits)
        res = fit_rational_multi(X, [metric_values[mt] for mt in metrics], variables,
                                 [bounds.get(mt, default_bounds(len(variables))) for mt in metrics],
                                 rank_tol, device)
        for metric, r in zip(metrics, res):
            if isinstance(r, Exception):
                out[metric] = str(r)
            else:
                f, rep = r
                out[metric] = (f, {"residual_norm": rep.residual_norm,
                                   "numerical_rank": rep.numerical_rank,
                                   "truncated": rep.truncated,
                                   "singular_values": list(rep.singular_values)})
        return out
    for metric in metrics:
        nb, db = bounds.get(metric, default_bounds(len(variables)))
        try:
            f, rep = fit_fn(X, metric_values[metric], variables, nb, db, rank_tol)
            out[metric] = (f, {"residual_norm": rep.residual_norm,
                               "numerical_rank": rep.numerical_rank,
                               "truncated": rep.truncated,
                               "singular_values": list(rep.singular_values)})
        except (DegenerateFit, SvdFailure) as e:
            out[metric] = str(e)
    return out


def assemble_model_set(variables: Sequence[str], constants: Dict[str, float],
                       outcomes: Dict[str, object]) -> F.MetricModelSet:
    """Collects per-metric outcomes into a MetricModelSet in metric-name order;
    a total wipeout raises AllMetricsFailed (pipeline.hpp:178-183)."""
    out = F.MetricModelSet(list(variables), {}, {}, dict(constants), {})
    for metric in sorted(outcomes):
        o = outcomes[metric]
        if isinstance(o, str):
            out.failures[metric] = o
        else:
            out.models[metric], out.reports[metric] = o
    if not out.models:
        raise AllMetricsFailed("no metric could be fitted:" +
                               "".join(f" [{k}: {v}]" for k, v in sorted(out.failures.items())))
    return out


def fit_all_metrics(X, metric_values: Dict[str, np.ndarray], variables: Sequence[str],
                    bounds: Dict[str, Tuple[List[int], List[int]]],
                    constants: Dict[str, float], rank_tol: float = K_DEFAULT_RANK_TOL,
                    device: int = 0) -> F.MetricModelSet:
    """pipe::fit_all_metrics (pipeline.hpp:145-184): one fit per metric
    column; numerical failures are recorded per metric, a total wipeout
    raises AllMetricsFailed."""
    order = check_metric_inputs(X, metric_values, variables, bounds, constants)
    return assemble_model_set(variables, constants,
                              fit_metrics(X, metric_values, variables, bounds, order, rank_tol, device))
