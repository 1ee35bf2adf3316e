"""ORACLE O3 — TEST INFRASTRUCTURE ONLY.

numpy/LAPACK restatement of the reference's least-squares rational fit,
``poly::fit_rational`` (polyfit.hpp:337-427), with every helper it uses:

* build_sample_matrix            polyfit.hpp:139-154
* equilibrate_columns            polyfit.hpp:219-229
* svd (JacobiSVD ThinU|FullV)    polyfit.hpp:162-169 — here LAPACK gesdd/gesvd
* numerical_rank                 polyfit.hpp:171-177
* make_ratfunc_from_coeffs       polyfit.hpp:185-213
* positive_den_minimizer         polyfit.hpp:242-311 (log-barrier Newton, KKT)
* the positivity safeguard       polyfit.hpp:369-414
* fit_polynomial                 polyfit.hpp:432-465

Eigen's JacobiSVD and LAPACK differ bitwise, so parity with the reference and
with the GPU fit is pinned by the reference's own properties and tolerances
(tests/test_oracle_fit.py), not bit patterns.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from paper_1906_00142_b200 import formats as F

K_DEFAULT_RANK_TOL = 1e-10
K_DEN_PINCH_TRIGGER = 1e-4
K_REWEIGHT_ROUNDS = 3


class DegenerateFit(RuntimeError):
    pass


class SvdFailure(RuntimeError):
    pass


def eval_monomials(basis: Sequence[Tuple[int, ...]], X: np.ndarray) -> np.ndarray:
    """eval_monomial for every point and basis element (m x len(basis)):
    per variable p = x*x*...*x from 1.0, m *= p in variable order."""
    m = X.shape[0]
    out = np.empty((m, len(basis)))
    for j, mono in enumerate(basis):
        acc = np.ones(m)
        for i, e in enumerate(mono):
            p = np.ones(m)
            for _ in range(e):
                p = p * X[:, i]
            acc = acc * p
        out[:, j] = acc
    return out


def build_sample_matrix(X, y, num_bounds, den_bounds):
    nb = F.monomial_basis(num_bounds)
    db = F.monomial_basis(den_bounds)
    A = np.empty((len(y), len(nb) + len(db)))
    A[:, : len(nb)] = eval_monomials(nb, X)
    A[:, len(nb):] = -np.asarray(y)[:, None] * eval_monomials(db, X)
    return A, nb, db


def equilibrate_columns(A: np.ndarray):
    A = A.copy()
    scale = np.ones(A.shape[1])
    for j in range(A.shape[1]):
        n = np.linalg.norm(A[:, j])
        if n > 0.0:
            scale[j] = 1.0 / n
            A[:, j] *= scale[j]
    return A, scale


@dataclass
class SvdResult:
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray  # full n x n


def svd(A: np.ndarray) -> SvdResult:
    if not np.all(np.isfinite(A)):
        raise SvdFailure("svd: matrix has non-finite entries")
    m, n = A.shape
    try:
        # thin U; V must be full n x n (only m < n needs full_matrices)
        U, s, Vh = np.linalg.svd(A, full_matrices=m < n)
    except np.linalg.LinAlgError:
        raise SvdFailure("svd: decomposition did not converge") from None
    k = len(s)
    return SvdResult(U[:, :k], s, Vh.T)


def numerical_rank(sigma: np.ndarray, rank_tol: float) -> int:
    if len(sigma) == 0 or sigma[0] <= 0.0:
        return 0
    return int(np.sum(sigma >= rank_tol * sigma[0]))


def make_ratfunc_from_coeffs(variables, num_basis, den_basis, c: np.ndarray) -> F.RationalFunction:
    nn, nd = len(num_basis), len(den_basis)
    norm = np.linalg.norm(c)
    if norm == 0.0:
        raise DegenerateFit("all-zero coefficient vector")
    c = c / norm
    first = -1
    for j in range(nd):
        if abs(c[nn + j]) > 1e-10:
            first = j
            break
    if first < 0:
        raise DegenerateFit("recovered denominator is identically zero")
    if c[nn + first] < 0.0:
        c = -c
    return F.RationalFunction(F.Polynomial(list(variables), list(num_basis), list(c[:nn])),
                              F.Polynomial(list(variables), list(den_basis), list(c[nn:])))


def positive_den_minimizer(A_eq, col_scale, den_values, num_size, start_raw):
    """polyfit.hpp:242-311."""
    m, n = A_eq.shape
    nd = den_values.shape[1]
    Q = np.zeros((m, n))
    Q[:, num_size: num_size + nd] = den_values * col_scale[num_size: num_size + nd]
    g = Q.sum(axis=0)
    c = start_raw / col_scale
    q = Q @ c
    if not (q.min() > 0.0):
        return None
    s = m / g.dot(c)
    if not (s > 0.0) or not math.isfinite(s):
        return None
    c = c * s
    q = q * s
    H0 = A_eq.T @ A_eq
    mu = max(float(np.sum((A_eq @ c) ** 2)), 1e-30) / m

    def phi(v, qv):
        return float(np.sum((A_eq @ v) ** 2)) - mu * float(np.sum(np.log(qv)))

    K = np.zeros((n + 1, n + 1))
    rhs = np.zeros(n + 1)
    for _outer in range(16):
        for _inner in range(40):
            qinv = 1.0 / q
            # Q is zero outside the denominator block: same algebra, den block only
            Qd = Q[:, num_size: num_size + nd]
            qt = np.zeros(n)
            qt[num_size: num_size + nd] = Qd.T @ qinv
            grad = 2.0 * (H0 @ c) - mu * qt
            H = 2.0 * H0
            H[num_size: num_size + nd, num_size: num_size + nd] += mu * (Qd.T * (qinv ** 2)) @ Qd
            K[:] = 0.0
            K[:n, :n] = H
            K[:n, n] = g
            K[n, :n] = g
            rhs[:n] = -grad
            rhs[n] = 0.0
            try:
                sol = np.linalg.solve(K, rhs)
            except np.linalg.LinAlgError:
                return None
            if not np.all(np.isfinite(sol)):
                return None
            dc = sol[:n]
            decrement = -grad.dot(dc)
            phi0 = phi(c, q)
            if not (decrement > 1e-14 * (1.0 + abs(phi0))):
                break
            stepped = False
            alpha = 1.0
            while alpha > 1e-18:
                cn = c + alpha * dc
                qn = Q @ cn
                if qn.min() > 0.0 and phi(cn, qn) <= phi0 - 1e-4 * alpha * decrement:
                    c, q = cn, qn
                    stepped = True
                    break
                alpha *= 0.5
            if not stepped:
                break
        mu *= 0.1
    raw = c * col_scale
    if not np.all(np.isfinite(raw)):
        return None
    return raw


@dataclass
class FitReport:
    residual_norm: float = 0.0
    numerical_rank: int = 0
    singular_values: List[float] = field(default_factory=list)
    truncated: bool = False
    safeguard: bool = False


def fit_rational(X, y, variables, num_bounds, den_bounds, rank_tol=K_DEFAULT_RANK_TOL,
                 trace=None):
    """polyfit.hpp:337-427.  ``trace`` (dict, optional): the safeguard's
    stages as rpg_fit_rational_traced reports them ("stages": unconstrained
    vector, first minimizer result, accepted reweighted rounds — raw
    coordinates; "round_qmin"; "stop")."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if len(y) == 0:
        raise ValueError("fit_rational: no samples")
    A_raw, nb, db = build_sample_matrix(X, y, num_bounds, den_bounds)
    nn, nd = len(nb), len(db)
    m = len(y)
    A, col_scale = equilibrate_columns(A_raw)
    dec = svd(A)
    cols = A.shape[1]
    c = dec.V[:, cols - 1] * col_scale
    if trace is not None:
        trace.update(stages=[c.copy()], round_qmin=[], stop="no_safeguard")
    den_values = eval_monomials(db, X)
    q = den_values @ c[nn:]
    sign_mixed = q.min() < 0.0 and q.max() > 0.0
    mean_mag = float(np.mean(np.abs(q)))
    pinched = mean_mag > 0.0 and float(np.min(np.abs(q))) < K_DEN_PINCH_TRIGGER * mean_mag
    safeguard = bool(sign_mixed or pinched)
    if safeguard:
        V = eval_monomials(nb, X)
        vd = svd(V)
        vrank = numerical_rank(vd.sigma, rank_tol)
        uty = vd.U.T @ y
        start = np.zeros(cols)
        for i in range(vrank):
            start[:nn] += vd.V[:, i] * (uty[i] / vd.sigma[i])
        start[nn] = 1.0
        refined = positive_den_minimizer(A, col_scale, den_values, nn, start)
        if trace is not None:
            trace["stop"] = "rounds" if refined is not None else "first_empty"
            if refined is not None:
                trace["stages"].append(refined.copy())
        rnd = 0
        while refined is not None and rnd < K_REWEIGHT_ROUNDS:
            qprev = den_values @ refined[nn:]
            if trace is not None:
                trace["round_qmin"].append(float(qprev.min()))
            if not (qprev.min() > 0.0):
                if trace is not None:
                    trace["stop"] = "qmin"
                break
            Aw = A_raw / (np.maximum(1.0, np.abs(y)) * qprev)[:, None]
            Aw, scale_w = equilibrate_columns(Aw)
            nxt = positive_den_minimizer(Aw, scale_w, den_values, nn, refined)
            if nxt is None:
                if trace is not None:
                    trace["stop"] = "empty"
                break
            refined = nxt
            if trace is not None:
                trace["stages"].append(refined.copy())
            rnd += 1
        if refined is not None:
            c = refined
    f = make_ratfunc_from_coeffs(variables, nb, db, c)
    rep = FitReport()
    rep.singular_values = list(dec.sigma)
    rep.numerical_rank = numerical_rank(dec.sigma, rank_tol)
    rep.truncated = rep.numerical_rank < cols - 1
    rep.residual_norm = float(dec.sigma[cols - 1]) if len(dec.sigma) >= cols else 0.0
    rep.safeguard = safeguard
    return f, rep


def fit_polynomial(X, y, variables, bounds, rank_tol=K_DEFAULT_RANK_TOL):
    """polyfit.hpp:432-465."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    basis = F.monomial_basis(bounds)
    A = eval_monomials(basis, X)
    dec = svd(A)
    rank = numerical_rank(dec.sigma, rank_tol)
    uty = dec.U.T @ np.asarray(y, dtype=np.float64)
    x = np.zeros(A.shape[1])
    for i in range(rank):
        x += dec.V[:, i] * (uty[i] / dec.sigma[i])
    rep = FitReport(singular_values=list(dec.sigma), numerical_rank=rank,
                    truncated=rank < A.shape[1],
                    residual_norm=float(np.linalg.norm(A @ x - y)))
    return F.Polynomial(list(variables), basis, list(x)), rep


def eval_ratfunc(f: F.RationalFunction, X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[None, :]
    p = eval_monomials(f.num.basis, X) @ np.asarray(f.num.coeffs)
    q = eval_monomials(f.den.basis, X) @ np.asarray(f.den.coeffs)
    return p / q
