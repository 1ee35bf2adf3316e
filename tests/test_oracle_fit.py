"""Pins O3 (numpy restatement of poly::fit_rational) to the reference's fit
tests (test_polyfit.cpp, acceptance.cpp criteria 3-4, test_pipeline.cpp) —
properties and tolerances, since Eigen JacobiSVD and LAPACK differ bitwise."""
import numpy as np
import pytest

from oracle import o3_fit as O3
from paper_1906_00142_b200 import formats as F


def g(x):
    return (x * x + 1.0) / (x + 2.0)


def univariate(count, lo, hi, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(lo, hi, count)
    y = g(x)
    if noise > 0:
        y = y * (1.0 + rng.uniform(-noise, noise, count))
    return x[:, None], y


def test_basis_and_svd_contract():
    # test_polyfit.cpp:108-140
    d = O3.svd(np.eye(3))
    assert np.allclose(d.sigma, 1.0)
    A = np.zeros((2, 2)); A[0, 0] = 3.0
    d = O3.svd(A)
    assert d.sigma[0] == pytest.approx(3.0) and abs(d.sigma[1]) < 1e-14
    rng = np.random.default_rng(7)
    A = rng.uniform(-1, 1, (20, 8))
    d = O3.svd(A)
    R = d.U @ np.diag(d.sigma) @ d.V[:, : len(d.sigma)].T
    assert np.linalg.norm(R - A) <= 1e-10 * d.sigma[0]
    assert np.all(np.diff(d.sigma) <= 0) and np.all(d.sigma >= 0)
    with pytest.raises(O3.SvdFailure):
        O3.svd(np.array([[np.nan]]))


def test_recovers_exact_generator():
    # test_polyfit.cpp:142-157
    X, y = univariate(20, 0.0, 4.0, 11)
    f, rep = O3.fit_rational(X, y, ["x"], [2], [1])
    assert rep.residual_norm < 1e-10 and not rep.truncated
    xs = np.random.default_rng(12).uniform(0, 4, 100)
    assert np.max(np.abs(O3.eval_ratfunc(f, xs[:, None]) - g(xs)) / np.abs(g(xs))) < 1e-8


def test_constant_data():
    # test_polyfit.cpp:159-168
    X = np.arange(6, dtype=float)[:, None]
    f, rep = O3.fit_rational(X, np.full(6, 5.0), ["x"], [0], [0])
    assert O3.eval_ratfunc(f, [[3.3]])[0] == pytest.approx(5.0)
    assert rep.residual_norm < 1e-12


def test_relative_noise():
    # test_polyfit.cpp:170-182
    X, y = univariate(200, 0.0, 4.0, 21, 0.01)
    f, _ = O3.fit_rational(X, y, ["x"], [2], [1])
    xs = np.random.default_rng(22).uniform(0, 4, 100)
    assert np.max(np.abs(O3.eval_ratfunc(f, xs[:, None]) - g(xs)) / np.abs(g(xs))) < 0.05


def test_scale_invariance():
    # test_polyfit.cpp:184-196
    X, y = univariate(40, 0.5, 3.5, 31)
    f1, _ = O3.fit_rational(X, y, ["x"], [2], [1])
    f2, _ = O3.fit_rational(X, 17.5 * y, ["x"], [2], [1])
    a, b = O3.eval_ratfunc(f1, X), O3.eval_ratfunc(f2, X)
    assert np.all(np.abs(b - 17.5 * a) <= 1e-8 * np.abs(17.5 * a))


def test_minimizes_homogeneous_residual():
    # test_polyfit.cpp:198-214
    X, y = univariate(30, 0.0, 4.0, 41, 0.05)
    f, _ = O3.fit_rational(X, y, ["x"], [2], [1])
    A, _, _ = O3.build_sample_matrix(X, y, [2], [1])
    cfit = np.array(f.num.coeffs + f.den.coeffs)
    best = np.linalg.norm(A @ cfit)
    rng = np.random.default_rng(43)
    for _ in range(1000):
        c = rng.uniform(-1, 1, A.shape[1])
        c /= np.linalg.norm(c)
        assert best <= np.linalg.norm(A @ c) + 1e-12


def test_exact_interpolation():
    # test_polyfit.cpp:216-228
    x = 0.5 + np.arange(5.0)
    f, rep = O3.fit_rational(x[:, None], g(x), ["x"], [2], [1])
    assert rep.residual_norm < 1e-10 * np.sqrt(np.sum(g(x) ** 2))


def test_degenerate_denominators_rejected():
    # test_polyfit.cpp:230-250
    nb, db = F.monomial_basis([1]), F.monomial_basis([1])
    with pytest.raises(O3.DegenerateFit):
        O3.make_ratfunc_from_coeffs(["x"], nb, db, np.array([1.0, 0.5, 1e-14, -1e-15]))
    f = O3.make_ratfunc_from_coeffs(["x"], nb, db, np.array([1.0, 0.5, -0.25, 0.1]))
    assert f.den.coeffs[0] > 0
    assert sum(v * v for v in f.num.coeffs + f.den.coeffs) == pytest.approx(1.0)


def test_fit_polynomial_cases():
    # test_polyfit.cpp:252-299
    p, rep = O3.fit_polynomial(np.array([[0.0], [1.0], [2.0]]), np.array([1.0, 3.0, 5.0]), ["x"], [1])
    assert p.coeffs[0] == pytest.approx(1.0, abs=1e-12) and p.coeffs[1] == pytest.approx(2.0, abs=1e-12)
    assert not rep.truncated
    rng = np.random.default_rng(51)
    x = rng.uniform(0, 10, 40)
    y = 2 * x + 1 + rng.uniform(-0.1, 0.1, 40)
    p, rep = O3.fit_polynomial(x[:, None], y, ["x"], [1])
    A = np.stack([np.ones(40), x], 1)
    sol = np.linalg.solve(A.T @ A, A.T @ y)
    assert abs(p.coeffs[0] - sol[0]) < 1e-8 and abs(p.coeffs[1] - sol[1]) < 1e-8
    p, rep = O3.fit_polynomial(np.ones((4, 1)), np.full(4, 3.0), ["x"], [1])
    assert rep.truncated and rep.numerical_rank == 1


def three_var_target(x, y, z):
    return (x * x + 1) * (y * y + 1) * (z * z + 1) / ((x + 2) * (y + 2) * (z + 2))


def test_three_variable_recovery_and_noise():
    # acceptance.cpp:161-210 (criterion 3)
    rng = np.random.default_rng(5150)
    P = rng.uniform(1.0, 4.0, (200, 3))
    H = rng.uniform(1.0, 4.0, (50, 3))
    y = three_var_target(*P.T)
    f, _ = O3.fit_rational(P, y, ["x", "y", "z"], [2, 2, 2], [1, 1, 1])
    yh = three_var_target(*H.T)
    err = np.abs(O3.eval_ratfunc(f, H) - yh) / np.maximum(1.0, np.abs(yh))
    assert err.max() < 1e-8
    noisy = y * (1 + rng.uniform(-0.01, 0.01, len(y)))
    f, _ = O3.fit_rational(P, noisy, ["x", "y", "z"], [2, 2, 2], [1, 1, 1])
    err = np.abs(O3.eval_ratfunc(f, H) - yh) / np.maximum(1.0, np.abs(yh))
    assert err.max() < 0.05


def stencil_samples(sizes):
    spec = F.load_kernel_spec("data/stencil2d.kernel.json")
    cfg = F.enumerate_configs()
    pts = np.array([(d, bx, by) for d in sizes for (bx, by, _) in cfg], dtype=float)
    return spec, pts


def test_rank_deficient_fit_truncates():
    # acceptance.cpp:214-246 (criterion 4)
    spec, pts = stencil_samples([64, 128, 256, 512])
    truth = spec.ground_truth[F.METRIC_COMP]
    y = O3.eval_ratfunc(truth, pts)
    f, rep = O3.fit_rational(pts, y, spec.variables, [2, 2, 0], [1, 1, 0])
    assert rep.truncated and rep.numerical_rank > 0
    assert rep.residual_norm < 1e-6
    assert all(np.isfinite(f.num.coeffs)) and all(np.isfinite(f.den.coeffs))
    for p in ([64, 8, 4], [512, 128, 2]):
        v = O3.eval_ratfunc(f, [p])[0]
        t = O3.eval_ratfunc(truth, [p])[0]
        assert abs(v - t) / max(1.0, abs(t)) < 1e-6


def test_stencil_metrics_recovered_on_holdout():
    # test_pipeline.cpp:199-237
    spec, pts = stencil_samples([64, 128, 256, 512])
    _, hold = stencil_samples([48, 96, 1536])
    bounds = {F.METRIC_COMP: ([1, 1, 0], [0, 1, 0]), F.METRIC_UNCOAL: ([0, 1, 0], [0, 1, 0]),
              F.METRIC_COAL: ([0, 0, 0], [0, 0, 0]), F.METRIC_SYNCH: ([1, 0, 0], [0, 1, 0]),
              F.METRIC_TOTAL_BLOCKS: ([2, 0, 0], [0, 1, 1])}
    for name, (nb, db) in bounds.items():
        truth = spec.ground_truth[name]
        y = O3.eval_ratfunc(truth, pts)
        f, rep = O3.fit_rational(pts, y, spec.variables, nb, db)
        assert rep.residual_norm <= 1e-9 * max(1.0, rep.singular_values[0])
        assert not rep.truncated
        got = O3.eval_ratfunc(f, hold)
        want = O3.eval_ratfunc(truth, hold)
        assert np.all(np.abs(got - want) <= 1e-9 * np.abs(want)), name


def test_safeguard_path_runs_on_noisy_multivariate_data():
    """A noisy 3-variable sample whose unconstrained denominator changes sign
    exercises positive_den_minimizer (polyfit.hpp:369-414)."""
    rng = np.random.default_rng(7)
    P = rng.uniform(1.0, 4.0, (300, 3))
    y = three_var_target(*P.T) * (1 + rng.uniform(-0.05, 0.05, 300))
    f, rep = O3.fit_rational(P, y, ["x", "y", "z"], [2, 2, 2], [1, 1, 1])
    q = O3.eval_monomials(f.den.basis, P) @ np.array(f.den.coeffs)
    if rep.safeguard:
        assert q.min() > 0 or q.max() < 0
