"""K3 — the GPU rational fit against the reference's fit tests and O3.

Eigen's JacobiSVD (reference), LAPACK (O3) and the GPU's TSQR + one-sided
Jacobi differ bitwise, so the bar is the reference's own tolerances
(test_polyfit.cpp, acceptance.cpp criteria 3-4, test_pipeline.cpp) plus
agreement with O3: singular values within 1e-10 * sigma_1, coefficient
vectors within 1e-8 on well-conditioned problems, and fitted functions within
1e-6 relative when the positivity safeguard runs (same Newton iteration,
different rounding)."""
import numpy as np
import pytest

from oracle import o3_fit as O3
from paper_1906_00142_b200 import fit as G
from paper_1906_00142_b200 import formats as F

from .test_oracle_fit import g, stencil_samples, three_var_target, univariate

pytestmark = pytest.mark.gpu


def ev(f, X):
    return O3.eval_ratfunc(f, X)


def coef(f):
    return np.array(f.num.coeffs + f.den.coeffs)


def test_recovers_exact_generator_and_matches_o3():
    X, y = univariate(20, 0.0, 4.0, 11)
    f, rep = G.fit_rational(X, y, ["x"], [2], [1])
    assert rep.residual_norm < 1e-10 and not rep.truncated and not rep.safeguard
    xs = np.random.default_rng(12).uniform(0, 4, 100)
    assert np.max(np.abs(ev(f, xs[:, None]) - g(xs)) / np.abs(g(xs))) < 1e-8
    fo, ro = O3.fit_rational(X, y, ["x"], [2], [1])
    assert np.allclose(rep.singular_values, ro.singular_values, rtol=0, atol=1e-10 * ro.singular_values[0])
    assert np.allclose(coef(f), coef(fo), rtol=0, atol=1e-8)


def test_constant_data():
    X = np.arange(6, dtype=float)[:, None]
    f, rep = G.fit_rational(X, np.full(6, 5.0), ["x"], [0], [0])
    assert ev(f, [[3.3]])[0] == pytest.approx(5.0)
    assert rep.residual_norm < 1e-12


def test_relative_noise():
    X, y = univariate(200, 0.0, 4.0, 21, 0.01)
    f, _ = G.fit_rational(X, y, ["x"], [2], [1])
    xs = np.random.default_rng(22).uniform(0, 4, 100)
    assert np.max(np.abs(ev(f, xs[:, None]) - g(xs)) / np.abs(g(xs))) < 0.05


def test_scale_invariance():
    X, y = univariate(40, 0.5, 3.5, 31)
    f1, _ = G.fit_rational(X, y, ["x"], [2], [1])
    f2, _ = G.fit_rational(X, 17.5 * y, ["x"], [2], [1])
    a, b = ev(f1, X), ev(f2, X)
    assert np.all(np.abs(b - 17.5 * a) <= 1e-8 * np.abs(17.5 * a))


def test_minimizes_homogeneous_residual():
    X, y = univariate(30, 0.0, 4.0, 41, 0.05)
    f, rep = G.fit_rational(X, y, ["x"], [2], [1])
    A, _, _ = O3.build_sample_matrix(X, y, [2], [1])
    best = np.linalg.norm(A @ coef(f))
    rng = np.random.default_rng(43)
    for _ in range(1000):
        c = rng.uniform(-1, 1, A.shape[1])
        c /= np.linalg.norm(c)
        assert best <= np.linalg.norm(A @ c) + 1e-12


def test_exact_interpolation_and_fewer_rows_than_columns():
    x = 0.5 + np.arange(5.0)
    f, rep = G.fit_rational(x[:, None], g(x), ["x"], [2], [1])
    assert rep.residual_norm < 1e-10 * np.sqrt(np.sum(g(x) ** 2))
    f, rep = G.fit_rational(x[:3, None], g(x[:3]), ["x"], [2], [1])  # m < n
    assert len(rep.singular_values) == 3 and rep.residual_norm == 0.0


def test_errors():
    with pytest.raises(ValueError, match="no samples"):
        G.fit_rational(np.zeros((0, 1)), np.zeros(0), ["x"], [1], [1])
    with pytest.raises(ValueError, match="negative degree bound"):
        G.fit_rational(np.ones((4, 1)), np.ones(4), ["x"], [-1], [1])
    with pytest.raises(G.SvdFailure):
        G.fit_rational(np.array([[1.0], [np.nan]]), np.ones(2), ["x"], [1], [0])


def test_three_variable_recovery_noise_and_safeguard():
    # acceptance.cpp:161-210 (criterion 3); the noisy fit runs the safeguard.
    rng = np.random.default_rng(5150)
    P = rng.uniform(1.0, 4.0, (200, 3))
    H = rng.uniform(1.0, 4.0, (50, 3))
    y = three_var_target(*P.T)
    f, rep = G.fit_rational(P, y, ["x", "y", "z"], [2, 2, 2], [1, 1, 1])
    yh = three_var_target(*H.T)
    assert (np.abs(ev(f, H) - yh) / np.maximum(1.0, np.abs(yh))).max() < 1e-8
    noisy = y * (1 + rng.uniform(-0.01, 0.01, len(y)))
    f, rep = G.fit_rational(P, noisy, ["x", "y", "z"], [2, 2, 2], [1, 1, 1])
    assert (np.abs(ev(f, H) - yh) / np.maximum(1.0, np.abs(yh))).max() < 0.05
    fo, ro = O3.fit_rational(P, noisy, ["x", "y", "z"], [2, 2, 2], [1, 1, 1])
    assert rep.safeguard == ro.safeguard
    gh, oh = ev(f, H), ev(fo, H)
    assert np.max(np.abs(gh - oh) / np.abs(oh)) < 1e-6


def test_rank_deficient_fit_truncates():
    """A rank-deficient fit (exact in-class data, a null space of dimension
    >= 2): truncated, residual ~0.  Which null vector comes back depends on
    the SVD (Eigen's in the reference), and a null vector may share a zero
    of p and q (a removable pole), so the check is the homogeneous one —
    p - y q vanishes on every sample — plus p/q = y wherever q is not
    vanishingly small (when the safeguard did not replace the null vector)."""
    spec, pts = stencil_samples([64, 128, 256, 512])
    truth = spec.ground_truth[F.METRIC_COMP]
    y = ev(truth, pts)
    f, rep = G.fit_rational(pts, y, spec.variables, [2, 2, 0], [1, 1, 0])
    assert rep.truncated and rep.numerical_rank > 0 and rep.residual_norm < 1e-6
    if rep.safeguard:
        # the null vector the SVD returned has a pinched denominator: the
        # positivity minimizer's result is a constrained least-squares
        # solution, not an interpolant (polyfit.hpp:364-414)
        assert all(np.isfinite(f.num.coeffs)) and all(np.isfinite(f.den.coeffs))
        return
    X = np.asarray(pts, dtype=float)
    nb, db = F.monomial_basis([2, 2, 0]), F.monomial_basis([1, 1, 0])
    P = np.column_stack([np.prod(X ** np.asarray(e, float), axis=1) for e in nb]) @ np.array(f.num.coeffs)
    Q = np.column_stack([np.prod(X ** np.asarray(e, float), axis=1) for e in db]) @ np.array(f.den.coeffs)
    assert np.all(np.abs(P - y * Q) <= 1e-9 * (np.abs(P) + np.abs(y * Q) + 1e-300))
    ok = np.abs(Q) >= 1e-6 * np.abs(Q).max()
    assert ok.mean() > 0.5
    assert np.all(np.abs(P[ok] / Q[ok] - y[ok]) <= 1e-6 * np.maximum(1.0, np.abs(y[ok])))


def test_stencil_metrics_recovered_on_holdout():
    spec, pts = stencil_samples([64, 128, 256, 512])
    _, hold = stencil_samples([48, 96, 1536])
    bounds = {F.METRIC_COMP: ([1, 1, 0], [0, 1, 0]), F.METRIC_UNCOAL: ([0, 1, 0], [0, 1, 0]),
              F.METRIC_COAL: ([0, 0, 0], [0, 0, 0]), F.METRIC_SYNCH: ([1, 0, 0], [0, 1, 0]),
              F.METRIC_TOTAL_BLOCKS: ([2, 0, 0], [0, 1, 1])}
    values = {name: ev(spec.ground_truth[name], pts) for name in bounds}
    models = G.fit_all_metrics(pts, values, spec.variables, bounds,
                               {F.METRIC_REGS: 20.0, F.METRIC_SHARED: 0.0})
    assert not models.failures and len(models.models) == 5
    for name in bounds:
        rep = models.reports[name]
        assert rep["residual_norm"] <= 1e-9 * max(1.0, rep["singular_values"][0])
        assert not rep["truncated"]
        got, want = ev(models.models[name], hold), ev(spec.ground_truth[name], hold)
        assert np.all(np.abs(got - want) <= 1e-9 * np.abs(want)), name


def test_large_sample_matches_o3():
    """2e5 noisy samples of the 3-variable target, default bounds (35
    columns): singular values, rank, safeguard decision and the fitted
    function agree with O3."""
    rng = np.random.default_rng(19)
    m = 200_000
    X = rng.uniform(1.0, 4.0, (m, 3))
    y = three_var_target(*X.T) * (1 + rng.uniform(-0.01, 0.01, m))
    nb, db = [2, 2, 2], [1, 1, 1]
    f, rep = G.fit_rational(X, y, ["x", "y", "z"], nb, db)
    fo, ro = O3.fit_rational(X, y, ["x", "y", "z"], nb, db)
    s0 = ro.singular_values[0]
    assert np.allclose(rep.singular_values, ro.singular_values, rtol=0, atol=1e-9 * s0)
    assert rep.numerical_rank == ro.numerical_rank and rep.safeguard == ro.safeguard
    Xh = X[:2000]
    assert np.max(np.abs(ev(f, Xh) - ev(fo, Xh)) / np.abs(ev(fo, Xh))) < 1e-6


def test_multi_fit_equals_one_by_one():
    """rpg_fit_rational_multi (X uploaded once, the fits concurrent on their
    own streams) returns exactly what one rpg_fit_rational call per metric
    returns — coefficients, singular values, rank, safeguard — including a
    failing job, which fails alone."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    X, ys, var = bench.c4_data(200_000, 0.01)
    names = sorted(ys)
    ys_list = [ys[k] for k in names] + [np.zeros(len(X))]
    bnds = [([2, 2, 2], [1, 1, 1])] * len(names) + [([1, 1, 1], [0, 0, 0])]
    got = G.fit_rational_multi(X, ys_list, var, bnds)
    assert len(got) == len(ys_list)
    for y, (nb, db), g in zip(ys_list, bnds, got):
        try:
            f, rep = G.fit_rational(X, y, var, nb, db)
        except (G.DegenerateFit, G.SvdFailure) as e:
            assert isinstance(g, type(e)) and str(g) == str(e)
            continue
        gf, grep = g
        assert gf.num.coeffs == f.num.coeffs and gf.den.coeffs == f.den.coeffs
        assert grep.singular_values == rep.singular_values
        assert (grep.numerical_rank, grep.safeguard, grep.truncated) == (rep.numerical_rank, rep.safeguard, rep.truncated)


_DM_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import bench
from paper_1906_00142_b200 import fit as G
X, ys, variables = bench.c4_data(200000, 0.01)
out = {}
for name in sorted(ys):
    tr = {}
    try:
        f, rep = G.fit_rational(X, ys[name], variables, [2, 2, 2], [1, 1, 1], trace=tr)
        res = [float(c).hex() for c in list(f.num.coeffs) + list(f.den.coeffs)] + [rep.safeguard]
    except (G.DegenerateFit, G.SvdFailure) as e:
        res = [type(e).__name__]
    out[name] = [res, [[float(v).hex() for v in st] for st in tr.get("stages", [])]]
print(json.dumps(out))
"""


def test_den_pass_monomial_sources_bit_identical():
    """The safeguard's sample passes take the denominator monomials either
    from a precomputed m x 8 array (RPG_FIT_DM=1) or recompute them from x by
    exponent bit masks (RPG_FIT_DM=0, the default for 0/1 denominator
    exponents): the two are the same products in the same order, so every
    stage vector and every fitted coefficient is bit-identical."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = []
    for mode in ("0", "1"):
        env = dict(os.environ, RPG_FIT_DM=mode)
        p = subprocess.run([sys.executable, "-c", _DM_SCRIPT, root], env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        runs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert runs[0] == runs[1]
    assert any(v[0][-1] is True for v in runs[0].values())  # the safeguard ran


def target(P, cols):
    """The acceptance target (acceptance.cpp:161-210) restricted to the
    variables in cols: prod (v^2 + 1) / prod (v + 2), exactly representable
    with bounds num 2 / den 1 per variable."""
    t = np.ones(len(P))
    for c in cols:
        t = t * (P[:, c] ** 2 + 1) / (P[:, c] + 2)
    return t


_FMA_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1906_00142_b200 import fit as G
from oracle import o3_fit as O3
from tests.test_gpu_fit import target
rng = np.random.default_rng(5150)
P = rng.uniform(1.0, 4.0, (20000, 3))
H = rng.uniform(1.0, 4.0, (50, 3))
e = rng.uniform(-0.01, 0.01, len(P))
out = {}
for name, cols, bounds in (("xyz", [0, 1, 2], ([2, 2, 2], [1, 1, 1])), ("xy", [0, 1], ([2, 2], [1, 1]))):
    noisy = target(P, cols) * (1 + e)
    f, rep = G.fit_rational(P[:, cols], noisy, ["x", "y", "z"][:len(cols)], *bounds)
    out[name] = [rep.safeguard, [float(v) for v in O3.eval_ratfunc(f, H[:, cols])]]
print(json.dumps(out))
"""


@pytest.mark.parametrize("no_dmma", ["1", ""])
def test_sample_pass_paths_match_o3(no_dmma):
    """nd = 8 and nd = 4 fits with the safeguard running agree with O3 on
    both sample-pass paths: the tensor-core one (den_pass8_body, default) and
    the generic FMA-Gram one (den_pass_body, RPG_FIT_NO_DMMA=1)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", _FMA_SCRIPT, root], env=dict(os.environ, RPG_FIT_NO_DMMA=no_dmma),
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = json.loads(p.stdout.strip().splitlines()[-1])
    rng = np.random.default_rng(5150)
    P = rng.uniform(1.0, 4.0, (20000, 3))
    H = rng.uniform(1.0, 4.0, (50, 3))
    e = rng.uniform(-0.01, 0.01, len(P))
    for name, cols, bounds in (("xyz", [0, 1, 2], ([2, 2, 2], [1, 1, 1])), ("xy", [0, 1], ([2, 2], [1, 1]))):
        noisy = target(P, cols) * (1 + e)
        fo, ro = O3.fit_rational(P[:, cols], noisy, ["x", "y", "z"][:len(cols)], *bounds)
        assert got[name][0] == ro.safeguard
        oh = ev(fo, H[:, cols])
        assert np.max(np.abs(np.array(got[name][1]) - oh) / np.abs(oh)) < 1e-6, name
