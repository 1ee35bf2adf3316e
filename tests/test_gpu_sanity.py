"""GPU parity of the hot path's callers: batched
eval_ratfunc, synthesize, the direct model over collected metrics, per-tuple
subset search and sanity_report — against oracles O1/O5 and the reference's
own known answers (test_datakit.cpp:139-237, test_pipeline.cpp:581-625)."""
import math
import os

import numpy as np
import pytest

from oracle import o1
from oracle import o5_data as O5
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import fit as G
from paper_1906_00142_b200 import formats as F
from paper_1906_00142_b200 import samples as SM
from paper_1906_00142_b200 import sanity as SN
from paper_1906_00142_b200 import search as S

from . import zoo

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stencil_kernel(noise_rel=0.0):
    k = F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json"))
    k.noise_rel = noise_rel
    return k


STENCIL_BOUNDS = {  # test_pipeline.cpp:82-90
    F.METRIC_COMP: ([1, 1, 0], [0, 1, 0]), F.METRIC_UNCOAL: ([0, 1, 0], [0, 1, 0]),
    F.METRIC_COAL: ([0, 0, 0], [0, 0, 0]), F.METRIC_SYNCH: ([1, 0, 0], [0, 1, 0]),
    F.METRIC_TOTAL_BLOCKS: ([2, 0, 0], [0, 1, 1])}
STENCIL_CONSTANTS = {F.METRIC_REGS: 20.0, F.METRIC_SHARED: 0.0}


def test_eval_ratfunc_batch_bit_exact():
    rng = np.random.default_rng(5)
    for _ in range(6):
        f = zoo.random_ratfunc(rng, ["D1", "bx", "by"], [2, 2, 2], [1, 1, 1], positive=False)
        X = np.column_stack([rng.integers(1, 70000, 3000), rng.integers(1, 1025, 3000),
                             rng.integers(1, 1025, 3000)]).astype(float)
        X[:5, 1] = 0.0
        v, nz = SM.eval_ratfunc_batch(f, X)
        for i in range(len(X)):
            want = O5.eval_ratfunc(f, X[i].tolist())
            assert nz[i] == (want is None)
            if want is not None:
                assert v[i] == want
    # a denominator that vanishes at bx = 32 (test_datakit.cpp:209-210)
    f = F.make_ratfunc(["D1", "bx", "by"], [0, 0, 0], [9], [0, 1, 0], [-32, 1])
    v, nz = SM.eval_ratfunc_batch(f, np.array([[64, 32, 1], [64, 16, 2], [64, 64, 1]], float))
    assert nz.tolist() == [True, False, False] and v[1:].tolist() == [9 / -16, 9 / 32]


def test_synthesize_known_answers():
    data, cfg = SM.design_points([256], [(32, 8, 1), (64, 4, 1)])
    s = SM.synthesize(stencil_kernel(), data, cfg, 7)
    assert len(s) == 2
    assert s.metric_names == [F.METRIC_COAL, F.METRIC_COMP, F.METRIC_SYNCH,
                              F.METRIC_TOTAL_BLOCKS, F.METRIC_UNCOAL]
    assert s.provenance == SM.Provenance("synthetic", 7, 0.0)
    v = dict(zip(s.metric_names, s.values[0]))
    assert v[F.METRIC_COMP] == 84.0 and v[F.METRIC_UNCOAL] == 5.375 and v[F.METRIC_COAL] == 9.0
    assert v[F.METRIC_SYNCH] == 16.0 and v[F.METRIC_TOTAL_BLOCKS] == 256.0
    w = dict(zip(s.metric_names, s.values[1]))
    assert w[F.METRIC_COMP] == (20.0 * 64 + 8 * 256) / 64 and w[F.METRIC_TOTAL_BLOCKS] == 256.0

    spec = stencil_kernel()
    spec.ground_truth[F.METRIC_COAL] = F.make_ratfunc(spec.variables, [0, 0, 0], [9], [0, 1, 0], [-32, 1])
    data, cfg = SM.design_points([64], [(16, 2, 1), (32, 1, 1), (64, 1, 1)])
    skipped = []
    s = SM.synthesize(spec, data, cfg, 0, skipped)
    assert len(s) == 1 and tuple(s.configs[0]) == (64, 1, 1)
    assert len(skipped) == 2
    assert "negative" in skipped[0] and "16x2x1" in skipped[0]
    assert "singular" in skipped[1] and "32x1x1" in skipped[1]
    neg = stencil_kernel()
    neg.ground_truth[F.METRIC_SYNCH] = F.make_ratfunc(neg.variables, [0, 0, 0], [-3], [0, 0, 0], [1])
    skipped = []
    assert len(SM.synthesize(neg, data, cfg, 0, skipped)) == 0 and len(skipped) == 3
    with pytest.raises(ValueError):
        SM.synthesize(spec, *SM.design_points([64, 64], [(32, 1, 1)]), 0)


def test_synthesize_noise_stream_bit_exact_vs_oracle():
    sizes = [1 << k for k in range(3, 23)]
    data, cfg = SM.design_points(sizes, F.enumerate_configs())
    spec = stencil_kernel(0.01)
    spec.ground_truth[F.METRIC_COAL] = F.make_ratfunc(spec.variables, [0, 0, 0], [9], [0, 1, 0], [-32, 1])
    skipped = []
    a = SM.synthesize(spec, data, cfg, 42, skipped)
    names, rows, oskipped = O5.synthesize(spec, data, cfg, 42)
    assert a.metric_names == names and skipped == oskipped
    assert len(a) == len(rows)
    assert np.array_equal(a.values, np.array([r[2] for r in rows]))
    assert [tuple(c) for c in a.configs] == [r[1] for r in rows]
    b = SM.synthesize(spec, data, cfg, 42)
    c = SM.synthesize(spec, data, cfg, 43)
    assert np.array_equal(a.values, b.values) and not np.array_equal(a.values, c.values)
    spec.noise_rel = 0.0
    clean = SM.synthesize(spec, a.data, a.configs, 0)
    dev = np.abs(a.values / clean.values - 1.0)
    assert dev.max() <= 0.01 + 1e-12 and 0.004 < dev.mean() < 0.006


def test_mwpcwp_cycles_batch_matches_direct_model():
    rng = np.random.default_rng(8)
    for hw in (zoo.sample_hw(), zoo.random_hw(rng), zoo.b200_hw()):
        hws = A.profile_struct(hw)
        n = 4000
        M = np.column_stack([rng.choice([0.0, 16.0, 40.0, 255.0], n), rng.choice([0.0, 100.0, 9000.0], n),
                             rng.uniform(0, 500, n), rng.choice([0.0, 1.0, 7.5], n),
                             rng.choice([0.0, 3.0, 9.0], n), rng.uniform(0, 4, n),
                             rng.uniform(1, 1e6, n)])
        M[:20, 2] = -1.0  # ModelError rows
        cfg = np.array(F.integer_configs(dims=3))[rng.integers(0, 30343, n)]
        cfg[:30] = [1500, 1, 1]  # T > T_max: ZeroOccupancy
        for rep in ("real", "ceil"):
            total, b, w, tag, st = SN.mwpcwp_cycles_batch(hw, M, cfg, rep)
            rm = A.RPG_REP_CEIL if rep == "ceil" else A.RPG_REP_REAL
            for i in range(n):
                m = o1.metrics(M[i, 2], M[i, 3], M[i, 4], M[i, 5], M[i, 6], R=M[i, 0], Z=M[i, 1])
                rc, bd = o1.mwpcwp_cycles(hws, m, tuple(int(v) for v in cfg[i]), rm)
                assert st[i] == rc, i
                if rc == 0:
                    assert total[i] == bd.total_cycles and b[i] == bd.b_active
                    assert w[i] == bd.n_active_warps and tag[i] == bd.case_tag


def test_mwpcwp_breakdown_matches_direct_model():
    """Every MwpCwpBreakdown field (perfmodel.hpp:284-296) bit-exact vs O1's
    restatement, all three cases, compute-only rows, ceil/real, rejections."""
    rng = np.random.default_rng(21)
    fields = ("b_active", "n_active_warps", "mem_cycles", "comp_cycles", "mwp", "cwp", "rep",
              "case_tag", "cycles_pre_synch", "synch_cost", "total_cycles")
    for hw in (zoo.sample_hw(), zoo.random_hw(rng), zoo.b200_hw(), zoo.random_hw(rng)):
        hws = A.profile_struct(hw)
        n = 3000
        unc = rng.choice([0.0, 0.0, 1.0, 7.5, 40.0], n)
        coal = rng.choice([0.0, 3.0, 9.0, 0.25], n)
        KM = np.column_stack([rng.choice([0.0, 16.0, 40.0, 255.0], n),
                              rng.choice([0.0, 100.0, 9000.0], n),
                              rng.choice([0.0, 1.0, 30.0, 500.0], n) * rng.uniform(0, 1, n),
                              unc + coal, unc, coal, rng.uniform(0, 4, n), rng.uniform(1, 1e6, n)])
        KM[:20, 2] = -1.0          # ModelError: negative
        KM[20:40, 3] += 1.0        # ModelError: inconsistent mem
        cfg = np.array(F.integer_configs(dims=3))[rng.integers(0, 30343, n)]
        cfg[40:70] = [1500, 1, 1]  # ZeroOccupancy
        for rep in ("real", "ceil"):
            got = SN.mwpcwp_breakdown_batch(hw, KM, cfg, rep)
            rm = A.RPG_REP_CEIL if rep == "ceil" else A.RPG_REP_REAL
            seen = set()
            for i in range(n):
                m = o1.metrics(KM[i, 2], KM[i, 4], KM[i, 5], KM[i, 6], KM[i, 7], R=KM[i, 0], Z=KM[i, 1])
                m.mem_insts_per_thread = KM[i, 3]
                rc, bd = o1.mwpcwp_cycles(hws, m, tuple(int(v) for v in cfg[i]), rm)
                st = int(got[i]["status"])
                assert {0: 0, 1: 1, 4: 1, 2: 2, 3: 2}[st] == rc, i
                if i < 20:
                    assert st == 2
                elif i < 40:
                    assert st == 3
                if rc == 0:
                    for f in fields:
                        g, w = got[i][f], getattr(bd, f)
                        assert g == w or (np.isnan(g) and np.isnan(w)), (i, f, g, w)
                    seen.add(int(bd.case_tag))
            assert len(seen) >= 2, seen


@pytest.mark.parametrize("kernel", ["specialized", "generic"])
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_subset_search_matches_search_over_the_subset(kernel, arith):
    rng = np.random.default_rng(13)
    for case in zoo.cases()[::3]:
        opts = S.SearchOptions(regs_per_thread=case.regs_fallback,
                               shared_words_per_block=case.shared_fallback,
                               rep_mode=case.rep_mode, arith=arith, kernel=kernel)
        n = len(case.data)
        subsets = [np.sort(rng.choice(len(case.space), size=int(rng.integers(0, len(case.space) + 1)),
                                      replace=False)) for _ in range(n)]
        subsets[0] = np.arange(len(case.space))  # the full space as a subset
        offsets = np.concatenate([[0], np.cumsum([len(s) for s in subsets])])
        # any order within a subset (the lex tie-break uses the global rank)
        flat = np.concatenate([rng.permutation(x) for x in subsets]) if offsets[-1] else \
            np.zeros(0, np.int32)
        with S.Plan(case.spec, case.hw, case.space, opts) as plan:
            got = plan.search_batch_subsets(case.data, offsets, flat)
            full = plan.search_batch(case.data[:1])
        pk = A.PackedModel(case.spec, drop_zero_terms=False)
        for t in range(n):
            sub = [case.space[i] for i in subsets[t]]
            if not sub:
                assert got[t]["cfg_idx"] == -1 and got[t]["n_feasible"] == 0
                continue
            w, _ = o1.search_one(pk, A.profile_struct(case.hw), opts.struct(),
                                 A.config_array(sub), case.data[t])
            if arith == "fast":  # O1's FAST twin is exercised by the batch path
                continue
            want_idx = -1 if w.cfg_idx < 0 else int(subsets[t][w.cfg_idx])
            assert got[t]["cfg_idx"] == want_idx, (case.name, t)
            for f in ("ties", "n_feasible", "w_occ", "case_tag"):
                assert got[t][f] == getattr(w, f), (case.name, t, f)
            assert got[t]["ec"] == w.ec
        for f in ("cfg_idx", "ties", "n_feasible", "ec", "best_ec"):
            assert got[0][f] == full[0][f]


def test_subset_search_rejects_bad_lists():
    case = zoo.cases()[0]
    with S.Plan(case.spec, case.hw, case.space) as plan:
        d = case.data[:2]
        with pytest.raises(ValueError, match="listed twice"):
            plan.search_batch_subsets(d, [0, 2, 3], [1, 1, 4])
        with pytest.raises(ValueError, match="out of range"):
            plan.search_batch_subsets(d, [0, 1, 2], [0, 99999])
        with pytest.raises(ValueError, match="non-decreasing"):
            plan.search_batch_subsets(d, [0, 2, 1], [0, 1])


def _samples(sizes, seed, noise):
    data, cfg = SM.design_points(sizes, F.enumerate_configs())
    return SM.synthesize(stencil_kernel(noise), data, cfg, seed)


def test_sanity_report_reference_known_answers():
    """test_pipeline.cpp:581-625."""
    hw = zoo.sample_hw()
    s = _samples([64, 128, 256, 512], 11, 0.0)
    X = np.column_stack([s.data[:, 0], s.configs[:, 0], s.configs[:, 1]]).astype(float)
    models = G.fit_all_metrics(X, {m: s.column(m) for m in s.metric_names}, ["D1", "bx", "by"],
                               STENCIL_BOUNDS, STENCIL_CONSTANTS)
    r = SN.sanity_report(models, s, hw)
    assert len(r.rows) == 4 and r.param_names == ["D1"] and not r.notes
    prev = 0
    for row in r.rows:
        assert len(row.data_params) == 1 and row.data_params[0] > prev
        prev = row.data_params[0]
        assert row.measured_best[:2] == row.predicted_best[:2]
        assert abs(row.collected_cycles - row.predicted_best_cycles) <= 1e-6 * abs(row.predicted_best_cycles)
        assert abs(row.measured_best_cycles - row.collected_cycles) <= 1e-9 * abs(row.collected_cycles)
    csv = SN.format_sanity_csv(r)
    assert "D1,ci_bx,ci_by,ci_bz,Ec_i,cr_bx,cr_by,cr_bz,Ec_r,collected_Ec\n" in csv
    assert csv.count("\n") == 5 and csv == SN.format_sanity_csv(r)
    text = SN.format_sanity_text(r)
    assert "collected Ec" in text and "x1" in text
    with pytest.raises(F.PipelineError):
        SN.sanity_report(F.MetricModelSet(), s, hw)
    with pytest.raises(F.PipelineError):
        SN.sanity_report(models, SM.SampleSet(), hw)


@pytest.mark.parametrize("rep_mode", ["real", "ceil"])
def test_sanity_report_matches_oracle(rep_mode):
    hw = zoo.sample_hw()
    sizes = [64, 96, 128, 200, 256, 512, 1000, 2048]
    s = _samples(sizes, 5, 0.02)
    # drop some samples so groups have different configuration subsets, and
    # starve one group of feasible configurations
    rng = np.random.default_rng(2)
    keep = rng.uniform(size=len(s)) > 0.3
    s = SM.SampleSet(s.metric_names, s.data[keep], s.configs[keep], s.values[keep], s.provenance)
    X = np.column_stack([s.data[:, 0], s.configs[:, 0], s.configs[:, 1]]).astype(float)
    models = G.fit_all_metrics(X, {m: s.column(m) for m in s.metric_names}, ["D1", "bx", "by"],
                               STENCIL_BOUNDS, STENCIL_CONSTANTS)
    r = SN.sanity_report(models, s, hw, rep_mode)
    rows = [(tuple(d), tuple(c), list(v)) for d, c, v in zip(s.data, s.configs, s.values)]
    want, notes = O5.sanity_report(models, s.metric_names, rows, hw, rep_mode)
    assert r.notes == notes
    assert len(r.rows) == len(want)
    for got, (params, mcfg, mec, pcfg, pec, col) in zip(r.rows, want):
        assert got.data_params == params
        assert got.measured_best == mcfg and got.measured_best_cycles == mec
        assert got.predicted_best == pcfg and got.predicted_best_cycles == pec
        assert (math.isnan(got.collected_cycles) and math.isnan(col)) or got.collected_cycles == col
