"""Pins oracle O1 to the reference's own known-answer tests (CPU only).

Every vector below is restated from the reference test suite (file:line in
each test) — the reference cannot be built here (Eigen/Boost/Catch2 absent),
so these KATs are what makes O1 trustworthy as the GPU checker.
"""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F


def sample_hw():  # test_perfmodel.cpp:22-39
    return F.DeviceProfile(65536, 12288, 1024, 8, 48, 16, 1.3, 436, 4, 40, 144, 4, 128, 32)


def oracle_hw(**kw):  # test_perfmodel.cpp:43-60
    hw = F.DeviceProfile(100000, 100000, 1024, 4, 48, 1, 1, 300, 150, 50, 2, 4, 100, 5)
    for k, v in kw.items():
        setattr(hw, k, v)
    return hw


def tight_hw():  # test_perfmodel.cpp:200-204
    hw = sample_hw()
    hw.R_max, hw.Z_max, hw.W_max, hw.B_max = 8192, 4096, 24, 6
    return hw


def brute_force_blocks(hw, R, Z, T):  # test_perfmodel.cpp:64-75
    if T < 1 or T > hw.T_max:
        return 0
    wpb = (T + 31) // 32
    for b in range(hw.B_max, 0, -1):
        if b * wpb > hw.W_max:
            continue
        if R > 0 and b * R * T > hw.R_max:
            continue
        if Z > 0 and b * Z > hw.Z_max:
            continue
        return b
    return 0


def test_active_blocks_brute_force_grid():
    # test_perfmodel.cpp:198-226
    L = o1.lib()
    for hw in (sample_hw(), tight_hw(), oracle_hw()):
        s = A.profile_struct(hw)
        for T in (1, 16, 31, 32, 33, 64, 96, 128, 192, 256, 512, 768, 1024, 1025, 4096):
            for R in (0, 1, 2, 10, 16, 21, 40, 64):
                for Z in (0, 1, 100, 1000, 4096, 6144, 12288, 20000):
                    want = brute_force_blocks(hw, R, Z, T)
                    got = L.o1_active_blocks(C.byref(s), float(R), float(Z), T)
                    assert got == want, (T, R, Z)
                    w = L.o1_active_warps(C.byref(s), got, T)
                    assert w == (min(got * T // 32, hw.W_max) if got > 0 else 0)
                    occ = L.o1_occupancy(C.byref(s), float(R), float(Z), T)
                    assert 0.0 <= occ <= 1.0


def test_active_blocks_random_tuples():
    # acceptance.cpp:75-99 (10^4 random tuples; numpy draws replace the
    # libstdc++-specific uniform_int_distribution stream)
    L = o1.lib()
    hw = sample_hw()
    s = A.profile_struct(hw)
    rng = np.random.default_rng(2024)
    Rs = rng.integers(0, 97, 10000)
    Zs = rng.integers(0, 16385, 10000)
    Ts = rng.integers(1, hw.T_max + 129, 10000)
    for R, Z, T in zip(Rs.tolist(), Zs.tolist(), Ts.tolist()):
        b = brute_force_blocks(hw, R, Z, T)
        assert L.o1_active_blocks(C.byref(s), float(R), float(Z), T) == b
        w = 0 if b == 0 else min(b * T // 32, hw.W_max)
        assert L.o1_occupancy(C.byref(s), float(R), float(Z), T) == w / hw.W_max


def test_occupancy_basics():
    # test_perfmodel.cpp:228-251
    L = o1.lib()
    s = A.profile_struct(sample_hw())
    ab = lambda R, Z, T: L.o1_active_blocks(C.byref(s), float(R), float(Z), T)
    assert ab(20, 0, 256) == 6
    assert L.o1_active_warps(C.byref(s), 6, 256) == 48
    assert L.o1_occupancy(C.byref(s), 20.0, 0.0, 256) == 1.0
    assert ab(64, 0, 256) == 4
    assert ab(0, 5000, 256) == 2
    assert ab(20, 0, 2048) == 0
    assert ab(0, 0, 0) == 0
    assert ab(300, 0, 1024) == 0
    assert L.o1_occupancy(C.byref(s), 300.0, 0.0, 1024) == 0.0
    prev = 8
    for R in range(1, 81):
        b = ab(R, 0, 256)
        assert b <= prev
        prev = b


def _cycles(hw, m, cfg=(32, 1, 1), mode=A.RPG_REP_REAL):
    return o1.mwpcwp_cycles(A.profile_struct(hw), m, cfg, mode)


def test_cwp_bound_oracle():
    # test_perfmodel.cpp:253-270
    rc, r = _cycles(oracle_hw(), o1.metrics(18, 1, 1, 0, 4))
    assert rc == o1.O1_OK
    assert (r.b_active, r.n_active_warps) == (4, 4)
    assert r.mem_cycles == 800.0 and r.comp_cycles == 80.0
    assert r.mwp == 2.0 and r.cwp == 4.0 and r.rep == 1.0
    assert r.case_tag == A.RPG_CASE_CWP_BOUND
    assert r.cycles_pre_synch == 1640.0 and r.synch_cost == 0.0
    assert r.total_cycles == 1640.0


def test_both_saturated_oracle():
    # test_perfmodel.cpp:272-290
    rc, r = _cycles(oracle_hw(B_max=2, departure_del_coal_cycles=50),
                    o1.metrics(23, 0, 2, 3, 2))
    assert rc == o1.O1_OK
    assert (r.b_active, r.n_active_warps) == (2, 2)
    assert r.mem_cycles == 600.0 and r.comp_cycles == 100.0
    assert r.mwp == 2.0 and r.cwp == 2.0
    assert r.case_tag == A.RPG_CASE_BOTH_SATURATED
    assert r.cycles_pre_synch == 750.0 and r.synch_cost == 300.0
    assert r.total_cycles == 1050.0


def test_mwp_bound_oracle():
    # test_perfmodel.cpp:292-311
    hw = oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=75, mem_bandwidth_GBps=4)
    rc, r = _cycles(hw, o1.metrics(98, 0, 2, 0, 16))
    assert rc == o1.O1_OK
    assert (r.b_active, r.n_active_warps) == (8, 8)
    assert r.mem_cycles == 600.0 and r.comp_cycles == 400.0
    assert r.mwp == 4.0 and r.cwp == 2.5 and r.rep == 1.0
    assert r.case_tag == A.RPG_CASE_MWP_BOUND
    assert r.total_cycles == 3500.0


def test_mwp_bound_raw_latency_pin():
    # test_perfmodel.cpp:313-332
    hw = oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=30,
                   departure_del_uncoal_cycles=30, mem_bandwidth_GBps=4)
    rc, r = _cycles(hw, o1.metrics(98, 1, 1, 0, 16))
    assert r.mwp == 4.0
    assert r.case_tag == A.RPG_CASE_MWP_BOUND
    assert r.total_cycles == 3500.0


def test_compute_only():
    # test_perfmodel.cpp:334-353
    rc, r = _cycles(oracle_hw(), o1.metrics(50, 0, 0, 2, 4))
    assert (r.b_active, r.n_active_warps) == (4, 4)
    assert r.mem_cycles == 0.0 and r.comp_cycles == 200.0 and r.mwp == 4.0
    assert r.case_tag == A.RPG_CASE_CWP_BOUND
    assert r.cycles_pre_synch == 200.0
    assert r.synch_cost == 150.0 * 3 * 2 * 4
    assert r.total_cycles == 200.0 + 3600.0
    assert _cycles(oracle_hw(), o1.metrics(50, 0, 0, 0, 4))[1].total_cycles == 200.0


def test_rejects_inconsistent_or_unlaunchable():
    # test_perfmodel.cpp:355-383
    hw = oracle_hw()
    bad = o1.metrics(10, 1, 1, 0, 4)
    bad.mem_insts_per_thread = 3
    assert _cycles(hw, bad)[0] == o1.O1_MODEL_ERROR
    neg = o1.metrics(-1, 1, 1, 0, 4)
    assert _cycles(hw, neg)[0] == o1.O1_MODEL_ERROR
    assert _cycles(hw, o1.metrics(10, 1, 1, 0, 4), (64, 32, 1))[0] == o1.O1_ZERO_OCCUPANCY
    assert _cycles(oracle_hw(B_max=1), o1.metrics(10, 1, 1, 0, 4), (8, 1, 1))[0] == o1.O1_ZERO_OCCUPANCY
    assert _cycles(hw, o1.metrics(10, 1, 1, 0, 4, R=1e9))[0] == o1.O1_ZERO_OCCUPANCY


def test_rep_modes():
    # test_perfmodel.cpp:385-396
    rc, r = _cycles(oracle_hw(), o1.metrics(50, 0, 0, 0, 5), mode=A.RPG_REP_REAL)
    assert r.rep == 1.25 and r.total_cycles == 250.0
    rc, r = _cycles(oracle_hw(), o1.metrics(50, 0, 0, 0, 5), mode=A.RPG_REP_CEIL)
    assert r.rep == 2.0 and r.total_cycles == 400.0


def _spec_from_constants(comp, uncoal, coal, synch, blocks, R=0.0, Z=0.0):
    return F.MetricSpec(["D1", "bx", "by"], {}, {
        F.METRIC_COMP: comp, F.METRIC_UNCOAL: uncoal, F.METRIC_COAL: coal,
        F.METRIC_SYNCH: synch, F.METRIC_TOTAL_BLOCKS: blocks,
        F.METRIC_REGS: R, F.METRIC_SHARED: Z})


@pytest.mark.parametrize("name,hw,m,total", [
    ("cwp_bound", oracle_hw(), (18, 1, 1, 0, 4), 1640),
    ("both_saturated", oracle_hw(B_max=2, departure_del_coal_cycles=50), (23, 0, 2, 3, 2), 1050),
    ("mwp_bound", oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=75, mem_bandwidth_GBps=4),
     (98, 0, 2, 0, 16), 3500),
    ("raw_latency_pin", oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=30,
                                  departure_del_uncoal_cycles=30, mem_bandwidth_GBps=4),
     (98, 1, 1, 0, 16), 3500),
])
def test_program_point_reproduces_hand_oracles(name, hw, m, total):
    # test_perfmodel.cpp:440-497: the search-semantics point at (64, 32x1).
    packed = A.PackedModel(_spec_from_constants(*m))
    p = o1.eval_point(packed, A.profile_struct(hw), A.options_struct(), [64], (32, 1, 1))
    assert p.feasible and p.ec == total, name


def stencil_spec():  # test_perfmodel.cpp:113-129
    return F.kernel_to_metric_spec(F.load_kernel_spec("data/stencil2d.kernel.json"))


def test_program_point_matches_direct_on_stencil():
    # test_perfmodel.cpp:499-542 (program == direct within 1e-9; here both are
    # FP64 so the agreement is exact), both rep modes.
    hw = sample_hw()
    hws = A.profile_struct(hw)
    packed = A.PackedModel(stencil_spec(), drop_zero_terms=False)
    checked = 0
    for mode in (A.RPG_REP_REAL, A.RPG_REP_CEIL):
        opts = A.options_struct(rep_mode=mode)
        for d1 in (64, 256, 1024):
            bx = 1
            while bx <= 1024:
                by = 1
                while bx * by <= 2048:
                    x = (C.c_double * 3)(d1, bx, by)
                    m = o1.o1_metrics()
                    assert o1.lib().o1_evaluate_metrics(C.byref(packed.struct), x, C.byref(m)) == 0
                    rc, br = o1.mwpcwp_cycles(hws, m, (bx, by, 1), mode)
                    p = o1.eval_point(packed, hws, opts, [d1], (bx, by, 1))
                    if rc == o1.O1_ZERO_OCCUPANCY:
                        assert p.ec == -1.0 and not p.feasible
                    else:
                        assert rc == o1.O1_OK and p.feasible
                        assert p.ec == br.total_cycles
                        assert p.tag == br.case_tag
                        checked += 1
                    by *= 2
                bx *= 2
    assert checked >= 100


def test_singular_denominator_is_infeasible():
    # test_perfmodel.cpp:544-556: coal = 9 / (bx - 32).
    spec = stencil_spec()
    spec.models[F.METRIC_COAL] = F.make_ratfunc(["D1", "bx", "by"], [0, 0, 0], [9], [0, 1, 0], [-32, 1])
    packed = A.PackedModel(spec)
    hws = A.profile_struct(sample_hw())
    assert o1.eval_point(packed, hws, A.options_struct(), [64], (32, 2, 1)).ec == -1.0
    assert o1.eval_point(packed, hws, A.options_struct(), [64], (16, 2, 1)).ec != -1.0


def test_eval_poly_kats():
    # test_polyfit.cpp:57-87
    coef = np.array([1.0, 2.0])
    exps = np.array([[0], [1]], dtype=np.uint8)
    p = A.rpg_poly(2, 0, A.ptr(coef, C.c_double), A.ptr(exps, C.c_uint8))
    x = (C.c_double * 1)(3.0)
    assert o1.lib().o1_eval_poly(C.byref(p), 1, x) == 7.0
    # random (2,2,2) polynomial vs a term-by-term oracle within 1e-12
    rng = np.random.default_rng(42)
    basis = F.monomial_basis([2, 2, 2])
    coef = rng.uniform(-2, 2, len(basis))
    ex = np.array(basis, dtype=np.uint8)
    p = A.rpg_poly(len(basis), 0, A.ptr(coef, C.c_double), A.ptr(ex, C.c_uint8))
    for _ in range(20):
        pt = rng.uniform(-2, 2, 3)
        want = sum(c * pt[0] ** e[0] * pt[1] ** e[1] * pt[2] ** e[2] for c, e in zip(coef, basis))
        got = o1.lib().o1_eval_poly(C.byref(p), 3, (C.c_double * 3)(*pt))
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
    # eval_ratfunc 5/4 and the singular point x = -2
    nc, ne = np.array([1.0, 0.0, 1.0]), np.array([[0], [1], [2]], dtype=np.uint8)
    dc, de = np.array([2.0, 1.0]), np.array([[0], [1]], dtype=np.uint8)
    num = A.rpg_poly(3, 0, A.ptr(nc, C.c_double), A.ptr(ne, C.c_uint8))
    den = A.rpg_poly(2, 0, A.ptr(dc, C.c_double), A.ptr(de, C.c_uint8))
    out = C.c_double()
    assert o1.lib().o1_eval_ratfunc(C.byref(num), C.byref(den), 1, (C.c_double * 1)(2.0), C.byref(out)) == 0
    assert out.value == pytest.approx(1.25)
    assert o1.lib().o1_eval_ratfunc(C.byref(num), C.byref(den), 1, (C.c_double * 1)(-2.0), C.byref(out)) == o1.O1_DEN_NEAR_ZERO


def test_synth_kat_metrics():
    # test_datakit.cpp:139-163: stencil metrics at D1=256, 32x8.
    packed = A.PackedModel(stencil_spec(), drop_zero_terms=False)
    m = o1.o1_metrics()
    assert o1.lib().o1_evaluate_metrics(C.byref(packed.struct), (C.c_double * 3)(256, 32, 8), C.byref(m)) == 0
    assert m.comp_insts_per_thread == 84.0
    assert m.uncoal_mem_insts_per_thread == 5.375
    assert m.coal_mem_insts_per_thread == 9.0
    assert m.synch_insts_per_block == 16.0
    assert m.total_blocks == 256.0


def test_tie_break_prefers_occupancy_then_lex():
    # test_pipeline.cpp:464-493 — the flat landscape (Ec = 100 for every
    # config, R = Z = 0): ties = 51, best 1x256, head (1,256),(1,512),(2,128),(2,256).
    # A compute-only constant model with rep = 1 gives a config-independent
    # Ec: comp*issue*rep with total_blocks = b*num_SM is not constant, so use
    # RepMode::Ceil with total_blocks = 1 (rep = ceil(1/(b*16)) = 1).
    spec = _spec_from_constants(25, 0, 0, 0, 1)
    packed = A.PackedModel(spec)
    hws = A.profile_struct(sample_hw())
    space = A.config_array(F.enumerate_configs())
    w, order = o1.search_one(packed, hws, A.options_struct(rep_mode=A.RPG_REP_CEIL), space, [64])
    assert w.ties == 51 and w.n_feasible == 51
    assert w.ec == 100.0
    head = [tuple(space[i])[:2] for i in order[:4]]
    assert head == [(1, 256), (1, 512), (2, 128), (2, 256)]
    assert tuple(space[w.cfg_idx])[:2] == (1, 256)
    assert w.w_occ == 48
