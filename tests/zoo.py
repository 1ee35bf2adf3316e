"""Test-model zoo: metric specs, profiles, spaces and data tuples that
exercise every branch of the search semantics (all three MWP-CWP cases,
compute-only, guarded/infeasible points, singular and near-singular
denominators, negative fitted metrics, register/shared-memory models, bz
modelled or not, data variables after block variables, flat tie landscapes,
both repetition modes).

The reference's own fixture (stencil2d x sample_device) is degenerate —
every config is cwp_bound — hence the builder-authored cases.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from paper_1906_00142_b200 import formats as F

ROOT_DATA = __import__("os").path.join(
    __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))),
    "data")


@dataclass
class Case:
    name: str
    spec: F.MetricSpec
    hw: F.DeviceProfile
    space: List[Tuple[int, int, int]]
    data: np.ndarray
    rep_mode: str = "real"
    regs_fallback: float = 0.0
    shared_fallback: float = 0.0


def sample_hw() -> F.DeviceProfile:
    return F.DeviceProfile(65536, 12288, 1024, 8, 48, 16, 1.3, 436, 4, 40, 144, 4, 128, 32)


def oracle_hw(**kw) -> F.DeviceProfile:
    hw = F.DeviceProfile(100000, 100000, 1024, 4, 48, 1, 1, 300, 150, 50, 2, 4, 100, 5)
    for k, v in kw.items():
        setattr(hw, k, v)
    return hw


def b200_hw() -> F.DeviceProfile:
    return F.load_profile(f"{ROOT_DATA}/b200.profile")


def stencil_spec() -> F.MetricSpec:
    return F.kernel_to_metric_spec(F.load_kernel_spec(f"{ROOT_DATA}/stencil2d.kernel.json"))


def const_spec(comp, uncoal, coal, synch, blocks, R=0.0, Z=0.0, variables=("D1", "bx", "by")):
    return F.MetricSpec(list(variables), {}, {
        F.METRIC_COMP: comp, F.METRIC_UNCOAL: uncoal, F.METRIC_COAL: coal,
        F.METRIC_SYNCH: synch, F.METRIC_TOTAL_BLOCKS: blocks,
        F.METRIC_REGS: R, F.METRIC_SHARED: Z})


def random_ratfunc(rng, variables, num_bounds, den_bounds, scale=1.0, positive=True,
                   sparsity=0.0):
    nb = F.monomial_basis(num_bounds)
    db = F.monomial_basis(den_bounds)
    def coeffs(basis, mag):
        c = []
        for mono in basis:
            deg = sum(mono)
            v = rng.uniform(0.05, 1.0) * mag / (8.0 ** deg)
            if not positive and rng.uniform() < 0.25:
                v = -v
            if rng.uniform() < sparsity:
                v = 0.0
            c.append(float(v))
        return c
    nc = coeffs(nb, scale)
    dc = coeffs(db, 1.0)
    dc[0] = max(dc[0], 0.5)  # keep the denominator away from zero
    return F.make_ratfunc(variables, num_bounds, nc, den_bounds, dc)


def random_spec(rng, variables, num_bounds=None, den_bounds=None, R=None, Z=None,
                positive=True, sparsity=0.2) -> F.MetricSpec:
    nv = len(variables)
    nb = num_bounds or [2] * nv
    db = den_bounds or [1] * nv
    spec = F.MetricSpec(list(variables), {}, {})
    scales = {F.METRIC_COMP: 40.0, F.METRIC_UNCOAL: 4.0, F.METRIC_COAL: 8.0,
              F.METRIC_SYNCH: 2.0, F.METRIC_TOTAL_BLOCKS: 3000.0}
    for name, sc in scales.items():
        spec.models[name] = random_ratfunc(rng, variables, nb, db, sc, positive, sparsity)
    spec.constants[F.METRIC_REGS] = float(R if R is not None else rng.integers(8, 64))
    spec.constants[F.METRIC_SHARED] = float(Z if Z is not None else rng.choice([0, 0, 256, 2048]))
    return spec


def random_hw(rng) -> F.DeviceProfile:
    return F.DeviceProfile(
        int(rng.choice([32768, 65536])), int(rng.choice([12288, 24576, 49152])), 1024,
        int(rng.integers(2, 33)), int(rng.integers(8, 65)), int(rng.integers(1, 149)),
        float(rng.uniform(0.8, 2.0)), float(rng.uniform(200, 800)), float(rng.uniform(2, 40)),
        float(rng.uniform(10, 120)), float(rng.uniform(20, 8000)), float(rng.choice([1, 2, 4])),
        int(rng.choice([64, 128])), int(rng.choice([4, 8, 16, 32])))


def cases(small: bool = True) -> List[Case]:
    rng = np.random.default_rng(20240817)
    pow2 = F.enumerate_configs()
    dense = F.integer_configs()
    dense_sub = dense[::7] if small else dense
    out: List[Case] = []

    d1 = np.array([[64], [128], [256], [512], [1000], [1024], [2048], [4097], [8192]], dtype=np.int64)
    out.append(Case("stencil_truth_pow2", stencil_spec(), sample_hw(), pow2, d1))
    out.append(Case("stencil_truth_dense", stencil_spec(), sample_hw(), dense_sub, d1[::2]))
    out.append(Case("stencil_truth_ceil", stencil_spec(), sample_hw(), pow2, d1, rep_mode="ceil"))

    # The hand-computed oracles as constant models (test_perfmodel.cpp:440-497),
    # over the power-of-two space.
    out.append(Case("oracle_cwp", const_spec(18, 1, 1, 0, 4), oracle_hw(), pow2, d1[:2]))
    out.append(Case("oracle_both", const_spec(23, 0, 2, 3, 2), oracle_hw(B_max=2, departure_del_coal_cycles=50), pow2, d1[:2]))
    out.append(Case("oracle_mwp", const_spec(98, 0, 2, 0, 16),
                    oracle_hw(B_max=8, num_SM=2, departure_del_coal_cycles=75, mem_bandwidth_GBps=4), pow2, d1[:2]))
    out.append(Case("compute_only", const_spec(50, 0, 0, 2, 5), oracle_hw(), pow2, d1[:2]))
    # Flat landscape: every config ties (test_pipeline.cpp:464-493).
    out.append(Case("flat_ties", const_spec(25, 0, 0, 0, 1), sample_hw(), pow2, d1[:2], rep_mode="ceil"))

    # Singular denominator at bx = 32 (test_perfmodel.cpp:544-556) and a
    # near-singular one (DenominatorNearZero fallback occupancy).
    s = stencil_spec()
    s.models[F.METRIC_COAL] = F.make_ratfunc(["D1", "bx", "by"], [0, 0, 0], [9], [0, 1, 0], [-32, 1])
    out.append(Case("singular_coal", s, sample_hw(), pow2, d1[:4]))
    s = stencil_spec()
    s.models[F.METRIC_SYNCH] = F.make_ratfunc(["D1", "bx", "by"], [1, 0, 0], [1e13, 0.0], [0, 1, 0], [-16.0, 1.0])
    out.append(Case("near_singular_synch", s, sample_hw(), pow2, d1[:4], regs_fallback=40.0,
                    shared_fallback=1000.0))

    # Random dense 3-variable models (default bounds) on random profiles.
    for i in range(6):
        hw = random_hw(rng)
        spec = random_spec(rng, ["D1", "bx", "by"])
        data = np.sort(rng.integers(64, 65537, size=(12, 1)), axis=0)
        out.append(Case(f"random3_{i}", spec, hw, dense_sub if i % 2 else pow2, data))
    # Negative dips (fitted metrics can go below zero).
    for i in range(2):
        hw = random_hw(rng)
        spec = random_spec(rng, ["D1", "bx", "by"], positive=False)
        data = rng.integers(64, 4097, size=(8, 1))
        out.append(Case(f"negative_{i}", spec, hw, pow2, data))
    # Register and shared-memory pressure as fitted models.
    spec = random_spec(rng, ["D1", "bx", "by"])
    del spec.constants[F.METRIC_REGS]
    del spec.constants[F.METRIC_SHARED]
    spec.models[F.METRIC_REGS] = F.make_ratfunc(["D1", "bx", "by"], [0, 1, 1], [16.0, 0.01, 0.02, 0.0001], [0, 0, 0], [1.0])
    spec.models[F.METRIC_SHARED] = F.make_ratfunc(["D1", "bx", "by"], [0, 1, 1], [0.0, 0.0, 0.0, 4.0], [0, 0, 0], [1.0])
    out.append(Case("regs_shared_models", spec, sample_hw(), dense_sub, rng.integers(64, 8193, size=(6, 1))))
    # Five variables (C5 shape): D1, D2, bx, by, bz with a 3-D space.
    spec = random_spec(rng, ["D1", "D2", "bx", "by", "bz"], sparsity=0.5)
    space3 = F.integer_configs(dims=3)[:: (97 if small else 1)]
    data = rng.integers(16, 2049, size=(5, 2))
    out.append(Case("five_vars_3d", spec, b200_hw(), space3, data))
    # bz not modelled but present in the space (T uses bx*by only).
    spec = random_spec(rng, ["D1", "bx", "by"])
    out.append(Case("bz_unmodelled", spec, sample_hw(), F.enumerate_configs(1024, 32, 3), rng.integers(64, 4097, size=(4, 1))))
    # Data variable after the block variables.
    spec = random_spec(rng, ["bx", "by", "D1"])
    out.append(Case("data_after_blocks", spec, sample_hw(), pow2, rng.integers(64, 4097, size=(4, 1))))
    # Two data parameters, data tuple wider than the model needs.
    spec = random_spec(rng, ["D2", "bx", "by"])
    out.append(Case("skip_d1", spec, sample_hw(), pow2, rng.integers(64, 4097, size=(4, 3))))
    return out
