"""Oracle O1's FAST_CM twin (oracle/o1.c fast_cm_poly): the configuration-
major FMA order differs from EXACT only in rounding — Ec within 1e-12
relative on every point of a C2 model sample and the same winners (or the
EXACT winner inside the tie window)."""
import os

import numpy as np

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F

from .agree import assert_agrees_with_exact, threads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fast_cm_twin_agrees_with_exact():
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))
    hw = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "b200.profile")))
    space = A.config_array(F.integer_configs(1024, dims=2)[::7])
    pk = A.PackedModel(spec, drop_zero_terms=False)
    data = np.arange(64, 65537, 4099, dtype=np.int64).reshape(-1, 1)
    ec_x, tag_x, w_x = o1.evaluate_batch(pk, hw, A.options_struct(arith=A.RPG_ARITH_EXACT), space, data, 2)
    ec_c, tag_c, w_c = o1.evaluate_batch(pk, hw, A.options_struct(arith=A.RPG_ARITH_FAST_CM), space, data, 2)
    assert np.all(np.abs(ec_c / ec_x - 1) < 1e-12)
    assert np.array_equal(tag_x, tag_c) and np.array_equal(w_x, w_c)
    win_c = o1.search_batch(pk, hw, A.options_struct(arith=A.RPG_ARITH_FAST_CM), space, data, 2)
    # The north star's rule (tests/agree.py): every winner equal, or inside
    # the EXACT minimum's 1e-9 window; diagnostics bit-exact where equal.
    assert_agrees_with_exact(win_c, spec, F.load_profile(os.path.join(ROOT, "data", "b200.profile")),
                             F.integer_configs(1024, dims=2)[::7], data)


def test_fast_cm_twin_c2_models_every_61st_n():
    """O1's FAST_CM twin (the headline mode's operation order) against O1
    EXACT on all three C2 models, 1,074 N x 7,262 configs each, under the
    north star's rule."""
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    space = F.integer_configs(1024, dims=2)
    data = np.arange(64, 65537, 61, dtype=np.int64).reshape(-1, 1)
    for k in ("2dconv", "gemm", "atax1"):
        spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", f"{k}.models.json")))
        pk = A.PackedModel(spec, drop_zero_terms=False)
        win_c = o1.search_batch(pk, A.profile_struct(hw), A.options_struct(arith=A.RPG_ARITH_FAST_CM),
                                A.config_array(space), data, threads())
        assert_agrees_with_exact(win_c, spec, hw, space, data)
