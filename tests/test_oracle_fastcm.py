"""Oracle O1's FAST_CM twin (oracle/o1.c fast_cm_poly): the configuration-
major FMA order differs from EXACT only in rounding — Ec within 1e-12
relative on every point of a C2 model sample and the same winners (or the
EXACT winner inside the tie window)."""
import os

import numpy as np

from oracle import o1
from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F

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
    win_x = o1.search_batch(pk, hw, A.options_struct(arith=A.RPG_ARITH_EXACT), space, data, 2)
    win_c = o1.search_batch(pk, hw, A.options_struct(arith=A.RPG_ARITH_FAST_CM), space, data, 2)
    same = win_x["cfg_idx"] == win_c["cfg_idx"]
    assert same.mean() > 0.9
    for i in np.nonzero(~same)[0]:  # a different winner must be inside the tie window
        assert abs(win_x["best_ec"][i] / win_c["best_ec"][i] - 1) < 1e-12
