"""Several devices behind one call (rpg_plan_group_*): the
winners are byte-identical to one plan on one device, on the tuple axis
(contiguous tuple blocks, pipeline.hpp:602) and on the configuration axis
(fewer tuples than devices: global best -> tie group -> per-device ranking
-> key merge).  One GPU here: the device list repeats device 0, which runs
the same host logic (one plan per list entry)."""
import numpy as np
import pytest

from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import search as S

from . import zoo

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arith", ["exact", "fast", "fastcm"])
@pytest.mark.parametrize("G", [2, 5])
def test_group_matches_single_device(arith, G):
    n_cases = 0
    for case in zoo.cases()[::2]:
        opts = S.SearchOptions(regs_per_thread=case.regs_fallback,
                               shared_words_per_block=case.shared_fallback,
                               rep_mode=case.rep_mode, arith=arith)
        try:
            single = S.Plan(case.spec, case.hw, case.space, opts)
        except (A.RpgError, ValueError):
            continue  # fast_cm not applicable to this model
        n_cases += 1
        with single, S.PlanGroup(case.spec, case.hw, case.space, [0] * G, opts) as grp:
            assert grp.size == G
            for rows in (case.data, case.data[:1], case.data[: G - 1], case.data[: G + 1]):
                want = single.search_batch(rows)
                got = grp.search_batch(rows)
                assert got.tobytes() == want.tobytes(), (case.name, arith, G, len(rows))
    assert n_cases > 0


def test_group_config_axis_ties_and_infeasible():
    """Flat landscapes (every config tied) and tuples with no feasible
    configuration on the configuration-axis path."""
    for case in zoo.cases():
        if case.name not in ("flat_ties", "singular_coal", "near_singular_synch",
                             "regs_shared_models", "compute_only"):
            continue
        for arith in ("exact", "fast"):
            opts = S.SearchOptions(regs_per_thread=case.regs_fallback,
                                   shared_words_per_block=case.shared_fallback,
                                   rep_mode=case.rep_mode, arith=arith)
            with S.Plan(case.spec, case.hw, case.space, opts) as one, \
                    S.PlanGroup(case.spec, case.hw, case.space, [0, 0, 0, 0], opts) as grp:
                for t in range(min(3, len(case.data))):
                    row = case.data[t: t + 1]
                    assert grp.search_batch(row).tobytes() == one.search_batch(row).tobytes()
