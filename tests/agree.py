"""The north star's agreement rule (BASELINE.json north_star; SURVEY.md §8d
"Agreement"), shared by the tests that compare a non-reference arithmetic
mode (FAST, FAST_CM) with the reference's operation order (oracle O1 EXACT,
which restates polyfit.hpp:96-130 / perfmodel.hpp:298-395 mul by mul):

* the chosen configuration is the EXACT winner, or its EXACT cycle estimate
  is within 1e-9 relative of the EXACT minimum (a tie within the tolerance
  counts as agreement, pipeline.hpp:654-669);
* the minimum cycle estimate (best_ec) is within 1e-9 relative;
* wherever the winners are equal, the winner's Ec is within 1e-9 and its
  occupancy, block count and case tag are bit-exact (b_active, w_active,
  w_occ, case_tag), and the feasible-config count is equal.

Test infrastructure only (imports oracle O1 as the checker)."""
from __future__ import annotations

import os

import numpy as np

from oracle import o1
from paper_1906_00142_b200 import abi as A

TOL = 1e-9


def threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def exact_options(rep="real", regs=0.0, shared=0.0):
    return A.options_struct(arith=A.RPG_ARITH_EXACT, rep_mode=A.RPG_REP_CEIL if rep == "ceil" else A.RPG_REP_REAL,
                            regs_per_thread=regs, shared_words_per_block=shared)


def exact_winners(spec, hw, space, data, rep="real", regs=0.0, shared=0.0):
    opts = exact_options(rep, regs, shared)
    return o1.search_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), opts,
                           A.config_array(space), data, threads())


def assert_agrees_with_exact(got, spec, hw, space, data, exact=None, rep="real", regs=0.0, shared=0.0):
    """`got`: winner records of the mode under test for `data`.  Returns the
    number of tuples whose winner differs (inside the tolerance)."""
    if exact is None:
        exact = exact_winners(spec, hw, space, data, rep, regs, shared)
    assert len(got) == len(exact)
    # Feasibility and the empty case are integer facts.
    assert np.array_equal(got["n_feasible"], exact["n_feasible"]), "feasible counts differ"
    none = exact["cfg_idx"] < 0
    assert np.array_equal(got["cfg_idx"] < 0, none)
    live = ~none
    rel = np.abs(got["best_ec"][live] - exact["best_ec"][live]) / np.maximum(np.abs(exact["best_ec"][live]),
                                                                           np.finfo(float).tiny)
    assert rel.size == 0 or rel.max() <= TOL, ("best_ec", float(rel.max()))
    same = live & (got["cfg_idx"] == exact["cfg_idx"])
    for f in ("b_active", "w_active", "w_occ", "case_tag"):
        bad = np.nonzero(same & (got[f] != exact[f]))[0]
        assert len(bad) == 0, (f, data[bad[:3]].tolist(), got[bad[:3]], exact[bad[:3]])
    rel_w = np.abs(got["ec"][same] - exact["ec"][same]) / np.maximum(np.abs(exact["ec"][same]),
                                                                     np.finfo(float).tiny)
    assert rel_w.size == 0 or rel_w.max() <= TOL, ("winner ec", float(rel_w.max()))
    diff = np.nonzero(live & ~same)[0]
    if len(diff):
        opts = exact_options(rep, regs, shared)
        ec, _, _ = o1.evaluate_batch(A.PackedModel(spec, drop_zero_terms=False), A.profile_struct(hw), opts,
                                     A.config_array(space), np.ascontiguousarray(data[diff]), threads())
        for j, t in enumerate(diff):
            g = int(got["cfg_idx"][t])
            best = float(exact["best_ec"][t])
            assert ec[j, g] >= 0 and ec[j, g] <= best + abs(best) * TOL, (
                data[t].tolist(), g, float(ec[j, g]), best)
    return len(diff)
