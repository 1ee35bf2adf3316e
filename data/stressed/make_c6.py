"""C6: a non-degenerate search landscape (builder-authored, synthetic).

The C2 landscape is degenerate (every point feasible, 99.99 %
cwp_bound, no ties).  C6 keeps C2's shape — three kernels, D1 = N, integer
(bx, by) with bx*by <= 1024, the B200 profile, default-bound fitted form
(numerator (2,2,2) / denominator (1,1,1), pipeline.hpp:88-93) — but builds
metrics that

* make configurations infeasible: regs_per_thread = 80 leaves no resident
  block once 80 * bx * by > R_max = 65536 (T >= 820), and shared memory
  (4096 words per block) caps the resident blocks at 14;
* tie exactly: every monomial is T-symmetric (exponents (i, a, a): the
  block dimensions only enter through T = bx * by), so all (bx, by) with
  the same product evaluate to the same bits (the monomials are exact
  integers) — every tuple's winner has a tie group of all divisor pairs of
  its T, decided by the reference's occupancy / Ec / lex rule;
* cover all three MWP-CWP cases: compute vs memory per thread and the
  uncoalesced fraction vary over (N, T) so that mc / cc spans [1, > W] and
  r = uncoal / mem spans [0, 1].

Written in the reference's `ratprog-models-v1` format: every T-symmetric
basis monomial carries a small seeded positive coefficient (the dense form a
least-squares fit produces), the remaining basis entries are 0.
Run: python data/stressed/make_c6.py   (deterministic; seed 1906)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1906_00142_b200 import formats as F  # noqa: E402

VARS = ["D1", "bx", "by"]
NUM_B, DEN_B = [2, 2, 2], [1, 1, 1]
TYPICAL_N, TYPICAL_T = 4096.0, 128.0
EPS = 1e-3

# (i, a) -> coefficient of N^i T^a, numerator / denominator.
KERNELS = {
    "c6_stencil": {
        # comp = 2 + 0.05 N + 3000 / T (compute grows with N, falls with T)
        "comp_insts_per_thread": ({(0, 1): 2.0, (1, 1): 0.05, (0, 0): 3000.0}, {(0, 1): 1.0}),
        # uncoal = 0.5 + 200 / T: narrow blocks are uncoalesced
        "uncoal_mem_insts_per_thread": ({(0, 1): 0.5, (0, 0): 200.0}, {(0, 1): 1.0}),
        "coal_mem_insts_per_thread": ({(0, 0): 10.0, (1, 0): 0.002}, {(0, 0): 1.0}),
        "synch_insts_per_block": ({(0, 0): 2.0, (0, 1): 1.0 / 64.0}, {(0, 0): 1.0}),
        "total_blocks": ({(2, 0): 1.0}, {(0, 1): 1.0}),
    },
    "c6_kloop": {
        # memory-heavy k loop: mc / cc large for small N, compute catches up
        "comp_insts_per_thread": ({(0, 0): 20.0, (1, 0): 0.5}, {(0, 0): 1.0}),
        "uncoal_mem_insts_per_thread": ({(1, 0): 0.25, (0, 0): 8.0}, {(0, 0): 1.0, (0, 1): 0.125}),
        "coal_mem_insts_per_thread": ({(1, 0): 1.0, (0, 0): 4.0}, {(0, 0): 1.0}),
        "synch_insts_per_block": ({(0, 0): 0.0, (1, 0): 1.0 / 16.0}, {(0, 0): 1.0}),
        "total_blocks": ({(2, 0): 1.0}, {(0, 1): 1.0}),
    },
    "c6_reduce": {
        # compute-heavy reduction with a coalesced sweep: mwp-bound and
        # both-saturated regions
        "comp_insts_per_thread": ({(0, 0): 40.0, (1, 0): 0.03, (0, 1): 0.5}, {(0, 0): 1.0}),
        "uncoal_mem_insts_per_thread": ({(0, 0): 1.0}, {(0, 0): 1.0, (0, 1): 0.5}),
        "coal_mem_insts_per_thread": ({(0, 0): 60.0, (1, 0): 0.01}, {(0, 0): 1.0}),
        "synch_insts_per_block": ({(0, 0): 4.0, (0, 1): 0.25}, {(0, 0): 1.0, (0, 1): 0.01}),
        "total_blocks": ({(2, 0): 1.0}, {(0, 1): 1.0}),
    },
}
CONSTANTS = {"regs_per_thread": 80.0, "shared_words_per_block": 4096.0}


def coeffs(terms, bounds, rng):
    """Dense T-symmetric coefficient list over the graded-lex basis: the
    ground-truth terms plus EPS-relative positive perturbations on every
    (i, a, a) monomial the bounds allow."""
    basis = F.monomial_basis(bounds)
    scale = max(abs(c) * TYPICAL_N ** i * TYPICAL_T ** a for (i, a), c in terms.items()) or 1.0
    out = []
    for (i, bx, by) in basis:
        if bx != by:
            out.append(0.0)
            continue
        c = terms.get((i, bx), 0.0)
        c += EPS * scale * rng.uniform(0.5, 1.5) / (TYPICAL_N ** i * TYPICAL_T ** bx)
        out.append(float(c))
    return out


def main():
    rng = np.random.default_rng(1906)
    for name, metrics in KERNELS.items():
        doc = {"schema": "ratprog-models-v1", "variables": VARS, "constants": CONSTANTS,
               "metrics": {}, "failures": {}}
        for metric in sorted(metrics):
            num, den = metrics[metric]
            doc["metrics"][metric] = {"num_bounds": NUM_B, "num_coeffs": coeffs(num, NUM_B, rng),
                                      "den_bounds": DEN_B, "den_coeffs": coeffs(den, DEN_B, rng)}
        with open(os.path.join(HERE, f"{name}.models.json"), "w") as f:
            json.dump(doc, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
