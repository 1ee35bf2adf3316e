"""Builder-authored synthetic PolyBench-GPU metric models (BASELINE config C2).

The reference ships no PolyBench data, so these are
SYNTHETIC.  For each kernel a physically motivated ground truth
(per-thread instruction counts of the PolyBench-GPU CUDA kernel as a function
of the problem size N = D1 and the block shape bx x by) is written in the
reference's `ratprog-kernel-v1` format; a "fitted" companion in
`ratprog-models-v1` format expands every metric to the reference's default
degree bounds (numerator (2,2,2), denominator (1,1,1); pipeline.hpp:88-93)
with small positive seeded perturbations on every monomial — the dense
coefficient structure a least-squares fit of noisy profiles produces.
The fitted files are the benchmark workload (27 + 8 terms per metric).

Run: python data/polybench/make_specs.py   (deterministic; seed 1906)
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
TYPICAL = (4096.0, 32.0, 8.0)  # scale point for the perturbations
EPS = 1e-3


def poly(terms, bounds):
    """terms: {(a,b,c): coef} -> coefficient list over the graded-lex basis."""
    basis = F.monomial_basis(bounds)
    for t in terms:
        assert t in basis, (t, bounds)
    return [float(terms.get(m, 0.0)) for m in basis]


def ratfunc(num_terms, den_terms):
    return {"num": num_terms, "den": den_terms}


# Ground truths (N = D1).  Monomial keys are (N, bx, by) exponents.
KERNELS = {
    # 2DCONV (PolyBench-GPU kernel ID 1): one output pixel per thread, a 3x3
    # stencil (9 loads + 1 store); warps narrower than 32 columns split into
    # partially coalesced segments.
    "2dconv": {
        "regs": 16.0, "shared": 0.0,
        "comp_insts_per_thread": ratfunc({(0, 1, 1): 30.0, (0, 1, 0): 12.0, (0, 0, 1): 6.0}, {(0, 1, 1): 1.0}),
        "uncoal_mem_insts_per_thread": ratfunc({(0, 0, 0): 320.0}, {(0, 0, 0): 32.0, (0, 1, 0): 1.0}),
        "coal_mem_insts_per_thread": ratfunc({(0, 1, 0): 10.0}, {(0, 0, 0): 32.0, (0, 1, 0): 1.0}),
        "synch_insts_per_block": ratfunc({}, {(0, 0, 0): 1.0}),
        "total_blocks": ratfunc({(2, 0, 0): 1.0}, {(0, 1, 1): 1.0}),
    },
    # GEMM (kernel ID 6): one C element per thread, an N-long k loop; A[i][k]
    # is a broadcast when a warp stays in one row (bx >= 32), B[k][j] is
    # coalesced.
    "gemm": {
        "regs": 24.0, "shared": 0.0,
        "comp_insts_per_thread": ratfunc({(1, 0, 0): 4.0, (0, 0, 0): 20.0}, {(0, 0, 0): 1.0}),
        "uncoal_mem_insts_per_thread": ratfunc({(1, 0, 0): 32.0}, {(0, 0, 0): 32.0, (0, 1, 0): 1.0}),
        "coal_mem_insts_per_thread": ratfunc({(1, 1, 0): 2.0, (1, 0, 0): 32.0, (0, 1, 0): 2.0, (0, 0, 0): 64.0},
                                             {(0, 0, 0): 32.0, (0, 1, 0): 1.0}),
        "synch_insts_per_block": ratfunc({}, {(0, 0, 0): 1.0}),
        "total_blocks": ratfunc({(2, 0, 0): 1.0}, {(0, 1, 1): 1.0}),
    },
    # ATAX kernel 1 (kernel ID 8.1): tmp[i] = sum_j A[i][j] x[j]; one row per
    # thread, row-major A walks are uncoalesced, x[j] is a broadcast.
    "atax1": {
        "regs": 20.0, "shared": 0.0,
        "comp_insts_per_thread": ratfunc({(1, 0, 0): 3.0, (0, 0, 0): 10.0}, {(0, 0, 0): 1.0}),
        "uncoal_mem_insts_per_thread": ratfunc({(1, 0, 0): 1.0}, {(0, 0, 0): 1.0}),
        "coal_mem_insts_per_thread": ratfunc({(1, 0, 0): 1.0, (0, 0, 0): 1.0}, {(0, 0, 0): 1.0}),
        "synch_insts_per_block": ratfunc({}, {(0, 0, 0): 1.0}),
        "total_blocks": ratfunc({(1, 0, 0): 1.0}, {(0, 1, 1): 1.0}),
    },
}


def truth_bounds(terms):
    b = [0, 0, 0]
    for m in terms:
        for i, e in enumerate(m):
            b[i] = max(b[i], e)
    return b


def mono(m, x):
    return float(np.prod([xi ** e for xi, e in zip(x, m)]))


def dense(terms, bounds, rng):
    """Default-bound coefficients: truth + EPS-relative positive
    perturbations on every monomial (scaled at the typical point)."""
    basis = F.monomial_basis(bounds)
    scale = sum(abs(c) * mono(m, TYPICAL) for m, c in terms.items()) or 1.0
    out = []
    for m in basis:
        c = terms.get(m, 0.0)
        c += EPS * rng.uniform(0.1, 1.0) * scale / (len(basis) * mono(m, TYPICAL))
        out.append(float(c))
    return out


def main():
    rng = np.random.default_rng(1906)
    for name, k in KERNELS.items():
        truth = {"schema": "ratprog-kernel-v1", "name": name, "variables": VARS,
                 "constants": {"regs_per_thread": k["regs"], "shared_words_per_block": k["shared"]},
                 "noise_rel": 0.0, "metrics": {}}
        fitted = {"schema": "ratprog-models-v1", "variables": VARS,
                  "constants": {"regs_per_thread": k["regs"], "shared_words_per_block": k["shared"]},
                  "metrics": {}, "failures": {}}
        for metric in sorted(F.REQUIRED_METRICS):
            f = k[metric]
            nb = truth_bounds(f["num"]) if f["num"] else [0, 0, 0]
            db = truth_bounds(f["den"])
            truth["metrics"][metric] = {"num_bounds": nb, "num_coeffs": poly(f["num"], nb),
                                        "den_bounds": db, "den_coeffs": poly(f["den"], db)}
            fitted["metrics"][metric] = {"num_bounds": NUM_B, "num_coeffs": dense(f["num"], NUM_B, rng),
                                         "den_bounds": DEN_B, "den_coeffs": dense(f["den"], DEN_B, rng),
                                         "report": {"synthetic": True}}
        with open(os.path.join(HERE, f"{name}.kernel.json"), "w") as fh:
            json.dump(truth, fh, indent=1)
            fh.write("\n")
        with open(os.path.join(HERE, f"{name}.models.json"), "w") as fh:
            json.dump(fitted, fh, indent=1)
            fh.write("\n")
        F.load_kernel_spec(os.path.join(HERE, f"{name}.kernel.json"))
        F.models_to_metric_spec(F.read_models(os.path.join(HERE, f"{name}.models.json")))
        print("wrote", name)


if __name__ == "__main__":
    main()
