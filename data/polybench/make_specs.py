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


# ---------------------------------------------------------------------------
# The rest of the PolyBench-GPU suite (kernel IDs 2.1-15.3;
# config C3).  Built from a few access-pattern building blocks, since every
# PolyBench-GPU kernel is one of: an element-wise 2-D update, a k-loop
# matrix product, or a 1-D row/column walk.  Per-thread counts; N = D1.

def _k(regs, shared, comp, uncoal, coal, synch, blocks):
    return {"regs": regs, "shared": shared, "comp_insts_per_thread": comp,
            "uncoal_mem_insts_per_thread": uncoal, "coal_mem_insts_per_thread": coal,
            "synch_insts_per_block": synch, "total_blocks": blocks}


_NO_SYNCH = ratfunc({}, {(0, 0, 0): 1.0})
_BLOCKS_2D = ratfunc({(2, 0, 0): 1.0}, {(0, 1, 1): 1.0})    # N^2 / (bx by)
_BLOCKS_1D = ratfunc({(1, 0, 0): 1.0}, {(0, 1, 1): 1.0})    # N / (bx by)


def _narrow(c):
    """c accesses split into 32/(32+bx)-weighted partial segments (warps narrower than 32 columns)."""
    return ratfunc({(0, 0, 0): 32.0 * c}, {(0, 0, 0): 32.0, (0, 1, 0): 1.0})


def _wide(c):
    """the complementary coalesced share bx/(32+bx) of c accesses."""
    return ratfunc({(0, 1, 0): float(c)}, {(0, 0, 0): 32.0, (0, 1, 0): 1.0})


def _elementwise(regs, comp, loads):
    """2-D element-wise update (FDTD steps, CORR/COVAR reduce)."""
    return _k(regs, 0.0, ratfunc({(0, 1, 1): comp, (0, 1, 0): 8.0, (0, 0, 1): 4.0}, {(0, 1, 1): 1.0}),
              _narrow(loads), _wide(loads), _NO_SYNCH, _BLOCKS_2D)


def _kloop(regs, comp_per_k, loads_per_k, uncoal_per_k):
    """k-loop matrix product, one output element per thread (2MM/3MM/SYRK/SYR2K)."""
    return _k(regs, 0.0, ratfunc({(1, 0, 0): comp_per_k, (0, 0, 0): 24.0}, {(0, 0, 0): 1.0}),
              ratfunc({(1, 0, 0): 32.0 * uncoal_per_k}, {(0, 0, 0): 32.0, (0, 1, 0): 1.0}),
              ratfunc({(1, 1, 0): 2.0 * loads_per_k, (1, 0, 0): 32.0 * loads_per_k, (0, 1, 0): 2.0, (0, 0, 0): 64.0},
                      {(0, 0, 0): 32.0, (0, 1, 0): 1.0}),
              _NO_SYNCH, _BLOCKS_2D)


def _rowwalk(regs, comp_per_n, rows, const=10.0):
    """1-D kernel, one row per thread: row-major walks are uncoalesced (ATAX1, BICG2, MVT1, GESUMMV)."""
    return _k(regs, 0.0, ratfunc({(1, 0, 0): comp_per_n, (0, 0, 0): const}, {(0, 0, 0): 1.0}),
              ratfunc({(1, 0, 0): float(rows)}, {(0, 0, 0): 1.0}),
              ratfunc({(1, 0, 0): 1.0, (0, 0, 0): 1.0}, {(0, 0, 0): 1.0}), _NO_SYNCH, _BLOCKS_1D)


def _colwalk(regs, comp_per_n, cols, const=10.0, synch=None, blocks=None):
    """1-D kernel, one column per thread: column walks coalesce across the warp (ATAX2, BICG1, MVT2, means)."""
    return _k(regs, 0.0, ratfunc({(1, 0, 0): comp_per_n, (0, 0, 0): const}, {(0, 0, 0): 1.0}),
              ratfunc({(0, 0, 0): 1.0}, {(0, 0, 0): 1.0}),
              ratfunc({(1, 0, 0): float(cols + 1), (0, 0, 0): 2.0}, {(0, 0, 0): 1.0}),
              synch or _NO_SYNCH, blocks or _BLOCKS_1D)


KERNELS.update({
    # FDTD_2D (2.1-2.3): ey/ex/hz updates, 2-4 loads + 1 store per point.
    "fdtd2d_step1": _elementwise(18.0, 14.0, 4.0),
    "fdtd2d_step2": _elementwise(18.0, 14.0, 4.0 + 0.5),
    "fdtd2d_step3": _elementwise(22.0, 22.0, 6.0),
    # 2MM (3) / 3MM (4): tmp = A B with an alpha scale; 3MM's first product.
    "2mm1": _kloop(26.0, 5.0, 1.0, 1.0),
    "3mm1": _kloop(24.0, 4.0, 1.0, 1.0),
    # BICG (5.1 column walk, 5.2 row walk).
    "bicg1": _colwalk(20.0, 3.0, 1),
    "bicg2": _rowwalk(20.0, 3.0, 1),
    # 3D_CONVOLUTION (7): 2-D block over (j, k) of one i-slice, 27-point stencil
    # (11 distinct taps), N-slice loop on the host: N^2 / (bx by) blocks.
    "3dconv": _k(28.0, 0.0, ratfunc({(0, 1, 1): 60.0, (0, 1, 0): 16.0, (0, 0, 1): 8.0}, {(0, 1, 1): 1.0}),
                 _narrow(11.0), _wide(11.0), _NO_SYNCH, _BLOCKS_2D),
    # ATAX kernel 2 (8.2): y[j] = sum_i A[i][j] tmp[i].
    "atax2": _colwalk(20.0, 3.0, 1),
    # GESUMMV (9): two row walks (A and B).
    "gesummv": _rowwalk(24.0, 5.0, 2, 14.0),
    # SYRK (10): C[i][j] = beta C + alpha sum_k A[i][k] A[j][k]; A[j][k] with j
    # across the warp is uncoalesced.
    "syrk": _kloop(24.0, 5.0, 1.0, 1.0 + 1.0),
    # MVT (11.1 row walk, 11.2 column walk).
    "mvt1": _rowwalk(18.0, 3.0, 1),
    "mvt2": _colwalk(18.0, 3.0, 1),
    # SYR2K (12): two products per k, four loads.
    "syr2k": _kloop(30.0, 9.0, 2.0, 2.0 + 1.0),
    # CORR (13.1-13.4): corr_kernel is an O(N^2)-per-thread triangular loop;
    # mean/std walk columns; reduce is element-wise.
    "corr": _k(32.0, 0.0, ratfunc({(2, 0, 0): 3.0, (1, 0, 0): 6.0, (0, 0, 0): 20.0}, {(0, 0, 0): 2.0}),
               ratfunc({(2, 0, 0): 1.0, (1, 0, 0): 1.0}, {(0, 0, 0): 2.0}),
               ratfunc({(2, 0, 0): 1.0, (1, 0, 0): 3.0}, {(0, 0, 0): 2.0}), _NO_SYNCH, _BLOCKS_1D),
    "corr_mean": _colwalk(16.0, 2.0, 1, 12.0),
    "corr_reduce": _elementwise(16.0, 12.0, 3.0),
    "corr_std": _colwalk(18.0, 3.0, 1, 40.0),
    # COVAR (14.1-14.3): covar_kernel like corr without the normalisation.
    "covar": _k(30.0, 0.0, ratfunc({(2, 0, 0): 2.0, (1, 0, 0): 5.0, (0, 0, 0): 16.0}, {(0, 0, 0): 2.0}),
                ratfunc({(2, 0, 0): 1.0, (1, 0, 0): 1.0}, {(0, 0, 0): 2.0}),
                ratfunc({(2, 0, 0): 1.0, (1, 0, 0): 3.0}, {(0, 0, 0): 2.0}), _NO_SYNCH, _BLOCKS_1D),
    "covar_mean": _colwalk(16.0, 2.0, 1, 12.0),
    "covar_reduce": _elementwise(16.0, 10.0, 2.0),
    # GRAMSCHM (15.1-15.3): kernel1 is one block computing a column norm with
    # a shared-memory tree (block-count independent of N); kernel2 scales a
    # column; kernel3 is the O(N) projection per column with a block barrier.
    "gramschmidt1": _k(20.0, 256.0, ratfunc({(1, 0, 0): 3.0, (0, 1, 1): 8.0, (0, 0, 0): 30.0}, {(0, 1, 1): 1.0}),
                       ratfunc({(1, 0, 0): 1.0}, {(0, 1, 1): 1.0}), ratfunc({(0, 0, 0): 2.0}, {(0, 0, 0): 1.0}),
                       ratfunc({(0, 0, 0): 9.0}, {(0, 0, 0): 1.0}),
                       ratfunc({(0, 0, 0): 1.0}, {(0, 0, 0): 1.0})),
    "gramschmidt2": _colwalk(16.0, 0.0, 0, 14.0),
    "gramschmidt3": _colwalk(22.0, 6.0, 2, 16.0, synch=ratfunc({(1, 0, 0): 1.0}, {(0, 0, 0): 1.0})),
})


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


# ---------------------------------------------------------------------------
# C5 stress model: a 3-D stencil over an N x M x 64 grid (data parameters
# D1 = N, D2 = M) launched with 3-D blocks (bx, by, bz).  Variables
# (D1, D2, bx, by, bz); fitted form at the default bounds num (2,2,2,2,2) /
# den (1,1,1,1,1) = 243 + 32 coefficients per metric.

VARS5 = ["D1", "D2", "bx", "by", "bz"]
NUM_B5, DEN_B5 = [2] * 5, [1] * 5
TYPICAL5 = (4096.0, 4096.0, 16.0, 8.0, 4.0)

STRESS = {
    "stencil3d_nm": {
        "regs": 32.0, "shared": 0.0,
        "comp_insts_per_thread": ratfunc({(0, 0, 1, 1, 1): 48.0, (0, 0, 1, 1, 0): 8.0, (0, 0, 0, 1, 1): 6.0,
                                          (0, 0, 1, 0, 1): 4.0},
                                         {(0, 0, 1, 1, 1): 1.0}),
        "uncoal_mem_insts_per_thread": ratfunc({(0, 0, 0, 0, 0): 32.0 * 7.0, (0, 0, 0, 0, 1): 16.0},
                                               {(0, 0, 0, 0, 0): 32.0, (0, 0, 1, 0, 0): 1.0}),
        "coal_mem_insts_per_thread": ratfunc({(0, 0, 1, 0, 0): 7.0, (0, 0, 0, 0, 1): 1.0},
                                             {(0, 0, 0, 0, 0): 32.0, (0, 0, 1, 0, 0): 1.0}),
        "synch_insts_per_block": ratfunc({}, {(0, 0, 0, 0, 0): 1.0}),
        "total_blocks": ratfunc({(1, 1, 0, 0, 0): 64.0}, {(0, 0, 1, 1, 1): 1.0}),
    },
}


def dense5(terms, bounds, rng):
    basis = F.monomial_basis(bounds)
    scale = sum(abs(c) * mono(m, TYPICAL5) for m, c in terms.items()) or 1.0
    return [float(terms.get(m, 0.0) + EPS * rng.uniform(0.1, 1.0) * scale / (len(basis) * mono(m, TYPICAL5)))
            for m in basis]


def write_stress():
    rng = np.random.default_rng(19060)
    for name, k in STRESS.items():
        consts = {"regs_per_thread": k["regs"], "shared_words_per_block": k["shared"]}
        truth = {"schema": "ratprog-kernel-v1", "name": name, "variables": VARS5, "constants": consts,
                 "noise_rel": 0.0, "metrics": {}}
        fitted = {"schema": "ratprog-models-v1", "variables": VARS5, "constants": consts,
                  "metrics": {}, "failures": {}}
        for metric in sorted(F.REQUIRED_METRICS):
            f = k[metric]
            nb = [max((m[i] for m in f["num"]), default=0) for i in range(5)]
            db = [max((m[i] for m in f["den"]), default=0) for i in range(5)]
            truth["metrics"][metric] = {"num_bounds": nb, "num_coeffs": poly(f["num"], nb),
                                        "den_bounds": db, "den_coeffs": poly(f["den"], db)}
            fitted["metrics"][metric] = {"num_bounds": NUM_B5, "num_coeffs": dense5(f["num"], NUM_B5, rng),
                                         "den_bounds": DEN_B5, "den_coeffs": dense5(f["den"], DEN_B5, rng),
                                         "report": {"synthetic": True}}
        for suffix, obj in (("kernel", truth), ("models", fitted)):
            with open(os.path.join(HERE, "..", "stress", f"{name}.{suffix}.json"), "w") as fh:
                json.dump(obj, fh, indent=1)
                fh.write("\n")
        F.load_kernel_spec(os.path.join(HERE, "..", "stress", f"{name}.kernel.json"))
        F.models_to_metric_spec(F.read_models(os.path.join(HERE, "..", "stress", f"{name}.models.json")))
        print("wrote stress", name)


def main():
    write_stress()
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
