"""AltArr interop: the paper's per-metric polynomial
encoding <-> the reference's graded-lex rational functions,
through the C ABI (rpg_aa_*).  Host-only; the GPU test searches a model
imported from AltArr form and checks it against oracle O1 on the JSON
model."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import altarr as AA
from paper_1906_00142_b200 import formats as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gemm_spec():
    return F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "gemm.models.json")))


def _round_trip_spec(spec):
    out = F.MetricSpec(variables=list(spec.variables), models={}, constants=dict(spec.constants))
    for name, f in spec.models.items():
        out.models[name] = AA.ratfunc_from_altarr(AA.to_altarr(f.num), AA.to_altarr(f.den), spec.variables)
    return out


def test_pack_layout_variable0_most_significant():
    assert AA.pack_degs([1, 0, 0]) == 1 << 43          # w = 21 bits for 3 variables
    assert AA.pack_degs([0, 0, 1]) == 1 << 1
    assert AA.pack_degs([2, 1]) == (2 << 32) | (1 << 0)
    for nv in range(1, 9):
        rng = np.random.default_rng(nv)
        for _ in range(50):
            e = [int(x) for x in rng.integers(0, 256, size=nv)]
            assert AA.unpack_degs(AA.pack_degs(e), nv) == tuple(e)


def test_altarr_order_and_zero_drop():
    f = _gemm_spec().models[F.METRIC_COMP]
    a = AA.to_altarr(f.num)
    degs = [d for _, d in a.terms]
    assert degs == sorted(degs, reverse=True) and len(set(degs)) == len(degs)
    nonzero = [(m, c) for m, c in zip(f.num.basis, f.num.coeffs) if c != 0.0]
    assert a.struct.size == len(nonzero)
    back = AA.from_altarr(a, f.num.variables)
    assert list(zip(back.basis, back.coeffs)) == nonzero   # graded-lex basis order restored


def test_imported_model_evaluates_bit_identically():
    from oracle import o1
    spec = _gemm_spec()
    imp = _round_trip_spec(spec)
    hw = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "b200.profile")))
    space = A.config_array(F.integer_configs(1024, dims=2)[::13])
    data = np.array([[64], [1000], [4097], [65536]], dtype=np.int64)
    opts = A.options_struct()
    want = o1.evaluate_batch(A.PackedModel(spec), hw, opts, space, data, 4)
    got = o1.evaluate_batch(A.PackedModel(imp), hw, opts, space, data, 4)
    for w, g in zip(want, got):
        assert np.array_equal(w.view(np.uint8), g.view(np.uint8))


def test_rejects_non_canonical_altarr():
    a = AA.AltArr.from_terms(3, [(1.0, AA.pack_degs([0, 0, 1])), (2.0, AA.pack_degs([1, 0, 0]))])
    with pytest.raises(A.RpgError, match="decreasing degree order"):
        AA.from_altarr(a, ["D1", "bx", "by"])
    a = AA.AltArr.from_terms(3, [(1.0, AA.pack_degs([1, 0, 0])), (2.0, AA.pack_degs([1, 0, 0]))])
    with pytest.raises(A.RpgError, match="decreasing degree order"):
        AA.from_altarr(a, ["D1", "bx", "by"])
    a = AA.AltArr.from_terms(3, [(float("nan"), AA.pack_degs([1, 0, 0]))])
    with pytest.raises(A.RpgError, match="non-finite"):
        AA.from_altarr(a, ["D1", "bx", "by"])
    a = AA.AltArr.from_terms(3, [(1.0, 1 << 40)])          # exponent field wider than 8 bits
    with pytest.raises(A.RpgError, match="wider than 8 bits"):
        AA.from_altarr(a, ["D1", "bx", "by"])


def test_emitted_header_compiles_and_round_trips(tmp_path):
    f = _gemm_spec().models[F.METRIC_COAL]
    hdr = AA.emit_metric_header(f, "coal_mem_insts_per_thread")
    (tmp_path / "metric.h").write_text(hdr)
    main = tmp_path / "main.c"
    main.write_text('#include <stdio.h>\n#include "metric.h"\nint main(void){\n'
                    '  double c[64]; unsigned char e[192]; int n = 0;\n'
                    '  if (rpg_aa_to_poly(&coal_mem_insts_per_thread_num, c, e, 64, &n, 0, 0)) return 1;\n'
                    '  for (int k = 0; k < n; ++k) printf("%a %d %d %d\\n", c[k], e[3*k], e[3*k+1], e[3*k+2]);\n'
                    '  return 0;\n}\n')
    exe = tmp_path / "main"
    lib = os.path.join(ROOT, "paper_1906_00142_b200")
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-I", str(tmp_path),
                    str(main), "-o", str(exe), "-L", lib, "-lrpgpu", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = [(tuple(int(x) for x in l.split()[1:]), float.fromhex(l.split()[0])) for l in out if l]
    assert got == [(m, c) for m, c in zip(f.num.basis, f.num.coeffs) if c != 0.0]


@pytest.mark.gpu
def test_gpu_search_of_altarr_imported_model_matches_oracle():
    from oracle import o1
    from paper_1906_00142_b200 import search as S
    spec = _gemm_spec()
    imp = _round_trip_spec(spec)
    hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
    space = F.integer_configs(1024, dims=2)
    data = np.arange(64, 64 + 300 * 97, 97, dtype=np.int64).reshape(-1, 1)
    want = o1.search_batch(A.PackedModel(spec), A.profile_struct(hw), A.options_struct(arith=A.RPG_ARITH_EXACT),
                           A.config_array(space), data, 8)
    with S.Plan(imp, hw, space, S.SearchOptions(arith="exact")) as plan:
        got = plan.search_batch(data)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
