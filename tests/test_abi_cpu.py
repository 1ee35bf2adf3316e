"""CPU-side checks of the C ABI library and host logic (no GPU calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1906_00142_b200 import abi as A
from paper_1906_00142_b200 import formats as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rpg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|uint64_t|void|const char\*)\s+(rpg_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = A.load_library()
    names = declared_symbols()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert set(A.EXPORTED_SYMBOLS) <= set(names)
    assert b"sm_100a" in lib.rpg_version()


def test_struct_layouts_match_header():
    assert C.sizeof(A.rpg_profile) == 14 * 8
    assert C.sizeof(A.rpg_config) == 24
    assert C.sizeof(A.rpg_winner) == 48
    assert C.sizeof(A.rpg_poly) == 24
    assert C.sizeof(A.rpg_metric) == 16 + 2 * 24
    assert C.sizeof(A.rpg_options) == 40


def test_plan_create_rejects_bad_inputs_before_touching_the_device():
    lib = A.load_library()
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    pk = A.PackedModel(spec)
    hw = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "sample_device.profile")))
    opts = A.options_struct()
    err = C.create_string_buffer(256)
    h = C.c_void_p()
    rc = lib.rpg_plan_create(C.byref(pk.struct), C.byref(hw), None, 0, C.byref(opts), 0,
                             C.byref(h), err, 256)
    assert rc == A.RPG_E_INVALID and b"configuration space is empty" in err.value
    space = A.config_array(F.enumerate_configs())
    bad = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "sample_device.profile")))
    bad.T_max = 2048
    rc = lib.rpg_plan_create(C.byref(pk.struct), C.byref(bad), A.ptr(space, A.rpg_config),
                             len(space), C.byref(opts), 0, C.byref(h), err, 256)
    assert rc == A.RPG_E_PROFILE and b"1024" in err.value
    m = A.rpg_model()
    C.memmove(C.byref(m), C.byref(pk.struct), C.sizeof(m))
    m.var_kind[1] = 0  # bx -> D1: no bx variable any more
    rc = lib.rpg_plan_create(C.byref(m), C.byref(hw), A.ptr(space, A.rpg_config),
                             len(space), C.byref(opts), 0, C.byref(h), err, 256)
    assert rc == A.RPG_E_MODEL and b"bx and by" in err.value


def test_profile_parser_messages():
    good = F.format_profile(F.load_profile(os.path.join(ROOT, "data", "sample_device.profile")))
    assert F.parse_profile(good).W_max == 48
    assert F.parse_profile("# c\n\n" + good + "  \n# t\n").W_max == 48

    def drop(key):
        return "".join(l + "\n" for l in good.splitlines() if not l.startswith(key + " "))
    for text, frag in [(good + "bogus_key = 1\n", "unknown key"),
                       (good + "W_max = 48\n", "duplicate"),
                       (drop("num_SM"), "missing key 'num_SM'"),
                       (drop("B_max") + "B_max = -2\n", "positive"),
                       (drop("B_max") + "B_max = 2.5\n", "integer"),
                       (drop("W_max") + "W_max = 4x8\n", "bad numeric value"),
                       (drop("W_max") + "W_max 48\n", "expected 'key = value'"),
                       (drop("T_max") + "T_max = 2048\n", "1024")]:
        with pytest.raises(F.ProfileError, match=re.escape(frag)):
            F.parse_profile(text)


def test_monomial_basis_kats():
    # test_polyfit.cpp:34-55
    assert F.monomial_basis([2]) == [(0,), (1,), (2,)]
    assert F.monomial_basis([1, 1]) == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert len(F.monomial_basis([2, 1, 1])) == 12
    assert F.monomial_basis([]) == [()]
    assert F.monomial_basis([0, 0]) == [(0, 0)]
    with pytest.raises(ValueError):
        F.monomial_basis([-1])


def test_enumerate_configs_kats():
    # test_datakit.cpp:76-118
    g = F.enumerate_configs()
    assert len(g) == 51 and g == sorted(g)
    assert F.enumerate_configs(1024, 32, 1) == [(32 << i, 1, 1) for i in range(6)]
    assert F.enumerate_configs(32, 32, 2) == [(1, 32, 1), (2, 16, 1), (4, 8, 1), (8, 4, 1), (16, 2, 1), (32, 1, 1)]
    assert len(F.enumerate_configs(64, 64, 3)) == 28
    for bad in [(2048, 32, 2), (16, 32, 2), (1024, 0, 2), (1024, 32, 4)]:
        with pytest.raises(ValueError):
            F.enumerate_configs(*bad)
    assert len(F.integer_configs()) == 7262
    assert len(F.integer_configs(dims=3)) == 30343


def test_metric_spec_validation():
    # test_perfmodel.cpp:603-626
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    missing = F.MetricSpec(spec.variables, dict(spec.models), dict(spec.constants))
    del missing.models[F.METRIC_SYNCH]
    with pytest.raises(F.ModelError):
        F.check_metric_spec(missing)
    no_regs = F.MetricSpec(spec.variables, dict(spec.models), {F.METRIC_SHARED: 0.0})
    with pytest.raises(F.ModelError):
        F.check_metric_spec(no_regs)
    bad_vars = F.MetricSpec(["D1", "bx"], dict(spec.models), dict(spec.constants))
    with pytest.raises(F.ModelError):
        F.check_metric_spec(bad_vars)
    collide = F.MetricSpec(["W_max", "bx", "by"], {}, {k: 1.0 for k in F.METRIC_SLOTS})
    with pytest.raises(F.ModelError):
        F.check_metric_spec(collide)


def test_models_json_roundtrip():
    spec = F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json"))
    ms = F.MetricModelSet(spec.variables, dict(spec.ground_truth), {},
                          {F.METRIC_REGS: 20.0, F.METRIC_SHARED: 0.0}, {"phantom": "degenerate fit"})
    text = F.format_models(ms)
    back = F.parse_models(text)
    assert F.format_models(back) == text
    with pytest.raises(F.PipelineError, match="not valid JSON"):
        F.parse_models("{ not json")
    with pytest.raises(F.PipelineError, match="ratprog-models-v1"):
        F.parse_models('{"schema":"other-v9"}')
    with pytest.raises(F.PipelineError, match="metrics"):
        F.parse_models('{"schema":"ratprog-models-v1","variables":["D1","bx","by"]}')


@pytest.mark.parametrize("arith", [A.RPG_ARITH_EXACT, A.RPG_ARITH_FAST])
def test_specialized_kernel_source_compiles_for_sm100a(arith):
    """The per-model kernel source (rpg_emit_cuda_source) compiles with NVRTC
    for sm_100a on the CPU-only host (no device needed)."""
    lib = A.load_library()
    spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", "2dconv.models.json")))
    pk = A.PackedModel(spec)
    hw = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "b200.profile")))
    opts = A.options_struct(arith=arith)
    buf = C.create_string_buffer(1 << 20)
    err = C.create_string_buffer(4096)
    cubin = C.c_int64(0)
    n = lib.rpg_emit_cuda_source(C.byref(pk.struct), C.byref(hw), C.byref(opts), 1, buf, len(buf),
                                 C.byref(cubin), err, len(err))
    assert n > 0, err.value
    src = buf.value.decode()
    assert "rpg_jit_search" in src and "rpg_jit_evaluate" in src
    assert ("fma(" in src) == (arith == A.RPG_ARITH_FAST)
    assert cubin.value > 10000


@pytest.mark.parametrize("tol", [-1e-12, float("nan"), float("inf")])
def test_plan_create_rejects_bad_tie_tolerance(tol):
    lib = A.load_library()
    spec = F.kernel_to_metric_spec(F.load_kernel_spec(os.path.join(ROOT, "data", "stencil2d.kernel.json")))
    pk = A.PackedModel(spec)
    hw = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "sample_device.profile")))
    space = A.config_array(F.enumerate_configs())
    err = C.create_string_buffer(256)
    h = C.c_void_p()
    rc = lib.rpg_plan_create(C.byref(pk.struct), C.byref(hw), A.ptr(space, A.rpg_config), len(space),
                             C.byref(A.options_struct(tie_rel_tol=tol)), 0, C.byref(h), err, 256)
    assert rc == A.RPG_E_INVALID and b"tie_rel_tol" in err.value


def test_profile_values_follow_stod():
    """parse_profile's numeric values follow std::stod with a full-consumption
    check (perfmodel.hpp:139-147): hex floats accepted, underscores and
    out-of-range literals rejected, a non-finite count is a ProfileError."""
    from paper_1906_00142_b200 import formats as F
    assert F._stod("0x1.8p3") == 12.0 and F._stod("0X.8") == 0.5 and F._stod("5.") == 5.0
    for bad in ("1_000", "1e", "0x", " 1", "1e400", "1e-400", "0x1p-1080", "1.2.3"):
        with pytest.raises(ValueError):
            F._stod(bad)
    base = open(os.path.join(ROOT, "data", "sample_device.profile")).read()
    hexed = base.replace("W_max = 48", "W_max = 0x30")
    assert F.parse_profile(hexed).W_max == 48
    with pytest.raises(F.ProfileError, match="bad numeric value '4_8'"):
        F.parse_profile(base.replace("W_max = 48", "W_max = 4_8"))
    with pytest.raises(F.ProfileError, match="'W_max' must be an integer"):
        F.parse_profile(base.replace("W_max = 48", "W_max = inf"))
