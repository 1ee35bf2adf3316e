"""ctypes mirror of include/rpg.h and the loader for librpgpu.so.

The library is the product: a missing or unloadable ``librpgpu.so`` raises
``RuntimeError`` — there is no CPU fallback anywhere on this path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import formats as F

HERE = os.path.dirname(os.path.abspath(__file__))
# RPG_LIBRARY: another build of librpgpu.so (A/B measurements of build variants)
LIB_PATH = os.environ.get("RPG_LIBRARY") or os.path.join(HERE, "librpgpu.so")

RPG_MAX_VARS = 8
RPG_N_METRICS = 7
RPG_VAR_BX, RPG_VAR_BY, RPG_VAR_BZ = -1, -2, -3
RPG_CASE_BOTH_SATURATED, RPG_CASE_CWP_BOUND, RPG_CASE_MWP_BOUND, RPG_CASE_UNKNOWN = 0, 1, 2, 3
CASE_NAMES = {0: "both_saturated", 1: "cwp_bound", 2: "mwp_bound", 3: "-"}
RPG_REP_REAL, RPG_REP_CEIL = 0, 1
RPG_ARITH_EXACT, RPG_ARITH_FAST, RPG_ARITH_FAST_CM = 0, 1, 2
RPG_KERNEL_SPECIALIZED, RPG_KERNEL_GENERIC = 0, 1

RPG_OK = 0
RPG_E_INVALID = -1
RPG_E_MODEL = -2
RPG_E_PROFILE = -3
RPG_E_CUDA = -4
RPG_E_NO_FEASIBLE = -5
RPG_E_PIPELINE = -6
RPG_E_FIT = -7
RPG_E_EVAL = -8
RPG_E_CSV = -9


class rpg_profile(C.Structure):
    _fields_ = [(k, C.c_int64 if k in F._COUNT_KEYS else C.c_double)
                for k in F.PROFILE_KEYS]


class rpg_poly(C.Structure):
    _fields_ = [("n_terms", C.c_int32), ("reserved", C.c_int32),
                ("coef", C.POINTER(C.c_double)), ("exps", C.POINTER(C.c_uint8))]


class rpg_metric(C.Structure):
    _fields_ = [("is_const", C.c_int32), ("reserved", C.c_int32),
                ("value", C.c_double), ("num", rpg_poly), ("den", rpg_poly)]


class rpg_model(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("var_kind", C.c_int32 * RPG_MAX_VARS),
                ("metric", rpg_metric * RPG_N_METRICS)]


class rpg_config(C.Structure):
    _fields_ = [("bx", C.c_int64), ("by", C.c_int64), ("bz", C.c_int64)]


RPG_FIT_TRACE_STAGES = 5
RPG_FIT_MAX_COLS = 64
FIT_STOP_NAMES = {-1: "no_safeguard", 0: "rounds", 1: "qmin", 2: "empty", 3: "first_empty"}


class rpg_fit_trace(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stop_reason", C.c_int32),
                ("stage_coef", (C.c_double * RPG_FIT_MAX_COLS) * RPG_FIT_TRACE_STAGES),
                ("round_qmin", C.c_double * RPG_FIT_TRACE_STAGES)]


class rpg_fit_job(C.Structure):
    _fields_ = [("y", C.POINTER(C.c_double)), ("num_bounds", C.POINTER(C.c_int32)),
                ("den_bounds", C.POINTER(C.c_int32)), ("coef_out", C.POINTER(C.c_double)),
                ("sigma_out", C.POINTER(C.c_double)), ("rank_out", C.POINTER(C.c_int32)),
                ("truncated_out", C.POINTER(C.c_int32)), ("residual_out", C.POINTER(C.c_double)),
                ("safeguard_out", C.POINTER(C.c_int32)), ("trace", C.POINTER(rpg_fit_trace)),
                ("status", C.c_int32), ("message", C.c_char * 252)]


# perf::MwpCwpBreakdown (perfmodel.hpp:284-296) + call status (rpg.h).
BREAKDOWN_DTYPE = np.dtype([("b_active", "<i8"), ("n_active_warps", "<i8"),
                            ("mem_cycles", "<f8"), ("comp_cycles", "<f8"), ("mwp", "<f8"),
                            ("cwp", "<f8"), ("rep", "<f8"), ("case_tag", "<i4"),
                            ("status", "<i4"), ("cycles_pre_synch", "<f8"),
                            ("synch_cost", "<f8"), ("total_cycles", "<f8")])


class rpg_options(C.Structure):
    _fields_ = [("rep_mode", C.c_int32), ("arith", C.c_int32),
                ("tie_rel_tol", C.c_double), ("regs_per_thread", C.c_double),
                ("shared_words_per_block", C.c_double),
                ("kernel", C.c_int32), ("reserved", C.c_int32)]


class rpg_winner(C.Structure):
    _fields_ = [("ec", C.c_double), ("best_ec", C.c_double),
                ("cfg_idx", C.c_int32), ("ties", C.c_int32),
                ("n_feasible", C.c_int32), ("b_active", C.c_int32),
                ("w_active", C.c_int32), ("w_occ", C.c_int32),
                ("case_tag", C.c_int32), ("reserved", C.c_int32)]


WINNER_DTYPE = np.dtype([("ec", "<f8"), ("best_ec", "<f8"), ("cfg_idx", "<i4"),
                         ("ties", "<i4"), ("n_feasible", "<i4"),
                         ("b_active", "<i4"), ("w_active", "<i4"),
                         ("w_occ", "<i4"), ("case_tag", "<i4"),
                         ("reserved", "<i4")])
assert WINNER_DTYPE.itemsize == C.sizeof(rpg_winner) == 48
CONFIG_DTYPE = np.dtype([("bx", "<i8"), ("by", "<i8"), ("bz", "<i8")])


def profile_struct(hw: F.DeviceProfile) -> rpg_profile:
    s = rpg_profile()
    for k in F.PROFILE_KEYS:
        setattr(s, k, getattr(hw, k))
    return s


def options_struct(rep_mode: int = RPG_REP_REAL, arith: int = RPG_ARITH_EXACT,
                   tie_rel_tol: float = 1e-12, regs_per_thread: float = 0.0,
                   shared_words_per_block: float = 0.0,
                   kernel: int = RPG_KERNEL_SPECIALIZED) -> rpg_options:
    return rpg_options(rep_mode, arith, tie_rel_tol, regs_per_thread,
                       shared_words_per_block, kernel, 0)


def var_kind(name: str) -> int:
    if name == "bx":
        return RPG_VAR_BX
    if name == "by":
        return RPG_VAR_BY
    if name == "bz":
        return RPG_VAR_BZ
    return int(name[1:]) - 1  # D<k> -> k-1


class rpg_aa_elem(C.Structure):
    _fields_ = [("coef", C.c_double), ("degs", C.c_uint64)]


class rpg_altarr(C.Structure):
    _fields_ = [("size", C.c_int32), ("alloc", C.c_int32), ("nvar", C.c_int32),
                ("unpacked", C.c_int32), ("elems", C.POINTER(rpg_aa_elem))]


class PackedModel:
    """An rpg_model plus the numpy buffers its pointers reference.

    ``drop_zero_terms`` mirrors emit_ratfunc (perfmodel.hpp:521): exact-zero
    coefficients contribute nothing and are skipped."""

    def __init__(self, spec: F.MetricSpec, drop_zero_terms: bool = True):
        F.check_metric_spec(spec)
        nv = len(spec.variables)
        if nv > RPG_MAX_VARS:
            raise F.ModelError(f"at most {RPG_MAX_VARS} model variables are supported")
        self.spec = spec
        self.struct = rpg_model()
        self.struct.n_vars = nv
        for i, v in enumerate(spec.variables):
            self.struct.var_kind[i] = var_kind(v)
        self._keep: List[np.ndarray] = []
        for slot, name in enumerate(F.METRIC_SLOTS):
            m = self.struct.metric[slot]
            if name in spec.constants:  # constants take priority (perfmodel.hpp:463-465)
                m.is_const = 1
                m.value = float(spec.constants[name])
            else:
                f = spec.models[name]
                m.is_const = 0
                m.num = self._poly(f.num, nv, drop_zero_terms)
                m.den = self._poly(f.den, nv, drop_zero_terms)

    def _poly(self, p: F.Polynomial, nv: int, drop: bool) -> rpg_poly:
        keep = [k for k, c in enumerate(p.coeffs) if not (drop and c == 0.0)]
        coef = np.ascontiguousarray([p.coeffs[k] for k in keep], dtype=np.float64)
        exps = np.ascontiguousarray([p.basis[k] for k in keep],
                                    dtype=np.uint8).reshape(len(keep), nv)
        if any(e > 255 for k in keep for e in p.basis[k]):
            raise F.ModelError("exponents above 255 are not supported")
        self._keep += [coef, exps]
        out = rpg_poly()
        out.n_terms = len(keep)
        out.coef = coef.ctypes.data_as(C.POINTER(C.c_double)) if len(keep) else None
        out.exps = exps.ctypes.data_as(C.POINTER(C.c_uint8)) if len(keep) else None
        return out


def config_array(space: Sequence[Tuple[int, int, int]]) -> np.ndarray:
    arr = np.zeros(len(space), dtype=CONFIG_DTYPE)
    if len(space):
        a = np.asarray(space, dtype=np.int64).reshape(len(space), 3)
        arr["bx"], arr["by"], arr["bz"] = a[:, 0], a[:, 1], a[:, 2]
    return arr


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


_LIB: Optional[C.CDLL] = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads librpgpu.so.  Raises if it is absent: the product has no
    fallback evaluator."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA evaluator is required; there is no CPU fallback)")
    lib = C.CDLL(path)
    errbuf = (C.c_char_p, C.c_size_t)
    sig = {
        "rpg_version": (C.c_char_p, ()),
        "rpg_device_count": (C.c_int, ()),
        "rpg_plan_create": (C.c_int, (C.POINTER(rpg_model), C.POINTER(rpg_profile),
                                      C.POINTER(rpg_config), C.c_int64,
                                      C.POINTER(rpg_options), C.c_int32,
                                      C.POINTER(C.c_void_p)) + errbuf),
        "rpg_plan_destroy": (C.c_int, (C.c_void_p,)),
        "rpg_search_batch": (C.c_int, (C.c_void_p, C.POINTER(C.c_int64), C.c_int64,
                                       C.c_int32, C.c_void_p) + errbuf),
        "rpg_search_batch_device": (C.c_int, (C.c_void_p, C.c_void_p, C.c_int64,
                                              C.c_int32, C.c_void_p, C.c_void_p) + errbuf),
        "rpg_evaluate": (C.c_int, (C.c_void_p, C.POINTER(C.c_int64), C.c_int64,
                                   C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p) + errbuf),
        "rpg_evaluate_device": (C.c_int, (C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                          C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p) + errbuf),
        "rpg_emit_cuda_source": (C.c_int64, (C.POINTER(rpg_model), C.POINTER(rpg_profile),
                                             C.POINTER(rpg_options), C.c_int32, C.c_char_p,
                                             C.c_size_t, C.POINTER(C.c_int64)) + errbuf),
        "rpg_fit_rational": (C.c_int, (C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64,
                                       C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.c_double, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                       C.POINTER(C.c_int32)) + errbuf),
        "rpg_fit_rational_traced": (C.c_int, (C.POINTER(C.c_double), C.POINTER(C.c_double),
                                              C.c_int64, C.c_int32, C.POINTER(C.c_int32),
                                              C.POINTER(C.c_int32), C.c_double, C.c_int32,
                                              C.POINTER(C.c_double), C.POINTER(C.c_double),
                                              C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                              C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                              C.POINTER(rpg_fit_trace)) + errbuf),
        "rpg_fit_rational_multi": (C.c_int, (C.POINTER(C.c_double), C.c_int64, C.c_int32,
                                             C.POINTER(rpg_fit_job), C.c_int32, C.c_double,
                                             C.c_int32) + errbuf),
        "rpg_program_plan_create": (C.c_int, (C.c_void_p, C.POINTER(rpg_profile),
                                              C.POINTER(rpg_config), C.c_int64,
                                              C.POINTER(rpg_options), C.c_int32,
                                              C.POINTER(C.c_void_p)) + errbuf),
        "rpg_plan_poll_error": (C.c_int, (C.c_void_p, C.c_void_p) + errbuf),
        "rpg_plan_cert_counts": (C.c_int, (C.c_void_p, C.POINTER(C.c_int64)) + errbuf),
        "rpg_emit_program_cuda_source": (C.c_int64, (C.c_void_p, C.POINTER(rpg_profile),
                                                     C.POINTER(rpg_options), C.c_int32,
                                                     C.c_char_p, C.c_size_t,
                                                     C.POINTER(C.c_int64)) + errbuf),
        "rpg_search_batch_subsets": (C.c_int, (C.c_void_p, C.POINTER(C.c_int64), C.c_int64,
                                               C.c_int32, C.POINTER(C.c_int64),
                                               C.POINTER(C.c_int32), C.c_void_p) + errbuf),
        "rpg_search_batch_subsets_device": (C.c_int, (C.c_void_p, C.c_void_p, C.c_int64,
                                                      C.c_int32, C.c_void_p, C.c_void_p,
                                                      C.c_void_p, C.c_void_p) + errbuf),
        "rpg_mwpcwp_cycles_batch": (C.c_int, (C.POINTER(rpg_profile), C.POINTER(C.c_double),
                                              C.POINTER(rpg_config), C.c_int64, C.c_int32,
                                              C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p) + errbuf),
        "rpg_mwpcwp_breakdown_batch": (C.c_int, (C.POINTER(rpg_profile), C.POINTER(C.c_double),
                                                 C.POINTER(rpg_config), C.c_int64, C.c_int32,
                                                 C.c_int32, C.c_void_p) + errbuf),
        "rpg_eval_ratfunc_batch": (C.c_int, (C.POINTER(rpg_poly), C.POINTER(rpg_poly), C.c_int32,
                                             C.POINTER(C.c_double), C.c_int64, C.c_int32,
                                             C.POINTER(C.c_double), C.POINTER(C.c_int32)) + errbuf),
        "rpg_uniform_stream": (C.c_int, (C.c_uint64, C.c_int64, C.c_double, C.c_double,
                                         C.POINTER(C.c_double))),
        "rpg_aa_pack_degs": (C.c_uint64, (C.POINTER(C.c_uint8), C.c_int32)),
        "rpg_aa_unpack_degs": (None, (C.c_uint64, C.c_int32, C.POINTER(C.c_uint8))),
        "rpg_aa_from_poly": (C.c_int, (C.POINTER(rpg_poly), C.c_int32, C.POINTER(rpg_altarr)) + errbuf),
        "rpg_aa_to_poly": (C.c_int, (C.POINTER(rpg_altarr), C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                     C.c_int32, C.POINTER(C.c_int32)) + errbuf),
        "rpg_emit_altarr_header": (C.c_int64, (C.POINTER(rpg_poly), C.POINTER(rpg_poly), C.c_int32,
                                               C.POINTER(C.c_char_p), C.c_char_p, C.c_char_p,
                                               C.c_size_t) + errbuf),
        "rpg_plan_group_create": (C.c_int, (C.POINTER(rpg_model), C.POINTER(rpg_profile),
                                            C.POINTER(rpg_config), C.c_int64,
                                            C.POINTER(rpg_options), C.POINTER(C.c_int32), C.c_int32,
                                            C.POINTER(C.c_void_p)) + errbuf),
        "rpg_plan_group_destroy": (C.c_int, (C.c_void_p,)),
        "rpg_plan_group_size": (C.c_int32, (C.c_void_p,)),
        "rpg_search_batch_group": (C.c_int, (C.c_void_p, C.POINTER(C.c_int64), C.c_int64,
                                             C.c_int32, C.c_void_p) + errbuf),
        "rpg_samples_parse": (C.c_int, (C.c_char_p, C.c_size_t, C.c_int32,
                                        C.POINTER(C.c_void_p)) + errbuf),
        "rpg_samples_info": (C.c_int, (C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_double))),
        "rpg_samples_metric_name": (C.c_char_p, (C.c_void_p, C.c_int32)),
        "rpg_samples_copy": (C.c_int, (C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)),
        "rpg_samples_free": (None, (C.c_void_p,)),
        "rpg_samples_format": (C.c_int64, (C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                           C.POINTER(C.c_char_p), C.c_int32, C.c_int32, C.c_uint64,
                                           C.c_double, C.c_int32, C.c_char_p, C.c_size_t) + errbuf),
        "rpg_jit_stats": (None, (C.POINTER(C.c_int64), C.POINTER(C.c_int64))),
        "rpg_search": (C.c_int, (C.POINTER(rpg_model), C.POINTER(rpg_profile),
                                 C.POINTER(rpg_config), C.c_int64,
                                 C.POINTER(rpg_options), C.POINTER(C.c_int64),
                                 C.c_int64, C.c_int32, C.c_int32, C.c_void_p) + errbuf),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = list(args)
    _LIB = lib
    return lib


EXPORTED_SYMBOLS = ("rpg_version", "rpg_device_count", "rpg_plan_create",
                    "rpg_plan_destroy", "rpg_search_batch",
                    "rpg_search_batch_device", "rpg_evaluate",
                    "rpg_evaluate_device", "rpg_search", "rpg_emit_cuda_source",
                    "rpg_fit_rational", "rpg_program_plan_create",
                    "rpg_plan_poll_error", "rpg_emit_program_cuda_source",
                    "rpg_search_batch_subsets", "rpg_search_batch_subsets_device",
                    "rpg_mwpcwp_cycles_batch", "rpg_eval_ratfunc_batch", "rpg_uniform_stream",
                    "rpg_aa_pack_degs", "rpg_aa_unpack_degs", "rpg_aa_from_poly",
                    "rpg_aa_to_poly", "rpg_emit_altarr_header", "rpg_jit_stats",
                    "rpg_plan_group_create", "rpg_plan_group_destroy", "rpg_plan_group_size",
                    "rpg_search_batch_group", "rpg_fit_rational_traced", "rpg_fit_rational_multi",
                    "rpg_samples_parse", "rpg_samples_info", "rpg_samples_metric_name",
                    "rpg_samples_copy", "rpg_samples_free", "rpg_samples_format",
                    "rpg_mwpcwp_breakdown_batch", "rpg_plan_cert_counts")


class RpgError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def check(code: int, err) -> None:
    if code != RPG_OK:
        msg = err.value.decode(errors="replace") if err is not None else ""
        raise RpgError(code, msg)


def jit_stats() -> Tuple[int, int]:
    """(NVRTC compilations, on-disk cubin cache hits) of this process."""
    lib = load_library()
    c, h = C.c_int64(0), C.c_int64(0)
    lib.rpg_jit_stats(C.byref(c), C.byref(h))
    return c.value, h.value
