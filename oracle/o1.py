"""ORACLE O1 loader — TEST INFRASTRUCTURE ONLY.

ctypes bindings to oracle/build/libo1.so (oracle/o1.c, a CPU restatement of
the reference's FP64 path; see o1.h).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import this module, and only as the
checker / baseline — never as the measured or shipped path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

from paper_1906_00142_b200 import abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libo1.so")


class o1_metrics(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "regs_per_thread", "shared_words_per_block", "comp_insts_per_thread",
        "mem_insts_per_thread", "uncoal_mem_insts_per_thread",
        "coal_mem_insts_per_thread", "synch_insts_per_block", "total_blocks")]


class o1_breakdown(C.Structure):
    _fields_ = [("b_active", C.c_int64), ("n_active_warps", C.c_int64),
                ("mem_cycles", C.c_double), ("comp_cycles", C.c_double),
                ("mwp", C.c_double), ("cwp", C.c_double), ("rep", C.c_double),
                ("case_tag", C.c_int32), ("cycles_pre_synch", C.c_double),
                ("synch_cost", C.c_double), ("total_cycles", C.c_double)]


class o1_point(C.Structure):
    _fields_ = [("ec", C.c_double), ("feasible", C.c_int32),
                ("b_active", C.c_int32), ("w_active", C.c_int32),
                ("w_occ", C.c_int32), ("tag", C.c_int32), ("reserved", C.c_int32)]


O1_OK, O1_ZERO_OCCUPANCY, O1_MODEL_ERROR, O1_DEN_NEAR_ZERO = 0, 1, 2, 3

_lib: Optional[C.CDLL] = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    L = C.CDLL(LIB)
    P = C.POINTER
    L.o1_eval_monomial.restype = C.c_double
    L.o1_eval_monomial.argtypes = [P(C.c_uint8), P(C.c_double), C.c_int32]
    L.o1_eval_poly.restype = C.c_double
    L.o1_eval_poly.argtypes = [P(A.rpg_poly), C.c_int32, P(C.c_double)]
    L.o1_eval_ratfunc.restype = C.c_int
    L.o1_eval_ratfunc.argtypes = [P(A.rpg_poly), P(A.rpg_poly), C.c_int32,
                                  P(C.c_double), P(C.c_double)]
    L.o1_active_blocks.restype = C.c_int64
    L.o1_active_blocks.argtypes = [P(A.rpg_profile), C.c_double, C.c_double, C.c_int64]
    L.o1_active_warps.restype = C.c_int64
    L.o1_active_warps.argtypes = [P(A.rpg_profile), C.c_int64, C.c_int64]
    L.o1_occupancy.restype = C.c_double
    L.o1_occupancy.argtypes = [P(A.rpg_profile), C.c_double, C.c_double, C.c_int64]
    L.o1_mwpcwp_cycles.restype = C.c_int
    L.o1_mwpcwp_cycles.argtypes = [P(A.rpg_profile), P(o1_metrics), P(A.rpg_config),
                                   C.c_int32, P(o1_breakdown)]
    L.o1_evaluate_metrics.restype = C.c_int
    L.o1_evaluate_metrics.argtypes = [P(A.rpg_model), P(C.c_double), P(o1_metrics)]
    L.o1_eval_point.restype = C.c_int
    L.o1_eval_point.argtypes = [P(A.rpg_model), P(A.rpg_profile), P(A.rpg_options),
                                P(C.c_int64), C.c_int32, P(A.rpg_config), P(o1_point)]
    L.o1_search_one.restype = C.c_int
    L.o1_search_one.argtypes = [P(A.rpg_model), P(A.rpg_profile), P(A.rpg_options),
                                P(A.rpg_config), C.c_int64, P(C.c_int64), C.c_int32,
                                P(A.rpg_winner), P(C.c_int32)]
    L.o1_search_batch.restype = C.c_int
    L.o1_search_batch.argtypes = [P(A.rpg_model), P(A.rpg_profile), P(A.rpg_options),
                                  P(A.rpg_config), C.c_int64, P(C.c_int64), C.c_int64,
                                  C.c_int32, C.c_int32, C.c_void_p]
    L.o1_evaluate_batch.restype = C.c_int
    L.o1_evaluate_batch.argtypes = [P(A.rpg_model), P(A.rpg_profile), P(A.rpg_options),
                                    P(A.rpg_config), C.c_int64, P(C.c_int64), C.c_int64,
                                    C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
    _lib = L
    return L


def metrics(comp, uncoal, coal, synch, blocks, R=0.0, Z=0.0) -> o1_metrics:
    m = o1_metrics()
    m.comp_insts_per_thread = comp
    m.uncoal_mem_insts_per_thread = uncoal
    m.coal_mem_insts_per_thread = coal
    m.mem_insts_per_thread = uncoal + coal
    m.synch_insts_per_block = synch
    m.total_blocks = blocks
    m.regs_per_thread = R
    m.shared_words_per_block = Z
    return m


def mwpcwp_cycles(hw: A.rpg_profile, m: o1_metrics, cfg, rep_mode=A.RPG_REP_REAL):
    out = o1_breakdown()
    c = A.rpg_config(*cfg)
    rc = lib().o1_mwpcwp_cycles(C.byref(hw), C.byref(m), C.byref(c), rep_mode, C.byref(out))
    return rc, out


def search_batch(packed: A.PackedModel, hw: A.rpg_profile, opts: A.rpg_options,
                 space: np.ndarray, data: np.ndarray, n_threads: int) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.int64)
    n, d = data.shape
    out = np.zeros(n, dtype=A.WINNER_DTYPE)
    lib().o1_search_batch(C.byref(packed.struct), C.byref(hw), C.byref(opts),
                          A.ptr(space, A.rpg_config), len(space),
                          A.ptr(data, C.c_int64), n, d, n_threads,
                          out.ctypes.data_as(C.c_void_p))
    return out


def search_one(packed, hw, opts, space, data_params):
    data = np.ascontiguousarray(data_params, dtype=np.int64).reshape(-1)
    w = A.rpg_winner()
    order = np.full(len(space), -1, dtype=np.int32)
    lib().o1_search_one(C.byref(packed.struct), C.byref(hw), C.byref(opts),
                        A.ptr(space, A.rpg_config), len(space),
                        A.ptr(data, C.c_int64), len(data), C.byref(w),
                        A.ptr(order, C.c_int32))
    return w, order[: w.n_feasible]


def evaluate_batch(packed, hw, opts, space, data, n_threads=1):
    data = np.ascontiguousarray(data, dtype=np.int64)
    n, d = data.shape
    ec = np.zeros(n * len(space), dtype=np.float64)
    tag = np.zeros(n * len(space), dtype=np.uint8)
    wocc = np.zeros(n * len(space), dtype=np.int32)
    lib().o1_evaluate_batch(C.byref(packed.struct), C.byref(hw), C.byref(opts),
                            A.ptr(space, A.rpg_config), len(space),
                            A.ptr(data, C.c_int64), n, d, n_threads,
                            ec.ctypes.data_as(C.c_void_p), tag.ctypes.data_as(C.c_void_p),
                            wocc.ctypes.data_as(C.c_void_p))
    return ec.reshape(n, len(space)), tag.reshape(n, len(space)), wocc.reshape(n, len(space))


def eval_point(packed, hw, opts, data_params, cfg) -> o1_point:
    data = np.ascontiguousarray(data_params, dtype=np.int64).reshape(-1)
    p = o1_point()
    c = A.rpg_config(*cfg)
    lib().o1_eval_point(C.byref(packed.struct), C.byref(hw), C.byref(opts),
                        A.ptr(data, C.c_int64) if len(data) else None, len(data),
                        C.byref(c), C.byref(p))
    return p
