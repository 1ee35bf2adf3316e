"""Python mirror of the reference's search API over librpgpu.so.

``search_optimal`` keeps the signature and result shape of
``pipe::search_optimal`` (pipeline.hpp:575-680) for the ``--models`` path
(a metric spec + profile + config space + one data tuple); ``Plan`` exposes
the batched form (``search_optimal_batch``) that sweeps many data tuples per
launch.  Every number comes from the CUDA kernels; the only host work is
argument packing and, for the single-tuple drop-in, ordering the device's
per-config rows into the reference's ranking.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi as A
from . import formats as F
from . import program as P


class NoFeasibleConfig(RuntimeError):
    """pipe::NoFeasibleConfig (pipeline.hpp:51)."""


@dataclass
class SearchOptions:
    """pipe::SearchOptions (pipeline.hpp:438-452) plus the arithmetic mode."""
    regs_per_thread: float = 0.0
    shared_words_per_block: float = 0.0
    rep_mode: str = "real"          # real | ceil
    tie_rel_tol: float = 1e-12
    arith: str = "exact"            # exact | fast | fastcm (searches only)
    kernel: str = "specialized"     # specialized (per-model NVRTC kernel) | generic
    device: int = 0

    def struct(self) -> A.rpg_options:
        if self.rep_mode not in ("real", "ceil"):
            raise ValueError("rep_mode must be real or ceil")
        if self.arith not in ("exact", "fast", "fastcm"):
            raise ValueError("arith must be exact, fast or fastcm")
        if self.kernel not in ("specialized", "generic"):
            raise ValueError("kernel must be specialized or generic")
        return A.options_struct(
            A.RPG_REP_CEIL if self.rep_mode == "ceil" else A.RPG_REP_REAL,
            {"exact": A.RPG_ARITH_EXACT, "fast": A.RPG_ARITH_FAST, "fastcm": A.RPG_ARITH_FAST_CM}[self.arith],
            self.tie_rel_tol, self.regs_per_thread, self.shared_words_per_block,
            A.RPG_KERNEL_GENERIC if self.kernel == "generic" else A.RPG_KERNEL_SPECIALIZED)


@dataclass
class SearchRow:
    config: Tuple[int, int, int]
    estimated_cycles: float
    occupancy: float
    case_tag: str


@dataclass
class SearchResult:
    ranking: List[SearchRow] = field(default_factory=list)
    ties: int = 1
    evaluated: int = 0
    infeasible: int = 0

    def best(self) -> SearchRow:
        return self.ranking[0]


def _raise(code: int, err) -> None:
    msg = err.value.decode(errors="replace")
    if code == A.RPG_E_INVALID:
        raise ValueError(msg)
    if code in (A.RPG_E_MODEL,):
        raise F.ModelError(msg)
    if code == A.RPG_E_PROFILE:
        raise F.ProfileError(msg)
    if code == A.RPG_E_PIPELINE:
        raise F.PipelineError(msg)
    if code == A.RPG_E_NO_FEASIBLE:
        raise NoFeasibleConfig(msg)
    if code == A.RPG_E_EVAL:
        raise P.EvalError(msg)
    raise A.RpgError(code, msg)


class Plan:
    """A rational program plus profile and configuration space resident on
    one GPU.  ``source`` is a metric spec (the ``--models`` path: the
    emitted MWP-CWP program, pipeline.hpp:251-255) or a bare program
    (``program.Program`` / ``.rp`` text, the ``--rp`` path)."""

    def __init__(self, source, hw: F.DeviceProfile,
                 space: Sequence[Tuple[int, int, int]],
                 opts: Optional[SearchOptions] = None, step_limit: int = 1_000_000):
        self.lib = A.load_library()
        self.opts = opts or SearchOptions()
        self.hw = hw
        self.hw_struct = A.profile_struct(hw)
        self.space = A.config_array(list(space))
        self.n_space = len(self.space)
        self._handle = C.c_void_p()
        self.lowered: Optional[P.LoweredProgram] = None
        err = C.create_string_buffer(512)
        opts_s = self.opts.struct()
        space_p = A.ptr(self.space, A.rpg_config) if self.n_space else None
        if isinstance(source, (str, P.Program)):
            prog = P.parse(source) if isinstance(source, str) else source
            if self.n_space == 0:
                raise ValueError("search_optimal: configuration space is empty")
            self.spec = None
            self.lowered = P.LoweredProgram(prog, hw, step_limit)
            self.d = self.lowered.max_data_index() + 1
            rc = self.lib.rpg_program_plan_create(
                C.cast(C.pointer(self.lowered.struct), C.c_void_p), C.byref(self.hw_struct),
                space_p, self.n_space, C.byref(opts_s), self.opts.device,
                C.byref(self._handle), err, len(err))
        else:
            self.spec = source
            self.packed = A.PackedModel(source)
            self.d = F.data_param_count(source)
            rc = self.lib.rpg_plan_create(
                C.byref(self.packed.struct), C.byref(self.hw_struct), space_p,
                self.n_space, C.byref(opts_s), self.opts.device,
                C.byref(self._handle), err, len(err))
        if rc != A.RPG_OK:
            _raise(rc, err)

    def _check(self, rc: int, err, n_data: Optional[int] = None) -> None:
        if rc == A.RPG_OK:
            return
        if self.lowered is not None:
            if rc == A.RPG_E_EVAL:
                self.lowered.raise_eval_error(err.value.decode(errors="replace"))
            if rc == A.RPG_E_PIPELINE and n_data is not None:
                self.lowered.check_binding(n_data)
        _raise(rc, err)

    def poll_error(self, stream_ptr: int = 0) -> None:
        """Raises the first evaluation error of earlier _device calls on a
        bare-program plan (rpg_plan_poll_error)."""
        err = C.create_string_buffer(512)
        self._check(self.lib.rpg_plan_poll_error(self._handle, C.c_void_p(stream_ptr),
                                                 err, len(err)), err)

    def cert_counts(self) -> dict:
        """FAST_CM range certificate (rpg_plan_cert_counts): for each binade k
        of N ([2^k, 2^(k+1)]), how many configurations run pass 1 without
        per-point range checks ("free") and with the MWP-CWP case proven
        ("cwp", "mwp", "both").  All zero without a certificate."""
        out = (C.c_int64 * 256)()
        err = C.create_string_buffer(512)
        self._check(self.lib.rpg_plan_cert_counts(self._handle, out, err, len(err)), err)
        v = list(out)
        return {name: v[64 * m:64 * (m + 1)] for m, name in enumerate(("free", "cwp", "mwp", "both"))}

    def close(self) -> None:
        if self._handle:
            self.lib.rpg_plan_destroy(self._handle)
            self._handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _data(self, data) -> np.ndarray:
        a = np.ascontiguousarray(data, dtype=np.int64)
        if a.ndim == 1:
            a = a.reshape(-1, 1) if self.d <= 1 else a.reshape(1, -1)
        return a

    def search_batch(self, data, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Winners (structured array, abi.WINNER_DTYPE) for every data tuple
        (rows of ``data``); host buffers in and out.  ``out``: an optional
        preallocated C-contiguous WINNER_DTYPE array of n records to fill
        (e.g. in pinned memory) — returned."""
        a = self._data(data)
        n, d = a.shape
        if out is None:
            out = np.zeros(n, dtype=A.WINNER_DTYPE)
        elif out.dtype != A.WINNER_DTYPE or out.shape != (n,) or not out.flags.c_contiguous:
            raise ValueError("search_batch: out must be a C-contiguous WINNER_DTYPE array of n records")
        err = C.create_string_buffer(512)
        if self.lowered is not None:
            self.lowered.check_binding(d)
        rc = self.lib.rpg_search_batch(self._handle, A.ptr(a, C.c_int64), n, d,
                                       out.ctypes.data_as(C.c_void_p), err, len(err))
        self._check(rc, err, d)
        return out

    def search_batch_subsets(self, data, offsets, cfg_list) -> np.ndarray:
        """Winners when tuple t searches only the space indices
        cfg_list[offsets[t]:offsets[t+1]] (rpg_search_batch_subsets)."""
        a = self._data(data)
        n, d = a.shape
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        lst = np.ascontiguousarray(cfg_list, dtype=np.int32)
        if len(off) != n + 1:
            raise ValueError("search_batch_subsets: need n_tuples + 1 offsets")
        out = np.zeros(n, dtype=A.WINNER_DTYPE)
        err = C.create_string_buffer(512)
        if self.lowered is not None:
            self.lowered.check_binding(d)
        rc = self.lib.rpg_search_batch_subsets(
            self._handle, A.ptr(a, C.c_int64), n, d, A.ptr(off, C.c_int64),
            A.ptr(lst, C.c_int32) if len(lst) else None, out.ctypes.data_as(C.c_void_p),
            err, len(err))
        self._check(rc, err, d)
        return out

    def search_batch_device(self, d_data_ptr: int, n: int, d: int,
                            d_out_ptr: int, stream_ptr: int) -> None:
        """Device-resident variant (raw device pointers, cudaStream_t)."""
        err = C.create_string_buffer(512)
        rc = self.lib.rpg_search_batch_device(self._handle, C.c_void_p(d_data_ptr), n, d,
                                              C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr),
                                              err, len(err))
        self._check(rc, err, d)

    def evaluate(self, data):
        """Per-point table: (Ec, case tag, occupancy warps), tuple-major."""
        a = self._data(data)
        n, d = a.shape
        ec = np.zeros((n, self.n_space), dtype=np.float64)
        tag = np.zeros((n, self.n_space), dtype=np.uint8)
        wocc = np.zeros((n, self.n_space), dtype=np.int32)
        err = C.create_string_buffer(512)
        if self.lowered is not None:
            self.lowered.check_binding(d)
        rc = self.lib.rpg_evaluate(self._handle, A.ptr(a, C.c_int64), n, d,
                                   ec.ctypes.data_as(C.c_void_p), tag.ctypes.data_as(C.c_void_p),
                                   wocc.ctypes.data_as(C.c_void_p), err, len(err))
        self._check(rc, err, d)
        return ec, tag, wocc

    def evaluate_device(self, d_data_ptr: int, n: int, d: int, d_ec: int,
                        d_tag: int, d_wocc: int, stream_ptr: int) -> None:
        err = C.create_string_buffer(512)
        rc = self.lib.rpg_evaluate_device(self._handle, C.c_void_p(d_data_ptr), n, d,
                                          C.c_void_p(d_ec), C.c_void_p(d_tag),
                                          C.c_void_p(d_wocc), C.c_void_p(stream_ptr),
                                          err, len(err))
        self._check(rc, err, d)

    def config(self, idx: int) -> Tuple[int, int, int]:
        r = self.space[idx]
        return int(r["bx"]), int(r["by"]), int(r["bz"])


class PlanGroup:
    """One metric spec + profile + space resident on several GPUs of this
    process (rpg_plan_group_*; a device may repeat).  search_batch shards
    the tuples across the devices (or, with fewer tuples than devices, the
    configuration space with the two-phase reduction); the winners are
    byte-identical to Plan.search_batch on one device."""

    def __init__(self, spec: F.MetricSpec, hw: F.DeviceProfile,
                 space: Sequence[Tuple[int, int, int]], devices: Sequence[int],
                 opts: Optional[SearchOptions] = None):
        self.lib = A.load_library()
        self.opts = opts or SearchOptions()
        self.spec = spec
        self.packed = A.PackedModel(spec)
        self.hw_struct = A.profile_struct(hw)
        self.space = A.config_array(list(space))
        self.d = F.data_param_count(spec)
        dev = np.ascontiguousarray(list(devices), dtype=np.int32)
        self._handle = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = self.lib.rpg_plan_group_create(
            C.byref(self.packed.struct), C.byref(self.hw_struct),
            A.ptr(self.space, A.rpg_config) if len(self.space) else None, len(self.space),
            C.byref(self.opts.struct()), A.ptr(dev, C.c_int32), len(dev), C.byref(self._handle),
            err, len(err))
        if rc != A.RPG_OK:
            _raise(rc, err)

    @property
    def size(self) -> int:
        return int(self.lib.rpg_plan_group_size(self._handle))

    def search_batch(self, data) -> np.ndarray:
        a = np.ascontiguousarray(data, dtype=np.int64)
        if a.ndim == 1:
            a = a.reshape(-1, 1) if self.d <= 1 else a.reshape(1, -1)
        n, d = a.shape
        out = np.zeros(n, dtype=A.WINNER_DTYPE)
        err = C.create_string_buffer(512)
        rc = self.lib.rpg_search_batch_group(self._handle, A.ptr(a, C.c_int64), n, d,
                                             out.ctypes.data_as(C.c_void_p), err, len(err))
        if rc != A.RPG_OK:
            _raise(rc, err)
        return out

    def close(self) -> None:
        if self._handle:
            self.lib.rpg_plan_group_destroy(self._handle)
            self._handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def ranking_from_table(space: np.ndarray, ec: np.ndarray, tag: np.ndarray,
                       wocc: np.ndarray, W_max: int, tie_rel_tol: float) -> SearchResult:
    """Orders one tuple's device rows exactly as search_optimal does
    (pipeline.hpp:616-679): feasible = Ec >= 0; sort by (Ec, lex); tie group
    Ec <= best + best*tol; stable sort of the tie group by occupancy desc."""
    n = len(space)
    feas = [i for i in range(n) if ec[i] >= 0.0]
    res = SearchResult(evaluated=n, infeasible=n - len(feas))
    if not feas:
        raise NoFeasibleConfig(
            "no configuration in the search space can launch on this device")
    key = lambda i: (ec[i], int(space[i]["bx"]), int(space[i]["by"]), int(space[i]["bz"]), i)
    feas.sort(key=key)
    best = ec[feas[0]]
    bound = best + best * tie_rel_tol
    ties = 0
    while ties < len(feas) and ec[feas[ties]] <= bound:
        ties += 1
    head = sorted(feas[:ties], key=lambda i: -int(wocc[i]))  # stable
    order = head + feas[ties:]
    res.ties = ties
    for i in order:
        res.ranking.append(SearchRow(
            (int(space[i]["bx"]), int(space[i]["by"]), int(space[i]["bz"])),
            float(ec[i]), int(wocc[i]) / W_max, A.CASE_NAMES[int(tag[i])]))
    return res


def search_optimal(source, data_params: Sequence[int],
                   hw: F.DeviceProfile, space: Sequence[Tuple[int, int, int]],
                   opts: Optional[SearchOptions] = None,
                   step_limit: int = 1_000_000) -> SearchResult:
    """pipe::search_optimal (pipeline.hpp:575-680) for one data tuple;
    ``source`` is a metric spec or a bare program (``program.Program`` or
    ``.rp`` text)."""
    if len(space) == 0:
        raise ValueError("search_optimal: configuration space is empty")
    opts = opts or SearchOptions()
    with Plan(source, hw, space, opts, step_limit=step_limit) as plan:
        data = np.asarray([list(data_params)], dtype=np.int64).reshape(1, len(data_params))
        ec, tag, wocc = plan.evaluate(data)
        return ranking_from_table(plan.space, ec[0], tag[0], wocc[0], hw.W_max,
                                  opts.tie_rel_tol)


def search_optimal_batch(source, data: Sequence[Sequence[int]],
                         hw: F.DeviceProfile, space: Sequence[Tuple[int, int, int]],
                         opts: Optional[SearchOptions] = None) -> np.ndarray:
    """Batched search: one winner record per data tuple."""
    with Plan(source, hw, space, opts) as plan:
        return plan.search_batch(data)
