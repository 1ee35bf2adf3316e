"""Paper-artifact interop: fitted metrics as AltArr-form polynomials.

KLARAPTOR (arXiv 1906.00142) ships every low-level metric as a rational
function whose numerator and denominator are BPAS ``AltArr_t`` sparse
polynomials; the reference ``ratprog`` replaces that
encoding with dense graded-lex coefficient vectors (SPEC.md:14,
pipeline.hpp:996-1069).  This module converts between the two through the
C ABI (``rpg_aa_*`` in include/rpg.h, host code in csrc/rpg_altarr.cu), so a
KLARAPTOR-produced model plugs into the B200 evaluator unchanged:

* ``to_altarr`` / ``from_altarr``: one polynomial <-> an AltArr (decreasing
  packed-degree order, variable 0 most significant);
* ``ratfunc_from_altarr``: a metric's (num, den) AltArr pair -> the
  reference's ``RationalFunction`` with terms in graded-lex basis order (the
  reference's summation order, so the imported model evaluates
  bit-identically to the same model read from JSON);
* ``emit_metric_header``: the paper's per-metric C header.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import abi as A
from . import formats as F


class AltArr:
    """Owns an ``rpg_altarr`` and its element buffer."""

    def __init__(self, nvar: int, alloc: int):
        self.elems = (A.rpg_aa_elem * max(alloc, 1))()
        self.struct = A.rpg_altarr(0, max(alloc, 1), nvar, 0, self.elems)

    @classmethod
    def from_terms(cls, nvar: int, terms: Sequence[Tuple[float, int]]) -> "AltArr":
        """Raw (coef, packed degrees) elements, as a KLARAPTOR header lists them."""
        a = cls(nvar, len(terms))
        for i, (c, d) in enumerate(terms):
            a.elems[i].coef = float(c)
            a.elems[i].degs = int(d)
        a.struct.size = len(terms)
        return a

    @property
    def terms(self) -> List[Tuple[float, int]]:
        return [(self.elems[i].coef, int(self.elems[i].degs)) for i in range(self.struct.size)]


def pack_degs(exps: Sequence[int]) -> int:
    e = (C.c_uint8 * len(exps))(*exps)
    return int(A.load_library().rpg_aa_pack_degs(e, len(exps)))


def unpack_degs(degs: int, nvar: int) -> Tuple[int, ...]:
    e = (C.c_uint8 * nvar)()
    A.load_library().rpg_aa_unpack_degs(degs, nvar, e)
    return tuple(e)


def _poly_struct(p: F.Polynomial, nv: int):
    coef = np.ascontiguousarray(p.coeffs, dtype=np.float64)
    exps = np.ascontiguousarray(p.basis, dtype=np.uint8).reshape(len(p.coeffs), nv)
    s = A.rpg_poly()
    s.n_terms = len(p.coeffs)
    s.coef = coef.ctypes.data_as(C.POINTER(C.c_double)) if len(coef) else None
    s.exps = exps.ctypes.data_as(C.POINTER(C.c_uint8)) if len(coef) else None
    return s, (coef, exps)


def to_altarr(p: F.Polynomial) -> AltArr:
    nv = len(p.variables)
    s, keep = _poly_struct(p, nv)
    a = AltArr(nv, len(p.coeffs))
    err = C.create_string_buffer(512)
    A.check(A.load_library().rpg_aa_from_poly(C.byref(s), nv, C.byref(a.struct), err, len(err)), err)
    return a


def from_altarr(a: AltArr, variables: Sequence[str]) -> F.Polynomial:
    nv = a.struct.nvar
    if len(variables) != nv:
        raise ValueError("variable count does not match the AltArr's nvar")
    cap = max(a.struct.size, 1)
    coef = np.zeros(cap, dtype=np.float64)
    exps = np.zeros(cap * nv, dtype=np.uint8)
    n = C.c_int32(0)
    err = C.create_string_buffer(512)
    A.check(A.load_library().rpg_aa_to_poly(C.byref(a.struct), A.ptr(coef, C.c_double),
                                            A.ptr(exps, C.c_uint8), cap, C.byref(n), err, len(err)),
            err)
    k = n.value
    return F.Polynomial(list(variables), [tuple(int(e) for e in exps[i * nv:(i + 1) * nv]) for i in range(k)],
                        [float(c) for c in coef[:k]])


def ratfunc_from_altarr(num: AltArr, den: AltArr, variables: Sequence[str]) -> F.RationalFunction:
    return F.RationalFunction(from_altarr(num, variables), from_altarr(den, variables))


def emit_metric_header(f: F.RationalFunction, name: str) -> str:
    nv = len(f.num.variables)
    sn, k1 = _poly_struct(f.num, nv)
    sd, k2 = _poly_struct(f.den, nv)
    names = (C.c_char_p * nv)(*[v.encode() for v in f.num.variables])
    err = C.create_string_buffer(512)
    lib = A.load_library()
    n = lib.rpg_emit_altarr_header(C.byref(sn), C.byref(sd), nv, names, name.encode(), None, 0, err, len(err))
    A.check(0 if n >= 0 else int(n), err)
    buf = C.create_string_buffer(int(n) + 1)
    lib.rpg_emit_altarr_header(C.byref(sn), C.byref(sd), nv, names, name.encode(), buf, len(buf), err, len(err))
    return buf.value.decode()
