"""Host mirror of gblite's GraphBLAS operation layer (core.hpp:15-140,
ops.hpp) over libgbx's device implementation (csrc/ops.cu).

    A = ops.Matrix.from_csr(nrows, ncols, row_ptr, col, vals, Domain.Fp64)
    w = ops.mxv(w_prior, ops.Descriptor(mask=m, replace=True), Semiring.PlusTimes,
                Domain.Fp64, A, u)
    C = ops.mxm(C_prior, ops.Descriptor(mask=L, structural=True), Semiring.PlusPair,
                Domain.Uint64, L, U, )

Matrices live in HBM (gbx_mat handles); vectors are host `Vector`s (n, sorted
idx, vals, domain).  Results follow the reference bit for bit: the semirings of
ops.cpp:362-372, the operators of ops.cpp:52-203 and the mask / accumulator /
replace post-step of core.cpp:131-204.  Errors raise `Error` with gblite's
ErrCode.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import Optional

import numpy as np

from .graph import Domain, Graph, _ptr, call

_NPD = {Domain.Bool: np.uint8, Domain.Int64: np.int64, Domain.Uint64: np.uint64,
        Domain.Fp64: np.float64}


class Semiring(IntEnum):
    """ops.cpp:362-372 (the operand / result domain is a separate argument)."""
    PlusTimes = 0
    AnySecondi = 1
    MinPlus = 2
    PlusFirst = 3
    PlusSecond = 4
    PlusPair = 5
    MinSecond = 6


class Op(IntEnum):
    """Binary operators usable as the accumulator (ops.cpp:52-203)."""
    NoOp = 0
    Plus = 1
    Minus = 2
    Times = 3
    Div = 4
    Min = 5
    Max = 6
    First = 7
    Second = 8
    Pair = 9
    Any = 10
    Lor = 11
    Land = 12


class _Vec(C.Structure):
    _fields_ = [("n", C.c_int64), ("nvals", C.c_int64), ("idx", C.c_void_p),
                ("vals", C.c_void_p), ("domain", C.c_int)]


class _Desc(C.Structure):
    _fields_ = [("mask_vec", C.c_void_p), ("mask_mat", C.c_void_p), ("complement", C.c_int),
                ("structural", C.c_int), ("replace", C.c_int), ("accum", C.c_int),
                ("accum_domain", C.c_int), ("transpose_in1", C.c_int),
                ("transpose_in2", C.c_int)]


@dataclass
class Vector:
    """gblite::SparseVector: length n, ascending idx, vals in `domain`."""
    n: int
    idx: np.ndarray
    vals: np.ndarray
    domain: Domain

    @staticmethod
    def empty(n, domain):
        return Vector(n, np.zeros(0, np.int64), np.zeros(0, _NPD[Domain(domain)]), Domain(domain))

    def _c(self):
        self._idx = np.ascontiguousarray(self.idx, np.int64)
        self._vals = np.ascontiguousarray(self.vals, _NPD[Domain(self.domain)])
        return _Vec(self.n, len(self._idx), self._idx.ctypes.data if len(self._idx) else None,
                    self._vals.ctypes.data if len(self._vals) else None, int(self.domain))


class Matrix:
    """gblite::SparseMatrix resident in HBM (gbx_mat)."""

    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def from_csr(nrows, ncols, row_ptr, col, vals, domain) -> "Matrix":
        rp = np.ascontiguousarray(row_ptr, np.int64)
        c = np.ascontiguousarray(col, np.int64)
        v = np.ascontiguousarray(vals, _NPD[Domain(domain)])
        h = C.c_void_p()
        call("gbx_mat_new", C.byref(h), int(nrows), int(ncols), _ptr(rp),
             c.ctypes.data if len(c) else None, v.ctypes.data if len(v) else None, int(domain))
        return Matrix(h)

    @staticmethod
    def from_graph(g: Graph, transposed=False) -> "Matrix":
        h = C.c_void_p()
        call("gbx_mat_from_graph", C.byref(h), g.handle, 1 if transposed else 0)
        return Matrix(h)

    @property
    def handle(self):
        return self._h

    def info(self):
        nr, nc, nv, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        call("gbx_mat_info", self._h, C.byref(nr), C.byref(nc), C.byref(nv), C.byref(d))
        return nr.value, nc.value, nv.value, Domain(d.value)

    def export(self):
        nr, nc, nv, d = self.info()
        rp = np.empty(nr + 1, np.int64)
        col = np.empty(max(nv, 1), np.int64)
        vals = np.empty(max(nv, 1), _NPD[d])
        call("gbx_mat_export", self._h, _ptr(rp), _ptr(col), _ptr(vals))
        return rp, col[:nv], vals[:nv]

    def free(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            call("gbx_mat_free", C.byref(self._h))
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


@dataclass
class Descriptor:
    """Descriptor + MaskSpec (core.hpp:15-73)."""
    mask: Optional[object] = None   # Vector for vector ops, Matrix for mxm
    complement: bool = False
    structural: bool = False
    replace: bool = False
    accum: Op = Op.NoOp
    accum_domain: Domain = Domain.Fp64
    transpose_in1: bool = False
    transpose_in2: bool = False

    def _c(self):
        d = _Desc()
        self._mv = None
        if isinstance(self.mask, Vector):
            self._mv = self.mask._c()
            d.mask_vec = C.cast(C.pointer(self._mv), C.c_void_p)
        elif isinstance(self.mask, Matrix):
            d.mask_mat = self.mask.handle.value
        d.complement, d.structural, d.replace = int(self.complement), int(self.structural), \
            int(self.replace)
        d.accum, d.accum_domain = int(self.accum), int(self.accum_domain)
        d.transpose_in1, d.transpose_in2 = int(self.transpose_in1), int(self.transpose_in2)
        return d


def _vec_op(name, w: Vector, desc: Optional[Descriptor], semiring, domain, first, second):
    desc = desc or Descriptor()
    dc = desc._c()
    wc = w._c()
    n = w.n
    oi = np.empty(max(n, 1), np.int64)
    ov = np.empty(max(n, 1), _NPD[Domain(w.domain)])
    nv = C.c_int64()
    if name == "gbx_mxv":
        A, u = first, second
        uc = u._c()
        call(name, _ptr(oi), _ptr(ov), C.byref(nv), C.byref(wc), C.byref(dc), int(semiring),
             int(domain), A.handle, C.byref(uc))
    else:
        u, A = first, second
        uc = u._c()
        call(name, _ptr(oi), _ptr(ov), C.byref(nv), C.byref(wc), C.byref(dc), int(semiring),
             int(domain), C.byref(uc), A.handle)
    k = nv.value
    return Vector(n, oi[:k].copy(), ov[:k].copy(), Domain(w.domain))


def mxv(w: Vector, desc: Optional[Descriptor], semiring, domain, A: Matrix, u: Vector) -> Vector:
    """w<mask> accum= A ⊕.⊗ u (core.cpp:340-386); returns the new w."""
    return _vec_op("gbx_mxv", w, desc, semiring, domain, A, u)


def vxm(w: Vector, desc: Optional[Descriptor], semiring, domain, u: Vector, A: Matrix) -> Vector:
    """w<mask> accum= u ⊕.⊗ A (core.cpp:308-338); returns the new w."""
    return _vec_op("gbx_vxm", w, desc, semiring, domain, u, A)


def mxm(Cm: Matrix, desc: Optional[Descriptor], semiring, domain, A: Matrix, B: Matrix) -> Matrix:
    """C<mask> accum= A ⊕.⊗ B (core.cpp:267-306); returns the new C."""
    desc = desc or Descriptor()
    dc = desc._c()
    h = C.c_void_p()
    call("gbx_mxm", C.byref(h), Cm.handle, C.byref(dc), int(semiring), int(domain), A.handle,
         B.handle)
    return Matrix(h)
