"""Host mirror of gblite's Graph object (include/gblite/graph.hpp:16-60).

A `Graph` owns a device handle (gbx_graph) holding A and the cached properties
in HBM.  Function names, argument meaning and error behaviour follow the
reference: `graph_new` validates and takes the matrix (graph.cpp:16-28),
`property_*` fill caches (graph.cpp:30-102), advanced algorithms raise
`Error(MissingProperty)` when a cache is absent.
"""
from __future__ import annotations

import ctypes as C
from enum import IntEnum

import numpy as np

from ._lib import MSG_LEN, gbx_stats, lib
from .errors import Error


class Kind(IntEnum):
    DirectedAdjacency = 0
    UndirectedAdjacency = 1


class TriState(IntEnum):
    False_ = 0
    True_ = 1
    Unknown = -1


class Domain(IntEnum):
    Bool = 0
    Int64 = 1
    Uint64 = 2
    Fp64 = 3
    Int32 = 4


_NP = {Domain.Bool: np.uint8, Domain.Int64: np.int64, Domain.Uint64: np.uint64,
       Domain.Fp64: np.float64, Domain.Int32: np.int32}


def _ptr(a):
    return None if a is None else a.ctypes.data


def call(name, *args):
    msg = C.create_string_buffer(MSG_LEN)
    rc = getattr(lib(), name)(*args, msg)
    if rc < 0:
        raise Error(rc, msg.value.decode(errors="replace"))
    return rc


def _domain_of(vals):
    if vals is None:
        return Domain.Bool
    dt = np.asarray(vals).dtype
    if dt == np.float64 or dt == np.float32:
        return Domain.Fp64
    if dt == np.int32:
        return Domain.Int32
    if dt == np.uint64:
        return Domain.Uint64
    if dt == np.bool_ or dt == np.uint8:
        return Domain.Bool
    return Domain.Int64


class Graph:
    """gblite::Graph: adjacency A (CSR in HBM) + cached properties."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    # -- lifetime ---------------------------------------------------------
    def free(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            call("gbx_graph_free", C.byref(self._h))
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @property
    def handle(self):
        if self._h is None or not self._h.value:
            raise Error(-33, "graph was freed")
        return self._h

    # -- info -------------------------------------------------------------
    def info(self):
        n, nnz, kind, dom = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        call("gbx_graph_info", self.handle, C.byref(n), C.byref(nnz), C.byref(kind),
             C.byref(dom))
        return n.value, nnz.value, Kind(kind.value), Domain(dom.value)

    def n(self):
        return self.info()[0]

    def nvals(self):
        return self.info()[1]

    @property
    def kind(self):
        return self.info()[2]

    def properties(self):
        at, rd, cd, sym = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        nd = C.c_int64()
        call("gbx_graph_properties", self.handle, C.byref(at), C.byref(rd), C.byref(cd),
             C.byref(sym), C.byref(nd))
        return {"AT": bool(at.value), "row_degree": bool(rd.value),
                "col_degree": bool(cd.value), "pattern_is_symmetric": TriState(sym.value),
                "ndiag": nd.value}

    @property
    def has_AT(self):
        return self.properties()["AT"]

    @property
    def ndiag(self):
        return self.properties()["ndiag"]

    @property
    def pattern_is_symmetric(self):
        return self.properties()["pattern_is_symmetric"]

    def export(self):
        """(row_ptr int64[n+1], col int32[nnz], vals or None) copied back from HBM."""
        n, nnz, _, dom = self.info()
        rp = np.empty(n + 1, np.int64)
        col = np.empty(max(nnz, 1), np.int32)
        vals = np.empty(max(nnz, 1), _NP[dom]) if dom != Domain.Bool else None
        call("gbx_graph_export", self.handle, _ptr(rp), _ptr(col), _ptr(vals))
        return rp, col[:nnz], (vals[:nnz] if vals is not None else None)

    def row_degree(self):
        d = np.empty(max(self.n(), 1), np.int64)
        call("gbx_row_degree", self.handle, _ptr(d))
        return d[: self.n()]

    def col_degree(self):
        d = np.empty(max(self.n(), 1), np.int64)
        call("gbx_col_degree", self.handle, _ptr(d))
        return d[: self.n()]

    def stream(self):
        s = C.c_void_p()
        call("gbx_graph_stream", self.handle, C.byref(s))
        return s.value

    def prepare(self, which: str):
        call("gbx_prepare", self.handle, which.encode())

    def last_stats(self):
        st = gbx_stats()
        call("gbx_last_stats", self.handle, C.byref(st))
        return {"launches": st.launches, "hot_launches": st.hot_launches,
                "hot_bytes_per_launch": st.hot_bytes_per_launch,
                "work_units": st.work_units, "iterations": st.iterations, "hot_ms": st.hot_ms}

    def result_device(self, which: str):
        p = C.c_void_p()
        cnt = C.c_int64()
        call("gbx_result_device", self.handle, which.encode(), C.byref(p), C.byref(cnt))
        return p.value, cnt.value


def graph_new(row_ptr, col_idx, vals=None, kind=Kind.DirectedAdjacency, n=None) -> Graph:
    """graph_new(SparseMatrix&&, Kind) (graph.cpp:16-28) from CSR arrays."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    if n is None:
        n = len(rp) - 1
    if len(rp) != n + 1:
        raise Error(-4, "graph_new: row_ptr length is not nrows+1")
    col = np.asarray(col_idx)
    h = C.c_void_p()
    dom = _domain_of(vals)
    v = None if vals is None else np.ascontiguousarray(vals, _NP[dom])
    if col.dtype == np.int32:
        col = np.ascontiguousarray(col)
        call("gbx_graph_new32", C.byref(h), n, _ptr(rp), _ptr(col), _ptr(v), int(dom), int(kind))
    else:
        col = np.ascontiguousarray(col, np.int64)
        call("gbx_graph_new", C.byref(h), n, _ptr(rp), _ptr(col), _ptr(v), int(dom), int(kind))
    return Graph(h)


def generate_rmat(scale, edge_factor=16, seed=1, kind=Kind.DirectedAdjacency, a=0.57, b=0.19,
                  c=0.19, scramble=True) -> Graph:
    h = C.c_void_p()
    call("gbx_generate_rmat", C.byref(h), scale, edge_factor, a, b, c, seed,
         1 if scramble else 0, int(kind))
    return Graph(h)


def generate_er(logn, degree=16, seed=1, weighted=True) -> Graph:
    h = C.c_void_p()
    call("gbx_generate_er", C.byref(h), logn, degree, seed, 1 if weighted else 0)
    return Graph(h)


def property_at(g: Graph):
    call("gbx_property_at", g.handle)


def property_rowdegree(g: Graph):
    call("gbx_property_rowdegree", g.handle)


def property_coldegree(g: Graph):
    call("gbx_property_coldegree", g.handle)


def property_symmetric_pattern(g: Graph):
    call("gbx_property_symmetric_pattern", g.handle)


def property_ndiag(g: Graph):
    call("gbx_property_ndiag", g.handle)


def delete_properties(g: Graph):
    call("gbx_delete_properties", g.handle)


def check_graph(g: Graph):
    """Returns (code, message): 0 and "" when every cache is consistent."""
    msg = C.create_string_buffer(MSG_LEN)
    rc = lib().gbx_check_graph(g.handle, msg)
    return rc, msg.value.decode(errors="replace")


def sort_by_degree(g: Graph, ascending=True, by_row=True):
    n = g.n()
    p = np.empty(max(n, 1), np.int64)
    call("gbx_sort_by_degree", _ptr(p), g.handle, 1 if ascending else 0, 1 if by_row else 0)
    return p[:n]


def init(device=0):
    call("gbx_init", device)


def version():
    return lib().gbx_version().decode()
