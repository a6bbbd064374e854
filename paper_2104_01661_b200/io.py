"""Host mirror of gblite::io (include/gblite/io.hpp) and build_matrix
(containers.cpp:128-169), landing the matrix in HBM as a Graph.

The reference reads into a host SparseMatrix and then moves it into a Graph;
here the file goes straight to the device (libgbx.so, csrc/io.cu), so the
readers return a Graph.  Formats and error codes are the reference's:
  "bin" -- LAGK v1 (bin_read / bin_write, io.cpp:224-334),
  "mm"  -- Matrix Market coordinate (mm_read / mm_write, io.cpp:35-222).
"""
from __future__ import annotations

import ctypes as C
from enum import IntEnum

import numpy as np

from .graph import _NP, Domain, Graph, Kind, _domain_of, _ptr, call


class Dup(IntEnum):
    """Duplicate-tuple policy of build_matrix's `dup` BinaryOp."""
    Error = 0   # mm_read's trap (io.cpp:143-153)
    First = 1
    Second = 2
    Min = 3
    Max = 4
    Plus = 5


def read_matrix_file(path: str, format: str, kind=Kind.DirectedAdjacency) -> Graph:
    """read_matrix_file (io.cpp:336-343) + graph_new (graph.cpp:16-28)."""
    h = C.c_void_p()
    call("gbx_graph_read", C.byref(h), str(path).encode(), format.encode(), int(kind))
    return Graph(h)


def read_matrix_bytes(data: bytes, format: str, kind=Kind.DirectedAdjacency) -> Graph:
    """mm_read / bin_read of an in-memory stream (io.cpp:35, 282)."""
    buf = C.create_string_buffer(bytes(data), len(data))
    h = C.c_void_p()
    call("gbx_graph_read_buffer", C.byref(h), buf, len(data), format.encode(), int(kind))
    return Graph(h)


def write_matrix_file(g: Graph, path: str, format: str, symmetric: bool = False) -> None:
    """write_matrix_file (io.cpp:345-355); symmetric selects mm_write's lower-
    triangle form (io.cpp:162-222)."""
    call("gbx_graph_write", g.handle, str(path).encode(), format.encode(), 1 if symmetric else 0)


def build_graph(n: int, rows, cols, vals=None, dup=Dup.Error,
                kind=Kind.DirectedAdjacency) -> Graph:
    """build_matrix(n, n, rows, cols, vals, dup) (containers.cpp:128-169) +
    graph_new, on the device."""
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    if len(r) != len(c) or (vals is not None and len(vals) != len(r)):
        from .errors import Error
        raise Error(-1, "build_matrix tuple arrays disagree in length")
    dom = _domain_of(vals)
    if dom == Domain.Int32:
        dom = Domain.Int64
    v = None if vals is None else np.ascontiguousarray(vals, _NP[dom])
    h = C.c_void_p()
    call("gbx_graph_build", C.byref(h), int(n), len(r), _ptr(r), _ptr(c), _ptr(v), int(dom),
         int(dup), int(kind))
    return Graph(h)
