"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 hot path.

Python bindings for
  * ``_build/liborc.so``: the plain-C restatement of the reference algorithms
    (oracle.c, each function cites the reference file:line it follows), and
  * ``_ref/libgblite_ref.so``: the UNMODIFIED reference library compiled from
    /root/reference/proj/src by ``make -C oracle ref`` behind an extern "C"
    shim (ref_shim.cpp).  Optional: absent on boxes where it was not built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs may import this package.  The product library never
calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ORC_SO = os.path.join(_HERE, "_build", "liborc.so")
_REF_SO = os.path.join(_HERE, "_ref", "libgblite_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")

_lib = None
_ref = None


def build(ref: bool = False) -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    if ref:
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORC_SO):
            build()
        L = C.CDLL(_ORC_SO)
        L.orc_stream.restype = C.c_uint64
        L.orc_stream.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_draw.restype = C.c_uint64
        L.orc_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_scramble.restype = C.c_uint32
        L.orc_scramble.argtypes = [C.c_uint32, C.c_int, C.c_uint64]
        L.orc_rmat_edges.restype = C.c_int64
        L.orc_rmat_edges.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_uint64, C.c_int, _u32p, _u32p]
        L.orc_er_edges.restype = C.c_int64
        L.orc_er_edges.argtypes = [C.c_int, C.c_int, C.c_uint64, _u32p, _u32p, C.c_void_p]
        L.orc_build_csr.restype = C.c_int64
        L.orc_build_csr.argtypes = [C.c_int64, C.c_int64, _u32p, _u32p, C.c_void_p, C.c_int,
                                    _i64p, _i32p, C.c_void_p]
        L.orc_transpose.restype = None
        L.orc_transpose.argtypes = [C.c_int64, _i64p, _i32p, C.c_void_p, _i64p, _i32p,
                                    C.c_void_p]
        L.orc_bfs.restype = C.c_int
        L.orc_bfs.argtypes = [C.c_int64, _i64p, _i32p, C.c_int64, _i64p, _i64p]
        L.orc_pagerank.restype = C.c_int
        L.orc_pagerank.argtypes = [C.c_int64, _i64p, _i32p, _i64p, C.c_double, C.c_double,
                                   C.c_int, _f64p, C.POINTER(C.c_int), C.c_void_p]
        L.orc_triangle_count.restype = C.c_uint64
        L.orc_triangle_count.argtypes = [C.c_int64, _i64p, _i32p]
        for f in (L.orc_sssp_delta,):
            f.restype = C.c_int
            f.argtypes = [C.c_int64, _i64p, _i32p, _f64p, C.c_int64, C.c_double, _f64p]
        L.orc_dijkstra.restype = C.c_int
        L.orc_dijkstra.argtypes = [C.c_int64, _i64p, _i32p, _f64p, C.c_int64, _f64p]
        L.orc_bc.restype = C.c_int
        L.orc_bc.argtypes = [C.c_int64, _i64p, _i32p, _i64p, _i32p, _i64p, C.c_int64, _f64p]
        L.orc_cc.restype = C.c_int
        L.orc_cc.argtypes = [C.c_int64, _i64p, _i32p, _i64p]
        L.orc_sort_by_degree.restype = None
        L.orc_sort_by_degree.argtypes = [C.c_int64, _i64p, _i64p]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle error {code} {what}")
        self.code = code


def _chk(code, what=""):
    if code != 0:
        raise OracleError(code, what)


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def threads() -> int:
    return int(lib().orc_get_threads())


# ---- seeded synthetic inputs ------------------------------------------------

RMAT_ABC = (0.57, 0.19, 0.19)


def rmat_edges(scale, edge_factor=16, seed=1, a=0.57, b=0.19, c=0.19, scramble=True):
    m = edge_factor << scale
    u = np.empty(m, np.uint32)
    v = np.empty(m, np.uint32)
    lib().orc_rmat_edges(scale, edge_factor, a, b, c, seed, 1 if scramble else 0, u, v)
    return u, v


def er_edges(logn, degree=16, seed=1, weights=True):
    m = degree << logn
    u = np.empty(m, np.uint32)
    v = np.empty(m, np.uint32)
    w = np.empty(m, np.int32) if weights else None
    lib().orc_er_edges(logn, degree, seed, u, v, w.ctypes.data if weights else None)
    return u, v, w


def build_csr(n, u, v, w=None, symmetrize=False):
    m = len(u)
    cap = 2 * m if symmetrize else m
    rp = np.empty(n + 1, np.int64)
    col = np.empty(max(cap, 1), np.int32)
    wo = np.empty(max(cap, 1), np.int32) if w is not None else None
    u = np.ascontiguousarray(u, np.uint32)
    v = np.ascontiguousarray(v, np.uint32)
    wp = np.ascontiguousarray(w, np.int32) if w is not None else None
    nnz = lib().orc_build_csr(n, m, u, v, wp.ctypes.data if wp is not None else None,
                              1 if symmetrize else 0, rp, col,
                              wo.ctypes.data if wo is not None else None)
    col = col[:nnz].copy()
    if wo is not None:
        wo = wo[:nnz].copy()
    return rp, col, wo


def transpose(n, rp, col, w=None):
    nnz = int(rp[n])
    trp = np.empty(n + 1, np.int64)
    tcol = np.empty(max(nnz, 1), np.int32)
    tw = np.empty(max(nnz, 1), np.int32) if w is not None else None
    wp = np.ascontiguousarray(w, np.int32) if w is not None else None
    lib().orc_transpose(n, rp, col, wp.ctypes.data if wp is not None else None, trp, tcol,
                        tw.ctypes.data if tw is not None else None)
    return trp, tcol[:nnz].copy(), (tw[:nnz].copy() if tw is not None else None)


# ---- algorithms ---------------------------------------------------------------


def bfs(n, rp, col, src):
    parent = np.empty(n, np.int64)
    level = np.empty(n, np.int64)
    _chk(lib().orc_bfs(n, rp, col, int(src), parent, level), "bfs")
    return parent, level


def pagerank(n, at_rp, at_col, outdeg, damping=0.85, tol=1e-4, itermax=100, trace=False):
    rank = np.empty(max(n, 1), np.float64)
    it = C.c_int(0)
    tr = np.zeros((itermax, n), np.float64) if trace else None
    _chk(lib().orc_pagerank(n, at_rp, at_col, np.ascontiguousarray(outdeg, np.int64),
                            damping, tol, itermax, rank, C.byref(it),
                            tr.ctypes.data if tr is not None else None), "pagerank")
    rank = rank[:n]
    if trace:
        return rank, it.value, tr[: it.value]
    return rank, it.value


def triangle_count(n, rp, col):
    return int(lib().orc_triangle_count(n, rp, col))


def sssp_delta(n, rp, col, w, src, delta):
    dist = np.empty(n, np.float64)
    _chk(lib().orc_sssp_delta(n, rp, col, np.ascontiguousarray(w, np.float64), int(src),
                              float(delta), dist), "sssp")
    return dist


def dijkstra(n, rp, col, w, src):
    dist = np.empty(n, np.float64)
    _chk(lib().orc_dijkstra(n, rp, col, np.ascontiguousarray(w, np.float64), int(src), dist),
         "dijkstra")
    return dist


def bc(n, rp, col, at_rp, at_col, sources):
    cent = np.empty(max(n, 1), np.float64)
    s = np.ascontiguousarray(sources, np.int64)
    _chk(lib().orc_bc(n, rp, col, at_rp, at_col, s, len(s), cent), "bc")
    return cent[:n]


def cc(n, rp, col):
    lab = np.empty(max(n, 1), np.int64)
    _chk(lib().orc_cc(n, rp, col, lab), "cc")
    return lab[:n]


def sort_by_degree(deg):
    deg = np.ascontiguousarray(deg, np.int64)
    perm = np.empty(len(deg), np.int64)
    lib().orc_sort_by_degree(len(deg), deg, perm)
    return perm


# ---- the reference itself (oracle/_ref) -------------------------------------------


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            raise OracleError(-1, f"{_REF_SO} not built (make -C oracle ref)")
        L = C.CDLL(_REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_new.restype = C.c_int
        L.ref_graph_new.argtypes = [C.POINTER(C.c_void_p), C.c_int64, _i64p, _i32p,
                                    C.c_void_p, C.c_int]
        L.ref_graph_free.argtypes = [C.c_void_p]
        for nm in ("ref_property_at", "ref_property_rowdegree", "ref_property_ndiag",
                   "ref_property_symmetric"):
            getattr(L, nm).restype = C.c_int
            getattr(L, nm).argtypes = [C.c_void_p]
        L.ref_ndiag.restype = C.c_int64
        L.ref_ndiag.argtypes = [C.c_void_p]
        L.ref_symmetric.restype = C.c_int
        L.ref_symmetric.argtypes = [C.c_void_p]
        L.ref_bfs.restype = C.c_int
        L.ref_bfs.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int, _i64p,
                              _i64p]
        L.ref_pagerank.restype = C.c_int
        L.ref_pagerank.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, _f64p,
                                   C.POINTER(C.c_int), C.c_void_p]
        L.ref_triangle_count.restype = C.c_int
        L.ref_triangle_count.argtypes = [C.c_void_p, C.c_int, C.c_uint64,
                                         C.POINTER(C.c_uint64)]
        L.ref_sssp.restype = C.c_int
        L.ref_sssp.argtypes = [C.c_void_p, C.c_int64, C.c_double, _f64p]
        L.ref_sssp_default_delta.restype = C.c_double
        L.ref_sssp_default_delta.argtypes = [C.c_void_p]
        L.ref_bc.restype = C.c_int
        L.ref_bc.argtypes = [C.c_void_p, _i64p, C.c_int64, _f64p]
        L.ref_cc.restype = C.c_int
        L.ref_cc.argtypes = [C.c_void_p, _i64p, C.POINTER(C.c_int)]
        L.ref_sort_by_degree.restype = C.c_int
        L.ref_sort_by_degree.argtypes = [C.c_void_p, _i64p]
        L.ref_sample_degree.restype = C.c_int
        L.ref_sample_degree.argtypes = [C.c_void_p, C.c_int64, C.c_uint64,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_pr_mxv_sample.restype = C.c_int
        L.ref_pr_mxv_sample.argtypes = [C.c_int64, _i64p, _i32p, _i64p, C.c_double,
                                        C.c_int64, C.c_int64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        L.ref_verify_bfs_parents.restype = C.c_int
        L.ref_verify_bfs_parents.argtypes = [C.c_void_p, C.c_int64, _i64p,
                                             C.POINTER(C.c_int)]
        L.ref_io_convert.restype = C.c_int
        L.ref_io_convert.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def _rchk(code):
    if code != 0:
        raise RefError(code, ref().ref_last_error().decode())


class RefGraph:
    """A gblite::Graph built by the reference's own graph_new (graph.cpp:16-28)."""

    def __init__(self, n, rp, col, w=None, undirected=False):
        L = ref()
        self.n = n
        self._h = C.c_void_p()
        self._w = np.ascontiguousarray(w, np.float64) if w is not None else None
        _rchk(L.ref_graph_new(C.byref(self._h), n, np.ascontiguousarray(rp, np.int64),
                              np.ascontiguousarray(col, np.int32),
                              self._w.ctypes.data if self._w is not None else None,
                              1 if undirected else 0))

    def __del__(self):
        if getattr(self, "_h", None) and _ref is not None:
            _ref.ref_graph_free(self._h)
            self._h = None

    def property_at(self):
        _rchk(ref().ref_property_at(self._h))

    def property_rowdegree(self):
        _rchk(ref().ref_property_rowdegree(self._h))

    def property_ndiag(self):
        _rchk(ref().ref_property_ndiag(self._h))

    def property_symmetric(self):
        _rchk(ref().ref_property_symmetric(self._h))

    def bfs(self, src, direction=0, push_divisor=16, want_level=True):
        parent = np.empty(self.n, np.int64)
        level = np.empty(self.n, np.int64)
        _rchk(ref().ref_bfs(self._h, int(src), direction, push_divisor,
                            1 if want_level else 0, parent, level))
        return parent, level

    def pagerank(self, damping=0.85, tol=1e-4, itermax=100, trace=False):
        rank = np.empty(max(self.n, 1), np.float64)
        it = C.c_int(0)
        tr = np.zeros((itermax, self.n), np.float64) if trace else None
        _rchk(ref().ref_pagerank(self._h, damping, tol, itermax, rank, C.byref(it),
                                 tr.ctypes.data if tr is not None else None))
        if trace:
            return rank[: self.n], it.value, tr[: it.value]
        return rank[: self.n], it.value

    def triangle_count(self, presort=0, seed=7):
        c = C.c_uint64(0)
        _rchk(ref().ref_triangle_count(self._h, presort, seed, C.byref(c)))
        return int(c.value)

    def sssp(self, src, delta):
        d = np.empty(self.n, np.float64)
        _rchk(ref().ref_sssp(self._h, int(src), float(delta), d))
        return d

    def bc(self, sources):
        cent = np.empty(max(self.n, 1), np.float64)
        s = np.ascontiguousarray(sources, np.int64)
        _rchk(ref().ref_bc(self._h, s, len(s), cent))
        return cent[: self.n]

    def cc(self):
        lab = np.empty(max(self.n, 1), np.int64)
        it = C.c_int(0)
        _rchk(ref().ref_cc(self._h, lab, C.byref(it)))
        return lab[: self.n], it.value

    def sort_by_degree(self):
        p = np.empty(self.n, np.int64)
        _rchk(ref().ref_sort_by_degree(self._h, p))
        return p


def ref_pr_mxv_sample(n, at_rp, at_col, outdeg, damping, r0, r1):
    secs = C.c_double(0)
    cs = C.c_double(0)
    _rchk(ref().ref_pr_mxv_sample(n, at_rp, at_col, np.ascontiguousarray(outdeg, np.int64),
                                  damping, r0, r1, C.byref(secs), C.byref(cs)))
    return secs.value, cs.value


# ---- convenience graph builders (numpy CSR) ---------------------------------------


def rmat_graph(scale, edge_factor=16, seed=1, undirected=False, scramble=True):
    u, v = rmat_edges(scale, edge_factor, seed, scramble=scramble)
    rp, col, _ = build_csr(1 << scale, u, v, None, symmetrize=undirected)
    return rp, col


def er_graph(logn, degree=16, seed=1):
    u, v, w = er_edges(logn, degree, seed)
    rp, col, wo = build_csr(1 << logn, u, v, w, symmetrize=False)
    return rp, col, wo


def csr_from_dense(adj):
    """CSR (rp int64, col int32, vals float64|None) from a dense matrix-like of
    Python values where None / 0 means absent."""
    a = np.asarray(adj)
    n = a.shape[0]
    rp = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(a[i])[0]
        cols.extend(nz.tolist())
        vals.extend(a[i, nz].tolist())
        rp[i + 1] = len(cols)
    return rp, np.array(cols, np.int32), np.array(vals, np.float64)
