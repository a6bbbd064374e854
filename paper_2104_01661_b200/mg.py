"""Multi-GPU mirror (thin): the communicator, the distributed graph and the
sharded algorithms of libgbx.so (include/gbx.h: gbx_comm_* / gbx_dgraph_* /
gbx_*_mg).  The orchestration -- shard construction, exchanges, convergence --
is C++ inside the library; this module only moves handles and arrays.

  comm = Comm.from_torch(dist)        # one NCCL rank per process (torchrun)
  comm = Comm.local(nranks)           # nranks in-process ranks on ONE GPU
  g = DGraph.rmat(comm, 22, 16, seed=1, kind=Kind.DirectedAdjacency)
  rank, iters = g.pagerank()          # every rank: the full result

Result semantics are the single-GPU algo.* ones (the reference's,
algorithms.hpp:19-104)."""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from ._lib import gbx_stats
from .graph import Kind, call

COMM_ID_BYTES = 128
MG_AUTO, MG_NCCL, MG_P2P = 0, 1, 2


class Comm:
    def __init__(self, handle):
        self.handle = handle
        self._graphs = weakref.WeakSet()  # freed before the communicator
        n, r, nl = C.c_int(), C.c_int(), C.c_int()
        call("gbx_comm_info", handle, C.byref(n), C.byref(r), C.byref(nl))
        self.nranks, self.rank, self.nlocal = n.value, r.value, nl.value

    @staticmethod
    def local(nranks, device=0):
        h = C.c_void_p()
        call("gbx_comm_init_local", C.byref(h), nranks, device)
        return Comm(h)

    @staticmethod
    def nccl(nranks, rank, unique_id: bytes, device=0):
        h = C.c_void_p()
        buf = C.create_string_buffer(unique_id, COMM_ID_BYTES)
        call("gbx_comm_init", C.byref(h), nranks, rank, buf, device)
        return Comm(h)

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(COMM_ID_BYTES)
        call("gbx_comm_unique_id", buf)
        return buf.raw

    @staticmethod
    def from_torch(dist, device=None):
        """The library's own NCCL communicator over the ranks of an initialised
        torch.distributed group (rank 0's unique id is broadcast through it)."""
        import torch
        rank, world = dist.get_rank(), dist.get_world_size()
        dev = torch.cuda.current_device() if device is None else device
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Comm.nccl(world, rank, obj[0], dev)

    def free(self):
        if self.handle:
            for g in list(self._graphs):
                g.free()
            h = C.c_void_p(self.handle.value if isinstance(self.handle, C.c_void_p) else self.handle)
            call("gbx_comm_free", C.byref(h))
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DGraph:
    """gbx_dgraph: every rank holds only its row block (of A, and of AT when
    directed)."""

    def __init__(self, comm: Comm, handle):
        self.comm = comm
        self.handle = handle
        comm._graphs.add(self)
        n, nnz, k = C.c_int64(), C.c_int64(), C.c_int()
        call("gbx_dgraph_info", handle, C.byref(n), C.byref(nnz), C.byref(k))
        self.n, self.nnz, self.kind = n.value, nnz.value, Kind(k.value)

    @staticmethod
    def rmat(comm, scale, edge_factor=16, seed=1, kind=Kind.DirectedAdjacency, a=0.57, b=0.19,
             c=0.19, scramble=True):
        h = C.c_void_p()
        call("gbx_dgraph_generate_rmat", C.byref(h), comm.handle, scale, edge_factor, a, b, c,
             seed, 1 if scramble else 0, int(kind))
        return DGraph(comm, h)

    @staticmethod
    def from_blocks(comm, n, blocks, kind=Kind.DirectedAdjacency):
        """blocks: one (row_begin, row_end, row_ptr int64[rows+1], col int32) per
        local rank (any split of the rows; the library redistributes them)."""
        L = comm.nlocal
        assert len(blocks) == L
        rb = np.ascontiguousarray([b[0] for b in blocks], np.int64)
        re = np.ascontiguousarray([b[1] for b in blocks], np.int64)
        rps = [np.ascontiguousarray(b[2], np.int64) for b in blocks]
        cols = [np.ascontiguousarray(b[3], np.int32) for b in blocks]
        prp = (C.c_void_p * L)(*[a.ctypes.data for a in rps])
        pcol = (C.c_void_p * L)(*[a.ctypes.data for a in cols])
        h = C.c_void_p()
        call("gbx_dgraph_from_blocks", C.byref(h), comm.handle, n, rb.ctypes.data, re.ctypes.data,
             prp, pcol, int(kind))
        return DGraph(comm, h)

    def block(self, local=0):
        rb, re, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        call("gbx_dgraph_block", self.handle, local, C.byref(rb), C.byref(re), C.byref(nnz))
        return rb.value, re.value, nnz.value

    def export_block(self, local=0):
        rb, re, nnz = self.block(local)
        rp = np.empty(re - rb + 1, np.int64)
        col = np.empty(max(nnz, 1), np.int32)
        call("gbx_dgraph_export_block", self.handle, local, rp.ctypes.data, col.ctypes.data)
        return rb, re, rp, col[:nnz]

    def last_stats(self):
        st = gbx_stats()
        call("gbx_dgraph_last_stats", self.handle, C.byref(st))
        return {f: getattr(st, f) for f, _ in gbx_stats._fields_}

    # ---- algorithms (every rank gets the full result)
    def pagerank(self, damping=0.85, tol=1e-4, itermax=100, exchange=MG_AUTO, to_host=True):
        it = C.c_int(0)
        out = np.empty(self.n, np.float64) if to_host else None
        call("gbx_pagerank_mg", None if out is None else out.ctypes.data, C.byref(it), self.handle,
             damping, tol, itermax, exchange)
        return out, it.value

    def triangle_count(self):
        c = C.c_uint64(0)
        call("gbx_triangle_count_mg", C.byref(c), self.handle)
        return int(c.value)

    def bfs(self, source, to_host=True):
        p = np.empty(self.n, np.int64) if to_host else None
        lv = np.empty(self.n, np.int64) if to_host else None
        call("gbx_bfs_mg", None if p is None else p.ctypes.data,
             None if lv is None else lv.ctypes.data, self.handle, int(source))
        return p, lv

    def betweenness(self, sources, to_host=True):
        s = np.ascontiguousarray(sources, np.uint64)
        out = np.empty(self.n, np.float64) if to_host else None
        call("gbx_betweenness_mg", None if out is None else out.ctypes.data, self.handle,
             s.ctypes.data, len(s))
        return out

    def free(self):
        if self.handle:
            h = C.c_void_p(self.handle.value if isinstance(self.handle, C.c_void_p) else self.handle)
            call("gbx_dgraph_free", C.byref(h))
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
