"""Multi-GPU drivers written over torch.distributed.

The product multi-GPU path is the C++ one inside libgbx.so -- its own NCCL
communicator, distributed graphs built locally, gbx_*_mg -- wrapped by
paper_2104_01661_b200/mg.py (Comm / DGraph) and used by bench.py --gpus N.
This module keeps the same protocols as Python drivers over the lower-level
shard calls (gbx_pr_shard_*, gbx_bfs_shard_*, gbx_bc_shard_*): their host
logic is what tests/test_dist_gloo.py runs on CPU (world size 2 over gloo with
a numpy backend), and they serve callers that already hold a torch process
group and a replicated graph.

One process per GPU, torch.distributed (NCCL over NVLink/NVSwitch) for the
exchange, libgbx.so shard kernels for the compute.

PageRank (config 2): 1D row blocks of the in-degree-relabeled AT, balanced by
rows + nnz.  Per iteration every rank runs the fused shard step on its rows
(gbx_pr_shard_step: sums, teleport, next contributions, fp64 L1 partial), then
  * one all_gather_into_tensor of the x slices (fp32, padded to the longest
    block, so every slice lands in place) -> the full x for the next step; the
    slots' last 8 bytes carry the fp64 L1 partials, summed in rank order and
    compared against tol exactly as pagerank.cpp:65-74 does (same iteration
    count as the single-GPU path), one iteration behind so the host check
    overlaps the next queued iteration.
Triangle count (config 3): U replicated, middle vertices split by probe work
(gbx_tc_partition), one u64 all-reduce at the end.
BFS (scale >= 22): 1D row blocks (32-aligned), one frontier-bitmap all-gather
per level (sharded_bfs): every rank pulls its unvisited rows against the global
frontier, parents are the min-id frontier in-neighbour exactly as on one GPU.
Betweenness (config 5), two drivers:
  * sharded_betweenness_rows -- 1D row blocks: every rank owns a
    nnz-balanced vertex block and settles only its rows' path counts (forward)
    and dependencies (backward); after every BFS level the ranks all-gather
    the (vertex, lanes, sigma[4] | coef[4]) records of the vertices they
    settled, so the replicated level lists / maps / sigma / coef stay
    identical; one fp64 all-reduce of the centrality partials at the end.
    Scales past the config's 4 sources; equals the single GPU to rounding;
  * sharded_betweenness -- the sources dealt round-robin (each rank runs its
    own batched Brandes; at most #sources ranks busy) + the same all-reduce:
    the sum over sources is the reference's own reduction
    (betweenness.cpp:74-79).

The drivers only speak to a small backend interface, so the host logic (the
partition bookkeeping, the exchange, the convergence test) is exercised on CPU
by tests/test_dist_gloo.py with world_size 2 over gloo and a numpy backend.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def _gather_slices(dist, local, bounds, world, out):
    """All-gather variable-length 1-D slices: rank p owns out[bounds[p]:bounds[p+1]].
    NCCL all-gather wants equal sizes, so slices are padded to the longest."""
    import torch
    chunk = max(int(bounds[p + 1] - bounds[p]) for p in range(world))
    send = torch.zeros(chunk, dtype=local.dtype, device=local.device)
    send[: local.numel()] = local
    parts = [torch.empty(chunk, dtype=local.dtype, device=local.device) for _ in range(world)]
    dist.all_gather(parts, send)
    for p in range(world):
        b, e = int(bounds[p]), int(bounds[p + 1])
        if e > b:
            out[b:e] = parts[p][: e - b]
    return out


def sharded_pagerank(backend, dist, damping=0.85, tol=1e-4, itermax=100, to_host=True):
    """GAP PageRank over `world` ranks; returns (rank vector on every rank (numpy,
    original ids), iterations).  to_host=False: the gathered (padded,
    relabeled) rank vector stays on the device and is returned as is.

    Per iteration k: the shard step (library stream), then ONE
    all_gather_into_tensor of the chunk-long slices straight into the padded x
    (gbx_pr_shard_layout) -- every slot carries its rank's fp64 L1 partial in
    its last 8 bytes -- and an async copy of the world partials to the host,
    summed there in rank order (the same total on every rank).
    The convergence test of iteration k-1 (pagerank.cpp:74: stop when L1 < tol)
    runs on the host while iteration k is already queued, so the host never
    drains the device; r is double-buffered, so when k-1 converged the result
    is r of k-1 and the speculative step k is discarded.  The iteration count
    and ranks equal the sequential loop's."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    rb, re, n = backend.prepare(rank, world)
    chunk = backend.chunk
    assert re - rb <= chunk
    backend.init(damping)
    x_full = backend.x_full()
    assert x_full.numel() == world * chunk
    pending = None
    iters = 0
    for k in range(1, itermax + 1):
        backend.step(damping, k)                   # r, x slice + its L1 partial (tail)
        dist.all_gather_into_tensor(x_full, backend.x_new_slice())
        tok = backend.l1_post(k)                   # every rank's partial -> host (async)
        if pending is not None:
            kk, tk = pending
            if not (backend.l1_value(tk) >= tol):
                iters = kk
                break
        pending = (k, tok)
    else:
        iters = pending[0] if pending is not None else 0
    r_full = torch.empty(world * chunk, dtype=backend.r_local(iters).dtype, device=backend.device)
    dist.all_gather_into_tensor(r_full, backend.r_local(iters))
    if not to_host:
        return r_full, iters
    return backend.unpermute(r_full), iters


def sharded_pagerank_p2p(backend, dist, damping=0.85, tol=1e-4, itermax=100, to_host=True):
    """GAP PageRank over `world` ranks with the exchange FUSED into the iteration
    kernel (gbx_pr_shard_run_p2p): one cooperative launch per rank runs every
    iteration; each row epilogue stores its contribution straight into every
    rank's x over NVLink (peer pointers), the L1 partials go
    to every rank's slot table, and a device-side signal barrier separates
    iterations -- no host round trip and no NCCL call per iteration.  One NCCL
    all-gather of the local ranks at the end.  Same results and iteration
    count as sharded_pagerank.

    The kernel's wait for its peers is bounded (option p2p.timeout_ms): when
    any rank fails -- its launch raised, or a peer never arrived -- every rank
    learns it through one all-reduce and the run is redone with the NCCL
    exchange (sharded_pagerank), so a broken peer path degrades instead of
    hanging the job."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    rb, re, n = backend.prepare(rank, world)
    chunk = backend.chunk
    ok = 1
    iters = 0
    try:
        backend.p2p_setup(dist)
        backend.p2p_init(damping)      # x0 (every slot), r0; signal words zeroed
    except Exception:
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=backend.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)   # every rank zeroed before any rank signals
    if int(flag.item()) == 1:
        try:
            iters = backend.p2p_run(damping, tol, itermax)
        except Exception:
            ok = 0
        flag.fill_(ok)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0:
        backend.p2p_failed = True
        return sharded_pagerank(backend, dist, damping, tol, itermax, to_host)
    r_local = backend.p2p_result(iters)
    r_full = torch.empty(world * chunk, dtype=r_local.dtype, device=backend.device)
    dist.all_gather_into_tensor(r_full, r_local)
    if not to_host:
        return r_full, iters
    return backend.unpermute(r_full), iters


def sharded_triangle_count(backend, dist):
    """Triangle count with wedge-balanced row blocks of the oriented U."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    bounds = backend.tc_partition(world)
    local = backend.tc_rows(int(bounds[rank]), int(bounds[rank + 1]))
    t = torch.tensor([local], dtype=torch.int64, device=backend.device)
    dist.all_reduce(t)
    return int(t.item())


def sharded_betweenness(backend, dist, sources):
    """Batched Brandes over `world` ranks: rank r takes sources[r::world]; returns
    the centrality (numpy fp64, every rank)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    mine = [int(s) for s in list(sources)[rank::world]]
    part = backend.bc_partial(mine)            # fp64 tensor [n] (zeros if no sources)
    dist.all_reduce(part)
    return part.cpu().numpy().copy()


def sharded_bfs(backend, dist, source):
    """Row-sharded BFS from one source; returns (parent, level) numpy int64
    arrays (-1 = unreached) on every rank."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    rb, re, n = backend.bfs_begin(source, rank, world)
    dev = backend.device
    b = torch.tensor([rb, re], dtype=torch.int64, device=dev)
    allb = [torch.empty(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(allb, b)
    rows = [int(t[0]) for t in allb] + [int(allb[-1][1])]
    assert rows[0] == 0 and rows[-1] == n
    words = (n + 31) // 32
    wb = [r // 32 for r in rows[:-1]] + [words]          # word slices tile [0, words)
    front = torch.zeros(max(words, 1), dtype=torch.int32, device=dev)
    front[source >> 5] = torch.tensor(1 << (source & 31), dtype=torch.int64).to(torch.int32)
    nxt = torch.zeros(max(wb[rank + 1] - wb[rank], 1), dtype=torch.int32, device=dev)
    while True:
        found = backend.bfs_level(front, nxt)
        tot = torch.tensor([found], dtype=torch.int64, device=dev)
        dist.all_reduce(tot)
        if int(tot.item()) == 0:
            break
        _gather_slices(dist, nxt[: wb[rank + 1] - wb[rank]], wb, world, front)
    par, lev = backend.bfs_result()
    p_full = torch.empty(n, dtype=torch.int64, device=dev)
    l_full = torch.empty(n, dtype=torch.int64, device=dev)
    _gather_slices(dist, torch.as_tensor(par, device=dev), rows, world, p_full)
    _gather_slices(dist, torch.as_tensor(lev, device=dev), rows, world, l_full)
    return p_full.cpu().numpy(), l_full.cpu().numpy()


def _gather_records(dist, recs, nrec, rec_bytes=40):
    """All-gather variable-length record buffers (uint8 tensors of nrec *
    rec_bytes bytes) in rank order; returns (concatenated tensor, total)."""
    import torch
    world = dist.get_world_size()
    dev = recs.device
    cnt = torch.tensor([nrec], dtype=torch.int64, device=dev)
    cnts = [torch.empty(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    cnts = [int(c.item()) for c in cnts]
    mx = max(cnts)
    total = sum(cnts)
    if mx == 0:
        return torch.empty(0, dtype=torch.uint8, device=dev), 0
    send = torch.zeros(mx * rec_bytes, dtype=torch.uint8, device=dev)
    if nrec:
        send[: nrec * rec_bytes] = recs[: nrec * rec_bytes]
    parts = [torch.empty(mx * rec_bytes, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(parts, send)
    out = torch.cat([parts[p][: cnts[p] * rec_bytes] for p in range(world)])
    return out, total


def sharded_betweenness_rows(backend, dist, sources):
    """Row-partitioned batched Brandes (one record exchange per BFS level);
    returns the centrality (numpy fp64, every rank)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    srcs = [int(s) for s in sources]
    total = None
    for b0 in range(0, len(srcs), 4):
        backend.bc_begin(srcs[b0:b0 + 4], rank, world)
        while True:                                   # forward: depth by depth
            recs, nrec = backend.bc_forward()
            allr, tot = _gather_records(dist, recs, nrec)
            if backend.bc_forward_apply(allr, tot):
                break
        while True:                                   # backward: deepest first
            recs, nrec, done = backend.bc_backward()
            if done:
                break
            allr, tot = _gather_records(dist, recs, nrec)
            backend.bc_backward_apply(allr, tot)
        part = backend.bc_centrality().clone()
        total = part if total is None else total + part
    dist.all_reduce(total)
    return total.cpu().numpy().copy()


# buffers of the fused P2P PageRank (one-rank torch driver), keyed by (world, chunk, device)
_P2P_BUFFERS = {}


class _DeviceArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (n,),
                                         "typestr": typestr, "version": 3}


class GpuShardBackend:
    """libgbx.so shard kernels on this rank's GPU (vectors are torch CUDA tensors)."""

    def __init__(self, graph):
        import torch
        self.g = graph
        self.device = torch.device("cuda", torch.cuda.current_device())

    def prepare(self, rank, world):
        import torch

        from .graph import call
        rb, re, chunk = C.c_int64(), C.c_int64(), C.c_int64()
        call("gbx_pr_shard_prepare", self.g.handle, rank, world, C.byref(rb), C.byref(re))
        call("gbx_pr_shard_layout", self.g.handle, C.byref(chunk), None)
        self.rb, self.re, self.chunk = rb.value, re.value, chunk.value
        self.world = world
        self.n = self.g.n()
        dev = self.device
        self._x = torch.empty(world * self.chunk, dtype=torch.float32, device=dev)
        self._xs = torch.zeros(self.chunk, dtype=torch.float32, device=dev)
        self._r = [torch.zeros(self.chunk, dtype=torch.float32, device=dev) for _ in range(2)]
        self._l1h = [torch.zeros(world, 1, dtype=torch.float64).pin_memory() for _ in range(2)]
        self._ev = [torch.cuda.Event() for _ in range(2)]
        self._stream = torch.cuda.ExternalStream(self.g.stream())
        return self.rb, self.re, self.n

    def init(self, damping):
        from .graph import call
        call("gbx_pr_shard_init", self.g.handle, self._x.data_ptr(), self._r[0].data_ptr(),
             damping)

    def step(self, damping, k):
        """Iteration k (1-based): r_prev = buffer (k-1)&1, r_new = buffer k&1; the
        fp64 L1 partial goes to the slice's last 8 bytes."""
        import torch

        from .graph import call
        # the library stream must see the x gathered on torch's stream
        self._stream.wait_stream(torch.cuda.current_stream())
        call("gbx_pr_shard_step", self.g.handle, self._x.data_ptr(),
             self._r[(k - 1) & 1].data_ptr(), self._r[k & 1].data_ptr(), self._xs.data_ptr(),
             self._xs.data_ptr() + 4 * (self.chunk - 2), damping)
        # the collectives run on torch's stream: order them after the library's
        torch.cuda.current_stream().wait_stream(self._stream)

    def l1_post(self, k):
        """Queue the world's L1 partials of iteration k (gathered slot tails) for
        the host: one strided async copy into pinned memory."""
        import torch
        tails = self._x.view(self.world, self.chunk)[:, self.chunk - 2:].view(torch.float64)
        self._l1h[k & 1].copy_(tails, non_blocking=True)
        self._ev[k & 1].record(torch.cuda.current_stream())
        return k & 1

    def l1_value(self, tok):
        self._ev[tok].synchronize()
        parts = self._l1h[tok]
        tot = 0.0
        for q in range(self.world):  # rank order: the same sum on every rank
            tot += float(parts[q, 0])
        return tot

    def x_new_slice(self):
        return self._xs
    # ---- fused P2P run (gbx_pr_shard_run_p2p)
    def p2p_setup(self, dist):
        """x0 / x1 / slot table / signal buffers and the table of every rank's
        pointers to them.  This torch driver only serves a ONE-rank group (plain
        device buffers, the rank is its own peer): with more ranks the peer
        buffers come from the library's own communicator (CUDA IPC handles
        exchanged over gbx_comm), i.e. mg.Comm / DGraph.pagerank -- the C++ path
        -- so no private torch API is involved."""
        import torch
        if self.world != 1:
            raise NotImplementedError(
                "the torch driver of the fused exchange serves one rank; multi-rank runs go "
                "through paper_2104_01661_b200.mg (gbx_comm_init + gbx_pagerank_mg)")
        if getattr(self, "_p2p_world", None) == (self.world, self.chunk):
            return
        dev = self.device
        key = (self.world, self.chunk, str(dev))
        if key not in _P2P_BUFFERS:  # allocated once per layout
            bufs = [torch.empty(self.world * self.chunk, dtype=torch.float32, device=dev),
                    torch.empty(self.world * self.chunk, dtype=torch.float32, device=dev),
                    torch.empty(2 * self.world, dtype=torch.float64, device=dev),
                    torch.empty(4, dtype=torch.int32, device=dev)]
            ptr = [np.ascontiguousarray([t.data_ptr()], np.uint64) for t in bufs]
            _P2P_BUFFERS.clear()
            _P2P_BUFFERS[key] = (bufs, None, ptr)
        self._pbufs, self._phdl, self._pptr = _P2P_BUFFERS[key]
        for a in self._pptr:
            assert len(a) == self.world
        self._pr = [torch.zeros(self.chunk, dtype=torch.float32, device=dev) for _ in range(2)]
        self._p2p_world = (self.world, self.chunk)

    def p2p_init(self, damping):
        import torch

        from .graph import call
        self._pbufs[3].zero_()
        self._pbufs[2].zero_()
        torch.cuda.current_stream().synchronize()
        call("gbx_pr_shard_init", self.g.handle, self._pbufs[0].data_ptr(),
             self._pr[0].data_ptr(), damping)
        self._stream.synchronize()

    def p2p_run(self, damping, tol, itermax):
        from .graph import call
        it = C.c_int(0)
        p = self._pptr
        call("gbx_pr_shard_run_p2p", self.g.handle, p[0].ctypes.data, p[1].ctypes.data,
             p[2].ctypes.data, p[3].ctypes.data, self._pr[0].data_ptr(), self._pr[1].data_ptr(),
             damping, tol, itermax, C.byref(it))
        return it.value

    def p2p_result(self, iters):
        return self._pr[iters & 1]


    def x_full(self):
        return self._x

    def r_local(self, k):
        return self._r[k & 1]

    def unpermute(self, r_full):
        import torch

        from .graph import call
        torch.cuda.synchronize()
        out = np.empty(self.n, np.float64)
        call("gbx_pr_shard_unpermute", self.g.handle, r_full.data_ptr(), out.ctypes.data)
        return out

    # ---- triangle count
    def tc_partition(self, world):
        from .graph import call
        b = np.empty(world + 1, np.int64)
        call("gbx_tc_partition", b.ctypes.data, self.g.handle, world)
        return b

    def tc_rows(self, rb, re):
        from .graph import call
        c = C.c_uint64(0)
        call("gbx_triangle_count_rows", C.byref(c), self.g.handle, rb, re)
        return int(c.value)

    # ---- row-sharded BFS (gbx_bfs_shard_*)
    def bfs_begin(self, source, rank, world):
        from .graph import call
        rb, re = C.c_int64(), C.c_int64()
        call("gbx_bfs_shard_begin", self.g.handle, int(source), rank, world, C.byref(rb),
             C.byref(re))
        self.bfs_rb, self.bfs_re = rb.value, re.value
        return self.bfs_rb, self.bfs_re, self.g.n()

    def bfs_level(self, front, nxt):
        import torch

        from .graph import call
        torch.cuda.synchronize()  # the gathered frontier was written on torch's stream
        k = C.c_int64()
        call("gbx_bfs_shard_level", self.g.handle, front.data_ptr(), nxt.data_ptr(), C.byref(k))
        return k.value

    def bfs_result(self):
        from .graph import call
        m = self.bfs_re - self.bfs_rb
        par = np.empty(max(m, 1), np.int64)
        lev = np.empty(max(m, 1), np.int64)
        call("gbx_bfs_shard_result", self.g.handle, par.ctypes.data, lev.ctypes.data)
        return par[:m], lev[:m]

    # ---- betweenness, row-partitioned protocol (gbx_bc_shard_*)
    def bc_begin(self, sources, rank, world):
        from .graph import call
        src = np.ascontiguousarray(sources, np.uint64)
        rb, re = C.c_int64(), C.c_int64()
        call("gbx_bc_shard_begin", self.g.handle, src.ctypes.data, len(src), rank, world,
             C.byref(rb), C.byref(re))
        self.bc_rb, self.bc_re = rb.value, re.value
        return self.bc_rb, self.bc_re

    def _recs(self, ptr, nrec):
        import torch
        if nrec == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.device)
        return torch.as_tensor(_DeviceArray(ptr, nrec * 40, "|u1"), device=self.device)

    def bc_forward(self):
        from .graph import call
        p, k = C.c_void_p(), C.c_int64()
        call("gbx_bc_shard_forward", self.g.handle, C.byref(p), C.byref(k))
        return self._recs(p.value, k.value), k.value

    def bc_forward_apply(self, recs, nrec):
        import torch

        from .graph import call
        torch.cuda.synchronize()  # the gathered records were written on torch's stream
        done = C.c_int(0)
        call("gbx_bc_shard_forward_apply", self.g.handle, recs.data_ptr() if nrec else None,
             nrec, C.byref(done))
        return bool(done.value)

    def bc_backward(self):
        from .graph import call
        p, k, done = C.c_void_p(), C.c_int64(), C.c_int(0)
        call("gbx_bc_shard_backward", self.g.handle, C.byref(p), C.byref(k), C.byref(done))
        return self._recs(p.value, k.value), k.value, bool(done.value)

    def bc_backward_apply(self, recs, nrec):
        import torch

        from .graph import call
        torch.cuda.synchronize()
        call("gbx_bc_shard_backward_apply", self.g.handle, recs.data_ptr() if nrec else None, nrec)

    def bc_centrality(self):
        import torch

        from .graph import call
        p = C.c_void_p()
        call("gbx_bc_shard_centrality", self.g.handle, C.byref(p))
        return torch.as_tensor(_DeviceArray(p.value, self.g.n(), "<f8"), device=self.device)

    # ---- betweenness, sources dealt over ranks
    def bc_partial(self, sources):
        import torch

        from .graph import call
        n = self.g.n()
        if not sources:
            return torch.zeros(n, dtype=torch.float64, device=self.device)
        src = np.ascontiguousarray(sources, np.uint64)
        call("gbx_betweenness", None, self.g.handle, src.ctypes.data, len(src))
        ptr, cnt = self.g.result_device("bc")
        # the library's centrality buffer, reduced in place by NCCL (the call
        # above has synchronised its stream)
        return torch.as_tensor(_DeviceArray(ptr, cnt, "<f8"), device=self.device)
