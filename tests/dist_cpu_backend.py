"""TEST ONLY: a numpy shard backend with the semantics of libgbx's shard calls
(gbx_pr_shard_*, gbx_tc_partition, gbx_triangle_count_rows, gbx_betweenness),
so the
multi-process driver logic in paper_2104_01661_b200/dist.py runs over gloo on
CPU.  Identity relabeling; fp64 storage."""
import numpy as np
import torch


class CpuShardBackend:
    device = torch.device("cpu")

    def __init__(self, n, rp, col):
        self.n = n
        self.rp = np.asarray(rp, np.int64)
        self.col = np.asarray(col, np.int32)

    # ---- PageRank (rows of AT)
    def prepare(self, rank, world):
        import oracle as O
        self.trp, self.tcol, _ = O.transpose(self.n, self.rp, self.col)
        self.deg = np.diff(self.rp)
        nnz = int(self.trp[-1])

        def split(q):
            if q <= 0:
                return 0
            if q >= world:
                return self.n
            target = (self.n + nnz) * q // world
            lo, hi = 0, self.n
            while lo < hi:
                mid = (lo + hi) // 2
                if mid + self.trp[mid] < target:
                    lo = mid + 1
                else:
                    hi = mid
            return lo
        self.bounds = [0]
        for q in range(1, world + 1):
            self.bounds.append(max(self.bounds[-1], split(q)))
        self.rb, self.re = self.bounds[rank], self.bounds[rank + 1]
        # slot: the longest block + 1 fp64 for the rank's L1 partial (the GPU
        # backend's fp32 slots carry it in their last two floats)
        self.chunk = max(1, max(self.bounds[q + 1] - self.bounds[q] for q in range(world))) + 1
        self.world = world
        # padded exchange layout (gbx_pr_shard_layout): vertex i of owner q at
        # q * chunk + (i - bounds[q])
        own = np.searchsorted(np.asarray(self.bounds[1:]), np.arange(self.n), side="right")
        self.pad = own * self.chunk + (np.arange(self.n) - np.asarray(self.bounds)[own])
        self._x = torch.zeros(world * self.chunk, dtype=torch.float64)
        self._xs = torch.zeros(self.chunk, dtype=torch.float64)
        self._r = [torch.zeros(self.chunk, dtype=torch.float64) for _ in range(2)]
        return self.rb, self.re, self.n

    def init(self, damping):
        r0 = 1.0 / self.n
        x = np.where(self.deg > 0, r0 / (np.maximum(self.deg, 1) / damping), 0.0)
        xf = np.zeros(self.world * self.chunk)
        xf[self.pad] = x
        self._x[:] = torch.from_numpy(xf)
        self._r[0][: self.re - self.rb] = r0

    def step(self, damping, k):
        x = self._x.numpy()[self.pad]
        teleport = (1 - damping) / self.n
        rp, rn_buf = self._r[(k - 1) & 1], self._r[k & 1]
        l1 = 0.0
        for i in range(self.rb, self.re):
            s = float(x[self.tcol[self.trp[i]:self.trp[i + 1]]].sum())
            rn = teleport + s
            l1 += abs(float(rp[i - self.rb]) - rn)
            rn_buf[i - self.rb] = rn
            self._xs[i - self.rb] = rn * damping / self.deg[i] if self.deg[i] > 0 else 0.0
        self._xs[self.chunk - 1] = l1

    # ---- the fused run's orchestration (dist.sharded_pagerank_p2p): the
    # device kernel exchanges x through peer memory; here every rank runs the
    # same sequential iterations on its replicated graph and keeps its rows
    def p2p_setup(self, dist):
        self._p2p_ready = True

    def p2p_init(self, damping):
        assert self._p2p_ready
        self.init(damping)

    def p2p_run(self, damping, tol, itermax):
        import oracle as O
        want, iters = O.pagerank(self.n, self.trp, self.tcol, self.deg, damping, tol, itermax)
        self._p2p_r = torch.zeros(self.chunk, dtype=torch.float64)
        self._p2p_r[: self.re - self.rb] = torch.from_numpy(want[self.rb:self.re].copy())
        return iters

    def p2p_result(self, iters):
        return self._p2p_r

    def l1_post(self, k):
        parts = self._x.view(self.world, self.chunk)[:, self.chunk - 1]
        return sum(float(parts[q]) for q in range(self.world))

    def l1_value(self, tok):
        return tok

    def x_new_slice(self):
        return self._xs

    def x_full(self):
        return self._x

    def r_local(self, k):
        return self._r[k & 1]

    def unpermute(self, r_full):
        return r_full.numpy()[self.pad].copy()

    # ---- triangle count (rows of the id-oriented U)
    def _upper(self, i):
        r = self.col[self.rp[i]:self.rp[i + 1]]
        return r[r > i]

    def tc_partition(self, world):
        work = np.array([sum(len(self._upper(j)) for j in self._upper(i)) + len(self._upper(i))
                         for i in range(self.n)], np.int64)
        total = int(work.sum())
        bounds = [0]
        acc, i = 0, 0
        for p in range(1, world):
            target = total // world * p
            while i < self.n and acc + work[i] <= target:
                acc += work[i]
                i += 1
            bounds.append(i)
        bounds.append(self.n)
        return np.array(bounds, np.int64)

    def tc_rows(self, rb, re):
        c = 0
        for i in range(rb, re):
            ui = set(self._upper(i).tolist())
            for j in self._upper(i):
                c += len(ui.intersection(self._upper(j).tolist()))
        return c

    # ---- betweenness (undirected graph: AT = A)
    def bc_partial(self, sources):
        import oracle as O
        if not sources:
            return torch.zeros(self.n, dtype=torch.float64)
        c = O.bc(self.n, self.rp, self.col, self.rp, self.col, np.asarray(sources, np.int64))
        return torch.from_numpy(np.ascontiguousarray(c, np.float64))


REC = np.dtype([("v", "<i4"), ("lanes", "<u4"), ("x", "<f8", (4,))])  # the 40-byte record


class CpuBcRowsBackend:
    """TEST ONLY: numpy restatement of the gbx_bc_shard_* protocol (row-
    partitioned batched Brandes, betweenness.cpp:11-86): owned rows settle
    their path counts / dependencies, records are exchanged per level."""
    device = torch.device("cpu")

    def __init__(self, n, rp, col):
        self.n = n
        self.rp = np.asarray(rp, np.int64)
        self.col = np.asarray(col, np.int64)  # undirected: AT = A

    def _nb(self, v):
        return self.col[self.rp[v]:self.rp[v + 1]]

    def bc_begin(self, sources, rank, world):
        n, nnz = self.n, int(self.rp[-1])

        def split(q):
            if q <= 0:
                return 0
            if q >= world:
                return n
            target = (n + nnz) * q // world
            lo, hi = 0, n
            while lo < hi:
                mid = (lo + hi) // 2
                if mid + self.rp[mid] < target:
                    lo = mid + 1
                else:
                    hi = mid
            return lo
        self.rb, self.re = split(rank), max(split(rank), split(rank + 1))
        self.ns = len(sources)
        self.level = np.full((n, 4), -1, np.int64)
        self.sigma = np.zeros((n, 4))
        self.coef = np.zeros((n, 4))
        self.cent = np.zeros(n)
        first = []
        for b, s in enumerate(sources):
            self.level[s, b] = 0
            self.sigma[s, b] = 1.0
            if s not in first:
                first.append(s)
        self.order = [np.array(first, np.int64)]
        self.live = (1 << self.ns) - 1
        self.done_fwd = False
        self.bd = None
        return self.rb, self.re

    def _pack(self, vs, vals, lanes):
        r = np.zeros(len(vs), REC)
        r["v"], r["x"], r["lanes"] = vs, vals, lanes
        return torch.from_numpy(r.view(np.uint8).copy()), len(vs)

    def bc_forward(self):
        d = len(self.order)
        vs, lanes = [], []
        for v in range(self.rb, self.re):
            nm = 0
            for b in range(self.ns):
                if not (self.live >> b) & 1 or self.level[v, b] != -1:
                    continue
                u = self._nb(v)
                on = u[self.level[u, b] == d - 1]
                s = float(self.sigma[on, b].sum())
                if s > 0:
                    self.level[v, b] = d
                    self.sigma[v, b] = s
                    nm |= 1 << b
            if nm:
                vs.append(v)
                lanes.append(nm)
        return self._pack(np.array(vs, np.int64), self.sigma[vs] if vs else np.zeros((0, 4)),
                          np.array(lanes, np.uint32))

    def bc_forward_apply(self, recs, nrec):
        d = len(self.order)
        r = recs.numpy().view(REC) if nrec else np.zeros(0, REC)
        live = 0
        for rec in r:
            v, m = int(rec["v"]), int(rec["lanes"])
            live |= m
            if not (self.rb <= v < self.re):
                for b in range(4):
                    if (m >> b) & 1:
                        self.level[v, b] = d
                        self.sigma[v, b] = rec["x"][b]
        self.order.append(r["v"].astype(np.int64))
        self.live = live
        if nrec == 0:
            self.done_fwd = True
        return self.done_fwd

    def bc_backward(self):
        empty = (torch.empty(0, dtype=torch.uint8), 0)
        if self.bd is None:
            D = len(self.order)
            deepest = D - 1
            while deepest > 0 and len(self.order[deepest]) == 0:
                deepest -= 1
            for v in self.order[deepest] if deepest >= 1 else []:
                for b in range(self.ns):
                    if self.level[v, b] == deepest:
                        self.coef[v, b] = 1.0 / self.sigma[v, b]
            self.bd = deepest - 1
        while self.bd >= 1 and len(self.order[self.bd]) == 0:
            self.bd -= 1
        if self.bd < 1:
            return empty[0], 0, True
        d = self.bd
        own = [v for v in self.order[d] if self.rb <= v < self.re]
        for v in own:
            w = self._nb(v)
            for b in range(self.ns):
                if self.level[v, b] != d:
                    continue
                on = w[self.level[w, b] == d + 1]
                acc = float(self.coef[on, b].sum())
                dl = self.sigma[v, b] * acc
                self.cent[v] += dl
                self.coef[v, b] = (1.0 + dl) / self.sigma[v, b]
        t, k = self._pack(np.array(own, np.int64), self.coef[own] if own else np.zeros((0, 4)),
                          np.zeros(len(own), np.uint32))
        return t, k, False

    def bc_backward_apply(self, recs, nrec):
        d = self.bd
        r = recs.numpy().view(REC) if nrec else np.zeros(0, REC)
        for rec in r:
            v = int(rec["v"])
            if not (self.rb <= v < self.re):
                for b in range(4):
                    if self.level[v, b] == d:
                        self.coef[v, b] = rec["x"][b]
        self.bd -= 1

    def bc_centrality(self):
        return torch.from_numpy(self.cent.copy())


class CpuBfsRowsBackend:
    """TEST ONLY: numpy restatement of the gbx_bfs_shard_* protocol (row-
    sharded BFS, bfs.cpp:18-85): owned 32-aligned rows pulled against the
    global frontier bitmap; parent = the first (min-id) frontier in-neighbour."""
    device = torch.device("cpu")

    def __init__(self, n, rp, col):
        self.n = n
        self.rp = np.asarray(rp, np.int64)
        self.col = np.asarray(col, np.int64)  # undirected: AT = A

    def bfs_begin(self, source, rank, world):
        n, nnz = self.n, int(self.rp[-1])
        b = [0]
        for q in range(1, world):
            target = (n + nnz) * q // world
            lo, hi = 0, n
            while lo < hi:
                mid = (lo + hi) // 2
                if mid + self.rp[mid] < target:
                    lo = mid + 1
                else:
                    hi = mid
            b.append(max(b[-1], min(n, (lo + 31) // 32 * 32)))
        b.append(n)
        self.rb, self.re = b[rank], b[rank + 1]
        self.level = np.full(n, -1, np.int64)
        self.parent = np.full(n, -1, np.int64)
        if self.rb <= source < self.re:
            self.level[source] = 0
            self.parent[source] = source
        self.d = 0
        return self.rb, self.re, n

    def bfs_level(self, front, nxt):
        f = front.numpy().view(np.uint32)
        d = self.d + 1
        nxt.zero_()
        nx = nxt.numpy().view(np.uint32)
        found = 0
        for v in range(self.rb, self.re):
            if self.level[v] != -1:
                continue
            for u in self.col[self.rp[v]:self.rp[v + 1]]:
                if (f[u >> 5] >> (u & 31)) & 1:
                    self.level[v] = d
                    self.parent[v] = u
                    nx[(v >> 5) - (self.rb >> 5)] |= np.uint32(1 << (v & 31))
                    found += 1
                    break
        self.d = d
        return found

    def bfs_result(self):
        return self.parent[self.rb:self.re].copy(), self.level[self.rb:self.re].copy()
