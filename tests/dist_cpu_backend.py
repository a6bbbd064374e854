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
        self.rb, self.re = split(rank), max(split(rank), split(rank + 1))
        self._x = torch.zeros(self.n, dtype=torch.float64)
        self._xn = torch.zeros(self.n, dtype=torch.float64)
        self._r = torch.zeros(max(self.re - self.rb, 1), dtype=torch.float64)
        return self.rb, self.re, self.n

    def init(self, damping):
        r0 = 1.0 / self.n
        x = np.where(self.deg > 0, r0 / (np.maximum(self.deg, 1) / damping), 0.0)
        self._x[:] = torch.from_numpy(x)
        self._r[: self.re - self.rb] = r0

    def step(self, damping):
        x = self._x.numpy()
        teleport = (1 - damping) / self.n
        l1 = 0.0
        for i in range(self.rb, self.re):
            s = float(x[self.tcol[self.trp[i]:self.trp[i + 1]]].sum())
            rn = teleport + s
            l1 += abs(float(self._r[i - self.rb]) - rn)
            self._r[i - self.rb] = rn
            self._xn[i] = rn * damping / self.deg[i] if self.deg[i] > 0 else 0.0
        return torch.tensor([l1], dtype=torch.float64)

    def x_new_slice(self):
        return self._xn[self.rb:self.re]

    def x_full(self):
        return self._x

    def r_local(self):
        return self._r[: self.re - self.rb]

    def unpermute(self, r_full):
        return r_full.numpy().copy()

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
