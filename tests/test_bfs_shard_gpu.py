"""Row-sharded BFS (gbx_bfs_shard_*) on one GPU: P ranks simulated in one
process, each with its own graph handle, exchanging their next-frontier bitmap
slices by concatenation -- level-synchronous, no rank's kernel waits on
another's.  Parents and levels must equal the single-GPU gbx_bfs bit for bit."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.dist import GpuShardBackend


def _protocol(bes, source, n):
    world = len(bes)
    bounds = [be.bfs_begin(source, r, world)[:2] for r, be in enumerate(bes)]
    rows = [b[0] for b in bounds] + [bounds[-1][1]]
    assert rows[0] == 0 and rows[-1] == n
    assert all(r % 32 == 0 for r in rows[:-1])
    words = (n + 31) // 32
    wb = [r // 32 for r in rows[:-1]] + [words]
    front = torch.zeros(words, dtype=torch.int32, device="cuda")
    front[source >> 5] = torch.tensor(1 << (source & 31), dtype=torch.int64).to(torch.int32)
    levels = 0
    while True:
        nxts = [torch.zeros(max(wb[r + 1] - wb[r], 1), dtype=torch.int32, device="cuda")
                for r in range(world)]
        found = sum(be.bfs_level(front, nxt) for be, nxt in zip(bes, nxts))
        if found == 0:
            break
        front = torch.cat([nxts[r][: wb[r + 1] - wb[r]] for r in range(world)])
        levels += 1
    par = np.concatenate([be.bfs_result()[0] for be in bes])
    lev = np.concatenate([be.bfs_result()[1] for be in bes])
    return par, lev, levels


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_bfs_row_shards_equal_single_gpu(world):
    rp, col = O.rmat_graph(14, 16, seed=5, undirected=True)
    n = len(rp) - 1
    src = int(P.pick_sources(np.diff(rp), 1, 2)[0])
    graphs = []
    for _ in range(world):
        g = P.graph_new(rp, col, kind=P.Kind.UndirectedAdjacency)
        P.property_at(g)
        graphs.append(g)
    par, lev, levels = _protocol([GpuShardBackend(g) for g in graphs], src, n)
    from paper_2104_01661_b200 import algo
    ref = P.graph_new(rp, col, kind=P.Kind.UndirectedAdjacency)
    P.property_at(ref)
    want = algo.bfs_direction_optimizing(ref, src, algo.BfsConfig(want_level=True))
    assert levels >= 3
    assert np.array_equal(par, want.parent) and np.array_equal(lev, want.level)
    wp, wl = O.bfs(n, rp, col, src)
    assert np.array_equal(par, wp) and np.array_equal(lev, wl)
