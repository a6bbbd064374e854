"""Row-partitioned batched Brandes (gbx_bc_shard_*) on one GPU: P ranks are
simulated in one process, each with its own graph handle, exchanging their
per-level records by concatenation (rank order) -- level-synchronous, so no
rank's kernel ever waits on another's.  The summed partials must equal the
single-GPU gbx_betweenness (same per-vertex sums; hub rows' backward partials
are fp64 atomics in both, so agreement is to rounding, 1e-12 relative), and the
oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.dist import GpuShardBackend


def _protocol(bes, srcs):
    world = len(bes)
    for r, be in enumerate(bes):
        be.bc_begin(srcs, r, world)
    assert bes[0].bc_rb == 0 and bes[-1].bc_re == bes[0].g.n()
    for r in range(world - 1):
        assert bes[r].bc_re == bes[r + 1].bc_rb
    levels = 0
    while True:
        outs = [be.bc_forward() for be in bes]
        allr = torch.cat([t.clone() for t, _ in outs]) if any(k for _, k in outs) else \
            torch.empty(0, dtype=torch.uint8, device="cuda")
        tot = sum(k for _, k in outs)
        done = {be.bc_forward_apply(allr, tot) for be in bes}
        assert len(done) == 1
        levels += 1
        if done.pop():
            break
    while True:
        outs = [be.bc_backward() for be in bes]
        flags = {d for _, _, d in outs}
        assert len(flags) == 1
        if flags.pop():
            break
        allr = torch.cat([t.clone() for t, _, _ in outs])
        tot = sum(k for _, k, _ in outs)
        for be in bes:
            be.bc_backward_apply(allr, tot)
    total = sum(be.bc_centrality().clone() for be in bes)
    return total.cpu().numpy(), levels


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_bc_row_shards_equal_single_gpu(world):
    rp, col = O.rmat_graph(15, 16, seed=7, undirected=True)  # hub rows (> 2048) present
    n = len(rp) - 1
    deg = np.diff(rp)
    assert deg.max() > 2048
    srcs = [int(x) for x in P.pick_sources(deg, 4, 3)]
    graphs = []
    for _ in range(world):
        g = P.graph_new(rp, col, kind=P.Kind.UndirectedAdjacency)
        P.property_at(g)
        graphs.append(g)
    got, levels = _protocol([GpuShardBackend(g) for g in graphs], srcs)
    ref = P.graph_new(rp, col, kind=P.Kind.UndirectedAdjacency)
    P.property_at(ref)
    from paper_2104_01661_b200 import algo
    want = np.asarray(algo.betweenness_centrality(ref, srcs).centrality, np.float64)
    assert levels > 3
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max(), np.abs(got - want).max()
    oracle = O.bc(n, rp, col, rp, col, np.asarray(srcs, np.int64))
    assert np.abs(got - oracle).sum() / np.abs(oracle).sum() <= 1e-9
