"""BASELINE.json configs at their FULL sizes on the device: against the oracle
where it finishes within about a minute (PageRank scale 22, BFS scale 22,
triangle count scale 22, BC scale 24) and against a size-independent
certificate for SSSP at 2^24 (feasible potentials + a tight in-edge for every
reached vertex <=> exact shortest-path distances for positive weights).
Config 1 (BFS scale 16, 64 sources) is test_gpu_parity.py::
test_bfs_batch_64_sources_config1."""
import numpy as np
import pytest

import oracle as O
import paper_2104_01661_b200 as P
from paper_2104_01661_b200 import algo
from tests.gpu_util import rel_l1

pytestmark = pytest.mark.gpu


def test_config2_pagerank_scale22_vs_oracle():
    g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.DirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    got = algo.pagerank_gap(g, 0.85, 1e-4, 100)
    rp, col, _ = g.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    want, iters = O.pagerank(n, trp, tcol, np.diff(rp), 0.85, 1e-4, 100)
    assert got.iterations == iters
    assert rel_l1(got.rank, want) <= 1e-4          # north_star tolerance


def test_bfs_scale22_vs_oracle():
    g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    # the 8 sources bench.py times (pick_sources(deg, 64, 1)[:8])
    for s in P.pick_sources(g.row_degree(), 64, 1)[:8]:
        b = algo.bfs_direction_optimizing(g, int(s), algo.BfsConfig(want_level=True))
        wp, wl = O.bfs(n, rp, col, int(s))
        assert np.array_equal(b.level, wl)
        assert np.array_equal(b.parent, wp)        # min-id previous-level parent


def test_config3_triangle_count_scale22_vs_oracle():
    g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_rowdegree(g)
    P.property_ndiag(g)
    got = algo.triangle_count(g)
    rp, col, _ = g.export()
    assert got == O.triangle_count(len(rp) - 1, rp, col)


def test_config4_sssp_2e24_certificate():
    import torch
    g = P.generate_er(24, 16, seed=1)
    P.property_rowdegree(g)
    rp, col, w = g.export()
    n = len(rp) - 1
    dev = torch.device("cuda", 0)
    rows = torch.repeat_interleave(torch.arange(n, device=dev),
                                   torch.from_numpy(np.diff(rp)).to(dev))
    cols = torch.from_numpy(col.astype(np.int64)).to(dev)
    wt = torch.from_numpy(np.asarray(w, np.float64)).to(dev)
    for s in P.pick_sources(g.row_degree(), 16, 1):
        d = algo.sssp_delta_stepping(g, int(s), 64.0).dist
        D = torch.from_numpy(d).to(dev)
        assert float(D[int(s)]) == 0.0
        fin = torch.isfinite(D)
        assert bool((D[fin] == torch.round(D[fin])).all())      # exact integers
        du, dv = D[rows], D[cols]
        reach_u = torch.isfinite(du)
        # feasible: no edge out of a reached vertex can still improve its head
        assert bool((dv[reach_u] <= du[reach_u] + wt[reach_u]).all())
        # tight: every reached vertex but the source has an in-edge with
        # dist(v) = dist(u) + w, u reached (positive weights: these lead back to s)
        tight = reach_u & (dv == du + wt)
        has = torch.zeros(n, dtype=torch.int32, device=dev)
        has.index_fill_(0, cols[tight], 1)
        need = fin.clone()
        need[int(s)] = False
        assert bool((has[need] == 1).all())


def test_config5_betweenness_scale24_vs_oracle():
    g = P.generate_rmat(24, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    srcs = [int(x) for x in P.pick_sources(g.row_degree(), 4, 1)]
    got = algo.betweenness_centrality(g, srcs).centrality
    rp, col, _ = g.export()
    want = O.bc(len(rp) - 1, rp, col, rp, col, srcs)
    assert rel_l1(got, want) <= 1e-4                # north_star tolerance
