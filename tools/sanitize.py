"""Small fixtures for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every cooperative and hot kernel of libgbx.so on scale-8..10 graphs, results
checked against the oracle so a run that "passes" the tool also computed the
right answer.  One tool per gpurun call (the profiling recipe), e.g.

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (the checker)
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200 import algo  # noqa: E402
from paper_2104_01661_b200.mg import Comm, DGraph  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).sum() / max(np.abs(b).sum(), 1e-300))


def main():
    P.init(0)
    done = []
    # PageRank: k_pr_persist (fp32 and fp64 storage), host-looped k_pr_rows/k_pr_finish
    g = P.generate_rmat(10, 8, seed=1)
    P.property_at(g)
    P.property_rowdegree(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    want, it = O.pagerank(n, trp, tcol, np.diff(rp))
    r = algo.pagerank_gap(g)
    assert r.iterations == it and rel(r.rank, want) <= 1e-4
    r = algo.pagerank_gap(g, 0.85, 1e-9, 60)
    done.append("k_pr_persist")
    from paper_2104_01661_b200.graph import call
    import ctypes as C
    call("gbx_set_option", b"pagerank.host_loop", C.c_int64(1))
    r = algo.pagerank_gap(g)
    call("gbx_reset_option", b"pagerank.host_loop")
    assert r.iterations == it
    done.append("k_pr_rows/k_pr_finish")
    # BFS: k_bfs1 (push / pull / auto), k_bfs64
    u = P.generate_rmat(10, 8, seed=2, kind=P.Kind.UndirectedAdjacency)
    P.property_at(u)
    P.property_rowdegree(u)
    urp, ucol, _ = u.export()
    srcs = P.pick_sources(u.row_degree(), 8, 2)
    for s in srcs[:3]:
        wp, wl = O.bfs(n, urp, ucol, int(s))
        for d in (algo.Direction.Auto, algo.Direction.ForcePush, algo.Direction.ForcePull):
            b = algo.bfs_direction_optimizing(u, int(s), algo.BfsConfig(d, 16, True))
            assert np.array_equal(b.parent, wp) and np.array_equal(b.level, wl)
    par, lev = algo.bfs_batch(u, srcs)
    assert np.array_equal(lev[0], O.bfs(n, urp, ucol, int(srcs[0]))[1])
    done.append("k_bfs1/k_bfs64")
    # triangle count: k_tc_warp / k_tc_cta
    P.property_ndiag(u)
    assert algo.triangle_count(u) == O.triangle_count(n, urp, ucol)
    done.append("k_tc_*")
    # SSSP: k_sssp_b
    e = P.generate_er(10, 8, seed=3)
    P.property_rowdegree(e)
    erp, ecol, ew = e.export()
    s0 = int(P.pick_sources(e.row_degree(), 1, 3)[0])
    dd = algo.sssp_delta_stepping(e, s0, 64.0).dist
    wd = O.dijkstra(len(erp) - 1, erp, ecol, ew.astype(np.float64), s0)
    assert np.array_equal(np.nan_to_num(dd, posinf=-1), np.nan_to_num(wd, posinf=-1))
    done.append("k_sssp_b")
    # BC: push / pull / back + hub passes
    c = algo.betweenness_centrality(u, [int(x) for x in srcs[:4]])
    assert rel(c.centrality, O.bc(n, urp, ucol, urp, ucol, np.asarray(srcs[:4], np.int64))) <= 1e-9
    done.append("k_bc_*")
    # multi-GPU: the one-launch multi-rank fused PageRank + the mg protocols
    dg = DGraph.rmat(Comm.local(3), 10, 8, seed=1, kind=P.Kind.DirectedAdjacency)
    got, it2 = dg.pagerank()
    assert it2 == it and rel(got, want) <= 1e-4
    du = DGraph.rmat(Comm.local(2), 10, 8, seed=2, kind=P.Kind.UndirectedAdjacency)
    assert du.triangle_count() == O.triangle_count(n, urp, ucol)
    pp, ll = du.bfs(int(srcs[0]))
    assert np.array_equal(ll, O.bfs(n, urp, ucol, int(srcs[0]))[1])
    du.betweenness([int(x) for x in srcs[:2]])
    done.append("k_pr_persist_p2p_virt + mg")
    print("sanitize fixtures ok:", ", ".join(done))


if __name__ == "__main__":
    main()
