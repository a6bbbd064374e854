"""The C++ multi-GPU path (gbx_comm / gbx_dgraph / gbx_*_mg) on one B200.

Multi-rank runs use the in-process transport (gbx_comm_init_local: 2..8 ranks
on one GPU, the same protocols with the exchanges as device copies -- ranks
never wait on one another); the NCCL transport runs as a 1-rank communicator
(gbx_comm_init) here and in tests/cpp/mg_nccl.cpp.  Every result is checked
against the single-GPU library and the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2104_01661_b200 as P
from paper_2104_01661_b200 import algo
from paper_2104_01661_b200.mg import MG_AUTO, MG_NCCL, MG_P2P, Comm, DGraph
from tests.gpu_util import rel_l1

pytestmark = pytest.mark.gpu

U, D = P.Kind.UndirectedAdjacency, P.Kind.DirectedAdjacency


def _assemble(g: DGraph):
    """The union of every local rank's block as one CSR."""
    n = g.n
    rp = np.zeros(n + 1, np.int64)
    cols = []
    prev = 0
    for l in range(g.comm.nlocal):
        rb, re, brp, bcol = g.export_block(l)
        assert rb == prev
        prev = re
        rp[rb + 1: re + 1] = np.diff(brp)
        cols.append(bcol)
    assert prev == n
    return np.cumsum(rp), np.concatenate(cols) if cols else np.empty(0, np.int32)


@pytest.mark.parametrize("kind", [D, U])
@pytest.mark.parametrize("nr", [1, 2, 3, 4, 8])
def test_dgraph_blocks_are_the_graph(kind, nr):
    """Local construction (edge slices + all-to-all to the owners) yields the
    single-GPU generator's graph, split into 32-aligned row blocks."""
    P.init(0)
    g = DGraph.rmat(Comm.local(nr), 12, 16, seed=2, kind=kind)
    rp, col = _assemble(g)
    ref = P.generate_rmat(12, 16, seed=2, kind=kind)
    wrp, wcol, _ = ref.export()
    assert np.array_equal(rp, wrp) and np.array_equal(col, wcol)
    assert g.nnz == len(wcol)
    for l in range(nr):
        rb, re, _ = g.block(l)
        assert rb % 32 == 0 and (re % 32 == 0 or re == g.n)


@pytest.mark.parametrize("nr", [1, 2, 4, 8])
@pytest.mark.parametrize("exchange", [MG_AUTO, MG_NCCL, MG_P2P])
def test_pagerank_mg(nr, exchange):
    P.init(0)
    g = DGraph.rmat(Comm.local(nr), 14, 16, seed=1, kind=D)
    got, it = g.pagerank(0.85, 1e-4, 100, exchange)
    ref = P.generate_rmat(14, 16, seed=1, kind=D)
    P.property_at(ref)
    P.property_rowdegree(ref)
    want = algo.pagerank_gap(ref)
    assert it == want.iterations
    # the same relabeling and per-row summation order as the single GPU
    assert np.array_equal(got, want.rank)
    rp, col, _ = ref.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    orc, oit = O.pagerank(n, trp, tcol, np.diff(rp), 0.85, 1e-4, 100)
    assert it == oit and rel_l1(got, orc) <= 1e-4
    # a second call reuses the shard plans and exchange buffers
    got2, it2 = g.pagerank(0.85, 1e-4, 100, exchange)
    assert it2 == it and np.array_equal(got2, got)


def test_pagerank_mg_undirected_and_itermax():
    P.init(0)
    g = DGraph.rmat(Comm.local(3), 12, 8, seed=5, kind=U)
    ref = P.generate_rmat(12, 8, seed=5, kind=U)
    P.property_at(ref)
    P.property_rowdegree(ref)
    got, it = g.pagerank(0.85, 1e-6, 4)
    want = algo.pagerank_gap(ref, 0.85, 1e-6, 4)
    assert it == want.iterations == 4 and np.array_equal(got, want.rank)
    got, it = g.pagerank(0.85, 1e-4, -3)
    assert it == -3 and np.all(got == 1.0 / g.n)


@pytest.mark.parametrize("nr", [1, 2, 3, 8])
def test_triangle_count_mg(nr):
    P.init(0)
    g = DGraph.rmat(Comm.local(nr), 14, 16, seed=3, kind=U)
    ref = P.generate_rmat(14, 16, seed=3, kind=U)
    rp, col, _ = ref.export()
    want = O.triangle_count(len(rp) - 1, rp, col)
    assert g.triangle_count() == want
    assert g.triangle_count() == want  # cached plan


def test_triangle_count_mg_rejects_directed():
    P.init(0)
    g = DGraph.rmat(Comm.local(2), 10, 8, seed=3, kind=D)
    with pytest.raises(P.Error) as e:
        g.triangle_count()
    assert e.value.code == P.ErrCode.InvalidGraph


@pytest.mark.parametrize("push_div", [0, 1, 1 << 30])
@pytest.mark.parametrize("kind", [U, D])
@pytest.mark.parametrize("nr", [1, 2, 4, 8])
def test_bfs_mg(kind, nr, push_div):
    """push levels (candidate marks + a pull over the candidates) while the
    frontier is small, pull levels otherwise; push_div 0 = the edge rule, 1 =
    push (almost) every level, 2^30 = pull only: the same parents and levels
    as the oracle."""
    import ctypes as C

    from paper_2104_01661_b200.graph import call
    P.init(0)
    call("gbx_set_option", b"bfs_mg.push_div", C.c_int64(push_div))
    g = DGraph.rmat(Comm.local(nr), 13, 16, seed=4, kind=kind)
    ref = P.generate_rmat(13, 16, seed=4, kind=kind)
    P.property_rowdegree(ref)
    rp, col, _ = ref.export()
    n = len(rp) - 1
    for s in P.pick_sources(ref.row_degree(), 3, 4):
        par, lev = g.bfs(int(s))
        # along out-edges; parents are the min-id predecessor on the previous level
        wp, wl = O.bfs(n, rp, col, int(s))
        assert np.array_equal(lev, wl)
        assert np.array_equal(par, wp)
    call("gbx_reset_option", b"bfs_mg.push_div")


@pytest.mark.parametrize("nr", [1, 2, 3, 4])
def test_betweenness_mg(nr):
    P.init(0)
    g = DGraph.rmat(Comm.local(nr), 12, 16, seed=6, kind=U)
    ref = P.generate_rmat(12, 16, seed=6, kind=U)
    P.property_at(ref)
    P.property_rowdegree(ref)
    srcs = [int(x) for x in P.pick_sources(ref.row_degree(), 6, 6)]  # two batches (4 + 2)
    got = g.betweenness(srcs)
    want = algo.betweenness_centrality(ref, srcs).centrality
    assert rel_l1(got, want) <= 1e-12
    rp, col, _ = ref.export()
    orc = O.bc(len(rp) - 1, rp, col, rp, col, np.asarray(srcs, np.int64))
    assert rel_l1(got, orc) <= 1e-9


def test_from_blocks_redistributes():
    """Caller-held CSR blocks with an arbitrary (unaligned) split: the library
    shuffles them to its own layout; results match the whole graph."""
    P.init(0)
    ref = P.generate_rmat(12, 16, seed=7, kind=U)
    rp, col, _ = ref.export()
    n = len(rp) - 1
    cuts = [0, 1000, 1001, 3333, n]
    blocks = [(a, b, rp[a:b + 1] - rp[a], col[rp[a]:rp[b]]) for a, b in zip(cuts[:-1], cuts[1:])]
    g = DGraph.from_blocks(Comm.local(4), n, blocks, kind=U)
    arp, acol = _assemble(g)
    assert np.array_equal(arp, rp) and np.array_equal(acol, col)
    assert g.triangle_count() == O.triangle_count(n, rp, col)
    s = int(np.argmax(np.diff(rp)))
    par, lev = g.bfs(s)
    wp, wl = O.bfs(n, rp, col, s)
    assert np.array_equal(par, wp) and np.array_equal(lev, wl)


def test_from_blocks_errors():
    P.init(0)
    c = Comm.local(2)
    rp = np.array([0, 1], np.int64)
    with pytest.raises(P.Error) as e:
        DGraph.from_blocks(c, 4, [(0, 1, rp, np.array([9], np.int32)), (1, 4, np.zeros(4, np.int64), np.zeros(0, np.int32))])
    assert e.value.code == P.ErrCode.IndexOutOfBounds


def test_nccl_transport_one_rank():
    """gbx_comm_init over NCCL (1 rank): every algorithm through the NCCL
    collectives and the IPC peer-buffer path equals the single GPU."""
    P.init(0)
    c = Comm.nccl(1, 0, Comm.unique_id(), 0)
    g = DGraph.rmat(c, 12, 16, seed=1, kind=D)
    ref = P.generate_rmat(12, 16, seed=1, kind=D)
    P.property_at(ref)
    P.property_rowdegree(ref)
    want = algo.pagerank_gap(ref)
    for ex in (MG_P2P, MG_NCCL):
        got, it = g.pagerank(exchange=ex)
        assert it == want.iterations and np.array_equal(got, want.rank)
    u = DGraph.rmat(c, 12, 16, seed=1, kind=U)
    refu = P.generate_rmat(12, 16, seed=1, kind=U)
    rp, col, _ = refu.export()
    assert u.triangle_count() == O.triangle_count(len(rp) - 1, rp, col)
    s = int(np.argmax(np.diff(rp)))
    par, lev = u.bfs(s)
    wp, wl = O.bfs(len(rp) - 1, rp, col, s)
    assert np.array_equal(par, wp) and np.array_equal(lev, wl)
    P.property_at(refu)
    bc = u.betweenness([s, 1, 2])
    assert rel_l1(bc, algo.betweenness_centrality(refu, [s, 1, 2]).centrality) <= 1e-12
