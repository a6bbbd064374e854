"""Parity of the CUDA library (through the C ABI) against the reference's own
outputs (tests/golden) and the oracle restatement.  Needs a B200."""
import ctypes as C
import numpy as np
import pytest

import oracle as O
import paper_2104_01661_b200 as P
from paper_2104_01661_b200 import algo
from paper_2104_01661_b200.graph import call
from tests.golden_util import Golden, case_ids
from tests.gpu_util import graph_of, rel_l1

pytestmark = pytest.mark.gpu
G = Golden()
CASES = {c.name: c for c in G.cases}


# ---------------------------------------------------------------- BFS
@pytest.mark.parametrize("name", case_ids("bfs"))
def test_bfs_golden(name):
    c = CASES[name]
    g = graph_of(c)
    src = c.params["src"]
    r = algo.bfs_push(g, src, want_level=True)
    assert np.array_equal(r.parent, c.out["parent_pushonly"])
    assert np.array_equal(r.level, c.out["level_pushonly"])
    P.property_at(g)
    for d, tag in ((algo.Direction.Auto, "auto"), (algo.Direction.ForcePush, "push"),
                   (algo.Direction.ForcePull, "pull")):
        r = algo.bfs_direction_optimizing(g, src, algo.BfsConfig(d, 16, True))
        assert np.array_equal(r.parent, c.out[f"parent_{tag}"]), tag
        assert np.array_equal(r.level, c.out[f"level_{tag}"]), tag


@pytest.mark.parametrize("name", case_ids("bfs"))
def test_bfs_batch_golden(name):
    c = CASES[name]
    g = graph_of(c)
    P.property_at(g)
    src = c.params["src"]
    sources = [src] * 3 + list(range(min(c.n, 5)))
    parent, level = algo.bfs_batch(g, sources)
    for b, s in enumerate(sources):
        wp, wl = O.bfs(c.n, c.rp, c.col, s)
        assert np.array_equal(parent[b], wp) and np.array_equal(level[b], wl), b


def test_bfs_errors():
    c = CASES["bfs_path3"]
    g = graph_of(c)
    with pytest.raises(P.Error) as e:
        algo.bfs_direction_optimizing(g, 0)
    assert e.value.code == P.ErrCode.MissingProperty
    assert not g.has_AT  # no silent computation (test_bfs.cpp:53-64)
    with pytest.raises(P.Error) as e:
        algo.bfs_push(g, 3)
    assert e.value.code == P.ErrCode.SourceOutOfRange
    r = algo.basic.bfs_direction_optimizing(g, 0, algo.BfsConfig(want_level=True))
    assert g.has_AT and r.level.tolist() == [0, 1, 2]


@pytest.mark.parametrize("scale,seed", [(14, 1), (16, 2)])
def test_bfs_rmat_vs_oracle(scale, seed):
    g = P.generate_rmat(scale, 16, seed=seed, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    P.property_rowdegree(g)
    srcs = P.pick_sources(g.row_degree(), 8, seed)
    for s in srcs:
        wp, wl = O.bfs(n, rp, col, s)
        for d in (algo.Direction.Auto, algo.Direction.ForcePush, algo.Direction.ForcePull):
            r = algo.bfs_direction_optimizing(g, int(s), algo.BfsConfig(d, 16, True))
            assert np.array_equal(r.level, wl) and np.array_equal(r.parent, wp)
    parent, level = algo.bfs_batch(g, srcs)
    for b, s in enumerate(srcs):
        wp, wl = O.bfs(n, rp, col, s)
        assert np.array_equal(parent[b], wp) and np.array_equal(level[b], wl)


def test_bfs_batch_64_sources_config1():
    """BASELINE config 1 shape: R-MAT scale 16 undirected, 64 seeded sources."""
    g = P.generate_rmat(16, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    srcs = P.pick_sources(g.row_degree(), 64, 1)
    parent, level = algo.bfs_batch(g, srcs)
    for b in range(64):  # every source of the config (the bench times all 64)
        wp, wl = O.bfs(n, rp, col, srcs[b])
        assert np.array_equal(parent[b], wp) and np.array_equal(level[b], wl)


# ---------------------------------------------------------------- PageRank
@pytest.mark.parametrize("name", case_ids("pagerank"))
def test_pagerank_golden(name):
    c = CASES[name]
    g = graph_of(c)
    P.property_at(g)
    P.property_rowdegree(g)
    prm = c.params
    r = algo.pagerank_gap(g, prm["damping"], prm["tol"], prm["itermax"])
    assert r.iterations == int(c.out["iters"])
    want = c.out["rank"]
    assert rel_l1(r.rank, want) <= 1e-4
    assert np.max(np.abs(r.rank - want)) <= 1e-6


def test_pagerank_fixed_points():
    # test_pr.cpp:24-38: 2- and 3-cycles settle at the uniform fixpoint
    for name, v in (("pr_cycle2", 0.5), ("pr_cycle3", 1.0 / 3)):
        g = graph_of(CASES[name])
        r = algo.basic.pagerank_gap(g, 0.85, 1e-8, 100)
        assert np.all(np.abs(r.rank - v) <= 1e-7)


def test_pagerank_errors_and_cap():
    g = graph_of(CASES["pr_cycle3"])
    with pytest.raises(P.Error) as e:
        algo.pagerank_gap(g)
    assert e.value.code == P.ErrCode.MissingProperty
    P.property_at(g)
    with pytest.raises(P.Error) as e:
        algo.pagerank_gap(g)
    assert e.value.code == P.ErrCode.MissingProperty
    P.property_rowdegree(g)
    for bad in (0.0, -0.5):
        with pytest.raises(P.Error) as e:
            algo.pagerank_gap(g, bad)
        assert e.value.code == P.ErrCode.NonPositiveDamping
    assert algo.pagerank_gap(g, 0.85, 0.0, 7).iterations == 7


@pytest.mark.parametrize("scale", [16, 18])
def test_pagerank_rmat_vs_oracle(scale):
    g = P.generate_rmat(scale, 16, seed=5, kind=P.Kind.DirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    r = algo.pagerank_gap(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    want, iters = O.pagerank(n, trp, tcol, np.diff(rp))
    assert r.iterations == iters
    assert rel_l1(r.rank, want) <= 1e-4


def test_pagerank_repeatable():
    g = P.generate_rmat(14, 16, seed=9)
    P.property_at(g)
    P.property_rowdegree(g)
    a = algo.pagerank_gap(g)
    b = algo.pagerank_gap(g)
    assert a.iterations == b.iterations
    assert np.array_equal(a.rank, b.rank)


# ---------------------------------------------------------------- CC
@pytest.mark.parametrize("name", case_ids("cc"))
def test_cc_golden(name):
    c = CASES[name]
    g = graph_of(c)
    r = algo.connected_components_fastsv(g)
    assert np.array_equal(r.label, c.out["label"])


def test_cc_rmat_vs_oracle():
    g = P.generate_rmat(16, 4, seed=3, kind=P.Kind.UndirectedAdjacency)
    rp, col, _ = g.export()
    r = algo.connected_components_fastsv(g)
    assert np.array_equal(r.label, O.cc(len(rp) - 1, rp, col))
    again = algo.connected_components_fastsv(g)
    assert np.array_equal(again.label, r.label)


# ---------------------------------------------------------------- graph layer
@pytest.mark.parametrize("und", [False, True])
def test_generator_matches_oracle(und):
    for scale in (8, 12):
        g = P.generate_rmat(scale, 16, seed=7,
                            kind=P.Kind.UndirectedAdjacency if und else P.Kind.DirectedAdjacency)
        rp, col, _ = g.export()
        wrp, wcol = O.rmat_graph(scale, 16, seed=7, undirected=und)
        assert np.array_equal(rp, wrp) and np.array_equal(col, wcol)
    g = P.generate_er(12, 16, seed=3)
    rp, col, w = g.export()
    wrp, wcol, ww = O.er_graph(12, 16, seed=3)
    assert np.array_equal(rp, wrp) and np.array_equal(col, wcol) and np.array_equal(w, ww)


def test_graph_object_caches():
    c = CASES["bfs_randdi0"]
    g = graph_of(c)
    props = g.properties()
    assert not props["AT"] and not props["row_degree"] and props["ndiag"] == -1
    P.property_at(g)
    P.property_rowdegree(g)
    P.property_coldegree(g)
    P.property_ndiag(g)
    P.property_symmetric_pattern(g)
    assert P.check_graph(g)[0] == 0
    assert np.array_equal(g.row_degree(), np.diff(c.rp))
    assert np.array_equal(g.col_degree(), np.bincount(c.col, minlength=c.n))
    P.delete_properties(g)
    assert not g.has_AT and g.ndiag == -1


def test_graph_new_rejects_corrupt_matrix():
    # test_graph.cpp:24-32: an unsorted row
    with pytest.raises(P.Error) as e:
        P.graph_new(np.array([0, 2, 2]), np.array([1, 0]))
    assert e.value.code == P.ErrCode.InvalidMatrix
    with pytest.raises(P.Error) as e:
        P.graph_new(np.array([0, 1, 1]), np.array([5]))
    assert e.value.code == P.ErrCode.InvalidMatrix


def test_graph_new32_chunked_upload():
    """graph_new (graph.cpp:16-28) from a host CSR larger than one upload chunk
    (8 Mi int32 columns): the chunks are validated and counted as they arrive
    (csrc/graph.cu build_from_host).  The round trip is exact, a fault ON a chunk
    boundary is found (containers.cpp:104-124), and PageRank on the uploaded
    graph equals PageRank on the same graph built on the device bit for bit (its
    plan reuses the column counts taken during the upload)."""
    gd = P.generate_rmat(20, 16, seed=5, kind=P.Kind.DirectedAdjacency)
    rp, col, _ = gd.export()
    col = np.ascontiguousarray(col, np.int32)
    chunk = 8 << 20
    assert len(col) > chunk + 1
    gh = P.graph_new(rp, col)
    rp2, col2, _ = gh.export()
    assert np.array_equal(rp2, rp) and np.array_equal(col2, col)
    for g in (gd, gh):
        P.property_at(g)
        P.property_rowdegree(g)
    a, b = algo.pagerank_gap(gd), algo.pagerank_gap(gh)
    assert a.iterations == b.iterations and np.array_equal(a.rank, b.rank)
    # entry `chunk` is the first of the second chunk: make it repeat its
    # predecessor inside one row, then point it out of range
    row = int(np.searchsorted(rp, chunk, side="right")) - 1
    if rp[row] == chunk:  # it starts a row: use the next entry pair inside a row instead
        row = next(r for r in range(row, len(rp) - 1) if rp[r + 1] - rp[r] >= 2 and rp[r] >= chunk)
    bad = col.copy()
    k = max(int(rp[row]) + 1, chunk)
    bad[k] = bad[k - 1]
    with pytest.raises(P.Error) as e:
        P.graph_new(rp, bad)
    assert e.value.code == P.ErrCode.InvalidMatrix
    bad = col.copy()
    bad[chunk] = len(rp) - 1  # == n: out of range
    with pytest.raises(P.Error) as e:
        P.graph_new(rp, bad)
    assert e.value.code == P.ErrCode.InvalidMatrix


@pytest.mark.parametrize("name", case_ids("sort_by_degree"))
def test_sort_by_degree_golden(name):
    c = CASES[name]
    g = graph_of(c)
    P.property_rowdegree(g)
    assert np.array_equal(P.sort_by_degree(g, True, True), c.out["perm"])


# ---------------------------------------------------------------- triangle count
def _tc_ready(c):
    g = graph_of(c)
    P.property_rowdegree(g)
    P.property_ndiag(g)
    return g


@pytest.mark.parametrize("name", case_ids("triangle_count"))
def test_tc_golden(name):
    c = CASES[name]
    g = _tc_ready(c)
    for ps, tag in ((algo.Presort.Auto, "auto"), (algo.Presort.Force, "force"),
                    (algo.Presort.Never, "never")):
        assert algo.triangle_count(g, algo.TriangleCountConfig(ps)) == int(c.out[f"count_{tag}"])


def test_tc_preconditions():
    c = CASES["tc_K3"]
    g = graph_of(c)
    P.property_rowdegree(g)
    with pytest.raises(P.Error) as e:
        algo.triangle_count(g)
    assert e.value.code == P.ErrCode.MissingProperty
    # self loop on a directed-kind graph marked symmetric (test_tc.cpp:100-112)
    rp = np.array([0, 2, 5, 7])
    col = np.array([1, 2, 0, 1, 2, 0, 1])
    bad = P.graph_new(rp, col, kind=P.Kind.DirectedAdjacency)
    P.property_symmetric_pattern(bad)
    P.property_ndiag(bad)
    P.property_rowdegree(bad)
    with pytest.raises(P.Error) as e:
        algo.triangle_count(bad)
    assert e.value.code == P.ErrCode.PreconditionViolated
    d = P.graph_new(np.array([0, 1, 2, 2]), np.array([1, 2]), kind=P.Kind.DirectedAdjacency)
    P.property_symmetric_pattern(d)
    P.property_ndiag(d)
    P.property_rowdegree(d)
    with pytest.raises(P.Error) as e:
        algo.triangle_count(d)
    assert e.value.code == P.ErrCode.PreconditionViolated
    fresh = graph_of(CASES["tc_K4"])
    assert algo.basic.triangle_count(fresh) == 4
    assert fresh.ndiag == 0


@pytest.mark.parametrize("scale", [14, 16])
def test_tc_rmat_vs_oracle(scale):
    g = P.generate_rmat(scale, 16, seed=4, kind=P.Kind.UndirectedAdjacency)
    rp, col, _ = g.export()
    want = O.triangle_count(len(rp) - 1, rp, col)
    assert algo.basic.triangle_count(g) == want


# ---------------------------------------------------------------- SSSP
@pytest.mark.parametrize("name", case_ids("sssp"))
def test_sssp_golden(name):
    c = CASES[name]
    g = graph_of(c)
    for d in c.params["deltas"]:
        r = algo.sssp_delta_stepping(g, c.params["src"], d)
        assert np.array_equal(r.dist, c.out[f"dist_{d:g}"]), d
    assert algo.sssp_default_delta(g) == c.params["default_delta"]


def test_sssp_errors():
    g = P.graph_new(np.array([0, 1, 1]), np.array([1]), np.array([1.0]))
    for src, delta, code in ((5, 1.0, P.ErrCode.SourceOutOfRange),
                             (0, 0.0, P.ErrCode.NonPositiveDelta),
                             (0, -1.0, P.ErrCode.NonPositiveDelta)):
        with pytest.raises(P.Error) as e:
            algo.sssp_delta_stepping(g, src, delta)
        assert e.value.code == code
    neg = P.graph_new(np.array([0, 1, 1]), np.array([1]), np.array([-2.0]))
    with pytest.raises(P.Error) as e:
        algo.sssp_delta_stepping(neg, 0, 1.0)
    assert e.value.code == P.ErrCode.NonPositiveWeight
    ints = P.graph_new(np.array([0, 1, 1]), np.array([1]), np.array([1], np.int64))
    with pytest.raises(P.Error) as e:
        algo.sssp_delta_stepping(ints, 0, 1.0)
    assert e.value.code == P.ErrCode.DomainMismatch
    # basic wrapper: delta = max / 2 (test_sssp.cpp:113-121)
    b = P.graph_new(np.array([0, 1, 2, 2]), np.array([1, 2]), np.array([3.0, 6.0]))
    assert algo.basic.sssp_delta_stepping(b, 0).dist[2] == 9.0


@pytest.mark.parametrize("logn", [12, 16])
def test_sssp_er_vs_oracle(logn):
    g = P.generate_er(logn, 16, seed=6)
    rp, col, w = g.export()
    n = len(rp) - 1
    P.property_rowdegree(g)
    for s in P.pick_sources(g.row_degree(), 3, 6):
        want = O.dijkstra(n, rp, col, w.astype(np.float64), s)
        for delta in (64.0, 16.0, 1000.0):
            got = algo.sssp_delta_stepping(g, int(s), delta).dist
            assert np.array_equal(got, want)


@pytest.mark.parametrize("pct", [1, 100, 0])
def test_sssp_heavy_pull_vs_oracle(pct):
    """the pull form of the heavy pass (sssp.pull_pct; 1: nearly every bucket,
    0: never) on uniform, sparse (unreachable vertices) and skewed graphs, with
    integral, power-of-two and non-integral deltas: distances equal Dijkstra"""
    from paper_2104_01661_b200.graph import call
    rng = np.random.default_rng(5)
    graphs = [P.generate_er(13, 16, seed=7), P.generate_er(12, 2, seed=8)]
    r0 = P.generate_rmat(12, 8, seed=9)
    rp0, col0, _ = r0.export()
    graphs.append(P.graph_new(rp0, col0, rng.integers(1, 256, len(col0)).astype(np.float64)))
    call("gbx_set_option", b"sssp.pull_pct", C.c_int64(pct))
    try:
        for g in graphs:
            rp, col, w = g.export()
            n = len(rp) - 1
            P.property_rowdegree(g)
            for s in P.pick_sources(g.row_degree(), 2, 4):
                want = O.dijkstra(n, rp, col, w.astype(np.float64), int(s))
                for delta in (64.0, 16.0, 37.5, 200.0, 3.0):
                    got = algo.sssp_delta_stepping(g, int(s), delta).dist
                    assert np.array_equal(got, want), (n, delta)
    finally:
        call("gbx_reset_option", b"sssp.pull_pct")


def test_sssp_fp64_weights_vs_oracle():
    rng = np.random.default_rng(3)
    g0 = P.generate_rmat(12, 8, seed=2)
    rp, col, _ = g0.export()
    w = rng.uniform(1e-3, 10.0, len(col))
    g = P.graph_new(rp, col, w)
    n = len(rp) - 1
    for s in (0, 1, 17):
        want = O.dijkstra(n, rp, col, w, s)
        for delta in (0.5, 2.0, 8.0):
            assert np.array_equal(algo.sssp_delta_stepping(g, s, delta).dist, want)


# ---------------------------------------------------------------- betweenness
@pytest.mark.parametrize("name", case_ids("bc"))
def test_bc_golden(name):
    c = CASES[name]
    g = graph_of(c)
    P.property_at(g)
    got = algo.betweenness_centrality(g, c.params["sources"]).centrality
    want = c.out["centrality"]
    # test_bc.cpp:74-91 accepts 1e-9 absolute against Brandes
    assert np.max(np.abs(got - want), initial=0.0) <= 1e-9


def test_bc_errors_and_basic():
    c = CASES["bc_path3"]
    g = graph_of(c)
    with pytest.raises(P.Error) as e:
        algo.betweenness_centrality(g, [0])
    assert e.value.code == P.ErrCode.MissingProperty
    P.property_at(g)
    with pytest.raises(P.Error) as e:
        algo.betweenness_centrality(g, [])
    assert e.value.code == P.ErrCode.EmptyBatch
    with pytest.raises(P.Error) as e:
        algo.betweenness_centrality(g, [7])
    assert e.value.code == P.ErrCode.SourceOutOfRange
    g2 = graph_of(CASES["bc_star4"])
    b = algo.basic.betweenness_centrality(g2, [0, 1, 2, 3, 4]).centrality
    assert np.allclose(b, CASES["bc_star4"].out["centrality"], atol=1e-12)


@pytest.mark.parametrize("und", [True, False])
def test_bc_rmat_vs_oracle(und):
    kind = P.Kind.UndirectedAdjacency if und else P.Kind.DirectedAdjacency
    g = P.generate_rmat(14, 16, seed=8, kind=kind)
    P.property_at(g)
    P.property_rowdegree(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    srcs = P.pick_sources(g.row_degree(), 6, 8)
    got = algo.betweenness_centrality(g, srcs).centrality
    want = O.bc(n, rp, col, trp, tcol, srcs)
    assert rel_l1(got, want) <= 1e-9


@pytest.mark.parametrize("und", [True, False])
def test_bc_rmat16_hubs_vs_oracle(und):
    """Scale 16: rows longer than the hub threshold take the chunked passes, and
    the middle levels are pulled."""
    kind = P.Kind.UndirectedAdjacency if und else P.Kind.DirectedAdjacency
    g = P.generate_rmat(16, 16, seed=3, kind=kind)
    P.property_at(g)
    P.property_rowdegree(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    assert np.diff(rp).max() > 2048 or np.diff(trp).max() > 2048
    srcs = P.pick_sources(g.row_degree(), 4, 3)
    got = algo.betweenness_centrality(g, srcs).centrality
    want = O.bc(n, rp, col, trp, tcol, srcs)
    assert rel_l1(got, want) <= 1e-9


def _undirected(n, edges):
    import scipy.sparse as sp
    e = np.asarray(edges, np.int64)
    r = np.concatenate([e[:, 0], e[:, 1]])
    c = np.concatenate([e[:, 1], e[:, 0]])
    m = sp.csr_matrix((np.ones(len(r)), (r, c)), shape=(n, n))
    m.sum_duplicates()
    m.sort_indices()
    return m.indptr.astype(np.int64), m.indices.astype(np.int32)


def test_bc_deep_path_and_components():
    """Depths past 254 (the one-byte level filter saturates) and a lane whose
    source sits in a small component (its lane dies early)."""
    n_path = 700
    edges = [(i, i + 1) for i in range(n_path - 1)]
    # a second component: a star with a tail, plus an isolated vertex
    base = n_path
    edges += [(base, base + k) for k in range(1, 40)] + [(base + 39, base + 40)]
    n = base + 42
    rp, col = _undirected(n, edges)
    g = P.graph_new(rp, col, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    trp, tcol = rp, col
    for srcs in ([0, 350, base + 5, 699], [3, base], [base + 41]):
        got = algo.betweenness_centrality(g, srcs).centrality
        want = O.bc(n, rp, col, trp, tcol, np.asarray(srcs, np.int64))
        assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, np.abs(want).max())


class _bc_relabeled:
    """bc.relabel_min_n = 0: every graph runs Brandes on its degree-sorted copy
    (csrc/bc.cu ensure_relabel; the default only does so from 2^18 vertices)."""

    def __enter__(self):
        call("gbx_set_option", b"bc.relabel_min_n", C.c_int64(0))

    def __exit__(self, *exc):
        call("gbx_reset_option", b"bc.relabel_min_n")


@pytest.mark.parametrize("name", case_ids("bc"))
def test_bc_golden_on_degree_sorted_copy(name):
    c = CASES[name]
    g = graph_of(c)
    P.property_at(g)
    with _bc_relabeled():
        got = algo.betweenness_centrality(g, c.params["sources"]).centrality
    assert np.max(np.abs(got - c.out["centrality"]), initial=0.0) <= 1e-9


@pytest.mark.parametrize("und", [True, False])
@pytest.mark.parametrize("scale,nsrc", [(14, 6), (16, 4)])
def test_bc_rmat_on_degree_sorted_copy(und, scale, nsrc):
    """The degree-sorted copy against the oracle and against the run on the
    original ids (same sums in another fp64 order), directed and undirected,
    with hub rows (scale 16) and two batches (6 sources)."""
    kind = P.Kind.UndirectedAdjacency if und else P.Kind.DirectedAdjacency
    g = P.generate_rmat(scale, 16, seed=8, kind=kind)
    P.property_at(g)
    P.property_rowdegree(g)
    rp, col, _ = g.export()
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    srcs = P.pick_sources(g.row_degree(), nsrc, 8)
    plain = algo.betweenness_centrality(g, srcs).centrality
    with _bc_relabeled():
        got = algo.betweenness_centrality(g, srcs).centrality
        again = algo.betweenness_centrality(g, srcs[:3]).centrality  # the copy is cached
    want = O.bc(n, rp, col, trp, tcol, srcs)
    assert rel_l1(got, want) <= 1e-9
    assert rel_l1(got, plain) <= 1e-12
    assert rel_l1(again, O.bc(n, rp, col, trp, tcol, srcs[:3])) <= 1e-9


@pytest.mark.parametrize("relabel", [False, True])
def test_bc_backward_push_form(relabel):
    """The backward sweep in push form (csrc/bc.cu k_bc_back_push: children add
    their coefficients into their parents' sums) forced at every depth
    (bc.back_push = 1 accepts any edge ratio >= 1, min depth 1), against the
    oracle and the pull form: goldens, R-MAT 14 / 16 directed and undirected."""
    try:
        call("gbx_set_option", b"bc.back_push", C.c_int64(1))
        call("gbx_set_option", b"bc.back_push_min_depth", C.c_int64(1))
        if relabel:
            call("gbx_set_option", b"bc.relabel_min_n", C.c_int64(0))
        for name in case_ids("bc"):
            c = CASES[name]
            g = graph_of(c)
            P.property_at(g)
            got = algo.betweenness_centrality(g, c.params["sources"]).centrality
            assert np.max(np.abs(got - c.out["centrality"]), initial=0.0) <= 1e-9, name
        for scale, und in ((14, True), (14, False), (16, True), (16, False)):
            kind = P.Kind.UndirectedAdjacency if und else P.Kind.DirectedAdjacency
            g = P.generate_rmat(scale, 16, seed=8, kind=kind)
            P.property_at(g)
            P.property_rowdegree(g)
            rp, col, _ = g.export()
            n = len(rp) - 1
            trp, tcol, _ = O.transpose(n, rp, col)
            srcs = P.pick_sources(g.row_degree(), 6, 8)
            got = algo.betweenness_centrality(g, srcs).centrality
            st = g.last_stats()
            assert rel_l1(got, O.bc(n, rp, col, trp, tcol, srcs)) <= 1e-9, (scale, und)
            call("gbx_set_option", b"bc.back_push", C.c_int64(0))
            pull = algo.betweenness_centrality(g, srcs).centrality
            assert g.last_stats()["launches"] != st["launches"]  # the push form did run
            call("gbx_set_option", b"bc.back_push", C.c_int64(1))
            assert rel_l1(got, pull) <= 1e-12, (scale, und)
    finally:
        for o in (b"bc.back_push", b"bc.back_push_min_depth", b"bc.relabel_min_n"):
            call("gbx_reset_option", o)


def test_bc_deep_path_on_degree_sorted_copy():
    n_path = 700
    edges = [(i, i + 1) for i in range(n_path - 1)]
    base = n_path
    edges += [(base, base + k) for k in range(1, 40)] + [(base + 39, base + 40)]
    n = base + 42
    rp, col = _undirected(n, edges)
    g = P.graph_new(rp, col, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    with _bc_relabeled():
        for srcs in ([0, 350, base + 5, 699], [3, base], [base + 41]):
            got = algo.betweenness_centrality(g, srcs).centrality
            want = O.bc(n, rp, col, rp, col, np.asarray(srcs, np.int64))
            assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, np.abs(want).max())


# ---------------------------------------------------------------- multi-GPU shard kernels
def test_bc_partials_compose_on_one_gpu():
    """The sharded BC driver's per-rank partials (dist.GpuShardBackend.bc_partial,
    a view of the library's device buffer) sum to the full batch."""
    import torch
    from paper_2104_01661_b200.dist import GpuShardBackend
    g = P.generate_rmat(13, 16, seed=4, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    srcs = [int(x) for x in P.pick_sources(g.row_degree(), 6, 4)]
    be = GpuShardBackend(g)
    parts = [be.bc_partial(srcs[r::2]).clone() for r in range(2)]
    assert parts[0].is_cuda and parts[0].dtype == torch.float64
    got = (parts[0] + parts[1]).cpu().numpy()
    want = algo.betweenness_centrality(g, srcs).centrality
    assert rel_l1(got, want) <= 1e-12
    assert float(be.bc_partial([]).abs().sum()) == 0.0


@pytest.mark.parametrize("world", [1, 2, 3])
def test_pr_shards_compose_on_one_gpu(world):
    """`world` shard plans stepped in lockstep with the padded all-gather done
    by hand equal the single-GPU PageRank: the shard kernels plus the
    driver's padded layout, double-buffered r and the lagged convergence test
    (dist.sharded_pagerank) without NCCL (the ranks never wait on each other)."""
    import torch
    from paper_2104_01661_b200.dist import GpuShardBackend
    bes = []
    for r in range(world):
        g = P.generate_rmat(14, 16, seed=5)
        P.property_at(g)
        P.property_rowdegree(g)
        be = GpuShardBackend(g)
        be.g_keep = g
        rb, re, n = be.prepare(r, world)
        bes.append(be)
    chunk = bes[0].chunk
    assert all(be.chunk == chunk for be in bes)
    assert bes[0].rb == 0 and bes[-1].re == n
    assert all(bes[q].re == bes[q + 1].rb for q in range(world - 1))
    assert all(be.re - be.rb <= chunk for be in bes)
    for be in bes:
        be.init(0.85)
    pending, iters = None, 0
    for k in range(1, 101):
        for be in bes:
            be.step(0.85, k)
        torch.cuda.synchronize()
        for be in bes:  # all_gather_into_tensor, by hand
            for q, src in enumerate(bes):
                be.x_full()[q * chunk:(q + 1) * chunk] = src.x_new_slice()
        torch.cuda.synchronize()
        l1s = [be.l1_value(be.l1_post(k)) for be in bes]
        assert all(v == l1s[0] for v in l1s)  # the same rank-order sum everywhere
        l1 = l1s[0]
        if pending is not None and not (pending[1] >= 1e-4):
            iters = pending[0]
            break
        pending = (k, l1)
    else:
        iters = pending[0]
    r_full = torch.cat([be.r_local(iters) for be in bes])
    got = bes[0].unpermute(r_full)
    ref = P.generate_rmat(14, 16, seed=5)
    P.property_at(ref)
    P.property_rowdegree(ref)
    want = algo.pagerank_gap(ref)
    assert iters == want.iterations
    assert rel_l1(got, want.rank) <= 1e-6


def test_tc_partition_rows_sum():
    g = P.generate_rmat(14, 16, seed=4, kind=P.Kind.UndirectedAdjacency)
    P.property_ndiag(g)
    from paper_2104_01661_b200.dist import GpuShardBackend
    be = GpuShardBackend(g)
    b = be.tc_partition(4)
    assert b[0] == 0 and np.all(np.diff(b) >= 0)
    parts = [be.tc_rows(int(b[p]), int(b[p + 1])) for p in range(4)]
    assert sum(parts) == algo.basic.triangle_count(g)


@pytest.mark.parametrize("with_zero_rows", [True, False])
def test_pagerank_bin_boundary_lengths(with_zero_rows):
    """In-degrees ON the plan's class boundaries (csrc/pagerank.cu: thread-per-row
    bins up to 80 nonzeros, warp-per-row up to 2048, 1024-nonzero chunks beyond;
    rows without in-edges claimed dynamically) against the oracle
    (pagerank.cpp:8-81): same iteration count, rel. L1 <= 1e-4 -- with and
    without empty rows, fp32 and fp64 storage."""
    rng = np.random.default_rng(11)
    n = 4096
    lens = [1, 2, 3, 4, 5, 31, 32, 33, 63, 64, 65, 79, 80, 81, 82, 127, 128, 129, 255, 256, 257,
            1023, 1024, 1025, 2047, 2048, 2049, 2050, 3071, 3072, 3073, 4000]
    if with_zero_rows:
        lens += [0] * 7
    indeg = np.array([lens[i % len(lens)] for i in range(n)], np.int64)
    # AT row i = indeg[i] distinct sources, ascending; A = its transpose
    trp = np.concatenate([[0], np.cumsum(indeg)])
    tcol = np.concatenate([np.sort(rng.choice(n, size=int(k), replace=False)) for k in indeg]
                          + [np.empty(0, np.int64)]).astype(np.int32)
    rp, col, _ = O.transpose(n, trp, tcol)
    g = P.graph_new(rp, col, kind=P.Kind.DirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    outdeg = np.diff(rp)
    for tol in (1e-4, 1e-9):  # fp32 and fp64 storage
        want, iters = O.pagerank(n, trp, tcol, outdeg, 0.85, tol, 100)
        r = algo.pagerank_gap(g, 0.85, tol, 100)
        assert r.iterations == iters, (tol, r.iterations, iters)
        assert rel_l1(r.rank, want) <= (1e-4 if tol == 1e-4 else 1e-9), tol


def test_pagerank_nonpositive_itermax_passes_through():
    """pagerank.cpp:52-75: iterations = min(k, itermax) with k = 1 when the loop
    never runs -- a non-positive itermax comes back unchanged, ranks stay 1/n."""
    g = P.generate_rmat(8, 8, seed=1)
    P.property_at(g)
    P.property_rowdegree(g)
    n = g.n()
    for itermax in (0, -1, -5):
        r = algo.pagerank_gap(g, 0.85, 1e-4, itermax)
        assert r.iterations == itermax
        assert np.all(r.rank == 1.0 / n)


def _sssp_batch(g, srcs, delta):
    from paper_2104_01661_b200.graph import call
    n = g.n()
    s = np.ascontiguousarray(srcs, np.uint64)
    out = np.empty((len(s), n), np.float64)
    call("gbx_sssp_batch", out.ctypes.data, g.handle, s.ctypes.data if len(s) else None, len(s),
         float(delta))
    return out


def test_sssp_batch_vs_oracle():
    """gbx_sssp_batch (the bench's config-4 call): every row equals Dijkstra
    and the one-source call."""
    g = P.generate_er(14, 16, seed=6)
    rp, col, w = g.export()
    n = len(rp) - 1
    P.property_rowdegree(g)
    srcs = P.pick_sources(g.row_degree(), 9, 6)
    for delta in (64.0, 1000.0, 7.0, 1.0):
        got = _sssp_batch(g, srcs, delta)
        for b, s in enumerate(srcs):
            want = O.dijkstra(n, rp, col, w.astype(np.float64), int(s))
            assert np.array_equal(got[b], want)
            assert np.array_equal(got[b], algo.sssp_delta_stepping(g, int(s), delta).dist)


def test_sssp_batch_fp64_and_errors():
    rng = np.random.default_rng(4)
    g0 = P.generate_rmat(11, 8, seed=3)
    rp, col, _ = g0.export()
    w = rng.uniform(1e-3, 10.0, len(col))
    g = P.graph_new(rp, col, w)
    n = len(rp) - 1
    got = _sssp_batch(g, [0, 5, 9], 2.0)
    for b, s in enumerate((0, 5, 9)):
        assert np.array_equal(got[b], O.dijkstra(n, rp, col, w, s))
    for srcs, delta, code in (([], 1.0, P.ErrCode.EmptyBatch), ([n], 1.0, P.ErrCode.SourceOutOfRange),
                              ([0], 0.0, P.ErrCode.NonPositiveDelta)):
        with pytest.raises(P.Error) as e:
            _sssp_batch(g, srcs, delta)
        assert e.value.code == code
