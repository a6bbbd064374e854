"""Pin the oracle restatement (oracle/oracle.c) against vectors produced by the
reference itself (tests/golden/, make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle as O
from tests.golden_util import Golden, case_ids

G = Golden()
CASES = {c.name: c for c in G.cases}


def _transpose(c):
    trp, tcol, _ = O.transpose(c.n, c.rp, c.col)
    return trp, tcol


@pytest.mark.parametrize("name", case_ids("bfs"))
def test_bfs(name):
    c = CASES[name]
    p, l = O.bfs(c.n, c.rp, c.col, c.params["src"])
    for tag in ("auto", "push", "pull", "pushonly"):
        assert np.array_equal(p, c.out[f"parent_{tag}"]), tag
        assert np.array_equal(l, c.out[f"level_{tag}"]), tag


@pytest.mark.parametrize("name", case_ids("pagerank"))
def test_pagerank(name):
    c = CASES[name]
    trp, tcol = _transpose(c)
    prm = c.params
    rank, iters, trace = O.pagerank(c.n, trp, tcol, np.diff(c.rp), prm["damping"], prm["tol"],
                                    prm["itermax"], trace=True)
    assert iters == int(c.out["iters"])
    # the restatement keeps the reference's fold order: bit-exact
    assert np.array_equal(rank, c.out["rank"])
    assert np.array_equal(trace, c.out["trace"])


@pytest.mark.parametrize("name", case_ids("triangle_count"))
def test_triangle_count(name):
    c = CASES[name]
    t = O.triangle_count(c.n, c.rp, c.col)
    for tag in ("auto", "force", "never"):
        assert t == int(c.out[f"count_{tag}"])


@pytest.mark.parametrize("name", case_ids("sssp"))
def test_sssp(name):
    c = CASES[name]
    for d in c.params["deltas"]:
        want = c.out[f"dist_{d:g}"]
        got = O.sssp_delta(c.n, c.rp, c.col, c.w, c.params["src"], d)
        assert np.array_equal(got, want)
        assert np.array_equal(O.dijkstra(c.n, c.rp, c.col, c.w, c.params["src"]), want)


@pytest.mark.parametrize("name", case_ids("bc"))
def test_bc(name):
    c = CASES[name]
    trp, tcol = _transpose(c)
    got = O.bc(c.n, c.rp, c.col, trp, tcol, c.params["sources"])
    want = c.out["centrality"]
    assert np.max(np.abs(got - want), initial=0.0) <= 1e-9


@pytest.mark.parametrize("name", case_ids("cc"))
def test_cc(name):
    c = CASES[name]
    assert np.array_equal(O.cc(c.n, c.rp, c.col), c.out["label"])


@pytest.mark.parametrize("name", case_ids("sort_by_degree"))
def test_sort_by_degree(name):
    c = CASES[name]
    assert np.array_equal(O.sort_by_degree(np.diff(c.rp)), c.out["perm"])


def test_generator_properties():
    """CSR invariants of the seeded generators (containers.cpp:104-124)."""
    for und in (False, True):
        rp, col = O.rmat_graph(10, 16, seed=4, undirected=und)
        n = 1 << 10
        assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == len(col)
        for i in range(n):
            r = col[rp[i]:rp[i + 1]]
            assert np.all(np.diff(r) > 0)
            assert not np.any(r == i)
        if und:
            trp, tcol, _ = O.transpose(n, rp, col)
            assert np.array_equal(trp, rp) and np.array_equal(tcol, col)
    rp, col, w = O.er_graph(10, 16, seed=5)
    assert w.min() >= 1 and w.max() <= 255
