"""World-size-2 gloo tests of the multi-GPU host logic (dist.py) on CPU:
row-block bookkeeping, the x all-gather, the L1 all-reduce and the stopping rule
(PageRank), and the wedge partition + count all-reduce (triangle count)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


BC_SOURCES = [3, 17, 40, 101, 250]
BFS_SOURCE = 17


def _worker(rank, world, port, q, what):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2104_01661_b200.dist import (sharded_betweenness, sharded_betweenness_rows,
                                            sharded_pagerank, sharded_triangle_count)
    from paper_2104_01661_b200.dist import sharded_bfs
    from tests.dist_cpu_backend import CpuBcRowsBackend, CpuBfsRowsBackend, CpuShardBackend
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        und = what in ("tc", "bc", "bcrows", "bfsrows")
        rp, col = O.rmat_graph(9, 8, seed=3, undirected=und)
        be = CpuShardBackend(len(rp) - 1, rp, col)
        if what == "pr":
            ranks, iters = sharded_pagerank(be, dist, 0.85, 1e-4, 100)
            q.put((rank, "pr", iters, ranks.tolist()))
        elif what == "prp2p":
            from paper_2104_01661_b200.dist import sharded_pagerank_p2p
            ranks, iters = sharded_pagerank_p2p(be, dist, 0.85, 1e-4, 100)
            q.put((rank, "prp2p", iters, ranks.tolist()))
        elif what == "prp2pfail":
            # rank 1's fused kernel gives up (a peer timeout): every rank must
            # redo the run over the NCCL-style exchange and agree
            from paper_2104_01661_b200.dist import sharded_pagerank_p2p
            if rank == 1:
                def boom(*a, **k):
                    raise RuntimeError("pr_shard_run_p2p: a peer rank did not arrive")
                be.p2p_run = boom
            ranks, iters = sharded_pagerank_p2p(be, dist, 0.85, 1e-4, 100)
            q.put((rank, "prp2pfail", iters, ranks.tolist(), bool(getattr(be, "p2p_failed", False))))
        elif what == "bc":
            c = sharded_betweenness(be, dist, BC_SOURCES)
            q.put((rank, "bc", None, c.tolist()))
        elif what == "bfsrows":
            p, lv = sharded_bfs(CpuBfsRowsBackend(len(rp) - 1, rp, col), dist, BFS_SOURCE)
            q.put((rank, "bfsrows", lv.tolist(), p.tolist()))
        elif what == "bcrows":
            c = sharded_betweenness_rows(CpuBcRowsBackend(len(rp) - 1, rp, col), dist, BC_SOURCES)
            q.put((rank, "bcrows", None, c.tolist()))
        else:
            q.put((rank, "tc", sharded_triangle_count(be, dist), None))
    finally:
        dist.destroy_process_group()


def _run(what, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, what)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_sharded_pagerank_gloo_matches_oracle():
    out = _run("pr")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=False)
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    want, iters = O.pagerank(n, trp, tcol, np.diff(rp))
    for _, _, it, ranks in out:
        assert it == iters
        got = np.array(ranks)
        assert np.abs(got - want).sum() / np.abs(want).sum() <= 1e-9


def test_sharded_pagerank_p2p_orchestration_gloo():
    """dist.sharded_pagerank_p2p's host side (layout, init, barrier, the final
    padded all-gather and the unpermute) over gloo; the fused kernel itself
    runs on the device (tests/test_pr_p2p_gpu.py)."""
    out = _run("prp2p")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=False)
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    want, iters = O.pagerank(n, trp, tcol, np.diff(rp))
    for _, _, it, ranks in out:
        assert it == iters
        assert np.array_equal(np.array(ranks), want)


def test_sharded_pagerank_p2p_failure_falls_back_gloo():
    """One rank's fused run fails: both ranks fall back to the exchange driver
    (no hang, no mixed results) and still match the oracle."""
    out = _run("prp2pfail")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=False)
    n = len(rp) - 1
    trp, tcol, _ = O.transpose(n, rp, col)
    want, iters = O.pagerank(n, trp, tcol, np.diff(rp))
    assert len(out) == 2
    for _, _, it, ranks, failed in out:
        assert failed
        assert it == iters
        assert np.abs(np.array(ranks) - want).sum() / np.abs(want).sum() <= 1e-9


def test_sharded_triangle_count_gloo_matches_oracle():
    out = _run("tc")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=True)
    want = O.triangle_count(len(rp) - 1, rp, col)
    assert all(c == want for _, _, c, _ in out)


def test_sharded_betweenness_gloo_matches_oracle():
    """Sources dealt round-robin (rank 0: 3 of them, rank 1: 2), partials
    all-reduced: equals the single-process batched Brandes."""
    out = _run("bc")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=True)
    n = len(rp) - 1
    want = O.bc(n, rp, col, rp, col, np.asarray(BC_SOURCES, np.int64))
    for _, _, _, c in out:
        got = np.array(c)
        assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())


def test_row_partitioned_betweenness_gloo_matches_oracle():
    """1D row blocks with one record exchange per BFS level (the protocol of
    gbx_bc_shard_*; 5 sources = a batch of 4 and a batch of 1): equals the
    single-process batched Brandes."""
    out = _run("bcrows")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=True)
    n = len(rp) - 1
    want = O.bc(n, rp, col, rp, col, np.asarray(BC_SOURCES, np.int64))
    for _, _, _, c in out:
        got = np.array(c)
        assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())


def test_row_partitioned_betweenness_single_process_protocol():
    """The same protocol with 3 simulated ranks in one process (records
    exchanged by concatenation): no rank ever waits on another."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tests.dist_cpu_backend import CpuBcRowsBackend
    rp, col = O.rmat_graph(8, 8, seed=5, undirected=True)
    n = len(rp) - 1
    srcs = [1, 9, 33, 77]
    world = 3
    bes = [CpuBcRowsBackend(n, rp, col) for _ in range(world)]
    for r, be in enumerate(bes):
        be.bc_begin(srcs, r, world)
    assert [be.rb for be in bes][0] == 0 and bes[-1].re == n
    while True:
        outs = [be.bc_forward() for be in bes]
        allr = torch.cat([t for t, _ in outs])
        tot = sum(k for _, k in outs)
        done = [be.bc_forward_apply(allr, tot) for be in bes]
        assert len(set(done)) == 1
        if done[0]:
            break
    while True:
        outs = [be.bc_backward() for be in bes]
        assert len({d for _, _, d in outs}) == 1
        if outs[0][2]:
            break
        allr = torch.cat([t for t, _, _ in outs])
        tot = sum(k for _, k, _ in outs)
        for be in bes:
            be.bc_backward_apply(allr, tot)
    got = sum(be.bc_centrality().numpy() for be in bes)
    want = O.bc(n, rp, col, rp, col, np.asarray(srcs, np.int64))
    assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())


def test_row_sharded_bfs_gloo_matches_oracle():
    """Row-sharded BFS, one frontier-bitmap all-gather per level: parents and
    levels bit-exact against the oracle (min-id parents)."""
    out = _run("bfsrows")
    rp, col = O.rmat_graph(9, 8, seed=3, undirected=True)
    n = len(rp) - 1
    wp, wl = O.bfs(n, rp, col, BFS_SOURCE)
    for _, _, lv, par in out:
        assert np.array_equal(np.array(par), wp) and np.array_equal(np.array(lv), wl)
