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


def _worker(rank, world, port, q, what):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2104_01661_b200.dist import (sharded_betweenness, sharded_pagerank,
                                            sharded_triangle_count)
    from tests.dist_cpu_backend import CpuShardBackend
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        und = what in ("tc", "bc")
        rp, col = O.rmat_graph(9, 8, seed=3, undirected=und)
        be = CpuShardBackend(len(rp) - 1, rp, col)
        if what == "pr":
            ranks, iters = sharded_pagerank(be, dist, 0.85, 1e-4, 100)
            q.put((rank, "pr", iters, ranks.tolist()))
        elif what == "bc":
            c = sharded_betweenness(be, dist, BC_SOURCES)
            q.put((rank, "bc", None, c.tolist()))
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
