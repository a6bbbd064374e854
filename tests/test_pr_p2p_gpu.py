"""The fused multi-GPU PageRank (gbx_pr_shard_run_p2p: x stored into every
rank's copy over peer pointers, device-side signal barrier per iteration) on a
one-rank NCCL group: the kernel, the symmetric-memory plumbing and the driver
(dist.sharded_pagerank_p2p) against the single-GPU PageRank and the NCCL-
exchange driver.  (Ranks > 1 need one GPU each: the kernels wait on each
other, so they are not simulated on one GPU.)"""
import os
import socket

import numpy as np
import pytest

import paper_2104_01661_b200 as P
from paper_2104_01661_b200 import algo

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def group():
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("scale,seed", [(10, 1), (14, 5)])
def test_p2p_pagerank_one_rank(group, scale, seed):
    from paper_2104_01661_b200.dist import (GpuShardBackend, sharded_pagerank,
                                            sharded_pagerank_p2p)
    P.init(0)
    g = P.generate_rmat(scale, 16, seed=seed)
    P.property_at(g)
    P.property_rowdegree(g)
    got, it = sharded_pagerank_p2p(GpuShardBackend(g), group, 0.85, 1e-4, 100)
    got2, it2 = sharded_pagerank(GpuShardBackend(g), group, 0.85, 1e-4, 100)
    want = algo.pagerank_gap(g)
    assert it == it2 == want.iterations
    assert np.array_equal(got, got2)
    assert np.abs(got - want.rank).sum() <= 1e-6 * np.abs(want.rank).sum()
    # a second run on the same buffers (signal words re-zeroed by the driver)
    got3, it3 = sharded_pagerank_p2p(GpuShardBackend(g), group, 0.85, 1e-4, 100)
    assert it3 == it and np.array_equal(got3, got)


def test_p2p_pagerank_itermax(group):
    from paper_2104_01661_b200.dist import GpuShardBackend, sharded_pagerank_p2p
    P.init(0)
    g = P.generate_rmat(10, 16, seed=2)
    P.property_at(g)
    P.property_rowdegree(g)
    _, it = sharded_pagerank_p2p(GpuShardBackend(g), group, 0.85, 1e-12, 3)
    assert it == 3
