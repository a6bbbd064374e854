"""The fused multi-GPU PageRank (gbx_pr_shard_run_p2p: x stored into every
rank's copy over peer pointers, device-side signal barrier per iteration) on a
one-rank NCCL group: the kernel, the peer-pointer plumbing and the driver
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


def _p2p_multi(g, nv, damping=0.85, tol=1e-4, itermax=100):
    """nv ranks of the fused exchange emulated in ONE cooperative launch on this
    GPU (gbx_pr_shard_run_p2p_multi): every rank its own shard handle and its own
    padded x0 / x1, slot table and signal word; peer pointers = the other
    ranks' buffers.  Returns (ranks in original order, iterations)."""
    import ctypes as C

    import torch

    from paper_2104_01661_b200.graph import call
    rp, col, _ = g.export()
    shards = []
    for v in range(nv):
        h = P.graph_new(rp, col, kind=P.Kind.DirectedAdjacency)
        P.property_at(h)
        P.property_rowdegree(h)
        rb, re = C.c_int64(), C.c_int64()
        call("gbx_pr_shard_prepare", h.handle, v, nv, C.byref(rb), C.byref(re))
        shards.append((h, rb.value, re.value))
    chunk = C.c_int64()
    call("gbx_pr_shard_layout", shards[0][0].handle, C.byref(chunk), None)
    chunk = chunk.value
    dev = torch.device("cuda", 0)
    x0 = [torch.zeros(nv * chunk, dtype=torch.float32, device=dev) for _ in range(nv)]
    x1 = [torch.zeros(nv * chunk, dtype=torch.float32, device=dev) for _ in range(nv)]
    l1 = [torch.zeros(2 * nv, dtype=torch.float64, device=dev) for _ in range(nv)]
    sig = [torch.zeros(4, dtype=torch.int32, device=dev) for _ in range(nv)]
    r0 = [torch.zeros(chunk, dtype=torch.float32, device=dev) for _ in range(nv)]
    r1 = [torch.zeros(chunk, dtype=torch.float32, device=dev) for _ in range(nv)]
    torch.cuda.synchronize()
    for v, (h, _, _) in enumerate(shards):
        call("gbx_pr_shard_init", h.handle, x0[v].data_ptr(), r0[v].data_ptr(), damping)
    for h, _, _ in shards:
        torch.cuda.ExternalStream(h.stream()).synchronize()
    ptrs = lambda ts: np.ascontiguousarray([t.data_ptr() for t in ts], np.uint64)  # noqa: E731
    px0, px1, pl1, psig = ptrs(x0), ptrs(x1), ptrs(l1), ptrs(sig)
    hs = (C.c_void_p * nv)(*[h.handle for h, _, _ in shards])
    pr0 = (C.c_void_p * nv)(*[t.data_ptr() for t in r0])
    pr1 = (C.c_void_p * nv)(*[t.data_ptr() for t in r1])
    it = C.c_int(0)
    call("gbx_pr_shard_run_p2p_multi", hs, nv, px0.ctypes.data, px1.ctypes.data,
         pl1.ctypes.data, psig.ctypes.data, pr0, pr1, damping, tol, itermax, C.byref(it))
    iters = it.value
    # every rank's x copies agree (each row's contribution went to every rank)
    xs = x0 if iters % 2 == 0 else x1
    for v in range(1, nv):
        assert torch.equal(xs[v], xs[0])
    res = r0 if iters % 2 == 0 else r1
    r_full = torch.zeros(nv * chunk, dtype=torch.float32, device=dev)
    for v, (_, rb, re) in enumerate(shards):
        r_full[v * chunk: v * chunk + (re - rb)] = res[v][: re - rb]
    torch.cuda.synchronize()
    out = np.empty(g.n(), np.float64)
    call("gbx_pr_shard_unpermute", shards[0][0].handle, r_full.data_ptr(), out.ctypes.data)
    return out, iters


@pytest.mark.parametrize("nv", [2, 3, 4, 8])
@pytest.mark.parametrize("scale,seed", [(12, 1), (16, 3)])
def test_p2p_pagerank_multi_rank_emulated(nv, scale, seed):
    """The fused exchange with 2..8 ranks (never run on real multi-GPU here):
    bit-identical ranks and the same iteration count as the single-GPU
    persistent kernel."""
    P.init(0)
    g = P.generate_rmat(scale, 16, seed=seed)
    P.property_at(g)
    P.property_rowdegree(g)
    got, it = _p2p_multi(g, nv)
    want = algo.pagerank_gap(g)
    assert it == want.iterations
    assert np.array_equal(got, want.rank)


def test_p2p_pagerank_multi_rank_itermax():
    P.init(0)
    g = P.generate_rmat(11, 16, seed=4)
    P.property_at(g)
    P.property_rowdegree(g)
    # tol 1e-6: still fp32 storage on one GPU (tighter switches it to fp64,
    # which the fp32-only shard path does not follow)
    got, it = _p2p_multi(g, 3, tol=1e-6, itermax=5)
    want = algo.pagerank_gap(g, 0.85, 1e-6, 5)
    assert it == want.iterations == 5
    assert np.array_equal(got, want.rank)


def test_p2p_peer_timeout_is_an_error():
    """A peer that never signals: the bounded spin gives up, the call returns
    GBX_CUDA_ERROR instead of hanging the cooperative grid."""
    import ctypes as C

    import torch

    from paper_2104_01661_b200 import Error
    from paper_2104_01661_b200.graph import call
    P.init(0)
    g = P.generate_rmat(10, 16, seed=1)
    P.property_at(g)
    P.property_rowdegree(g)
    rb, re, chunk = C.c_int64(), C.c_int64(), C.c_int64()
    # rank 0 of a 2-rank layout; rank 1 never runs: its buffers are scratch
    call("gbx_pr_shard_prepare", g.handle, 0, 2, C.byref(rb), C.byref(re))
    call("gbx_pr_shard_layout", g.handle, C.byref(chunk), None)
    ch = chunk.value
    dev = torch.device("cuda", 0)
    bufs = [[torch.zeros(2 * ch, dtype=torch.float32, device=dev) for _ in range(2)]
            for _ in range(2)]
    l1 = [torch.zeros(4, dtype=torch.float64, device=dev) for _ in range(2)]
    sig = [torch.zeros(4, dtype=torch.int32, device=dev) for _ in range(2)]
    r = [torch.zeros(ch, dtype=torch.float32, device=dev) for _ in range(2)]
    torch.cuda.synchronize()
    call("gbx_pr_shard_init", g.handle, bufs[0][0].data_ptr(), r[0].data_ptr(), 0.85)
    ptr = lambda ts: np.ascontiguousarray([t.data_ptr() for t in ts], np.uint64)  # noqa: E731
    px0, px1 = ptr([bufs[0][0], bufs[1][0]]), ptr([bufs[0][1], bufs[1][1]])
    pl1, psig = ptr(l1), ptr(sig)
    call("gbx_set_option", b"p2p.timeout_ms", C.c_int64(200))
    try:
        with pytest.raises(Error) as e:
            call("gbx_pr_shard_run_p2p", g.handle, px0.ctypes.data, px1.ctypes.data,
                 pl1.ctypes.data, psig.ctypes.data, r[0].data_ptr(), r[1].data_ptr(), 0.85,
                 1e-4, 100, C.byref(C.c_int(0)))
        assert e.value.code == P.ErrCode.CudaError
    finally:
        call("gbx_reset_option", b"p2p.timeout_ms")
    # the library and the device stay usable
    assert algo.pagerank_gap(g).iterations > 0
