"""Fused P2P sharded PageRank vs the NCCL-exchange driver and the single-GPU
run, under torchrun (any world size; on one GPU: --nproc-per-node 1)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200 import algo  # noqa: E402
from paper_2104_01661_b200.dist import (GpuShardBackend, sharded_pagerank,  # noqa: E402
                                        sharded_pagerank_p2p)

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
P.init(local)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
g = P.generate_rmat(scale, 16, seed=5)
P.property_at(g)
P.property_rowdegree(g)
got, it = sharded_pagerank_p2p(GpuShardBackend(g), dist, 0.85, 1e-4, 100)
got2, it2 = sharded_pagerank(GpuShardBackend(g), dist, 0.85, 1e-4, 100)
ref = P.generate_rmat(scale, 16, seed=5)
P.property_at(ref)
P.property_rowdegree(ref)
want = algo.pagerank_gap(ref)
rel = np.abs(got - want.rank).sum() / np.abs(want.rank).sum()
rel2 = np.abs(got - got2).sum() / np.abs(got2).sum()
be = GpuShardBackend(g)
rb, re, n = be.prepare(dist.get_rank(), dist.get_world_size())


class Prepared:  # plan built outside the timed region (as bench.py does)
    def __init__(self, b):
        self.b = b

    def prepare(self, rank, world):
        return rb, re, n

    def __getattr__(self, k):
        return getattr(self.b, k)


times = []
for _ in range(5):
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, itx = sharded_pagerank_p2p(Prepared(be), dist, 0.85, 1e-4, 100, to_host=False)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
if dist.get_rank() == 0:
    print(f"p2p iters {it} nccl iters {it2} single iters {want.iterations} relL1 vs single "
          f"{rel:.2e} vs nccl {rel2:.2e}; p2p run {min(times):.3f} ms")
ok = it == want.iterations == it2 and rel <= 1e-6
dist.destroy_process_group()
sys.exit(0 if ok else 1)
