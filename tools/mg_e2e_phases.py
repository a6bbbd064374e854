"""Phases of the multi-GPU PageRank e2e path on a 1-rank NCCL communicator:
gbx_dgraph_from_blocks (host CSR in), first gbx_pagerank_mg (plan + exchange
buffers + run + D2H), second call (run only)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200.mg import MG_AUTO, MG_NCCL, Comm, DGraph  # noqa: E402
import torch  # noqa: E402

P.init(0)
c = Comm.nccl(1, 0, Comm.unique_id(), 0)
ref = P.generate_rmat(22, 16, seed=1)
rp, col, _ = ref.export()
n = len(rp) - 1
rp_h = torch.from_numpy(rp).pin_memory().numpy()
col_h = torch.from_numpy(col).pin_memory().numpy()
for ex in (MG_AUTO, MG_NCCL):
    for rep in range(3):
        t = [time.perf_counter()]
        g = DGraph.from_blocks(c, n, [(0, n, rp_h, col_h)])
        t.append(time.perf_counter())
        r, it = g.pagerank(exchange=ex)
        t.append(time.perf_counter())
        r, it = g.pagerank(exchange=ex)
        t.append(time.perf_counter())
        g.free()
        t.append(time.perf_counter())
        print(f"exchange {ex}: from_blocks {1e3 * (t[1] - t[0]):.1f} ms, first pagerank_mg "
              f"{1e3 * (t[2] - t[1]):.1f} ms, second {1e3 * (t[3] - t[2]):.1f} ms, free "
              f"{1e3 * (t[4] - t[3]):.1f} ms ({it} iterations)", flush=True)
