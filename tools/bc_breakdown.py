"""BC config-5 time breakdown: device time of one batch (events) vs the sum of
its kernels (from an ncu launch list run separately) -- the gap is host
round trips between levels."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import call

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P.init(0)
g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_at(g)
P.property_rowdegree(g)
srcs = np.ascontiguousarray(P.pick_sources(g.row_degree(), 4, 1), np.uint64)
st = torch.cuda.ExternalStream(g.stream())
for _ in range(3):
    call("gbx_betweenness", None, g.handle, srcs.ctypes.data, 4)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    call("gbx_betweenness", None, g.handle, srcs.ctypes.data, 4)
    e1.record(st)
    e1.synchronize()
    ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
print("device ms / wall ms per batch:", ts)
print("stats", g.last_stats())
