"""Host wall time per gbx_bfs call vs device time (diagnostic)."""
import time
import numpy as np
import torch
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import call

P.init(0)
g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_at(g); P.property_rowdegree(g)
srcs = P.pick_sources(g.row_degree(), 64, 1)
for s in srcs[:4]:
    call("gbx_bfs", None, None, g.handle, int(s), 0, 16)
for s in srcs[:8]:
    t0 = time.perf_counter()
    call("gbx_bfs", None, None, g.handle, int(s), 0, 16)
    t1 = time.perf_counter()
    print("src", s, "wall %.1f us" % ((t1 - t0) * 1e6), "iters", g.last_stats()["iterations"])
st = torch.cuda.ExternalStream(g.stream())
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for s in srcs[:8]:
    call("gbx_bfs", None, None, g.handle, int(s), 0, 16)
e1.record(st); e1.synchronize()
print("8 calls events ms", e0.elapsed_time(e1))
