"""SSSP device time per source vs delta on the config-4 graph (ER 2^24, deg 16)
-- exploration only: the BASELINE config fixes delta = 64."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import call

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P.init(0)
g = P.generate_er(logn, 16, seed=1)
P.property_rowdegree(g)
g.prepare("sssp")
srcs = P.pick_sources(g.row_degree(), 4, 1)
st = torch.cuda.ExternalStream(g.stream())
for delta in (8.0, 16.0, 32.0, 64.0, 128.0):
    for s in srcs[:1]:
        call("gbx_sssp", None, g.handle, int(s), delta)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for s in srcs:
        call("gbx_sssp", None, g.handle, int(s), delta)
    e1.record(st)
    e1.synchronize()
    print(f"delta {delta:6.1f}: {e0.elapsed_time(e1) / len(srcs):.2f} ms/source, "
          f"near iterations {g.last_stats()['iterations']}")
