"""Config 4 timing (ER 2^24, 16 sources, gbx_sssp_batch): median of 5 after
warm-up; GBX_LIB selects a library variant (tools/build_variant.sh)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200.graph import call  # noqa: E402
import torch  # noqa: E402

P.init(0)
g = P.generate_er(24, 16, seed=1)
P.property_rowdegree(g)
g.prepare("sssp")
srcs = np.ascontiguousarray(P.pick_sources(g.row_degree(), 16, 1), np.uint64)
stream = torch.cuda.ExternalStream(g.stream())
ts = []
for rep in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call("gbx_sssp_batch", None, g.handle, srcs.ctypes.data, len(srcs), 64.0)
    e1.record(stream)
    e1.synchronize()
    if rep >= 2:
        ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{os.environ.get('GBX_LIB', 'libgbx.so')}: {ts[len(ts) // 2]:.2f} ms per 16 sources")
