"""Per-depth host timing of the batched Brandes (option bc.trace) on config 5."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200.graph import call  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P.init(0)
g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_at(g)
P.property_rowdegree(g)
s = np.ascontiguousarray(P.pick_sources(g.row_degree(), 4, 1), np.uint64)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    call("gbx_set_option", k.encode(), C.c_int64(int(v)))
for _ in range(3):
    call("gbx_betweenness", None, g.handle, s.ctypes.data, 4)
call("gbx_set_option", b"bc.trace", C.c_int64(1))
t0 = time.perf_counter()
call("gbx_betweenness", None, g.handle, s.ctypes.data, 4)
print(f"total {1e3 * (time.perf_counter() - t0):.2f} ms (traced: synchronised per depth)", file=sys.stderr)
