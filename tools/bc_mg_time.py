"""gbx_betweenness_mg on in-process ranks vs gbx_betweenness (config 5 shape):
python tools/bc_mg_time.py [ranks] [scale]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200.graph import call  # noqa: E402
from paper_2104_01661_b200.mg import Comm, DGraph  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 24
P.init(0)
ref = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_at(ref)
P.property_rowdegree(ref)
srcs = [int(x) for x in P.pick_sources(ref.row_degree(), 4, 1)]
s = np.ascontiguousarray(srcs, np.uint64)
want = np.empty(ref.n(), np.float64)
call("gbx_betweenness", want.ctypes.data, ref.handle, s.ctypes.data, 4)
ref.free()
g = DGraph.rmat(Comm.local(nr), scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
got = g.betweenness(srcs)
print("rel diff vs single GPU", np.abs(got - want).sum() / np.abs(want).sum())
for _ in range(3):
    t0 = time.perf_counter()
    g.betweenness(srcs, to_host=False)
    print(f"{nr} ranks: {1e3 * (time.perf_counter() - t0):.2f} ms, {g.last_stats()['iterations']} levels, "
          f"{g.last_stats()['hot_launches']} candidate levels", flush=True)
