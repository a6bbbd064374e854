"""Per-level trace of the multi-GPU BFS (gbx_bfs_mg, option bfs.trace) on
in-process ranks: python tools/bfs_mg_levels.py [ranks] [scale]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200.graph import call  # noqa: E402
from paper_2104_01661_b200.mg import Comm, DGraph  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
P.init(0)
g = DGraph.rmat(Comm.local(nr), scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
ref = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_rowdegree(ref)
import time  # noqa: E402
srcs = P.pick_sources(ref.row_degree(), 64, 1)[:8]
g.bfs(int(srcs[0]), to_host=False)
call("gbx_set_option", b"bfs.trace", C.c_int64(1))
for s in srcs:
    t0 = time.perf_counter()
    g.bfs(int(s), to_host=False)
    print(f"source {int(s)}: {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
