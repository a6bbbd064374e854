"""Profiling driver: run one algorithm once (after one warm-up) on its BASELINE-shaped graph."""
import sys
import ctypes as C
import numpy as np
sys.path.insert(0, ".")
import paper_2104_01661_b200 as P
from paper_2104_01661_b200 import algo
from paper_2104_01661_b200.graph import call


def opt_args(argv):
    """name=value arguments -> library options (gbx_set_option); the rest returned"""
    rest = []
    for a in argv:
        if "=" in a:
            k, v = a.split("=", 1)
            call("gbx_set_option", k.encode(), C.c_int64(int(v)))
        else:
            rest.append(a)
    return rest


sys.argv = [sys.argv[0]] + opt_args(sys.argv[1:])

w = sys.argv[1]
scale = int(sys.argv[2])
P.init(0)
if w == "tc":
    g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_rowdegree(g); P.property_ndiag(g); g.prepare("tc")
    run = lambda: algo.triangle_count(g)
elif w == "sssp":
    g = P.generate_er(scale, 16, seed=1)
    P.property_rowdegree(g); g.prepare("sssp")
    src = int(P.pick_sources(g.row_degree(), 1, 1)[0])
    run = lambda: call("gbx_sssp", None, g.handle, src, 64.0)
elif w in ("bfs", "bfs64"):
    g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g); P.property_rowdegree(g)
    srcs = P.pick_sources(g.row_degree(), 64, 1)
    if w == "bfs":
        run = lambda: call("gbx_bfs", None, None, g.handle, int(srcs[0]), 0, 16)
    else:
        arr = np.ascontiguousarray(srcs, np.uint64)
        run = lambda: call("gbx_bfs_batch", None, None, g.handle, arr.ctypes.data, 64)
elif w == "bc":
    g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
    P.property_at(g); P.property_rowdegree(g)
    s = np.ascontiguousarray(P.pick_sources(g.row_degree(), 4, 1), np.uint64)
    run = lambda: call("gbx_betweenness", None, g.handle, s.ctypes.data, 4)
run()
print(run() if w == "tc" else "ran", g.last_stats())
