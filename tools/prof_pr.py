"""Profiling driver: one PageRank run (itermax iterations) on the R-MAT graph."""
import sys
import ctypes as C
sys.path.insert(0, ".")
import paper_2104_01661_b200 as P
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

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
itermax = int(sys.argv[2]) if len(sys.argv) > 2 else 4
P.init(0)
g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.DirectedAdjacency)
P.property_at(g)
P.property_rowdegree(g)
g.prepare("pagerank")
it = C.c_int(0)
for _ in range(2):
    call("gbx_pagerank", None, C.byref(it), g.handle, 0.85, 1e-4, itermax)
print("iters", it.value, g.last_stats())
