"""Per-level trace of one BFS source (diagnostic): python tools/bfs_one.py IDX"""
import sys
import ctypes as C
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

P.init(0)
g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_at(g); P.property_rowdegree(g)
srcs = P.pick_sources(g.row_degree(), 64, 1)
s = int(srcs[int(sys.argv[1])])
deg = g.row_degree()
print("source", s, "degree", int(deg[s]), file=sys.stderr)
for _ in range(3):
    call("gbx_bfs", None, None, g.handle, s, 0, 16)
