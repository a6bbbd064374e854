"""Per-level trace of one BFS source (diagnostic): python tools/bfs_one.py IDX"""
import sys
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import call

P.init(0)
g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
P.property_at(g); P.property_rowdegree(g)
srcs = P.pick_sources(g.row_degree(), 64, 1)
s = int(srcs[int(sys.argv[1])])
deg = g.row_degree()
print("source", s, "degree", int(deg[s]), file=sys.stderr)
for _ in range(3):
    call("gbx_bfs", None, None, g.handle, s, 0, 16)
