"""Phases of the PageRank plan build (option pagerank.trace) at scale 22."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200.graph import call  # noqa: E402

P.init(0)
for rep in range(3):
    g = P.generate_rmat(22, 16, seed=1)
    P.property_at(g)
    P.property_rowdegree(g)
    if rep == 2:
        call("gbx_set_option", b"pagerank.trace", C.c_int64(1))
    g.prepare("pagerank")
    g.free()
