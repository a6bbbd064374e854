"""Phase timing of the PageRank e2e path (graph_new32 -> basic PR -> D2H)."""
import ctypes as C, time, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import call

P.init(0)
g = P.generate_rmat(22, 16, seed=1, kind=P.Kind.DirectedAdjacency)
rp, col, _ = g.export()
n = len(rp) - 1
rp_h = torch.from_numpy(rp).pin_memory(); col_h = torch.from_numpy(col).pin_memory()
rank_h = torch.empty(n, dtype=torch.float64).pin_memory()
it = C.c_int(0)
for rep in range(6):
    t = [time.perf_counter()]
    h = C.c_void_p()
    call("gbx_graph_new32", C.byref(h), n, rp_h.data_ptr(), col_h.data_ptr(), None, 0, 0); t.append(time.perf_counter())
    call("gbx_property_at", h); t.append(time.perf_counter())
    call("gbx_property_rowdegree", h); t.append(time.perf_counter())
    call("gbx_prepare", h, b"pagerank"); t.append(time.perf_counter())
    call("gbx_pagerank", None, C.byref(it), h, 0.85, 1e-4, 100); t.append(time.perf_counter())
    call("gbx_pagerank", rank_h.data_ptr(), C.byref(it), h, 0.85, 1e-4, 100); t.append(time.perf_counter())
    call("gbx_graph_free", C.byref(h)); t.append(time.perf_counter())
    names = ["graph_new32", "property_at", "rowdegree", "prepare(pr)", "pagerank", "pagerank+D2H", "free"]
    print(" ".join(f"{nm}={1e3*(t[i+1]-t[i]):.1f}ms" for i, nm in enumerate(names)))
