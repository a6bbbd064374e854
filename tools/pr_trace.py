"""PageRank scale-22 per-phase breakdown (option pagerank.trace): row phase,
barrier 1, long-row finish, barrier 2, L1 fold -- %globaltimer means per
iteration, printed by the library.  Usage: python tools/pr_trace.py [scale] [opt=val ...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01661_b200 as P  # noqa: E402
from paper_2104_01661_b200 import algo  # noqa: E402
from paper_2104_01661_b200.graph import call  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
P.init(0)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    call("gbx_set_option", k.encode(), C.c_int64(int(v)))
g = P.generate_rmat(scale, 16, seed=1)
P.property_at(g)
P.property_rowdegree(g)
g.prepare("pagerank")
for _ in range(3):
    algo.pagerank_gap(g)
import torch  # noqa: E402
stream = torch.cuda.ExternalStream(g.stream())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
it = C.c_int(0)
ts = []
for _ in range(20):
    with torch.cuda.stream(stream):
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call("gbx_pagerank", None, C.byref(it), g.handle, 0.85, 1e-4, 100)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{os.environ.get('GBX_LIB', 'libgbx.so')}: {it.value} iterations, median {ts[10]:.3f} ms/run "
      f"= {ts[10] / it.value * 1e3:.1f} us/iter, rows {g.last_stats()['hot_ms'] * 1e3:.1f} us")
call("gbx_set_option", b"pagerank.trace", C.c_int64(1))
r = algo.pagerank_gap(g)
