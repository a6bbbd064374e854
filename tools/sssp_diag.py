"""SSSP diagnostics: stats (near iterations, relaxations) and wall time per source."""
import sys, time
import ctypes as C
import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import call


def opt_args(argv):
    """name=value arguments -> library options (gbx_set_option); the rest returned"""
    rest = []
    for a in argv:
        if a.startswith("delta="):
            global DELTA
            DELTA = float(a.split("=", 1)[1])
        elif "=" in a:
            k, v = a.split("=", 1)
            call("gbx_set_option", k.encode(), C.c_int64(int(v)))
        else:
            rest.append(a)
    return rest


DELTA = 64.0
sys.argv = [sys.argv[0]] + opt_args(sys.argv[1:])

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P.init(0)
g = P.generate_er(logn, 16, seed=1)
P.property_rowdegree(g)
g.prepare("sssp")
n, nnz, _, _ = g.info()
srcs = P.pick_sources(g.row_degree(), 16, 1)
for s in srcs[:2]:
    call("gbx_sssp", None, g.handle, int(s), DELTA)
for s in srcs[:4]:
    t0 = time.perf_counter()
    call("gbx_sssp", None, g.handle, int(s), DELTA)
    t1 = time.perf_counter()
    st = g.last_stats()
    print(f"src {s} wall {1e3*(t1-t0):.2f} ms near_iters {st['iterations']} relax {st['work_units']} ({st['work_units']/nnz:.2f} x nnz)")
