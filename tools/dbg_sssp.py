import sys, numpy as np
sys.path.insert(0, ".")
import oracle as O
import paper_2104_01661_b200 as P
from paper_2104_01661_b200 import algo
case = sys.argv[1]
if case == "path":
    g = P.graph_new(np.array([0, 1, 2, 2]), np.array([1, 2]), np.array([1.0, 1.0]))
    print(algo.sssp_delta_stepping(g, 0, 2.0).dist, flush=True)
elif case == "er10":
    g = P.generate_er(10, 16, seed=6)
    rp, col, w = g.export()
    want = O.dijkstra(len(rp) - 1, rp, col, w.astype(np.float64), 0)
    got = algo.sssp_delta_stepping(g, 0, 64.0).dist
    print("er10 equal", np.array_equal(got, want), flush=True)
elif case == "er10d16":
    g = P.generate_er(10, 16, seed=21)
    rp, col, w = g.export()
    want = O.dijkstra(len(rp) - 1, rp, col, w.astype(np.float64), 0)
    got = algo.sssp_delta_stepping(g, 0, float(sys.argv[2])).dist
    print("equal", np.array_equal(got, want), flush=True)
