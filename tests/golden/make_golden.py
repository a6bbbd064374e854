"""Generate tests/golden/golden.npz + manifest.json by running the REFERENCE ITSELF.

This script runs only in the build container, where /root/reference exists: it
calls the unmodified gblite library (compiled from /root/reference/proj/src by
``make -C oracle ref``) through oracle/ref_shim.cpp on
  * the reference's own named fixtures and known answers (tests/test_*.cpp and
    proj/data/*.mtx; the known answers are asserted here as well), and
  * seeded synthetic graphs (our R-MAT / Erdos-Renyi generator at small scales,
    and numpy-seeded random graphs shaped like tests/test_helpers.hpp's),
and stores inputs and reference outputs.  The oracle restatement and the CUDA
library are both checked against these vectors (tests/test_oracle_golden.py,
tests/test_gpu_parity.py); the GPU box never needs /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
INF = float("inf")


def dense_csr(n, edges, weights=None):
    """CSR from an edge list (sorted rows, strictly ascending columns)."""
    rows = [[] for _ in range(n)]
    for k, (i, j) in enumerate(edges):
        rows[i].append((j, weights[k] if weights is not None else 1.0))
    rp = np.zeros(n + 1, np.int64)
    col, val = [], []
    for i in range(n):
        d = dict(rows[i])
        for j in sorted(d):
            col.append(j)
            val.append(d[j])
        rp[i + 1] = len(col)
    return rp, np.array(col, np.int32), np.array(val, np.float64)


def undirected(n, pairs):
    e = []
    for i, j in pairs:
        e.append((i, j))
        e.append((j, i))
    return dense_csr(n, e)


def star(leaves):
    return undirected(leaves + 1, [(0, l) for l in range(1, leaves + 1)])


def complete(n):
    return dense_csr(n, [(i, j) for i in range(n) for j in range(n) if i != j])


def cycle(n, und=False):
    e = [(i, (i + 1) % n) for i in range(n)]
    if und:
        e += [((i + 1) % n, i) for i in range(n)]
    return dense_csr(n, e)


def mtx(path):
    """Tiny Matrix Market reader for the three reference data files."""
    with open(path) as f:
        header = f.readline().split()
        symmetric = header[-1] == "symmetric"
        real = header[3] == "real"
        line = f.readline()
        while line.startswith("%"):
            line = f.readline()
        n, _, nz = map(int, line.split())
        edges, w = [], []
        for _ in range(nz):
            t = f.readline().split()
            i, j = int(t[0]) - 1, int(t[1]) - 1
            x = float(t[2]) if real else 1.0
            edges.append((i, j))
            w.append(x)
            if symmetric and i != j:
                edges.append((j, i))
                w.append(x)
    return (n,) + dense_csr(n, edges, w)


def rand_digraph(rng, n, density):
    e = [(i, j) for i in range(n) for j in range(n) if i != j and rng.random() < density]
    return dense_csr(n, e)


def rand_undirected(rng, n, density):
    return undirected(n, [(i, j) for i in range(n) for j in range(i + 1, n)
                          if rng.random() < density])


def rand_weighted(rng, n, density):
    e, w = [], []
    for i in range(n):
        for j in range(n):
            if i != j and rng.random() < density:
                e.append((i, j))
                w.append(float(rng.uniform(1e-3, 10.0)))
    return dense_csr(n, e, w)


class Store:
    def __init__(self):
        self.arrays = {}
        self.cases = []

    def add(self, name, algo, params, graph, outputs):
        n, rp, col, w, und = graph
        self.arrays[f"{name}/rp"] = np.asarray(rp, np.int64)
        self.arrays[f"{name}/col"] = np.asarray(col, np.int32)
        if w is not None:
            self.arrays[f"{name}/w"] = np.asarray(w, np.float64)
        for k, v in outputs.items():
            self.arrays[f"{name}/{k}"] = np.asarray(v)
        self.cases.append({"name": name, "algo": algo, "n": int(n), "undirected": bool(und),
                           "weighted": w is not None, "params": params,
                           "outputs": sorted(outputs)})

    def save(self):
        np.savez_compressed(os.path.join(OUT, "golden.npz"), **self.arrays)
        with open(os.path.join(OUT, "manifest.json"), "w") as f:
            json.dump({"generator": "tests/golden/make_golden.py",
                       "reference": "gblite (/root/reference/proj) via oracle/ref_shim.cpp",
                       "cases": self.cases}, f, indent=1)


def G(n, csr, und, weighted=False):
    rp, col, w = csr
    return (n, rp, col, w if weighted else None, und)


def ref_graph(g):
    n, rp, col, w, und = g
    return O.RefGraph(n, rp, col, w, undirected=und)


def main():
    O.build(ref=True)
    S = Store()
    rng = np.random.default_rng(20260401)
    rmat = {}
    for scale in (6, 8, 10):
        rp, col = O.rmat_graph(scale, 16, seed=11, undirected=True)
        rmat[("u", scale)] = G(1 << scale, (rp, col, None), True)
        rp, col = O.rmat_graph(scale, 16, seed=12, undirected=False)
        rmat[("d", scale)] = G(1 << scale, (rp, col, None), False)

    # ---------------- BFS ----------------
    bfs_graphs = [
        ("star3", G(4, star(3), True), 0, [0, 0, 0, 0], None),          # test_bfs.cpp:27-34
        ("path3", G(3, dense_csr(3, [(0, 1), (1, 2)]), False), 0,        # test_bfs.cpp:36-43
         [0, 0, 1], [0, 1, 2]),
        ("empty2", G(2, dense_csr(2, []), False), 1, [-1, 1], None),      # :45-51
        ("star4_src2", G(5, star(4), True), 2, None, None),              # :78-90
        ("disconnected", G(4, dense_csr(4, [(0, 1), (2, 3)]), False), 0,  # :119-129
         [0, 0, -1, -1], None),
    ]
    for k in range(6):
        n = int(rng.integers(1, 65))
        g = G(n, rand_digraph(rng, n, float(rng.uniform(0.02, 0.2))), False)
        bfs_graphs.append((f"randdi{k}", g, int(rng.integers(0, n)), None, None))
    for scale in (8, 10):
        for kind in ("u", "d"):
            g = rmat[(kind, scale)]
            deg = np.diff(g[1])
            bfs_graphs.append((f"rmat{scale}{kind}", g, int(np.argmax(deg)), None, None))
    for name, g, src, want_parent, want_level in bfs_graphs:
        R = ref_graph(g)
        R.property_at()
        outs = {}
        for d, tag in ((0, "auto"), (1, "push"), (2, "pull"), (3, "pushonly")):
            p, l = R.bfs(src, d, 16, True)
            outs[f"parent_{tag}"] = p
            outs[f"level_{tag}"] = l
        if want_parent is not None:
            assert outs["parent_pushonly"].tolist() == want_parent, name
        if want_level is not None:
            assert outs["level_pushonly"].tolist() == want_level, name
        S.add(f"bfs_{name}", "bfs", {"src": src}, g, outs)

    # ---------------- PageRank ----------------
    pr_cases = [
        ("cycle2", G(2, cycle(2), False), dict(damping=0.85, tol=1e-8, itermax=100)),
        ("cycle3", G(3, cycle(3), False), dict(damping=0.85, tol=1e-8, itermax=100)),
        ("path3", G(3, dense_csr(3, [(0, 1), (1, 2)]), False),
         dict(damping=0.85, tol=1e-8, itermax=50)),
        ("cycle2_cap7", G(2, cycle(2), False), dict(damping=0.85, tol=0.0, itermax=7)),
    ]
    for k in range(5):
        n = int(rng.integers(2, 65))
        pr_cases.append((f"randdi{k}", G(n, rand_digraph(rng, n, float(rng.uniform(0.05, 0.3))),
                                         False), dict(damping=0.85, tol=1e-4, itermax=100)))
    for scale in (8, 10):
        pr_cases.append((f"rmat{scale}d", rmat[("d", scale)],
                         dict(damping=0.85, tol=1e-4, itermax=100)))
    for name, g, prm in pr_cases:
        R = ref_graph(g)
        R.property_at()
        R.property_rowdegree()
        rank, iters, trace = R.pagerank(prm["damping"], prm["tol"], prm["itermax"], trace=True)
        if name == "cycle2":
            assert abs(rank[0] - 0.5) <= 1e-12 and rank[0] == rank[1]
        if name == "cycle2_cap7":
            assert iters == 7
        S.add(f"pr_{name}", "pagerank", prm, g,
              {"rank": rank, "iters": np.array(iters), "trace": trace})

    # ---------------- Triangle count ----------------
    n_k4, *k4 = mtx("/root/reference/proj/data/k4.mtx")
    skew = dense_csr(33, [(i, j) for i in range(3) for j in range(3) if i != j])
    tc_cases = [("K3", G(3, complete(3), True), 1), ("K4", G(4, complete(4), True), 4),
                ("C4", G(4, cycle(4, True), True), 0), ("k4mtx", G(n_k4, k4, True), 4),
                ("skew33", G(33, skew, True), 1), ("C16", G(16, cycle(16, True), True), 0)]
    for k in range(6):
        n = int(rng.integers(1, 101))
        tc_cases.append((f"randu{k}", G(n, rand_undirected(rng, n, float(rng.uniform(0.02, 0.25))),
                                        True), None))
    for scale in (8, 10):
        tc_cases.append((f"rmat{scale}u", rmat[("u", scale)], None))
    for name, g, want in tc_cases:
        R = ref_graph(g)
        R.property_rowdegree()
        R.property_ndiag()
        outs = {f"count_{t}": np.array(R.triangle_count(p, 7), np.uint64)
                for p, t in ((0, "auto"), (1, "force"), (2, "never"))}
        if want is not None:
            assert int(outs["count_auto"]) == want, name
        S.add(f"tc_{name}", "triangle_count", {}, g, outs)

    # ---------------- SSSP ----------------
    n_wd, *wd = mtx("/root/reference/proj/data/wdiamond.mtx")
    sssp_cases = [
        ("path", G(3, dense_csr(3, [(0, 1), (1, 2)], [1.0, 1.0]), False, True), 0, [2.0],
         [0.0, 1.0, 2.0]),                                                  # test_sssp.cpp:34-44
        ("diamond", G(3, dense_csr(3, [(0, 1), (0, 2), (1, 2)], [1.0, 4.0, 1.0]), False, True),
         0, [2.0], [0.0, 1.0, 2.0]),                                        # :46-54
        ("unreached", G(4, dense_csr(4, [(0, 1), (2, 3)], [1.0, 1.0]), False, True), 0, [1.0],
         [0.0, 1.0, INF, INF]),                                             # :56-65
        ("defaultdelta", G(3, dense_csr(3, [(0, 1), (1, 2)], [3.0, 6.0]), False, True), 0,
         [3.0], [0.0, 3.0, 9.0]),                                           # :113-121
        ("wdiamond", G(n_wd, wd, False, True), 0, [1.0, 2.5, 8.0], None),
    ]
    for k in range(6):
        n = int(rng.integers(2, 65))
        g = G(n, rand_weighted(rng, n, float(rng.uniform(0.05, 0.3))), False, True)
        sssp_cases.append((f"randw{k}", g, int(rng.integers(0, n)), [0.5, 2.0, 8.0], None))
    for logn in (8, 10):
        rp, col, w = O.er_graph(logn, 16, seed=21)
        g = (1 << logn, rp, col, w.astype(np.float64), False)
        sssp_cases.append((f"er{logn}", g, 0, [64.0, 16.0], None))
    for name, g, src, deltas, want in sssp_cases:
        R = ref_graph(g)
        outs = {}
        for d in deltas:
            outs[f"dist_{d:g}"] = R.sssp(src, d)
        if want is not None:
            for d in deltas:
                assert outs[f"dist_{d:g}"].tolist() == want, name
        S.add(f"sssp_{name}", "sssp", {"src": src, "deltas": deltas,
                                        "default_delta": R_default_delta(R)}, g, outs)

    # ---------------- Betweenness ----------------
    bc_cases = [("path3", G(3, undirected(3, [(0, 1), (1, 2)]), True), [0, 1, 2]),
                ("isolated1", G(1, dense_csr(1, []), True), [0]),
                ("K3", G(3, complete(3), True), [0, 1, 2]),
                ("star4", G(5, star(4), True), [0, 1, 2, 3, 4])]
    for k in range(6):
        n = int(rng.integers(2, 49))
        dens = float(rng.uniform(0.04, 0.25))
        und = k % 2 == 0
        csr = rand_undirected(rng, n, dens) if und else rand_digraph(rng, n, dens)
        bc_cases.append((f"rand{k}", G(n, csr, und), list(range(n))))
    g30 = G(30, rand_undirected(rng, 30, 0.15), True)
    bc_cases.append(("batch30", g30, [3, 11, 17, 29]))                      # test_bc.cpp:93-103
    for scale in (8, 10):
        g = rmat[("u", scale)]
        deg = np.diff(g[1])
        srcs = [int(x) for x in np.argsort(-deg, kind="stable")[:2]] + [1, 5]
        bc_cases.append((f"rmat{scale}u", g, srcs))
    g = rmat[("d", 8)]
    bc_cases.append(("rmat8d", g, [0, 1, 2, 3]))
    for name, g, srcs in bc_cases:
        R = ref_graph(g)
        R.property_at()
        cent = R.bc(srcs)
        if name == "path3":
            assert cent.tolist() == [0.0, 2.0, 0.0]
        S.add(f"bc_{name}", "bc", {"sources": srcs}, g, {"centrality": cent})

    # ---------------- Connected components ----------------
    cc_cases = [("twoedges", G(4, undirected(4, [(0, 1), (2, 3)]), True), [0, 0, 2, 2]),
                ("path5", G(5, undirected(5, [(i, i + 1) for i in range(4)]), True), [0] * 5),
                ("isolated3", G(3, dense_csr(3, []), True), [0, 1, 2])]
    for k in range(6):
        n = int(rng.integers(1, 129))
        cc_cases.append((f"randu{k}", G(n, rand_undirected(rng, n, float(rng.uniform(0.005, 0.08))),
                                        True), None))
    for scale in (8, 10):
        cc_cases.append((f"rmat{scale}u", rmat[("u", scale)], None))
    for name, g, want in cc_cases:
        R = ref_graph(g)
        lab, iters = R.cc()
        if want is not None:
            assert lab.tolist() == want, name
        S.add(f"cc_{name}", "cc", {}, g, {"label": lab, "iters": np.array(iters)})

    # ---------------- degree sort (TC relabel) ----------------
    for scale in (8, 10):
        g = rmat[("u", scale)]
        R = ref_graph(g)
        R.property_rowdegree()
        S.add(f"sortdeg_rmat{scale}u", "sort_by_degree", {}, g, {"perm": R.sort_by_degree()})

    S.save()
    print(f"wrote {len(S.cases)} cases")


def R_default_delta(R):
    return float(O.ref().ref_sssp_default_delta(R._h))


if __name__ == "__main__":
    main()
