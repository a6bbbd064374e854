import numpy as np

import paper_2104_01661_b200 as P


def graph_of(case):
    kind = P.Kind.UndirectedAdjacency if case.undirected else P.Kind.DirectedAdjacency
    return P.graph_new(case.rp, case.col, case.w, kind=kind)


def rel_l1(got, want):
    den = np.abs(want).sum()
    return float(np.abs(got - want).sum() / den) if den > 0 else float(np.abs(got - want).sum())
