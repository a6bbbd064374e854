"""The GraphBLAS operation layer (csrc/ops.cu) against the reference itself.

tests/golden/ops/ holds 570 cases of mxv / vxm / mxm (with transposes) over
the reference's seven semirings, its four domains, the five mask kinds of its
fuzz table (tests/fuzz_core.hpp:61-110: none, valued, complemented valued,
structural, complemented structural), replace and accumulators, plus error
cases -- each with the REFERENCE's result (make_ops_golden.py, gblite through
oracle/_ref).  The device results must be identical bit for bit (Fp64 values
compared as raw bits: every fold runs in the reference's order).
"""
import json
import os

import numpy as np
import pytest

import paper_2104_01661_b200 as P
from paper_2104_01661_b200.graph import Domain
from paper_2104_01661_b200.ops import Descriptor, Matrix, Vector, mxm, mxv, vxm

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ops")
MANIFEST = json.load(open(os.path.join(GOLD, "manifest.json")))["cases"]
_ARR = None


def arr():
    global _ARR
    if _ARR is None:
        _ARR = dict(np.load(os.path.join(GOLD, "ops.npz")))
    return _ARR


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def test_grid_covers_reference_fuzz_axes():
    ops = {c["op"] for c in MANIFEST}
    assert {"mxv", "vxm", "mxm", "mxm_tb", "mxv_ta", "vxm_tb", "mxm_ta"} <= ops
    assert {c["semiring"] for c in MANIFEST} == set(range(7))
    assert {c["dom"] for c in MANIFEST} == {0, 1, 2, 3}
    kinds = {(c["has_mask"], c["complement"], c["structural"]) for c in MANIFEST}
    assert len(kinds) == 5
    assert {c["code"] for c in MANIFEST} == {0, -1, -2}


def _case_inputs(c):
    a = arr()
    k = f"c{c['id']}_"
    A = Matrix.from_csr(c["ashape"][0], c["ashape"][1], a[k + "arp"], a[k + "acol"], a[k + "aval"],
                        c["dom"])
    return a, k, A


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [c["id"] for c in MANIFEST])
def test_op_matches_reference(cid):
    c = next(x for x in MANIFEST if x["id"] == cid)
    a, k, A = _case_inputs(c)
    odom = Domain(c["sdom"])
    if c.get("error_case") == "outdom":
        odom = Domain.Int64
    desc = Descriptor(complement=bool(c["complement"]), structural=bool(c["structural"]),
                      replace=bool(c["replace"]), accum=c["accum"],
                      accum_domain=Domain(c["accum_domain"]),
                      transpose_in1=c["op"] in ("mxv_ta", "mxm_ta"),
                      transpose_in2=c["op"] in ("vxm_tb", "mxm_tb"))
    if c["op"].startswith(("mxv", "vxm")):
        udom = 3 if "error_case" in c else c["dom"]
        u = Vector(c["un"], a[k + "uidx"], a[k + "uval"], Domain(udom))
        wdom = 3 if "error_case" in c else c["sdom"]
        w = Vector(c["wn"], a[k + "widx"], a[k + "wval"], Domain(wdom))
        if c["has_mask"]:
            desc.mask = Vector(c.get("mn", c["wn"]), a[k + "midx"], a[k + "mval"], Domain(c["mdom"]))
        f = mxv if c["op"].startswith("mxv") else vxm
        args = (A, u) if f is mxv else (u, A)
        if c["code"] != 0:
            with pytest.raises(P.Error) as e:
                f(w, desc, c["semiring"], c["sdom"], *args)
            assert e.value.code == c["code"], e.value
            return
        got = f(w, desc, c["semiring"], c["sdom"], *args)
        assert np.array_equal(got.idx, a[k + "oidx"])
        assert np.array_equal(bits(got.vals), bits(a[k + "oval"]))
    else:
        B = Matrix.from_csr(c["bshape"][0], c["bshape"][1], a[k + "brp"], a[k + "bcol"],
                            a[k + "bval"], c["dom"])
        cdom = int(odom)
        Cm = Matrix.from_csr(c["cshape"][0], c["cshape"][1], a[k + "crp"], a[k + "ccol"],
                             a[k + "cval"], cdom)
        if c["has_mask"]:
            ms = c.get("mshape", c["cshape"])
            desc.mask = Matrix.from_csr(ms[0], ms[1], a[k + "mrp"], a[k + "mcol"], a[k + "mval"],
                                        c["mdom"])
        if c["code"] != 0:
            with pytest.raises(P.Error) as e:
                mxm(Cm, desc, c["semiring"], c["sdom"], A, B)
            assert e.value.code == c["code"], e.value
            return
        out = mxm(Cm, desc, c["semiring"], c["sdom"], A, B)
        rp, col, vals = out.export()
        assert np.array_equal(rp, a[k + "orp"])
        assert np.array_equal(col, a[k + "ocol"])
        assert np.array_equal(bits(vals), bits(a[k + "oval"]))


@pytest.mark.gpu
def test_masked_plus_pair_counts_triangles():
    """C<L> = L plus.pair U' (triangle.cpp:30-64) through the op layer equals the
    fused triangle-count kernel and the oracle on an R-MAT graph."""
    import oracle as O
    from paper_2104_01661_b200 import algo
    g = P.generate_rmat(10, 8, seed=4, kind=P.Kind.UndirectedAdjacency)
    rp, col, _ = g.export()
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    lo = col < rows
    L_rp = np.zeros(n + 1, np.int64)
    L_rp[1:] = np.cumsum(np.bincount(rows[lo], minlength=n))
    L = Matrix.from_csr(n, n, L_rp, col[lo], np.ones(lo.sum(), np.uint8), Domain.Bool)
    up = col > rows
    U_rp = np.zeros(n + 1, np.int64)
    U_rp[1:] = np.cumsum(np.bincount(rows[up], minlength=n))
    U = Matrix.from_csr(n, n, U_rp, col[up], np.ones(up.sum(), np.uint8), Domain.Bool)
    C0 = Matrix.from_csr(n, n, np.zeros(n + 1, np.int64), [], [], Domain.Uint64)
    T = mxm(C0, Descriptor(mask=L, structural=True, transpose_in2=True), 5, Domain.Uint64, L, U)
    # C<L> = L * U' over plus.pair: T(i,j) = |L(i,:) ∩ U(j,:)|, j < i
    _, _, v = T.export()
    P.property_ndiag(g)
    P.property_rowdegree(g)
    want = O.triangle_count(n, rp, col)
    assert int(v.sum()) == want == algo.triangle_count(g)
