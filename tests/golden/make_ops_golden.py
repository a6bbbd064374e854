"""Generate tests/golden/ops/: random mxv / vxm / mxm cases over the reference's
semirings, domains, masks (none / valued / complemented valued / structural /
complemented structural), replace and accumulators -- the grid of the
reference's own fuzz table (tests/fuzz_core.hpp:526-601) for these three ops --
and the REFERENCE's results for them (gblite::mxv / vxm / mxm through
oracle/_ref).  tests/test_ops.py replays every case on the device and demands
bit-identical output (values compared as raw bits, Fp64 included).

    python tests/golden/make_ops_golden.py      (needs /root/reference; run here)
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "ops")
NPD = {0: np.uint8, 1: np.int64, 2: np.uint64, 3: np.float64}
SEMIRINGS = 7
# accumulators per domain (ops.cpp): value operators, lor/land on bool
ACCUMS = {0: [1, 5, 6, 7, 8, 11, 12], 1: [1, 2, 3, 4, 5, 6, 7, 8, 10],
          2: [1, 2, 3, 4, 5, 6, 7, 8, 10], 3: [1, 2, 3, 4, 5, 6, 7, 8, 9, 10]}


def rvals(rng, m, dom):
    if dom == 0:
        return rng.integers(0, 2, m).astype(np.uint8)
    if dom == 1:
        v = rng.integers(-1000, 1000, m).astype(np.int64)
        if m and rng.random() < 0.3:
            v[rng.integers(0, m)] = np.int64(2**62 + 12345)  # wrapping products / sums
        return v
    if dom == 2:
        v = rng.integers(0, 1000, m).astype(np.uint64)
        if m and rng.random() < 0.3:
            v[rng.integers(0, m)] = np.uint64(2**63 + 7)
        return v
    v = rng.standard_normal(m) * 10.0
    if m and rng.random() < 0.2:
        v[rng.integers(0, m)] = 0.0
    return v


def rmat(rng, nr, nc, dens, dom):
    a = rng.random((nr, nc)) < dens
    rp = np.zeros(nr + 1, np.int64)
    rp[1:] = np.cumsum(a.sum(1))
    col = np.nonzero(a)[1].astype(np.int64)
    return rp, col, rvals(rng, len(col), dom)


def rvec(rng, n, dens, dom):
    idx = np.flatnonzero(rng.random(n) < dens).astype(np.int64)
    return idx, rvals(rng, len(idx), dom)


def p(a):
    return a.ctypes.data if a is not None and len(a) else None


def main():
    os.makedirs(OUT, exist_ok=True)
    L = O.ref()
    L.ref_vec_op.restype = C.c_int
    L.ref_mxm.restype = C.c_int
    i64, vp, I = C.c_int64, C.c_void_p, C.c_int
    L.ref_vec_op.argtypes = [I, I, I, i64, i64, vp, vp, vp, I, i64, i64, vp, vp, I, i64, i64, vp, vp,
                             I, I, i64, i64, vp, vp, I, I, I, I, I, I, I, I, vp, vp, vp]
    L.ref_mxm.argtypes = [I, I, i64, i64, vp, vp, vp, I, i64, i64, vp, vp, vp, I, i64, i64, vp, vp,
                          vp, I, I, vp, vp, vp, I, I, I, I, I, I, I, I, vp]
    L.ref_mxm2.restype = C.c_int
    L.ref_mxm2.argtypes = [I, I, i64, i64, vp, vp, vp, I, i64, i64, vp, vp, vp, I, i64, i64, vp,
                           vp, vp, I, I, i64, i64, vp, vp, vp, I, I, I, I, I, I, I, I, vp]
    L.ref_mxm_fetch.restype = None
    L.ref_mxm_fetch.argtypes = [vp, vp, vp]
    rng = np.random.default_rng(20210403)
    arrays, cases = {}, []
    cid = 0
    ops = ["mxv", "vxm", "mxm", "mxm_tb", "mxv_ta", "vxm_tb", "mxm_ta"]
    for op in ops:
        for dom in range(4):
            for maskvar in range(5):
                for ra in range(4):
                    cid += 1
                    sr = cid % SEMIRINGS
                    sdom = 2 if sr == 1 else dom
                    odom = sdom
                    replace, use_acc = ra & 1, (ra >> 1) & 1
                    acc = int(rng.choice(ACCUMS[odom])) if use_acc else 0
                    dens = [0.1, 0.3, 0.5][cid % 3]
                    nr, kk, nc = (int(rng.integers(1, 13)) for _ in range(3))
                    comp = int(maskvar in (2, 4))
                    structural = int(maskvar >= 3)
                    mdom = int(rng.integers(0, 4))
                    case = {"id": cid, "op": op, "semiring": sr, "sdom": sdom, "dom": dom,
                            "replace": replace, "accum": acc, "accum_domain": odom,
                            "has_mask": int(maskvar > 0), "complement": comp,
                            "structural": structural, "mdom": mdom}
                    k = f"c{cid}_"
                    if op.startswith("mxv") or op.startswith("vxm"):
                        tr = op.endswith("_ta") or op.endswith("_tb")
                        if op.startswith("mxv"):
                            # T = op(A) u: op(A) is nr x kk
                            ar, ac = (kk, nr) if tr else (nr, kk)
                            un, wn = kk, nr
                        else:
                            ar, ac = (nc, kk) if tr else (kk, nc)
                            un, wn = kk, nc
                        arp, acol, aval = rmat(rng, ar, ac, dens, dom)
                        uidx, uval = rvec(rng, un, dens, dom)
                        widx, wval = rvec(rng, wn, 0.4, odom)
                        midx, mval = rvec(rng, wn, 0.5, mdom)
                        oi = np.empty(max(wn, 1), np.int64)
                        ov = np.empty(max(wn, 1), NPD[odom])
                        nv = C.c_int64()
                        rc = L.ref_vec_op(0 if op.startswith("mxv") else 1, sr, sdom, ar, ac,
                                          p(arp), p(acol), p(aval), dom, un, len(uidx), p(uidx),
                                          p(uval), dom, wn, len(widx), p(widx), p(wval), odom,
                                          case["has_mask"], wn, len(midx), p(midx), p(mval), mdom,
                                          comp, structural, replace, acc, odom,
                                          int(op == "mxv_ta"), int(op == "vxm_tb"),
                                          oi.ctypes.data, ov.ctypes.data, C.byref(nv))
                        case.update({"ashape": [ar, ac], "un": un, "wn": wn, "code": rc})
                        for nm, a in (("arp", arp), ("acol", acol), ("aval", aval), ("uidx", uidx),
                                      ("uval", uval), ("widx", widx), ("wval", wval),
                                      ("midx", midx), ("mval", mval)):
                            arrays[k + nm] = a
                        if rc == 0:
                            arrays[k + "oidx"] = oi[:nv.value].copy()
                            arrays[k + "oval"] = ov[:nv.value].copy()
                    else:
                        ta, tb = op == "mxm_ta", op == "mxm_tb"
                        ar, ac = (kk, nr) if ta else (nr, kk)
                        br, bc = (nc, kk) if tb else (kk, nc)
                        arp, acol, aval = rmat(rng, ar, ac, dens, dom)
                        brp, bcol, bval = rmat(rng, br, bc, dens, dom)
                        crp, ccol, cval = rmat(rng, nr, nc, 0.4, odom)
                        mrp, mcol, mval = rmat(rng, nr, nc, 0.5, mdom)
                        nnz = C.c_int64()
                        rc = L.ref_mxm(sr, sdom, ar, ac, p(arp), p(acol), p(aval), dom, br, bc,
                                       p(brp), p(bcol), p(bval), dom, nr, nc, p(crp), p(ccol),
                                       p(cval), odom, case["has_mask"], p(mrp), p(mcol), p(mval),
                                       mdom, comp, structural, replace, acc, odom, int(ta),
                                       int(tb), C.byref(nnz))
                        case.update({"ashape": [ar, ac], "bshape": [br, bc], "cshape": [nr, nc],
                                     "code": rc})
                        for nm, a in (("arp", arp), ("acol", acol), ("aval", aval), ("brp", brp),
                                      ("bcol", bcol), ("bval", bval), ("crp", crp),
                                      ("ccol", ccol), ("cval", cval), ("mrp", mrp),
                                      ("mcol", mcol), ("mval", mval)):
                            arrays[k + nm] = a
                        if rc == 0:
                            orp = np.empty(nr + 1, np.int64)
                            ocol = np.empty(max(nnz.value, 1), np.int64)
                            oval = np.empty(max(nnz.value, 1), NPD[odom])
                            L.ref_mxm_fetch(orp.ctypes.data, ocol.ctypes.data, oval.ctypes.data)
                            arrays[k + "orp"] = orp
                            arrays[k + "ocol"] = ocol[:nnz.value].copy()
                            arrays[k + "oval"] = oval[:nnz.value].copy()
                    cases.append(case)
    # error cases: each perturbs one precondition of a valid call
    errs = [("mxv", "domain"), ("vxm", "domain"), ("mxm", "domain"), ("mxv", "ulen"),
            ("vxm", "wlen"), ("mxm", "inner"), ("mxv", "masklen"), ("mxm", "maskshape"),
            ("mxv", "accumdom"), ("mxm", "outdom")]
    for op, what in errs:
        cid += 1
        k = f"c{cid}_"
        dom, sr = 3, 0  # plus_times over fp64
        nr, kk, nc = 5, 4, 6
        acc = 1 if what == "accumdom" else 0
        accdom = 1 if what == "accumdom" else 3
        adom = 1 if what == "domain" else 3
        odom = 1 if what == "outdom" else 3
        case = {"id": cid, "op": op, "semiring": sr, "sdom": dom, "dom": adom, "replace": 0,
                "accum": acc, "accum_domain": accdom, "has_mask": int(what.startswith("mask")),
                "complement": 0, "structural": 0, "mdom": 3, "error_case": what}
        if op in ("mxv", "vxm"):
            ar, ac = (nr, kk) if op == "mxv" else (kk, nc)
            un = (kk if op == "mxv" else kk) + (1 if what == "ulen" else 0)
            wn = (nr if op == "mxv" else nc) + (1 if what == "wlen" else 0)
            arp, acol, aval = rmat(rng, ar, ac, 0.5, adom)
            uidx, uval = rvec(rng, un, 0.5, 3)
            widx, wval = rvec(rng, wn, 0.4, 3)
            mn = wn + (2 if what == "masklen" else 0)
            midx, mval = rvec(rng, mn, 0.5, 3)
            oi = np.empty(max(wn, 1), np.int64)
            ov = np.empty(max(wn, 1), np.float64)
            nv = C.c_int64()
            # the reference's SparseVector mask carries its own length
            rc = L.ref_vec_op(0 if op == "mxv" else 1, sr, dom, ar, ac, p(arp), p(acol), p(aval),
                              adom, un, len(uidx), p(uidx), p(uval), 3, wn, len(widx), p(widx),
                              p(wval), 3, case["has_mask"], mn, len(midx), p(midx), p(mval), 3, 0, 0,
                              0, acc, accdom, 0, 0, oi.ctypes.data, ov.ctypes.data, C.byref(nv))
            case.update({"ashape": [ar, ac], "un": un, "wn": wn, "mn": mn, "code": rc})
            for nm, a in (("arp", arp), ("acol", acol), ("aval", aval), ("uidx", uidx),
                          ("uval", uval), ("widx", widx), ("wval", wval), ("midx", midx),
                          ("mval", mval)):
                arrays[k + nm] = a
        else:
            kb = kk + (1 if what == "inner" else 0)
            arp, acol, aval = rmat(rng, nr, kk, 0.5, adom)
            brp, bcol, bval = rmat(rng, kb, nc, 0.5, adom)
            crp, ccol, cval = rmat(rng, nr, nc, 0.4, odom)
            mr, mc = (nr + 1, nc) if what == "maskshape" else (nr, nc)
            mrp, mcol, mval = rmat(rng, mr, mc, 0.5, 3)
            nnz = C.c_int64()
            rc = L.ref_mxm2(sr, dom, nr, kk, p(arp), p(acol), p(aval), adom, kb, nc, p(brp),
                            p(bcol), p(bval), adom, nr, nc, p(crp), p(ccol), p(cval), odom,
                            case["has_mask"], mr, mc, p(mrp), p(mcol), p(mval), 3, 0, 0, 0, acc,
                            accdom, 0, 0, C.byref(nnz))
            case.update({"ashape": [nr, kk], "bshape": [kb, nc], "cshape": [nr, nc],
                         "mshape": [mr, mc], "code": rc})
            for nm, a in (("arp", arp), ("acol", acol), ("aval", aval), ("brp", brp),
                          ("bcol", bcol), ("bval", bval), ("crp", crp), ("ccol", ccol),
                          ("cval", cval), ("mrp", mrp), ("mcol", mcol), ("mval", mval)):
                arrays[k + nm] = a
        cases.append(case)
    np.savez_compressed(os.path.join(OUT, "ops.npz"), **arrays)
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_ops_golden.py",
                   "reference": "gblite mxv / vxm / mxm (core.cpp:267-386) via oracle/_ref",
                   "cases": cases}, f, indent=0)
    codes = {}
    for c in cases:
        codes[c["code"]] = codes.get(c["code"], 0) + 1
    print(len(cases), "cases; reference codes:", codes)


if __name__ == "__main__":
    main()
