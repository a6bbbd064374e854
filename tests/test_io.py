"""Graph ingest / export (csrc/io.cu) against the reference's own gblite::io.

tests/golden/io/ holds hand-written Matrix Market / LAGK inputs and what the
REFERENCE did with each (make_io_golden.py, run through oracle/_ref): its
error code, or the LAGK / Matrix Market bytes it writes back (bin_write,
mm_write, mm_write(symmetric)).  Our reader lands the matrix in HBM; our
writers must then reproduce the reference's bytes exactly, which pins every
index, value and domain the reader produced.
"""
import json
import os

import numpy as np
import pytest

import paper_2104_01661_b200 as P
from paper_2104_01661_b200.io import (Dup, build_graph, read_matrix_bytes, read_matrix_file,
                                      write_matrix_file)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
MANIFEST = json.load(open(os.path.join(GOLD, "manifest.json")))["cases"]
CASES = sorted(MANIFEST)


def _bytes(name):
    with open(os.path.join(GOLD, name), "rb") as f:
        return f.read()


def test_manifest_covers_reference_error_codes():
    codes = {c["code"] for c in MANIFEST.values()}
    # ParseError, IndexOutOfBounds, DuplicateEntry, BadMagic, UnsupportedVersion,
    # TruncatedStream, InvalidMatrix, InvalidValue (error.hpp:13-41)
    assert {0, -13, -3, -14, -16, -17, -18, -4, -21} <= codes
    for c in MANIFEST.values():
        assert os.path.exists(os.path.join(GOLD, c["input"]))
        if c["code"] == 0:
            assert c["bin"]["code"] == 0 and c["mm"]["code"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_read_matches_reference(name, tmp_path):
    c = MANIFEST[name]
    data = _bytes(c["input"])
    if c["code"] != 0:
        with pytest.raises(P.Error) as e:
            read_matrix_bytes(data, c["format"])
        assert e.value.code == c["code"], (e.value, c["error"])
        return
    g = read_matrix_bytes(data, c["format"])
    for ofmt, sym in (("bin", False), ("mm", False), ("mm_sym", True)):
        want = c[ofmt]
        out = tmp_path / f"out.{ofmt}"
        fmt = "bin" if ofmt == "bin" else "mm"
        if want["code"] != 0:
            with pytest.raises(P.Error) as e:
                write_matrix_file(g, str(out), fmt, symmetric=sym)
            assert e.value.code == want["code"]
        else:
            write_matrix_file(g, str(out), fmt, symmetric=sym)
            assert out.read_bytes() == _bytes(want["file"]), ofmt


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in CASES if MANIFEST[n]["code"] == 0])
def test_file_read_equals_buffer_read(name, tmp_path):
    c = MANIFEST[name]
    g1 = read_matrix_file(os.path.join(GOLD, c["input"]), c["format"])
    g2 = read_matrix_bytes(_bytes(c["input"]), c["format"])
    a, b = g1.export(), g2.export()
    assert g1.info() == g2.info()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.gpu
def test_missing_file_is_io_failure(tmp_path):
    with pytest.raises(P.Error) as e:
        read_matrix_file(str(tmp_path / "nope.mtx"), "mm")
    assert e.value.code == P.ErrCode.IoFailure
    with pytest.raises(P.Error) as e:
        read_matrix_file(os.path.join(GOLD, MANIFEST["pattern_general"]["input"]), "xml")
    assert e.value.code == P.ErrCode.InvalidValue


def _rand_tuples(rng, n, m):
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    return r, c


def _expected_csr(n, r, c, v, how):
    """numpy restatement of build_matrix's stable sort + in-order dup fold."""
    order = np.lexsort((np.arange(len(r)), c, r))
    r, c = r[order], c[order]
    v = None if v is None else v[order]
    key = r * n + c
    head = np.ones(len(key), bool)
    head[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(head)
    ends = np.append(starts[1:], len(key))
    out = None
    if v is not None:
        out = np.empty(len(starts), v.dtype)
        for i, (s, e) in enumerate(zip(starts, ends)):
            seg = v[s:e]
            if how == Dup.First:
                out[i] = seg[0]
            elif how == Dup.Second:
                out[i] = seg[-1]
            elif how == Dup.Min:
                out[i] = seg.min()
            elif how == Dup.Max:
                out[i] = seg.max()
            else:
                acc = seg[0]
                for x in seg[1:]:
                    acc = acc + x
                out[i] = acc
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r[starts] + 1, 1)
    return np.cumsum(rp), c[starts].astype(np.int32), out


@pytest.mark.gpu
@pytest.mark.parametrize("how", list(Dup)[1:])
@pytest.mark.parametrize("dtype", [np.float64, np.int64])
def test_build_duplicate_policies(how, dtype):
    rng = np.random.default_rng(int(how) * 7 + (dtype == np.int64))
    n, m = 300, 5000
    r, c = _rand_tuples(rng, n, m)
    v = (rng.standard_normal(m) * 100).astype(dtype) if dtype == np.float64 else \
        rng.integers(-1000, 1000, m).astype(dtype)
    g = build_graph(n, r, c, v, dup=how)
    rp, col, vals = g.export()
    wrp, wcol, wv = _expected_csr(n, r, c, v, how)
    assert np.array_equal(rp, wrp) and np.array_equal(col, wcol)
    assert np.array_equal(vals, wv)  # bit-exact: in-order fold, same association


@pytest.mark.gpu
def test_build_errors():
    with pytest.raises(P.Error) as e:
        build_graph(4, [0, 1, 0], [1, 2, 1])
    assert e.value.code == P.ErrCode.DuplicateEntry
    with pytest.raises(P.Error) as e:
        build_graph(4, [0, 4], [1, 2])
    assert e.value.code == P.ErrCode.IndexOutOfBounds
    g = build_graph(4, [], [])
    assert g.info()[:2] == (4, 0)


@pytest.mark.gpu
def test_large_mm_multithreaded_parse(tmp_path):
    """A few MB of entries (parsed by several host threads) against numpy."""
    rng = np.random.default_rng(5)
    n, m = 1 << 15, 400_000
    r, c = _rand_tuples(rng, n, m)
    key = np.unique(r * n + c)
    rng.shuffle(key)
    r, c = key // n, key % n
    v = rng.standard_normal(len(r))
    lines = "\n".join(f"{a + 1} {b + 1} {x:.17g}" for a, b, x in zip(r, c, v))
    text = f"%%MatrixMarket matrix coordinate real general\n{n} {n} {len(r)}\n{lines}\n"
    path = tmp_path / "big.mtx"
    path.write_text(text)
    g = read_matrix_file(str(path), "mm")
    rp, col, vals = g.export()
    wrp, wcol, wv = _expected_csr(n, r, c, v, Dup.First)
    assert np.array_equal(rp, wrp) and np.array_equal(col, wcol) and np.array_equal(vals, wv)
    # LAGK round trip is bit-exact and feeds the algorithms
    out = tmp_path / "big.lagk"
    write_matrix_file(g, str(out), "bin")
    g2 = read_matrix_file(str(out), "bin")
    rp2, col2, vals2 = g2.export()
    assert np.array_equal(rp2, rp) and np.array_equal(col2, col) and np.array_equal(vals2, vals)


@pytest.mark.gpu
def test_read_graph_runs_algorithms(tmp_path):
    """An R-MAT graph written to LAGK and read back gives the same BFS."""
    from paper_2104_01661_b200 import algo
    g = P.generate_rmat(12, 16, seed=9, kind=P.Kind.UndirectedAdjacency)
    out = tmp_path / "g.lagk"
    write_matrix_file(g, str(out), "bin")
    h = read_matrix_file(str(out), "bin", kind=P.Kind.UndirectedAdjacency)
    for x in (g, h):
        P.property_at(x)
    src = int(np.argmax(np.diff(g.export()[0])))
    a = algo.bfs_direction_optimizing(g, src, algo.BfsConfig(want_level=True))
    b = algo.bfs_direction_optimizing(h, src, algo.BfsConfig(want_level=True))
    assert np.array_equal(a.parent, b.parent) and np.array_equal(a.level, b.level)
