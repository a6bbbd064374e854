"""Generate tests/golden/io/: Matrix Market / LAGK inputs and the REFERENCE's
own results for them (gblite::io, io.cpp:35-355, run through oracle/_ref).

For every case the reference reads the input (read_matrix_file) and, when that
succeeds and the matrix is square (graph_new), writes it back as LAGK
(bin_write), as general Matrix Market (mm_write) and as symmetric Matrix Market
(mm_write(symmetric=true), which may fail).  manifest.json records the codes;
the written files are the byte-exact expectations for libgbx's readers and
writers (tests/test_io.py).  The inputs are hand-written here.

    python tests/golden/make_io_golden.py      (needs /root/reference; run here)
"""
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "io")

MM = {
    "pattern_general": "%%MatrixMarket matrix coordinate pattern general\n% a comment\n"
                       "4 4 5\n1 2\n2 3\n3 1\n4 4\n1 4\n",
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n2 1\n3 1\n2 2\n",
    "integer_general": "%%MatrixMarket matrix coordinate integer general\n3 3 4\n"
                       "1 1 -5\n3 2 7\n2 3 0\n1 3 9223372036854775807\n",
    "real_general": "%%MatrixMarket matrix coordinate real general\n3 3 5\n1 2 0.1\n"
                    "2 1 -2.5e-300\n3 3 3.14159265358979\n1 1 1e300\n2 2 -0\n",
    "real_symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n2 1 0.5\n"
                      "3 3 2\n4 2 -1.25\n4 1 3\n",
    "domain_uint64": "%%MatrixMarket matrix coordinate integer general\n%%domain uint64\n"
                     "2 2 2\n1 1 18\n2 1 3\n",
    "domain_bool": "%%MatrixMarket matrix coordinate integer general\n%%domain bool\n"
                   "3 3 3\n1 2 0\n2 3 5\n3 1 1\n",
    "domain_bool_alltrue": "%%MatrixMarket matrix coordinate integer general\n%%domain bool\n"
                           "2 2 2\n1 2 1\n2 1 7\n",
    "domain_fp64_on_integer": "%%MatrixMarket matrix coordinate integer general\n%%domain fp64\n"
                              "2 2 1\n1 2 4\n",
    "pattern_ignores_domain": "%%MatrixMarket matrix coordinate pattern general\n%%domain int64\n"
                              "2 2 1\n2 1\n",
    "crlf_blank_comments": "%%MatrixMarket matrix coordinate integer general\r\n\r\n% c1\r\n\r\n"
                           "%c2\r\n3 3 3\r\n3 3 1\r\n1 1 2\r\n2 1 3\r\n",
    "extra_lines_ignored": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\n"
                           "garbage that is never read\n",
    "unordered_entries": "%%MatrixMarket matrix coordinate integer general\n4 4 6\n4 1 1\n"
                         "1 4 2\n2 2 3\n1 1 4\n4 4 5\n3 2 6\n",
    "tabs_and_spaces": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n 1\t2  -3\n"
                       "2 1\t4 trailing\n",
    "empty_matrix": "%%MatrixMarket matrix coordinate pattern general\n3 3 0\n",
    "zero_by_zero": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "no_trailing_newline": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1",
    # errors (codes as the reference reports them)
    "err_missing_banner": "%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n",
    "err_object": "%%MatrixMarket vector coordinate pattern general\n2 2 1\n1 1\n",
    "err_format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "err_field": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n",
    "err_symmetry": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "err_size_line": "%%MatrixMarket matrix coordinate pattern general\n2 2\n1 1\n",
    "err_no_size_line": "%%MatrixMarket matrix coordinate pattern general\n% only comments\n",
    "err_index_zero": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n0 1\n",
    "err_index_big": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n2 3\n",
    "err_duplicate": "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 1 1\n2 2 2\n1 1 3\n",
    "err_sym_duplicate": "%%MatrixMarket matrix coordinate pattern symmetric\n2 2 2\n2 1\n1 2\n",
    "err_short": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n1 1\n2 2\n",
    "err_missing_value": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 1 4\n2 2\n",
    "err_negative_uint64": "%%MatrixMarket matrix coordinate integer general\n%%domain uint64\n"
                           "2 2 1\n1 1 -3\n",
    "err_unknown_domain": "%%MatrixMarket matrix coordinate integer general\n%%domain int8\n"
                          "2 2 1\n1 1 1\n",
    "err_bad_indices": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\nx 1\n",
    "err_empty_line_entry": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n\n2 2\n",
    "err_nonsquare": "%%MatrixMarket matrix coordinate pattern general\n3 4 2\n1 4\n3 1\n",
    "err_empty_stream": "",
}


def lagk(domain, nrows, ncols, rp, col, vals_bytes):
    b = b"LAGK" + struct.pack("<IB", 1, domain) + struct.pack("<QQQ", nrows, ncols, len(col))
    b += np.asarray(rp, "<u8").tobytes() + np.asarray(col, "<u8").tobytes() + vals_bytes
    return b


def bin_cases():
    good = lagk(3, 3, 3, [0, 2, 2, 3], [0, 2, 1], np.array([1.5, -2.0, 7.25], "<f8").tobytes())
    return {
        "bin_fp64": good,
        "bin_bool_values": lagk(0, 2, 2, [0, 1, 2], [1, 0], bytes([0, 9])),
        "bin_int64": lagk(1, 2, 2, [0, 2, 2], [0, 1], np.array([-1, 2**62], "<i8").tobytes()),
        "bin_empty": lagk(0, 0, 0, [0], [], b""),
        "err_bin_magic": b"LAGX" + good[4:],
        "err_bin_version": good[:4] + struct.pack("<I", 2) + good[8:],
        "err_bin_tag": good[:8] + bytes([9]) + good[9:],
        "err_bin_truncated": good[:-5],
        "err_bin_truncated_header": good[:20],
        "err_bin_unsorted": lagk(1, 2, 2, [0, 2, 2], [1, 0], np.array([1, 2], "<i8").tobytes()),
        "err_bin_rowptr": lagk(1, 2, 2, [0, 2, 1], [0, 1], np.array([1, 2], "<i8").tobytes()),
        "err_bin_col_range": lagk(1, 2, 2, [0, 1, 1], [5], np.array([1], "<i8").tobytes()),
        "err_bin_nonsquare": lagk(0, 2, 3, [0, 1, 1], [2], bytes([1])),
    }


def main():
    os.makedirs(OUT, exist_ok=True)
    L = O.ref()
    cases = {}
    inputs = [(k, "mm", v.encode()) for k, v in MM.items()] + \
             [(k, "bin", v) for k, v in bin_cases().items()]
    for name, fmt, data in inputs:
        src = os.path.join(OUT, f"{name}.{'mtx' if fmt == 'mm' else 'lagk'}")
        with open(src, "wb") as f:
            f.write(data)
        rc = L.ref_io_convert(src.encode(), fmt.encode(), None, None, 1)
        entry = {"input": os.path.basename(src), "format": fmt, "code": rc,
                 "error": L.ref_last_error().decode() if rc else ""}
        if rc == 0:
            for ofmt, ext in (("bin", "ref.lagk"), ("mm", "ref.mtx"), ("mm_sym", "ref_sym.mtx")):
                dst = os.path.join(OUT, f"{name}.{ext}")
                c = L.ref_io_convert(src.encode(), fmt.encode(), dst.encode(), ofmt.encode(), 0)
                entry[ofmt] = {"code": c, "file": os.path.basename(dst) if c == 0 else None}
                if c != 0 and os.path.exists(dst):
                    os.remove(dst)
        cases[name] = entry
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_io_golden.py",
                   "reference": "gblite::io via oracle/_ref (io.cpp:35-355)",
                   "cases": cases}, f, indent=1, sort_keys=True)
    print(f"{len(cases)} cases, {sum(1 for c in cases.values() if c['code'] == 0)} readable")


if __name__ == "__main__":
    main()
