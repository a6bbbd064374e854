"""CPU-only checks of the C-ABI library: it loads, and exports every entry point
include/gbx.h declares (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gbx.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gbx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("gbx_graph_new", "gbx_property_at", "gbx_property_rowdegree", "gbx_bfs",
                 "gbx_pagerank", "gbx_triangle_count", "gbx_sssp", "gbx_betweenness",
                 "gbx_connected_components", "gbx_basic_pagerank"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2104_01661_b200 as P
    lib = C.CDLL(P.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2104_01661_b200._lib import exported_symbols
    assert set(declared()) == set(exported_symbols())


def test_version_string():
    import paper_2104_01661_b200 as P
    assert "sm_100a" in P.version()


def test_errcodes_mirror_reference():
    # gblite::ErrCode (error.hpp:13-41)
    from paper_2104_01661_b200 import ErrCode
    assert ErrCode.MissingProperty == -6 and ErrCode.SourceOutOfRange == -7
    assert ErrCode.InvalidValue == -21 and ErrCode.NoValue == 1


def test_null_handle_is_an_error_not_a_crash():
    # no GPU needed: the handle check fires before any CUDA call
    import paper_2104_01661_b200 as P
    from paper_2104_01661_b200.graph import call
    with pytest.raises(P.Error) as e:
        call("gbx_graph_info", None, None, None, None, None)
    assert e.value.code == P.ErrCode.NullArgument


def test_sm100a_cubin_present():
    import subprocess
    import paper_2104_01661_b200 as P
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_options_registry():
    """gbx_set_option / gbx_get_option: documented names, range checks, reset to
    the measured default (no GPU needed)."""
    import paper_2104_01661_b200 as P
    from paper_2104_01661_b200._lib import lib
    from paper_2104_01661_b200.graph import call
    names = []
    i = 0
    while lib().gbx_option_name(i) is not None:
        names.append(lib().gbx_option_name(i).decode())
        i += 1
    assert "pagerank.l1_window_kb" in names and "p2p.timeout_ms" in names
    v = C.c_int64()
    call("gbx_get_option", b"pagerank.l1_window_kb", C.byref(v))
    assert v.value == 144
    call("gbx_set_option", b"pagerank.l1_window_kb", C.c_int64(96))
    call("gbx_get_option", b"pagerank.l1_window_kb", C.byref(v))
    assert v.value == 96
    call("gbx_reset_option", b"pagerank.l1_window_kb")
    call("gbx_get_option", b"pagerank.l1_window_kb", C.byref(v))
    assert v.value == 144
    with pytest.raises(P.Error) as e:
        call("gbx_set_option", b"no.such.option", C.c_int64(1))
    assert e.value.code == P.ErrCode.InvalidValue
    with pytest.raises(P.Error) as e:
        call("gbx_set_option", b"p2p.timeout_ms", C.c_int64(0))
    assert e.value.code == P.ErrCode.InvalidValue
