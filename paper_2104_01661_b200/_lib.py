"""ctypes binding of libgbx.so (include/gbx.h).  Loads the in-tree build and
fails loudly when it is missing: there is no CPU fallback."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GBX_LIB") or os.path.join(_HERE, "libgbx.so")
MSG_LEN = 256

_lib = None


class gbx_stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("hot_launches", C.c_int64),
                ("hot_bytes_per_launch", C.c_double), ("work_units", C.c_int64),
                ("iterations", C.c_int), ("hot_ms", C.c_double)]


_vp = C.c_void_p
_i64 = C.c_int64
_u64 = C.c_uint64
_int = C.c_int
_dbl = C.c_double
_cp = C.c_char_p
_pp = C.POINTER(C.c_void_p)

# name: (argtypes) -- every function returns int and takes char* msg last
_SIGS = {
    "gbx_init": [_int],
    "gbx_set_option": [_cp, _i64],
    "gbx_reset_option": [_cp],
    "gbx_get_option": [_cp, _vp],
    "gbx_graph_new": [_pp, _i64, _vp, _vp, _vp, _int, _int],
    "gbx_graph_new32": [_pp, _i64, _vp, _vp, _vp, _int, _int],
    "gbx_graph_free": [_pp],
    "gbx_generate_rmat": [_pp, _int, _int, _dbl, _dbl, _dbl, _u64, _int, _int],
    "gbx_generate_er": [_pp, _int, _int, _u64, _int],
    "gbx_graph_info": [_vp, _vp, _vp, _vp, _vp],
    "gbx_graph_export": [_vp, _vp, _vp, _vp],
    "gbx_property_at": [_vp],
    "gbx_property_rowdegree": [_vp],
    "gbx_property_coldegree": [_vp],
    "gbx_property_symmetric_pattern": [_vp],
    "gbx_property_ndiag": [_vp],
    "gbx_delete_properties": [_vp],
    "gbx_graph_properties": [_vp, _vp, _vp, _vp, _vp, _vp],
    "gbx_row_degree": [_vp, _vp],
    "gbx_col_degree": [_vp, _vp],
    "gbx_check_graph": [_vp],
    "gbx_sort_by_degree": [_vp, _vp, _int, _int],
    "gbx_bfs_push": [_vp, _vp, _vp, _u64],
    "gbx_bfs": [_vp, _vp, _vp, _u64, _int, _u64],
    "gbx_bfs_batch": [_vp, _vp, _vp, _vp, _u64],
    "gbx_pagerank": [_vp, _vp, _vp, _dbl, _dbl, _int],
    "gbx_triangle_count": [_vp, _vp, _int, _u64],
    "gbx_sssp": [_vp, _vp, _u64, _dbl],
    "gbx_sssp_default_delta": [_vp, _vp],
    "gbx_sssp_batch": [_vp, _vp, _vp, _u64, _dbl],
    "gbx_betweenness": [_vp, _vp, _vp, _u64],
    "gbx_connected_components": [_vp, _vp, _vp],
    "gbx_basic_bfs_push": [_vp, _vp, _vp, _u64],
    "gbx_basic_bfs": [_vp, _vp, _vp, _u64, _int, _u64],
    "gbx_basic_pagerank": [_vp, _vp, _vp, _dbl, _dbl, _int],
    "gbx_basic_triangle_count": [_vp, _vp, _int, _u64],
    "gbx_basic_sssp": [_vp, _vp, _u64, _dbl],
    "gbx_basic_betweenness": [_vp, _vp, _vp, _u64],
    "gbx_basic_connected_components": [_vp, _vp, _vp],
    "gbx_graph_stream": [_vp, _pp],
    "gbx_prepare": [_vp, _cp],
    "gbx_result_device": [_vp, _cp, _pp, _vp],
    "gbx_last_stats": [_vp, C.POINTER(gbx_stats)],
    "gbx_pr_shard_prepare": [_vp, _int, _int, _vp, _vp],
    "gbx_pr_shard_init": [_vp, _vp, _vp, _dbl],
    "gbx_pr_shard_unpermute": [_vp, _vp, _vp],
    "gbx_pr_shard_step": [_vp, _vp, _vp, _vp, _vp, _vp, _dbl],
    "gbx_pr_shard_layout": [_vp, _vp, _vp],
    "gbx_pr_shard_run_p2p": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _int, _vp],
    "gbx_pr_shard_run_p2p_multi": [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _int,
                                   _vp],
    "gbx_partition_rows": [_vp, _vp, _int, _int],
    "gbx_triangle_count_rows": [_vp, _vp, _i64, _i64],
    "gbx_tc_partition": [_vp, _vp, _int],
    "gbx_graph_build": [_pp, _i64, _i64, _vp, _vp, _vp, _int, _int, _int],
    "gbx_graph_read": [_pp, _cp, _cp, _int],
    "gbx_graph_read_buffer": [_pp, _vp, C.c_size_t, _cp, _int],
    "gbx_graph_write": [_vp, _cp, _cp, _int],
    "gbx_mat_new": [_pp, _i64, _i64, _vp, _vp, _vp, _int],
    "gbx_mat_from_graph": [_pp, _vp, _int],
    "gbx_mat_info": [_vp, _vp, _vp, _vp, _vp],
    "gbx_mat_export": [_vp, _vp, _vp, _vp],
    "gbx_mat_free": [_pp],
    "gbx_mxv": [_vp, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp],
    "gbx_vxm": [_vp, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp],
    "gbx_mxm": [_pp, _vp, _vp, _int, _int, _vp, _vp],
    "gbx_bc_shard_begin": [_vp, _vp, _u64, _int, _int, _vp, _vp],
    "gbx_bfs_shard_begin": [_vp, _u64, _int, _int, _vp, _vp],
    "gbx_bfs_shard_level": [_vp, _vp, _vp, _vp],
    "gbx_bfs_shard_result": [_vp, _vp, _vp],
    "gbx_bc_shard_forward": [_vp, _pp, _vp],
    "gbx_bc_shard_forward_apply": [_vp, _vp, _i64, _vp],
    "gbx_bc_shard_backward": [_vp, _pp, _vp, _vp],
    "gbx_bc_shard_backward_apply": [_vp, _vp, _i64],
    "gbx_bc_shard_centrality": [_vp, _pp],
    "gbx_comm_unique_id": [_vp],
    "gbx_comm_init": [_pp, _int, _int, _vp, _int],
    "gbx_comm_init_local": [_pp, _int, _int],
    "gbx_comm_free": [_pp],
    "gbx_comm_info": [_vp, _vp, _vp, _vp],
    "gbx_dgraph_generate_rmat": [_pp, _vp, _int, _int, _dbl, _dbl, _dbl, _u64, _int, _int],
    "gbx_dgraph_from_blocks": [_pp, _vp, _i64, _vp, _vp, _vp, _vp, _int],
    "gbx_dgraph_free": [_pp],
    "gbx_dgraph_info": [_vp, _vp, _vp, _vp],
    "gbx_dgraph_block": [_vp, _int, _vp, _vp, _vp],
    "gbx_dgraph_export_block": [_vp, _int, _vp, _vp],
    "gbx_dgraph_last_stats": [_vp, C.POINTER(gbx_stats)],
    "gbx_pagerank_mg": [_vp, _vp, _vp, _dbl, _dbl, _int, _int],
    "gbx_triangle_count_mg": [_vp, _vp],
    "gbx_bfs_mg": [_vp, _vp, _vp, _u64],
    "gbx_betweenness_mg": [_vp, _vp, _vp, _u64],
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (make -C paper_2104_01661_b200/csrc).  There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = list(args) + [C.c_char_p]
            f.restype = C.c_int
        L.gbx_version.restype = C.c_char_p
        L.gbx_version.argtypes = []
        L.gbx_option_name.restype = C.c_char_p
        L.gbx_option_name.argtypes = [C.c_int]
        _lib = L
    return _lib


def exported_symbols():
    return sorted(list(_SIGS) + ["gbx_version", "gbx_option_name"])
