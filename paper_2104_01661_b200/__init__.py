"""paper_2104_01661_b200 -- B200-native (sm_100a) hot path of the LAGraph paper's
graph algorithms, a drop-in for gblite's Graph object and algo:: entry points.

The compute path is libgbx.so (csrc/, C ABI in include/gbx.h); this package is
the host-side mirror of the reference interface.  Importing it loads the CUDA
library; there is no CPU fallback.
"""
from . import algo, io, ops
from ._lib import LIB_PATH, lib
from .errors import ErrCode, Error
from .graph import (Domain, Graph, Kind, TriState, check_graph, delete_properties,
                    generate_er, generate_rmat, graph_new, init, property_at,
                    property_coldegree, property_ndiag, property_rowdegree,
                    property_symmetric_pattern, sort_by_degree, version)
from .sources import pick_sources

lib()  # fail loudly at import when the CUDA library is missing

__all__ = ["algo", "io", "ops", "Domain", "ErrCode", "Error", "Graph", "Kind", "TriState", "check_graph",
           "delete_properties", "generate_er", "generate_rmat", "graph_new", "init",
           "property_at", "property_coldegree", "property_ndiag", "property_rowdegree",
           "property_symmetric_pattern", "sort_by_degree", "version", "pick_sources", "LIB_PATH"]
