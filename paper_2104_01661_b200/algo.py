"""Host mirror of gblite::algo (include/gblite/algorithms.hpp:12-104).

Advanced forms never touch the caches and raise Error(MissingProperty);
`basic.*` fill the missing caches, then delegate.  Results are dense numpy
arrays: unreached BFS vertices are -1, unreached SSSP vertices +inf (the
reference returns sparse vectors with those entries absent).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import Optional

import numpy as np

from .graph import Graph, _ptr, call


class Direction(IntEnum):
    Auto = 0
    ForcePush = 1
    ForcePull = 2


@dataclass
class BfsConfig:
    direction: Direction = Direction.Auto
    push_divisor: int = 16
    want_level: bool = False


@dataclass
class BfsResult:
    parent: np.ndarray
    level: Optional[np.ndarray] = None


class Presort(IntEnum):
    Auto = 0
    Force = 1
    Never = 2


@dataclass
class TriangleCountConfig:
    presort: Presort = Presort.Auto
    sample_seed: int = 7


@dataclass
class PageRankResult:
    rank: np.ndarray
    iterations: int


@dataclass
class SsspResult:
    dist: np.ndarray


@dataclass
class CentralityResult:
    centrality: np.ndarray


@dataclass
class ComponentResult:
    label: np.ndarray
    iterations: int


def _bfs_out(n, want_level):
    return np.empty(max(n, 1), np.int64), (np.empty(max(n, 1), np.int64) if want_level else None)


def bfs_push(g: Graph, source: int, want_level: bool = False, _fn="gbx_bfs_push") -> BfsResult:
    n = g.n()
    parent, level = _bfs_out(n, want_level)
    call(_fn, _ptr(parent), _ptr(level), g.handle, int(source))
    return BfsResult(parent[:n], level[:n] if level is not None else None)


def bfs_direction_optimizing(g: Graph, source: int, config: BfsConfig = BfsConfig(),
                             _fn="gbx_bfs") -> BfsResult:
    n = g.n()
    parent, level = _bfs_out(n, config.want_level)
    call(_fn, _ptr(parent), _ptr(level), g.handle, int(source), int(config.direction),
         int(config.push_divisor))
    return BfsResult(parent[:n], level[:n] if level is not None else None)


def bfs_batch(g: Graph, sources, want_level: bool = True):
    """B200 extension: ns BFS runs in one 64-lane sweep -> parent/level [ns, n]."""
    n = g.n()
    s = np.ascontiguousarray(sources, np.uint64)
    parent = np.empty((len(s), max(n, 1)), np.int64)
    level = np.empty((len(s), max(n, 1)), np.int64) if want_level else None
    call("gbx_bfs_batch", _ptr(parent), _ptr(level), g.handle, _ptr(s), len(s))
    return parent[:, :n], (level[:, :n] if level is not None else None)


def pagerank_gap(g: Graph, damping: float = 0.85, tol: float = 1e-4, itermax: int = 100,
                 _fn="gbx_pagerank") -> PageRankResult:
    n = g.n()
    rank = np.empty(max(n, 1), np.float64)
    it = C.c_int(0)
    call(_fn, _ptr(rank), C.byref(it), g.handle, float(damping), float(tol), int(itermax))
    return PageRankResult(rank[:n], it.value)


def triangle_count(g: Graph, config: TriangleCountConfig = TriangleCountConfig(),
                   _fn="gbx_triangle_count") -> int:
    c = C.c_uint64(0)
    call(_fn, C.byref(c), g.handle, int(config.presort), int(config.sample_seed))
    return int(c.value)


def sssp_delta_stepping(g: Graph, source: int, delta: float, _fn="gbx_sssp") -> SsspResult:
    n = g.n()
    dist = np.empty(max(n, 1), np.float64)
    call(_fn, _ptr(dist), g.handle, int(source), float(delta))
    return SsspResult(dist[:n])


def sssp_default_delta(g: Graph) -> float:
    d = C.c_double(0)
    call("gbx_sssp_default_delta", C.byref(d), g.handle)
    return d.value


def betweenness_centrality(g: Graph, sources, _fn="gbx_betweenness") -> CentralityResult:
    n = g.n()
    s = np.ascontiguousarray(sources, np.uint64)
    cent = np.empty(max(n, 1), np.float64)
    call(_fn, _ptr(cent), g.handle, _ptr(s) if len(s) else None, len(s))
    return CentralityResult(cent[:n])


def connected_components_fastsv(g: Graph, _fn="gbx_connected_components") -> ComponentResult:
    n = g.n()
    lab = np.empty(max(n, 1), np.int64)
    it = C.c_int(0)
    call(_fn, _ptr(lab), C.byref(it), g.handle)
    return ComponentResult(lab[:n], it.value)


class basic:
    """gblite::algo::basic -- compute missing caches, then delegate."""

    @staticmethod
    def bfs_push(g, source, want_level=False):
        return bfs_push(g, source, want_level, _fn="gbx_basic_bfs_push")

    @staticmethod
    def bfs_direction_optimizing(g, source, config=BfsConfig()):
        return bfs_direction_optimizing(g, source, config, _fn="gbx_basic_bfs")

    @staticmethod
    def pagerank_gap(g, damping=0.85, tol=1e-4, itermax=100):
        return pagerank_gap(g, damping, tol, itermax, _fn="gbx_basic_pagerank")

    @staticmethod
    def triangle_count(g, config=TriangleCountConfig()):
        return triangle_count(g, config, _fn="gbx_basic_triangle_count")

    @staticmethod
    def sssp_delta_stepping(g, source, delta=None):
        return sssp_delta_stepping(g, source, -1.0 if delta is None else delta,
                                   _fn="gbx_basic_sssp")

    @staticmethod
    def betweenness_centrality(g, sources):
        return betweenness_centrality(g, sources, _fn="gbx_basic_betweenness")

    @staticmethod
    def connected_components_fastsv(g):
        return connected_components_fastsv(g, _fn="gbx_basic_connected_components")
