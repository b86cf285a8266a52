"""Host-side compressed-row NeighborGraph (graph.hpp:31-54).

`Graph` owns numpy CSR arrays and hands the flat `gmt_graph_view` of
include/gmt_b200.h to either the product library or the oracle.  For
Euclidean graphs the in-lists equal the out-lists bit for bit
(graph.cpp:184-186), so one array pair serves both (`directed=False`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi


class Graph:
    def __init__(self, n: int, radius: float, out_ptr, out_col, out_cost, dim: int = 0,
                 directed: bool = False, in_ptr=None, in_col=None, in_cost=None,
                 out_path=None, in_path=None, path_ptr=None, path_pts=None):
        self.n = int(n)
        self.radius = float(radius)
        self.dim = int(dim)
        self.directed = bool(directed)
        self.out_ptr = abi.i64(out_ptr)
        self.out_col = abi.i32(out_col)
        self.out_cost = abi.f64(out_cost)
        self.in_ptr = None if in_ptr is None else abi.i64(in_ptr)
        self.in_col = None if in_col is None else abi.i32(in_col)
        self.in_cost = None if in_cost is None else abi.f64(in_cost)
        self.out_path = None if out_path is None else abi.i32(out_path)
        self.in_path = None if in_path is None else abi.i32(in_path)
        self.path_ptr = None if path_ptr is None else abi.i64(path_ptr)
        self.path_pts = None if path_pts is None else abi.f64(path_pts)

    @property
    def num_edges(self) -> int:
        return int(self.out_ptr[-1])

    def view(self) -> abi.GraphView:
        v = abi.GraphView()
        v.n = self.n
        v.dim = self.dim
        v.radius = self.radius
        v.directed = 1 if self.directed else 0
        v.out_ptr = abi.ptr(self.out_ptr, C.c_int64)
        v.out_col = abi.ptr(self.out_col, C.c_int32)
        v.out_cost = abi.ptr(self.out_cost, C.c_double)
        v.out_path = abi.ptr(self.out_path, C.c_int32)
        v.in_ptr = abi.ptr(self.in_ptr, C.c_int64)
        v.in_col = abi.ptr(self.in_col, C.c_int32)
        v.in_cost = abi.ptr(self.in_cost, C.c_double)
        v.in_path = abi.ptr(self.in_path, C.c_int32)
        v.num_paths = 0 if self.path_ptr is None else len(self.path_ptr) - 1
        v.path_ptr = abi.ptr(self.path_ptr, C.c_int64)
        v.path_pts = abi.ptr(self.path_pts, C.c_double)
        return v

    def out_list(self, u: int):
        a, b = self.out_ptr[u], self.out_ptr[u + 1]
        return self.out_col[a:b], self.out_cost[a:b]

    def transpose(self) -> "Graph":
        """In-lists of a directed graph in ascending source order, the order
        build_neighbor_graph's sequential merge produces (graph.cpp:184-186)."""
        n = self.n
        src = np.repeat(np.arange(n, dtype=np.int32), np.diff(self.out_ptr))
        order = np.lexsort((src, self.out_col))
        in_col = src[order]
        in_cost = self.out_cost[order]
        counts = np.bincount(self.out_col, minlength=n)
        in_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        in_path = None if self.out_path is None else self.out_path[order]
        return in_ptr, in_col, in_cost, in_path

    def same_as(self, other: "Graph") -> bool:
        """Bitwise equality of the out-lists (indices and raw cost bits)."""
        return (np.array_equal(self.out_ptr, other.out_ptr)
                and np.array_equal(self.out_col, other.out_col)
                and self.out_cost.view(np.uint64).tobytes() == other.out_cost.view(np.uint64).tobytes())
