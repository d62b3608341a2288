"""CSR container and graph assembly (drop-in for the parts of
sketchlpa/graph.py the hot path consumes).

``Graph`` mirrors graph.py:35-104 (immutable CSR, same validation).
``build_graph`` mirrors graph.py:142-162 but assembles on the device
(sort + duplicate merge + both directions, slpa_graph.cu) with the
reference's rules, including np.add.reduceat's summation order.  The
engine accepts the reference's own ``Graph`` objects just as well.
"""

from __future__ import annotations

import math

import numpy as np

from .engine import default_engine


class GraphLoadError(ValueError):
    """graph.py:31-32."""


class Graph:
    """Immutable CSR adjacency structure (graph.py:35-74)."""

    __slots__ = ("num_vertices", "num_arcs", "offsets", "targets", "weights")

    def __init__(self, offsets, targets, weights):
        offsets = np.asarray(offsets, dtype=np.int64)
        targets = np.asarray(targets, dtype=np.int32)
        weights = np.asarray(weights)
        if offsets.ndim != 1 or offsets.size < 1 or offsets[0] != 0:
            raise ValueError("offsets must be a 1-d array starting at 0")
        if np.any(np.diff(offsets) < 0):
            raise ValueError("offsets must be non-decreasing")
        n = offsets.size - 1
        if targets.shape != weights.shape or targets.ndim != 1:
            raise ValueError("targets and weights must be 1-d arrays of equal length")
        if targets.size != offsets[-1]:
            raise ValueError("offsets[-1] must equal the arc count")
        if targets.size and (targets.min() < 0 or targets.max() >= n):
            raise ValueError("arc target out of range")
        if weights.size and not np.all(weights > 0):
            raise ValueError("arc weights must be positive")
        self.num_vertices = n
        self.num_arcs = int(targets.size)
        self.offsets = offsets
        self.targets = targets
        self.weights = weights
        for arr in (self.offsets, self.targets, self.weights):
            arr.setflags(write=False)

    def degree(self, i: int) -> int:
        return int(self.offsets[i + 1] - self.offsets[i])

    def neighbors(self, i: int):
        lo, hi = self.offsets[i], self.offsets[i + 1]
        return self.targets[lo:hi], self.weights[lo:hi]

    def weighted_degree(self, i: int) -> float:
        lo, hi = self.offsets[i], self.offsets[i + 1]
        return float(np.sum(self.weights[lo:hi], dtype=np.float64))

    def total_weight(self) -> float:
        return float(np.sum(self.weights, dtype=np.float64)) / 2.0

    def __eq__(self, other):
        if not isinstance(other, Graph):
            return NotImplemented
        return (self.num_vertices == other.num_vertices and np.array_equal(self.offsets, other.offsets)
                and np.array_equal(self.targets, other.targets) and np.array_equal(self.weights, other.weights))

    def __repr__(self):
        return f"Graph(num_vertices={self.num_vertices}, num_arcs={self.num_arcs})"


def build_graph(num_vertices: int, edges, weight_dtype=np.float32, *, engine=None) -> Graph:
    """graph.py:142-162: (i, j) or (i, j, w) tuples -> canonical Graph,
    assembled on the device."""
    src, dst, w = [], [], []
    for e in edges:
        if len(e) == 2:
            i, j = e
            wt = 1.0
        else:
            i, j, wt = e
        if not (0 <= i < num_vertices and 0 <= j < num_vertices):
            raise ValueError(f"edge ({i}, {j}) out of range for {num_vertices} vertices")
        if not (wt > 0 and math.isfinite(wt)):
            raise ValueError(f"edge ({i}, {j}) must have a positive finite weight")
        src.append(i)
        dst.append(j)
        w.append(wt)
    return build_graph_arrays(num_vertices, src, dst, w, weight_dtype, engine=engine)


def build_graph_arrays(num_vertices, src, dst, w=None, weight_dtype=np.float32, *, engine=None) -> Graph:
    eng = engine or default_engine()
    eng.build(int(num_vertices), np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64),
              None if w is None else np.asarray(w, dtype=np.float64), weight_dtype)
    off, tgt, wts = eng.download()
    return Graph(off, tgt, wts.astype(weight_dtype, copy=False))
