"""ctypes front end of the CPU oracle (``lpa_oracle.c``) plus a numpy
restatement of the reference's graph assembly.  TEST INFRASTRUCTURE ONLY:
imported by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` arm -- never by the product package.

Function map (reference file:line each restates):

* ``Oracle.lpa_run``     -> ``sketchlpa/lpa.py:262-308`` (worker_count == 0)
* ``Oracle.lpa_move``    -> ``sketchlpa/lpa.py:227-241``
* ``Oracle.select``      -> ``sketchlpa/lpa.py:92-193`` (exact / bm / mg)
* ``Oracle.tally``       -> ``sketchlpa/metrics.py:34-49``
* ``Oracle.modularity``  -> ``sketchlpa/metrics.py:63-74``
* ``assemble``           -> ``sketchlpa/graph.py:107-139``
* ``build_graph``        -> ``sketchlpa/graph.py:142-162``
* ``HostGraph``          -> ``sketchlpa/graph.py:35-74`` (validation rules)
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblpa_oracle.so")

VARIANT_CODE = {"exact": 0, "bm": 1, "mg": 2}


def build(force: bool = False) -> str:
    """Compile lpa_oracle.c with gcc into oracle/liblpa_oracle.so."""
    src = os.path.join(HERE, "lpa_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", LIB_PATH, src, "-lm"]
        )
    return LIB_PATH


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("scan_double", ctypes.c_int32),
        ("sketch_slots", ctypes.c_int32),
        ("pickless_gap", ctypes.c_int32),
        ("tolerance", ctypes.c_double),
        ("max_iterations", ctypes.c_int32),
        ("degree_threshold", ctypes.c_int32),
        ("partial_groups", ctypes.c_int32),
        ("shared_sketch", ctypes.c_int32),
    ]


class _Graph(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("offsets", ctypes.c_void_p),
        ("targets", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("w_f64", ctypes.c_int32),
    ]


@dataclass
class OracleResult:
    labels: np.ndarray
    iterations: int
    delta_history: list
    converged: bool
    label_history: np.ndarray | None


class HostGraph:
    """Plain CSR holder with the reference ``Graph`` validation
    (graph.py:51-74).  Attributes mirror the reference: num_vertices,
    num_arcs, offsets (int64), targets (int32), weights (float32/64)."""

    __slots__ = ("num_vertices", "num_arcs", "offsets", "targets", "weights")

    def __init__(self, offsets, targets, weights):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        targets = np.ascontiguousarray(targets, dtype=np.int32)
        weights = np.ascontiguousarray(weights)
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
        self.offsets, self.targets, self.weights = offsets, targets, weights

    def degree(self, i):
        return int(self.offsets[i + 1] - self.offsets[i])


def assemble(n, src, dst, w, weight_dtype=np.float32) -> HostGraph:
    """numpy restatement of graph.py:107-139 (canonical pairs, lexsort,
    float64 duplicate sums with np.add.reduceat, self-loop once)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    a = np.minimum(src, dst)
    b = np.maximum(src, dst)
    order = np.lexsort((b, a))
    a, b, w = a[order], b[order], w[order]
    if a.size:
        new = np.empty(a.size, dtype=bool)
        new[0] = True
        new[1:] = (a[1:] != a[:-1]) | (b[1:] != b[:-1])
        starts = np.flatnonzero(new)
        pa, pb = a[starts], b[starts]
        pw = np.add.reduceat(w, starts)
    else:
        pa = pb = np.empty(0, dtype=np.int64)
        pw = np.empty(0, dtype=np.float64)
    loops = pa == pb
    arc_src = np.concatenate([pa, pb[~loops]])
    arc_dst = np.concatenate([pb, pa[~loops]])
    arc_w = np.concatenate([pw, pw[~loops]])
    order = np.lexsort((arc_dst, arc_src))
    arc_src, arc_dst, arc_w = arc_src[order], arc_dst[order], arc_w[order]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(arc_src, minlength=n), out=offsets[1:])
    return HostGraph(offsets, arc_dst.astype(np.int32), arc_w.astype(weight_dtype))


def build_graph(num_vertices, edges, weight_dtype=np.float32) -> HostGraph:
    """graph.py:142-162 -- (i, j) or (i, j, w) tuples."""
    src, dst, w = [], [], []
    for e in edges:
        if len(e) == 2:
            i, j = e
            wt = 1.0
        else:
            i, j, wt = e
        if not (0 <= i < num_vertices and 0 <= j < num_vertices):
            raise ValueError(f"edge ({i}, {j}) out of range for {num_vertices} vertices")
        if not (wt > 0 and np.isfinite(wt)):
            raise ValueError(f"edge ({i}, {j}) must have a positive finite weight")
        src.append(i)
        dst.append(j)
        w.append(wt)
    return assemble(num_vertices, src, dst, w, weight_dtype)


def _cfg_struct(cfg) -> _Cfg:
    return _Cfg(
        VARIANT_CODE[cfg.variant],
        1 if cfg.scan_mode == "double" else 0,
        cfg.sketch_slots,
        cfg.pickless_gap,
        float(cfg.tolerance),
        cfg.max_iterations,
        cfg.degree_threshold,
        cfg.partial_groups,
        1 if cfg.shared_sketch else 0,
    )


class Oracle:
    """Loaded liblpa_oracle.so."""

    def __init__(self, path: str | None = None):
        path = path or LIB_PATH
        if not os.path.exists(path):
            build()
        self.lib = ctypes.CDLL(path)
        L = self.lib
        vp, i64, i32, u64, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32
        L.orc_select.restype = i32
        L.orc_select.argtypes = [vp, vp, i64, vp]
        L.orc_lpa_move.restype = i64
        L.orc_lpa_move.argtypes = [vp, vp, vp, vp, i32, vp]
        L.orc_lpa_move_range.restype = i64
        L.orc_lpa_move_range.argtypes = [vp, vp, vp, vp, i32, vp, i64, i64]
        L.orc_lpa_run.restype = i32
        L.orc_lpa_run.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_reset_processed.argtypes = []
        L.orc_get_processed.argtypes = [vp]
        L.orc_tally.restype = i32
        L.orc_tally.argtypes = [vp, vp, vp, vp, vp]
        L.orc_aux_memory_estimate.restype = i64
        L.orc_aux_memory_estimate.argtypes = [i64, i32, vp, i32]
        L.orc_verify_sweep.restype = i64
        L.orc_verify_sweep.argtypes = [vp, vp, vp, vp, vp, vp, i32, vp, i64, vp]
        L.orc_perm.restype = u64
        L.orc_perm.argtypes = [u64, u64, u64]
        L.orc_rmat_edges.restype = i64
        L.orc_rmat_edges.argtypes = [i32, i64, u32, u32, u32, u64, i32, u64, vp, vp]
        L.orc_grid_edges.restype = i64
        L.orc_grid_edges.argtypes = [i64, i64, i32, u64, vp, vp]
        L.orc_kmer_edges.restype = i64
        L.orc_kmer_edges.argtypes = [i64, u32, u64, i32, u64, vp, vp]
        L.orc_assemble_unit.restype = i64
        L.orc_assemble_unit.argtypes = [i64, i64, vp, vp, vp, vp, vp]

    # -- graph marshalling
    @staticmethod
    def _graph(g):
        off = np.ascontiguousarray(g.offsets, dtype=np.int64)
        tgt = np.ascontiguousarray(g.targets, dtype=np.int32)
        w = np.ascontiguousarray(g.weights)
        if w.dtype not in (np.float32, np.float64):
            w = w.astype(np.float64)
        keep = (off, tgt, w)
        gs = _Graph(int(g.num_vertices), off.ctypes.data, tgt.ctypes.data, w.ctypes.data,
                    1 if w.dtype == np.float64 else 0)
        return gs, keep

    def select(self, g, labels, i, cfg) -> int:
        gs, keep = self._graph(g)
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        c = _cfg_struct(cfg)
        return int(self.lib.orc_select(ctypes.byref(gs), lab.ctypes.data, int(i), ctypes.byref(c)))

    def lpa_move(self, g, labels, unprocessed, cfg, pickless, order=None) -> int:
        """Mutates labels (int32) and unprocessed (bool/uint8) in place."""
        assert labels.dtype == np.int32 and labels.flags.c_contiguous
        flags = unprocessed.view(np.uint8) if unprocessed.dtype == np.bool_ else unprocessed
        gs, keep = self._graph(g)
        c = _cfg_struct(cfg)
        o = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        return int(self.lib.orc_lpa_move(ctypes.byref(gs), labels.ctypes.data, flags.ctypes.data,
                                         ctypes.byref(c), 1 if pickless else 0,
                                         None if o is None else o.ctypes.data))

    def lpa_move_range(self, g, labels, unprocessed, cfg, pickless, lo, hi) -> int:
        flags = unprocessed.view(np.uint8) if unprocessed.dtype == np.bool_ else unprocessed
        gs, keep = self._graph(g)
        c = _cfg_struct(cfg)
        return int(self.lib.orc_lpa_move_range(ctypes.byref(gs), labels.ctypes.data, flags.ctypes.data,
                                               ctypes.byref(c), 1 if pickless else 0, None,
                                               int(lo), int(hi)))

    def lpa_run(self, g, cfg, order=None, keep_history=False) -> OracleResult:
        n = int(g.num_vertices)
        gs, keep = self._graph(g)
        c = _cfg_struct(cfg)
        labels = np.empty(n, dtype=np.int32)
        delta = np.zeros(cfg.max_iterations, dtype=np.int64)
        iters = ctypes.c_int32(0)
        conv = ctypes.c_int32(0)
        hist = np.empty((cfg.max_iterations, n), dtype=np.int32) if keep_history else None
        o = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        self.lib.orc_lpa_run(ctypes.byref(gs), ctypes.byref(c),
                             None if o is None else o.ctypes.data,
                             labels.ctypes.data, delta.ctypes.data,
                             ctypes.byref(iters), ctypes.byref(conv),
                             None if hist is None else hist.ctypes.data)
        it = iters.value
        return OracleResult(labels, it, [int(x) for x in delta[:it]], bool(conv.value),
                            None if hist is None else hist[:it].copy())

    def processed(self, reset=False):
        """(vertices, arcs) processed by the sweeps since the last reset
        (lpa.py:212-214: flag set when the vertex is reached)."""
        if reset:
            self.lib.orc_reset_processed()
            return (0, 0)
        out = np.zeros(2, dtype=np.int64)
        self.lib.orc_get_processed(out.ctypes.data)
        return int(out[0]), int(out[1])

    def verify_sweep(self, g, L0, F0, L1, F1, cfg, pickless, vertices=None):
        """Check a GPU sweep (L0,F0) -> (L1,F1) vertex by vertex (ascending
        order, symmetric graph).  Returns (mismatches, first_bad_vertex)."""
        gs, keep = self._graph(g)
        c = _cfg_struct(cfg)
        arrs = [np.ascontiguousarray(L0, dtype=np.int32), np.ascontiguousarray(F0).view(np.uint8),
                np.ascontiguousarray(L1, dtype=np.int32), np.ascontiguousarray(F1).view(np.uint8)]
        vs = None if vertices is None else np.ascontiguousarray(vertices, dtype=np.int64)
        count = int(g.num_vertices) if vs is None else int(vs.size)
        first = ctypes.c_int64(-1)
        bad = self.lib.orc_verify_sweep(ctypes.byref(gs), arrs[0].ctypes.data, arrs[1].ctypes.data,
                                        arrs[2].ctypes.data, arrs[3].ctypes.data, ctypes.byref(c),
                                        1 if pickless else 0, None if vs is None else vs.ctypes.data,
                                        count, ctypes.byref(first))
        return int(bad), int(first.value)

    def tally(self, g, labels):
        n = int(g.num_vertices)
        gs, keep = self._graph(g)
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        sizes = np.zeros(n, dtype=np.int64)
        internal = np.zeros(n, dtype=np.float64)
        incident = np.zeros(n, dtype=np.float64)
        rc = self.lib.orc_tally(ctypes.byref(gs), lab.ctypes.data, sizes.ctypes.data,
                                internal.ctypes.data, incident.ctypes.data)
        if rc != 0:
            raise ValueError("label out of range")
        return sizes, internal, incident

    def modularity(self, g, labels) -> float:
        _, internal, incident = self.tally(g, labels)
        total = incident.sum()
        if total <= 0:
            raise ValueError("modularity is undefined on a graph with no edges")
        frac = incident / total
        return float(np.sum(internal / total - frac * frac))

    def aux_memory_estimate(self, g, cfg) -> int:
        c = _cfg_struct(cfg)
        return int(self.lib.orc_aux_memory_estimate(int(g.num_vertices), int(np.dtype(g.weights.dtype).itemsize),
                                                    ctypes.byref(c), int(cfg.worker_count)))

    # -- generators
    def perm(self, x, n, key) -> int:
        return int(self.lib.orc_perm(int(x), int(n), int(key)))

    def _assemble_unit(self, n, src, dst) -> HostGraph:
        ne = src.size
        off = np.zeros(n + 1, dtype=np.int64)
        tgt = np.zeros(max(2 * ne, 1), dtype=np.int32)
        w = np.zeros(max(2 * ne, 1), dtype=np.float32)
        m = self.lib.orc_assemble_unit(n, ne, src.ctypes.data, dst.ctypes.data, off.ctypes.data,
                                       tgt.ctypes.data, w.ctypes.data)
        return HostGraph(off, tgt[:m].copy(), w[:m].copy())

    def rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True,
             perm_key=7) -> HostGraph:
        ne = edge_factor << scale
        ta, tab, tabc = rmat_thresholds(a, b, c)
        src = np.empty(ne, dtype=np.uint32)
        dst = np.empty(ne, dtype=np.uint32)
        k = self.lib.orc_rmat_edges(scale, ne, ta, tab, tabc, seed, 1 if permute else 0, perm_key,
                                    src.ctypes.data, dst.ctypes.data)
        return self._assemble_unit(1 << scale, src[:k], dst[:k])

    def grid(self, rows, cols, permute=True, perm_key=7) -> HostGraph:
        ne = max(rows * (cols - 1) + (rows - 1) * cols, 0)
        src = np.empty(max(ne, 1), dtype=np.uint32)
        dst = np.empty(max(ne, 1), dtype=np.uint32)
        k = self.lib.orc_grid_edges(rows, cols, 1 if permute else 0, perm_key, src.ctypes.data, dst.ctypes.data)
        return self._assemble_unit(rows * cols, src[:k], dst[:k])

    def kmer(self, n, keep=0.95, seed=1, permute=True, perm_key=7) -> HostGraph:
        cap = n + n // 20 + 1
        src = np.empty(cap, dtype=np.uint32)
        dst = np.empty(cap, dtype=np.uint32)
        k = self.lib.orc_kmer_edges(n, keep_threshold(keep), seed, 1 if permute else 0, perm_key,
                                    src.ctypes.data, dst.ctypes.data)
        return self._assemble_unit(n, src[:k], dst[:k])


def rmat_thresholds(a, b, c):
    """Integer quadrant thresholds shared by the C and CUDA generators."""
    def t(x):
        return min(int(x * 4294967296.0), 0xFFFFFFFF)
    return t(a), t(a + b), t(a + b + c)


def keep_threshold(p):
    return min(int(p * 4294967296.0), 0xFFFFFFFF)


_ORACLE = None


def get_oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        build()
        _ORACLE = Oracle()
    return _ORACLE
