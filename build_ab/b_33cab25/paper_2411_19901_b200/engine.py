"""Device context: one B200, one stream, one resident graph.

``Engine`` is the resident-graph handle (upload once, run many times) that
``lpa_run`` / ``lpa_move`` / ``modularity`` use under the hood.  It owns an
``slpa_ctx`` from libslpa_b200.so; all device memory lives there.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _lib
from ._lib import HOOK_FN, PROF_CLASSES, SlpaConfig, SlpaProfile, SlpaRunStats, check

VARIANT_CODE = {"exact": 0, "bm": 1, "mg": 2}
SCAN_CODE = {"single": 0, "double": 1}


def config_struct(cfg) -> SlpaConfig:
    return SlpaConfig(
        VARIANT_CODE[cfg.variant],
        SCAN_CODE[cfg.scan_mode],
        int(cfg.sketch_slots),
        int(cfg.pickless_gap),
        float(cfg.tolerance),
        int(cfg.max_iterations),
        int(cfg.degree_threshold),
        int(cfg.partial_groups),
        int(cfg.worker_count),
        1 if cfg.shared_sketch else 0,
    )


def _graph_arrays(g):
    """(n, offsets int64, targets int32, weights f32|f64) of any Graph-like object."""
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(g.targets, dtype=np.int32)
    w = np.ascontiguousarray(g.weights)
    if w.dtype not in (np.float32, np.float64):
        w = w.astype(np.float64)
    n = int(off.size - 1)
    return n, off, tgt, w


def _destroy(lib, ctx):
    lib.slpa_destroy(ctx)


class Engine:
    """Resident-graph label propagation on one device.

    >>> eng = Engine(device=0)
    >>> eng.upload(g)                       # a sketchlpa.Graph or any CSR holder
    >>> res = eng.run(LpaConfig())          # lpa.py:262 semantics
    """

    def __init__(self, device: int = 0):
        self.lib = _lib.load_library()
        ctx = ctypes.c_void_p()
        rc = self.lib.slpa_create(int(device), ctypes.byref(ctx))
        check(self.lib, None, rc)
        self.ctx = ctx
        self.device = device
        self.n = 0
        self.m = 0
        self.weights_dtype = np.dtype(np.float32)
        self._finalizer = weakref.finalize(self, _destroy, self.lib, ctx)

    def close(self):
        self._finalizer()

    # ------------------------------------------------------------------ graphs
    def upload(self, g, order=None):
        n, off, tgt, w = _graph_arrays(g)
        o = None
        if order is not None:
            o = np.ascontiguousarray(order, dtype=np.int64)
        rc = self.lib.slpa_graph_upload(self.ctx, n, int(tgt.size), off.ctypes.data, tgt.ctypes.data,
                                        w.ctypes.data, 1 if w.dtype == np.float64 else 0,
                                        None if o is None else o.ctypes.data)
        check(self.lib, self.ctx, rc)
        self._refresh()
        return self

    def upload_device(self, offsets, targets, weights, order=None):
        """Upload from CUDA tensors (torch) -- buffer hand-off by data_ptr()."""
        n = int(offsets.numel()) - 1
        f64 = str(weights.dtype) == "torch.float64"
        rc = self.lib.slpa_graph_upload_device(self.ctx, n, int(targets.numel()), offsets.data_ptr(),
                                               targets.data_ptr(), weights.data_ptr(), 1 if f64 else 0,
                                               None if order is None else order.data_ptr())
        check(self.lib, self.ctx, rc)
        self._refresh()
        return self

    def set_order(self, order=None):
        o = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        rc = self.lib.slpa_graph_set_order(self.ctx, None if o is None else o.ctypes.data)
        check(self.lib, self.ctx, rc)

    def _refresh(self):
        n, m, f64, sym = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        check(self.lib, self.ctx, self.lib.slpa_graph_info(self.ctx, ctypes.byref(n), ctypes.byref(m),
                                                           ctypes.byref(f64), ctypes.byref(sym)))
        self.n, self.m = n.value, m.value
        self.weights_dtype = np.dtype(np.float64 if f64.value else np.float32)
        self.symmetric = bool(sym.value)

    def download(self):
        """Resident CSR as host arrays (offsets, targets, weights)."""
        off = np.empty(self.n + 1, dtype=np.int64)
        tgt = np.empty(max(self.m, 1), dtype=np.int32)
        w = np.empty(max(self.m, 1), dtype=self.weights_dtype)
        check(self.lib, self.ctx, self.lib.slpa_graph_download(self.ctx, off.ctypes.data, tgt.ctypes.data,
                                                               w.ctypes.data))
        return off, tgt[: self.m], w[: self.m]

    def validate(self):
        """validate_graph on the resident graph: (code, vertex, deg_sum, total)."""
        code, vertex = ctypes.c_int32(), ctypes.c_int64()
        ds, tot = ctypes.c_double(), ctypes.c_double()
        check(self.lib, self.ctx, self.lib.slpa_validate_graph(self.ctx, ctypes.byref(code), ctypes.byref(vertex),
                                                               ctypes.byref(ds), ctypes.byref(tot)))
        return code.value, vertex.value, ds.value, tot.value

    def gen_rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True, perm_key=7):
        ta, tab, tabc = rmat_thresholds(a, b, c)
        rc = self.lib.slpa_gen_rmat(self.ctx, int(scale), int(edge_factor) << int(scale), ta, tab, tabc,
                                    int(seed), 1 if permute else 0, int(perm_key))
        check(self.lib, self.ctx, rc)
        self._refresh()
        return self

    def gen_grid(self, rows, cols, permute=True, perm_key=7):
        check(self.lib, self.ctx, self.lib.slpa_gen_grid(self.ctx, int(rows), int(cols), 1 if permute else 0,
                                                         int(perm_key)))
        self._refresh()
        return self

    def gen_kmer(self, n, keep=0.95, seed=1, permute=True, perm_key=7):
        check(self.lib, self.ctx, self.lib.slpa_gen_kmer(self.ctx, int(n), keep_threshold(keep), int(seed),
                                                         1 if permute else 0, int(perm_key)))
        self._refresh()
        return self

    def build(self, n, src, dst, w=None, weight_dtype=np.float32):
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        wp = None
        if w is not None:
            w = np.ascontiguousarray(w, dtype=np.float64)
            wp = w.ctypes.data
        rc = self.lib.slpa_build_graph(self.ctx, int(n), int(src.size), src.ctypes.data, dst.ctypes.data, wp,
                                       1 if np.dtype(weight_dtype) == np.float64 else 0)
        check(self.lib, self.ctx, rc)
        self._refresh()
        return self

    # ------------------------------------------------------------------ runs
    def run(self, cfg, hook=None, fetch_labels=True):
        """lpa_run on the resident graph.  Returns (labels|None, iterations,
        delta_history, converged)."""
        c = config_struct(cfg)
        delta = np.zeros(max(int(cfg.max_iterations), 1), dtype=np.int64)
        iters, conv = ctypes.c_int32(0), ctypes.c_int32(0)
        if hook is not None:
            fetch_labels = True  # the hook sees the live result array
        labels = np.empty(max(self.n, 1), dtype=np.int32) if fetch_labels else None
        live = labels[: self.n] if labels is not None else None
        err = []
        cb = HOOK_FN()
        if hook is not None:
            # lpa.py:271-273, :297-298: the hook receives the live labels array --
            # the same object every sweep and the one returned; the library
            # writes it before the call and uploads any edit the hook makes.

            def _tramp(user, it, pickless, ptr):
                try:
                    hook(int(it), bool(pickless), live)
                    return 0
                except BaseException as e:  # re-raised after the C call returns
                    err.append(e)
                    return 1

            cb = HOOK_FN(_tramp)
        rc = self.lib.slpa_run(self.ctx, ctypes.byref(c), None if labels is None else labels.ctypes.data,
                               delta.ctypes.data, ctypes.byref(iters), ctypes.byref(conv), cb, None)
        if rc == _lib.SLPA_EHOOK and err:
            raise err[0]
        check(self.lib, self.ctx, rc)
        it = iters.value
        return live, it, [int(x) for x in delta[:it]], bool(conv.value)

    def move(self, cfg, labels, unprocessed, pickless):
        """lpa_move on the resident graph; mutates labels/unprocessed in place."""
        c = config_struct(cfg)
        changed = ctypes.c_int64(0)
        lab = labels if (labels.dtype == np.int32 and labels.flags.c_contiguous) else None
        if lab is None:
            raise ValueError("labels must be a contiguous int32 array")
        if unprocessed.dtype == np.bool_:
            flags = unprocessed.view(np.uint8)
        elif unprocessed.dtype == np.uint8:
            flags = unprocessed
        else:
            raise ValueError("unprocessed must be a bool or uint8 array")
        if not flags.flags.c_contiguous:
            raise ValueError("unprocessed must be contiguous")
        rc = self.lib.slpa_move(self.ctx, ctypes.byref(c), lab.ctypes.data, flags.ctypes.data,
                                1 if pickless else 0, ctypes.byref(changed))
        check(self.lib, self.ctx, rc)
        return int(changed.value)

    def labels(self):
        out = np.empty(max(self.n, 1), dtype=np.int32)
        check(self.lib, self.ctx, self.lib.slpa_get_labels(self.ctx, out.ctypes.data))
        return out[: self.n]

    def stats(self) -> dict:
        s = SlpaRunStats()
        check(self.lib, self.ctx, self.lib.slpa_last_run_stats(self.ctx, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in SlpaRunStats._fields_}

    def set_profiling(self, on: bool):
        check(self.lib, self.ctx, self.lib.slpa_set_profiling(self.ctx, 1 if on else 0))

    def profile(self) -> dict:
        """Per-kernel-class {launches, ms, evals, arcs} accumulated while profiling."""
        p = SlpaProfile()
        check(self.lib, self.ctx, self.lib.slpa_get_profile(self.ctx, ctypes.byref(p)))
        return {name: {"launches": p.launches[i], "ms": p.ms[i], "evals": p.evals[i], "arcs": p.arcs[i]}
                for i, name in enumerate(PROF_CLASSES) if name != "unused"}

    def tally(self, labels=None, want_arrays=True):
        """(q, num_communities, sizes, internal, incident) -- metrics.py:34-74."""
        q = ctypes.c_double(0.0)
        nc = ctypes.c_int64(0)
        lab = None
        if labels is not None:
            lab = np.ascontiguousarray(labels, dtype=np.int32)
        sizes = internal = incident = None
        if want_arrays:
            sizes = np.zeros(max(self.n, 1), dtype=np.int64)
            internal = np.zeros(max(self.n, 1), dtype=np.float64)
            incident = np.zeros(max(self.n, 1), dtype=np.float64)
        rc = self.lib.slpa_modularity(self.ctx, None if lab is None else lab.ctypes.data, ctypes.byref(q),
                                      ctypes.byref(nc),
                                      None if sizes is None else sizes.ctypes.data,
                                      None if internal is None else internal.ctypes.data,
                                      None if incident is None else incident.ctypes.data)
        if rc != 0:
            msg = self.lib.slpa_last_error(self.ctx).decode()
            if "no edges" in msg:
                q = None
            else:
                check(self.lib, self.ctx, rc)
        if want_arrays:
            sizes, internal, incident = sizes[: self.n], internal[: self.n], incident[: self.n]
        return (None if q is None else q.value), nc.value, sizes, internal, incident

    # ------------------------------------------------------------------ partition (multi-GPU)
    def part_gen_rmat(self, scale, v_begin, v_end, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True,
                      perm_key=7):
        """This rank's rows [v_begin, v_end) of the RMAT graph gen_rmat builds."""
        ta, tab, tabc = rmat_thresholds(a, b, c)
        rc = self.lib.slpa_part_gen_rmat(self.ctx, int(scale), int(edge_factor) << int(scale), ta, tab, tabc,
                                         int(seed), 1 if permute else 0, int(perm_key), int(v_begin), int(v_end))
        check(self.lib, self.ctx, rc)
        return self._part_refresh()

    def rmat_cuts(self, scale, world, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True, perm_key=7):
        """Arc-balanced contiguous ranges [(begin, end)] of the RMAT graph over
        `world` ranks (the same on every rank; computed on this device)."""
        ta, tab, tabc = rmat_thresholds(a, b, c)
        cuts = np.zeros(int(world) + 1, dtype=np.int64)
        rc = self.lib.slpa_rmat_cuts(self.ctx, int(scale), int(edge_factor) << int(scale), ta, tab, tabc, int(seed),
                                     1 if permute else 0, int(perm_key), int(world), cuts.ctypes.data)
        check(self.lib, self.ctx, rc)
        return [(int(cuts[r]), int(cuts[r + 1])) for r in range(int(world))]

    def part_arc_hash(self):
        """The 4 symmetry hash sums of this rank's rows (uint64, add up over ranks)."""
        h = np.zeros(4, dtype=np.uint64)
        check(self.lib, self.ctx, self.lib.slpa_part_arc_hash(self.ctx, h.ctypes.data))
        return h

    def part_set_symmetric(self, symmetric: bool):
        check(self.lib, self.ctx, self.lib.slpa_part_set_symmetric(self.ctx, 1 if symmetric else 0))

    def part_upload(self, n, v_begin, v_end, row_offsets, targets, weights):
        """Rows [v_begin, v_end): row_offsets int64[v_end-v_begin+1] (from 0),
        targets int32 (global ids), weights float32|float64."""
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        tg = np.ascontiguousarray(targets, dtype=np.int32)
        w = np.ascontiguousarray(weights)
        if w.dtype not in (np.float32, np.float64):
            w = w.astype(np.float64)
        rc = self.lib.slpa_part_upload(self.ctx, int(n), int(v_begin), int(v_end), ro.ctypes.data, tg.ctypes.data,
                                       w.ctypes.data, 1 if w.dtype == np.float64 else 0)
        check(self.lib, self.ctx, rc)
        return self._part_refresh()

    def _part_refresh(self):
        n, m, vb, ve = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self.lib, self.ctx, self.lib.slpa_part_info(self.ctx, ctypes.byref(n), ctypes.byref(m),
                                                          ctypes.byref(vb), ctypes.byref(ve)))
        self.n, self.m, self.v_begin, self.v_end = n.value, m.value, vb.value, ve.value
        return self

    def part_begin(self, cfg):
        c = config_struct(cfg)
        check(self.lib, self.ctx, self.lib.slpa_part_begin(self.ctx, ctypes.byref(c)))

    def part_sweep(self, cfg, pickless) -> int:
        c = config_struct(cfg)
        ch = ctypes.c_int64(0)
        check(self.lib, self.ctx, self.lib.slpa_part_sweep(self.ctx, ctypes.byref(c), 1 if pickless else 0,
                                                           ctypes.byref(ch)))
        return int(ch.value)

    def part_end_exchange(self):
        check(self.lib, self.ctx, self.lib.slpa_part_end_exchange(self.ctx))

    # deterministic partitioned sweep (worker_count == 0), one round per call
    def part_det_round(self, cfg, pickless, rnd):
        c = config_struct(cfg)
        check(self.lib, self.ctx, self.lib.slpa_part_det_round(self.ctx, ctypes.byref(c), 1 if pickless else 0,
                                                               int(rnd)))

    def part_det_import(self) -> int:
        t = ctypes.c_int64(0)
        check(self.lib, self.ctx, self.lib.slpa_part_det_import(self.ctx, ctypes.byref(t)))
        return int(t.value)

    def part_det_commit(self, cfg) -> int:
        c = config_struct(cfg)
        ch = ctypes.c_int64(0)
        check(self.lib, self.ctx, self.lib.slpa_part_det_commit(self.ctx, ctypes.byref(c), ctypes.byref(ch)))
        return int(ch.value)

    def part_det_buffers(self):
        """(lab_new, dirty) as zero-copy torch CUDA tensors: the speculative
        end-of-sweep label words (int32 view of uint32[n], bit 31 = changed)
        and the dirty marks as bytes (uint8[n])."""
        lp, dp = ctypes.c_uint64(0), ctypes.c_uint64(0)
        check(self.lib, self.ctx, self.lib.slpa_part_det_buffers(self.ctx, ctypes.byref(lp), ctypes.byref(dp)))
        return (device_tensor(lp.value, self.n, "<i4", self.device), device_tensor(dp.value, self.n, "|u1", self.device))

    def part_buffers(self):
        """(labels, flags) as zero-copy torch CUDA tensors over the context's
        label replica (int32[n]) and flag array (uint8[n])."""
        lp, fp = ctypes.c_uint64(0), ctypes.c_uint64(0)
        check(self.lib, self.ctx, self.lib.slpa_part_buffers(self.ctx, ctypes.byref(lp), ctypes.byref(fp)))
        return (device_tensor(lp.value, self.n, "<i4", self.device), device_tensor(fp.value, self.n, "|u1", self.device))

    def part_tally(self):
        """(internal weight of owned rows, incident float64[n] tensor, sizes int64[n] tensor)."""
        iw = ctypes.c_double(0.0)
        ip, sp = ctypes.c_uint64(0), ctypes.c_uint64(0)
        check(self.lib, self.ctx, self.lib.slpa_part_tally(self.ctx, ctypes.byref(iw), ctypes.byref(ip),
                                                           ctypes.byref(sp)))
        return (iw.value, device_tensor(ip.value, self.n, "<f8", self.device),
                device_tensor(sp.value, self.n, "<i8", self.device))

    def part_modularity(self, internal_total) -> float:
        q = ctypes.c_double(0.0)
        rc = self.lib.slpa_part_modularity(self.ctx, float(internal_total), ctypes.byref(q))
        check(self.lib, self.ctx, rc)
        return q.value

    def stream(self) -> int:
        s = ctypes.c_uint64(0)
        check(self.lib, self.ctx, self.lib.slpa_stream(self.ctx, ctypes.byref(s)))
        return s.value


class _CudaArray:
    """__cuda_array_interface__ view of device memory owned by the library."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_tensor(ptr, n, typestr, device):
    import torch
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device=f"cuda:{device}")


def rmat_thresholds(a, b, c):
    """Integer quadrant thresholds, shared with the oracle."""
    def t(x):
        return min(int(x * 4294967296.0), 0xFFFFFFFF)
    return t(a), t(a + b), t(a + b + c)


def keep_threshold(p):
    return min(int(p * 4294967296.0), 0xFFFFFFFF)


_tls = threading.local()


def default_engine(device: int = 0) -> Engine:
    """One cached Engine per (thread, device) for the functional API."""
    engines = getattr(_tls, "engines", None)
    if engines is None:
        engines = _tls.engines = {}
    eng = engines.get(device)
    if eng is None:
        eng = engines[device] = Engine(device)
    return eng
