"""Graph files: ``load_graph``, ``write_edgelist``, ``write_matrix_market``,
``validate_graph`` (drop-in for sketchlpa/graph.py:165-403).

Parsing runs in libslpa_b200.so (csrc/slpa_io.cpp: memory-mapped file, one
thread per chunk of lines, the reference's per-line rules and error order),
the parsed entries go to the device assembly (``Engine.build``: graph.py:107-
139 rules incl. np.add.reduceat's summation order), and the writers format
rows in parallel in the same library.  ``validate_graph`` runs on the device
(csrc/slpa_validate.cu).

Files whose text needs Python's own decoding or integer rules (non-ASCII
bytes, digit underscores, ids beyond 18 digits; the library answers
SLPA_IO_EXOTIC) are parsed here by ``_parse_text`` -- a restatement of the
reference parsers -- and assembled on the device like any other.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _lib
from .engine import default_engine
from .graph import Graph, GraphLoadError

FORMAT_ALIASES = {  # graph.py:291-298
    "edge-list": "edge-list",
    "edgelist": "edge-list",
    "el": "edge-list",
    "matrix-market": "matrix-market",
    "mm": "matrix-market",
    "mtx": "matrix-market",
}
_FORMAT_CODE = {"edge-list": 0, "matrix-market": 1}

IO_EL_FIELDS, IO_EL_NONINT, IO_EL_NEGATIVE, IO_EL_BADWEIGHT, IO_EL_WEIGHT, IO_NO_EDGES = range(101, 107)
(IO_MM_HEADER, IO_MM_LAYOUT, IO_MM_FIELD, IO_MM_SYMMETRY, IO_MM_NOSIZE, IO_MM_SIZE_FIELDS, IO_MM_SIZE_NONINT,
 IO_MM_NOT_SQUARE, IO_MM_EMPTY, IO_MM_ENTRY_FIELDS, IO_MM_NONINT, IO_MM_RANGE, IO_MM_BADVALUE, IO_MM_VALUE,
 IO_MM_COUNT) = range(110, 125)
IO_EXOTIC, IO_OSERROR, IO_NOMEM = 190, 191, 192

# error code -> message tail; {L} = "{path}:{line}", {P} = "{path}"  (graph.py:165-288)
_MESSAGES = {
    IO_EL_FIELDS: "{L}: expected 'src dst [weight]', got {a} fields",
    IO_EL_NONINT: "{L}: non-integer vertex id",
    IO_EL_NEGATIVE: "{L}: negative vertex id",
    IO_EL_BADWEIGHT: "{L}: malformed weight",
    IO_EL_WEIGHT: "{L}: weight must be positive and finite",
    IO_NO_EDGES: "{P}: no edges found",
    IO_MM_HEADER: "{P}: not a MatrixMarket matrix file",
    IO_MM_LAYOUT: "{P}: only coordinate layout is supported",
    IO_MM_FIELD: "{P}: only pattern or real fields are supported",
    IO_MM_SYMMETRY: "{P}: only general or symmetric structure is supported",
    IO_MM_NOSIZE: "{P}: missing size line",
    IO_MM_SIZE_FIELDS: "{L}: size line must be 'rows cols nnz'",
    IO_MM_SIZE_NONINT: "{L}: non-integer size line",
    IO_MM_NOT_SQUARE: "{P}: matrix must be square ({a}x{b})",
    IO_MM_EMPTY: "{P}: empty graph (no vertices)",
    IO_MM_ENTRY_FIELDS: "{L}: expected {a} fields per entry",
    IO_MM_NONINT: "{L}: non-integer index",
    IO_MM_RANGE: "{L}: index out of declared range",
    IO_MM_BADVALUE: "{L}: malformed value",
    IO_MM_VALUE: "{L}: value must be positive and finite",
    IO_MM_COUNT: "{P}: declared {a} entries, found {b}",
}


def sniff_format(path) -> str:
    """graph.py:301-307: extension first, then the first line."""
    ext = os.path.splitext(path)[1].lower()
    if ext in (".mtx", ".mm"):
        return "matrix-market"
    with open(path, "r") as f:
        first = f.readline()
    return "matrix-market" if first.lower().startswith("%%matrixmarket") else "edge-list"


def _native_parse(path, fmt, threads=0):
    """(status, src, dst, w, n, raw_ids|None, (line, aux, aux2))."""
    lib = _lib.load_library()
    h = ctypes.c_void_p()
    rc = lib.slpa_edges_parse(os.fsencode(path), _FORMAT_CODE[fmt], int(threads), ctypes.byref(h))
    if rc == IO_OSERROR and not h.value:
        return rc, None, None, None, 0, None, (0, 0, 0)
    try:
        cnt, n, rem, err = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        line, aux, aux2 = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.slpa_edges_info(h, ctypes.byref(cnt), ctypes.byref(n), ctypes.byref(rem), ctypes.byref(err),
                            ctypes.byref(line), ctypes.byref(aux), ctypes.byref(aux2))
        if rc != 0:
            return rc, None, None, None, 0, None, (line.value, aux.value, aux2.value)
        c = cnt.value
        src = np.empty(max(c, 1), dtype=np.int64)
        dst = np.empty(max(c, 1), dtype=np.int64)
        w = np.empty(max(c, 1), dtype=np.float64)
        raw = np.empty(max(n.value, 1), dtype=np.int64) if rem.value else None
        lib.slpa_edges_copy(h, src.ctypes.data, dst.ctypes.data, w.ctypes.data,
                            None if raw is None else raw.ctypes.data)
        return 0, src[:c], dst[:c], w[:c], n.value, (None if raw is None else raw[: n.value]), (0, 0, 0)
    finally:
        lib.slpa_edges_free(h)


# ---------------------------------------------------------------- Python restatement (exotic text)
def _remap(src, dst):
    """_remap_ids (graph.py:200-218)."""
    seen = set(src)
    seen.update(dst)
    top = max(seen)
    if len(seen) == top + 1:
        return src, dst, top + 1, {v: v for v in sorted(seen)}
    mapping = {}
    for a, b in zip(src, dst):
        for v in (a, b):
            if v not in mapping:
                mapping[v] = len(mapping)
    return [mapping[v] for v in src], [mapping[v] for v in dst], len(mapping), mapping


def _parse_text(f, path, fmt):
    """Both reference parsers (graph.py:165-197, :221-288) over a text stream.
    Returns (n, src, dst, w, mapping|None)."""
    mm = fmt == "matrix-market"
    lineno = 0
    rows = None
    want = 2
    if mm:
        tok = f.readline().lower().split()
        lineno = 1
        if len(tok) != 5 or tok[0] != "%%matrixmarket" or tok[1] != "matrix":
            raise GraphLoadError(f"{path}: not a MatrixMarket matrix file")
        if tok[2] != "coordinate":
            raise GraphLoadError(f"{path}: only coordinate layout is supported")
        if tok[3] not in ("pattern", "real"):
            raise GraphLoadError(f"{path}: only pattern or real fields are supported")
        if tok[4] not in ("general", "symmetric"):
            raise GraphLoadError(f"{path}: only general or symmetric structure is supported")
        want = 3 if tok[3] == "real" else 2
        size = None
        for raw in f:
            lineno += 1
            s = raw.strip()
            if s and not s.startswith("%"):
                size = s.split()
                break
        if size is None:
            raise GraphLoadError(f"{path}: missing size line")
        if len(size) != 3:
            raise GraphLoadError(f"{path}:{lineno}: size line must be 'rows cols nnz'")
        try:
            rows, cols, nnz = (int(x) for x in size)
        except ValueError:
            raise GraphLoadError(f"{path}:{lineno}: non-integer size line") from None
        if rows != cols:
            raise GraphLoadError(f"{path}: matrix must be square ({rows}x{cols})")
        if rows < 1:
            raise GraphLoadError(f"{path}: empty graph (no vertices)")
    src, dst, w = [], [], []
    for raw in f:
        lineno += 1
        s = raw.strip()
        if not s or s[0] == "%" or (not mm and s[0] == "#"):
            continue
        parts = s.split()
        where = f"{path}:{lineno}"
        if mm and len(parts) != want:
            raise GraphLoadError(f"{where}: expected {want} fields per entry")
        if not mm and len(parts) not in (2, 3):
            raise GraphLoadError(f"{where}: expected 'src dst [weight]', got {len(parts)} fields")
        try:
            i, j = int(parts[0]), int(parts[1])
        except ValueError:
            raise GraphLoadError(f"{where}: " + ("non-integer index" if mm else "non-integer vertex id")) from None
        if mm and not (1 <= i <= rows and 1 <= j <= rows):
            raise GraphLoadError(f"{where}: index out of declared range")
        if not mm and (i < 0 or j < 0):
            raise GraphLoadError(f"{where}: negative vertex id")
        wt = 1.0
        if len(parts) == 3:
            try:
                wt = float(parts[2])
            except ValueError:
                raise GraphLoadError(f"{where}: " + ("malformed value" if mm else "malformed weight")) from None
            if not (wt > 0 and math.isfinite(wt)):
                raise GraphLoadError(f"{where}: " + ("value must be positive and finite" if mm
                                                      else "weight must be positive and finite"))
        if mm:
            i, j = i - 1, j - 1
        src.append(i)
        dst.append(j)
        w.append(wt)
    if mm and len(src) != nnz:
        raise GraphLoadError(f"{path}: declared {nnz} entries, found {len(src)}")
    if not src:
        raise GraphLoadError(f"{path}: no edges found")
    if mm:
        return rows, src, dst, w, None
    src, dst, n, mapping = _remap(src, dst)
    return n, src, dst, w, mapping


def load_graph(path, fmt=None, *, weight_dtype=np.float32, return_mapping=False, engine=None, threads=0):
    """graph.py:310-349: parse a graph file and assemble it on the device."""
    if fmt is None:
        fmt = sniff_format(path)
    try:
        fmt = FORMAT_ALIASES[fmt.lower()]
    except KeyError:
        raise GraphLoadError(f"unknown graph format: {fmt!r}") from None
    with open(path, "r"):  # the reference's open(): same OSError for missing / unreadable paths
        pass
    rc, src, dst, w, n, raw, (line, aux, aux2) = _native_parse(path, fmt, threads)
    mapping = None
    if rc == IO_EXOTIC:
        with open(path, "r") as f:
            n, src, dst, w, mapping = _parse_text(f, path, fmt)
    elif rc == IO_OSERROR:
        with open(path, "r") as f:  # re-raise the OS error the way Python reports it
            f.read()
        raise OSError(f"cannot read {path}")
    elif rc == IO_NOMEM:
        raise MemoryError(f"{path}: out of host memory while parsing")
    elif rc != 0:
        msg = _MESSAGES[rc].format(L=f"{path}:{line}", P=f"{path}", a=aux, b=aux2)
        raise GraphLoadError(msg)
    elif fmt == "edge-list" and return_mapping:
        if raw is None:
            mapping = {v: v for v in range(n)}
        else:
            mapping = {int(r): d for d, r in enumerate(raw.tolist())}
    eng = engine or default_engine()
    eng.build(int(n), np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64),
              np.asarray(w, dtype=np.float64), weight_dtype)
    off, tgt, wts = eng.download()
    g = Graph(off, tgt, wts.astype(weight_dtype, copy=False))
    if return_mapping:
        return g, (mapping if fmt == "edge-list" else None)
    return g


# ---------------------------------------------------------------- writers
_ROWS_ARCS = 1 << 23  # arcs formatted per library call (bounded text buffers)


def _write_rows(g, out, lower):
    lib = _lib.load_library()
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(g.targets, dtype=np.int32)
    w = np.ascontiguousarray(g.weights)
    if w.dtype not in (np.float32, np.float64):
        w = w.astype(np.float64)
    n = off.size - 1
    r0 = 0
    while r0 < n:
        r1 = int(np.searchsorted(off, off[r0] + _ROWS_ARCS, side="right")) - 1
        r1 = min(max(r1, r0 + 1), n)
        buf, ln = ctypes.c_void_p(), ctypes.c_int64()
        rc = lib.slpa_format_rows(r0, r1, off.ctypes.data, tgt.ctypes.data, w.ctypes.data,
                                  1 if w.dtype == np.float64 else 0, int(lower), 0, ctypes.byref(buf),
                                  ctypes.byref(ln))
        if rc != 0:
            raise MemoryError("graph writer: out of host memory")
        if buf.value:
            try:
                out.write(ctypes.string_at(buf.value, ln.value).decode("ascii"))
            finally:
                lib.slpa_free_buffer(buf)
        r0 = r1


def write_edgelist(g, out) -> None:
    """graph.py:352-361: one 'i j w' line per undirected edge (i <= j)."""
    _write_rows(g, out, lower=0)


def write_matrix_market(g, out) -> None:
    """graph.py:364-375: real symmetric coordinate, lower triangle."""
    lib = _lib.load_library()
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(g.targets, dtype=np.int32)
    n = off.size - 1
    count = int(lib.slpa_format_count(n, off.ctypes.data, tgt.ctypes.data, 1))
    out.write("%%MatrixMarket matrix coordinate real symmetric\n")
    out.write(f"{g.num_vertices} {g.num_vertices} {count}\n")
    _write_rows(g, out, lower=1)


def validate_graph(g, *, engine=None) -> None:
    """graph.py:378-403 on the device: raises ValueError on the first breach,
    in the reference's check order."""
    eng = engine or default_engine()
    eng.upload(g)
    code, vertex, deg_sum, total = eng.validate()
    if code == 1:
        raise ValueError(f"vertex {vertex}: neighbor list not strictly increasing")
    if code == 2:
        raise ValueError("non-positive arc weight")
    if code == 3:
        raise ValueError("arc set is not symmetric")
    if not math.isclose(deg_sum, total, rel_tol=1e-9, abs_tol=1e-12):
        raise ValueError("degree sum does not match twice the total weight")
