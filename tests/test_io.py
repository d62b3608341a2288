"""Graph files: the native parsers and writers against the
reference's own loaders / writers (golden_io.json, made by
tests/golden/make_io_golden.py from sketchlpa/graph.py:165-375).

CPU tests: parsing and writing are host code in libslpa_b200.so
(csrc/slpa_io.cpp), so the raw entries, id maps, error messages and writer
text are checked here; the device assembly of the parsed entries is checked
in the GPU test at the bottom.
"""

import io
import json
import os

import numpy as np
import pytest

from paper_2411_19901_b200 import graph_io
from paper_2411_19901_b200.graph import Graph, GraphLoadError

with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_io.json")) as _f:
    CASES = json.load(_f)
IDS = [c["name"] for c in CASES]


def _write(tmp_path, case):
    p = tmp_path / case["name"]
    with open(p, "w", newline="") as f:
        f.write(case["text"])
    return str(p)


def _parse(path, fmt):
    """Native parse (the Python restatement for SLPA_IO_EXOTIC text)."""
    rc, src, dst, w, n, raw, (line, aux, aux2) = graph_io._native_parse(path, fmt, threads=3)
    if rc == graph_io.IO_EXOTIC:
        with open(path, "r") as f:
            n, src, dst, w, mapping = graph_io._parse_text(f, path, fmt)
        return "exotic", n, list(src), list(dst), list(w), mapping
    if rc != 0:
        raise GraphLoadError(graph_io._MESSAGES[rc].format(L=f"{path}:{line}", P=path, a=aux, b=aux2))
    mapping = None
    if fmt == "edge-list":
        mapping = ({v: v for v in range(n)} if raw is None else {int(r): d for d, r in enumerate(raw.tolist())})
    return "native", n, src.tolist(), dst.tolist(), w.tolist(), mapping


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_parse_matches_reference(tmp_path, case):
    path = _write(tmp_path, case)
    if case["ok"] or not case["error"].startswith("{dir}"):
        try:
            how, n, src, dst, w, mapping = _parse(path, case["fmt"])
        except GraphLoadError as exc:
            pytest.fail(f"unexpected GraphLoadError {exc}")
        except ValueError:
            assert not case["ok"]
            return
        if not case["ok"]:  # the reference failed later (Graph constructor / decoding)
            return
        assert n == case["n"]
        assert src == case["src"] and dst == case["dst"]
        assert w == case["w"]  # exact binary64 values
        if case["mapping"] is not None:
            assert mapping == {k: v for k, v in case["mapping"]}
    else:
        with pytest.raises(GraphLoadError) as ei:
            _parse(path, case["fmt"])
        assert str(ei.value) == case["error"].replace("{dir}", str(tmp_path))


def test_exotic_text_routes_to_python():
    # underscores, non-ASCII digits, >18-digit ids: the library defers, the
    # Python restatement decides (tested against the reference above)
    exotic = [c for c in CASES if any(s in c["text"] for s in ("_", "١", "٢", "123456789012345678901"))]
    assert len(exotic) >= 5


def test_native_parser_threads_and_line_numbers(tmp_path):
    # > 1 MiB so the file is split over threads; an error deep in the file
    # must name the same line number as a sequential parse
    rng = np.random.default_rng(5)
    lines = [f"{a} {b} {w}" for a, b, w in zip(rng.integers(0, 5000, 120000), rng.integers(0, 5000, 120000),
                                              rng.choice([0.5, 1.0, 2.0], 120000))]
    ends = ["\n", "\r\n", "\r"]
    for k, end in enumerate(ends):
        p = tmp_path / f"big{k}.el"
        txt = end.join(lines) + end
        p.write_bytes(txt.encode())
        rc, src, dst, w, n, raw, _ = graph_io._native_parse(str(p), "edge-list", threads=7)
        assert rc == 0 and src.size == 120000
        with open(p, "r") as f:
            n2, s2, d2, w2, _m = graph_io._parse_text(f, str(p), "edge-list")
        assert n == n2 and src.tolist() == s2 and dst.tolist() == d2 and w.tolist() == w2
        bad = list(lines)
        bad[97531] = "1 2 -1"
        p.write_bytes((end.join(bad) + end).encode())
        rc, *_rest, (line, aux, aux2) = graph_io._native_parse(str(p), "edge-list", threads=7)
        assert rc == graph_io.IO_EL_WEIGHT and line == 97532


@pytest.mark.parametrize("case", [c for c in CASES if c["ok"]], ids=[c["name"] for c in CASES if c["ok"]])
def test_writers_match_reference(case):
    g = Graph(np.array(case["offsets"], dtype=np.int64), np.array(case["targets"], dtype=np.int32),
              np.array(case["weights"], dtype=np.float32))
    e, mm = io.StringIO(), io.StringIO()
    graph_io.write_edgelist(g, e)
    graph_io.write_matrix_market(g, mm)
    assert e.getvalue() == case["edgelist"]
    assert mm.getvalue() == case["mm"]


def test_writer_chunking(monkeypatch):
    rng = np.random.default_rng(9)
    n = 3000
    src, dst = rng.integers(0, n, 20000), rng.integers(0, n, 20000)
    a, b = np.minimum(src, dst), np.maximum(src, dst)
    pairs = np.unique(np.stack([a, b], 1), axis=0)
    arcs = np.concatenate([pairs, pairs[pairs[:, 0] != pairs[:, 1]][:, ::-1]])
    arcs = arcs[np.lexsort((arcs[:, 1], arcs[:, 0]))]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(arcs[:, 0], minlength=n), out=off[1:])
    w = rng.choice(np.array([0.5, 1.5, 3.0, 0.1], dtype=np.float32), arcs.shape[0])
    g = Graph(off, arcs[:, 1].astype(np.int32), w)
    whole = io.StringIO()
    graph_io.write_edgelist(g, whole)
    monkeypatch.setattr(graph_io, "_ROWS_ARCS", 1000)
    parts = io.StringIO()
    graph_io.write_edgelist(g, parts)
    assert whole.getvalue() == parts.getvalue()
    expect = "".join(f"{i} {int(t)} {float(x):.6g}\n" for i in range(n)
                     for t, x in zip(g.targets[off[i]:off[i + 1]], g.weights[off[i]:off[i + 1]]) if i <= t)
    assert whole.getvalue() == expect


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(OSError):
        graph_io.load_graph(str(tmp_path / "absent.el"))


def test_unknown_format(tmp_path):
    p = tmp_path / "g.el"
    p.write_text("0 1\n")
    with pytest.raises(GraphLoadError, match="unknown graph format: 'xml'"):
        graph_io.load_graph(str(p), "xml")


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["ok"] or not c["error"].startswith("{dir}")],
                         ids=[c["name"] for c in CASES if c["ok"] or not c["error"].startswith("{dir}")])
def test_load_graph_device_assembly(tmp_path, case):
    import paper_2411_19901_b200 as slpa
    path = _write(tmp_path, case)
    if not case["ok"]:
        with pytest.raises(ValueError):
            slpa.load_graph(path, case["fmt"])
        return
    g, mapping = slpa.load_graph(path, case["fmt"], return_mapping=True)
    assert g.offsets.tolist() == case["offsets"]
    assert g.targets.tolist() == case["targets"]
    assert g.weights.dtype == np.float32
    assert np.array_equal(g.weights, np.array(case["weights"], dtype=np.float32))
    if case["mapping"] is None:
        assert mapping is None
    else:
        assert mapping == {k: v for k, v in case["mapping"]}
    slpa.validate_graph(g)
