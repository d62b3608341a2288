"""Golden fixtures for the graph-file path, made by running
the Python REFERENCE's loaders and writers (sketchlpa/graph.py:165-375).

    python tests/golden/make_io_golden.py

Writes tests/golden/golden_io.json: a list of cases, each a file text plus
what the reference does with it -- the raw parsed entries (src, dst, w after
id remapping / 0-basing), the vertex count, the id mapping, the assembled
CSR, or the GraphLoadError message -- and, for assembled graphs, the
canonical edge-list / MatrixMarket text the reference writers produce.
Hand cases cover every error branch and the text corner cases (CR / CRLF
line ends, exotic whitespace, signs, leading zeros, inf / nan / subnormal
weights, digit underscores, non-ASCII, >18-digit ids); random cases fuzz
the formatting.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import io
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True

from sketchlpa import GraphLoadError, load_graph, write_edgelist, write_matrix_market  # noqa: E402
from sketchlpa import graph as refgraph  # noqa: E402

HAND_EL = [
    "0 1\n1 2\n",
    "0 1 2.0\n1 0 3.0\n",
    "# a comment\n% another\n\n0 1\n",
    "0 0 2.0\n0 1\n",
    "10 30\n30 20\n",
    "2 1\n0 2\n",
    "", "# only comments\n", "0\n", "0 1 2 3\n", "a b\n", "0 -1\n", "0 1 0.0\n", "0 1 -2\n", "0 1 nan\n",
    "0 1\r\n1 2\r\n", "0 1\r1 2\r2 3", "0 1\r\n\r\n1 2\r\r\n", "0\t1\t0.5\n\x0b1\x0c2\x1c3\n",
    "  0   1  \n\t\n", "+0 +1 +1.5\n", "-0 1\n", "007 0010\n", "0 1 1e-320\n", "0 1 1e400\n", "0 1 inf\n",
    "0 1 Infinity\n", "0 1 .5\n0 2 5.\n", "0 1 1E3\n", "0 1 1e\n", "0 1 0x10\n", "0 1 1..2\n",
    "0 1 1_0\n", "0 1_0 2\n", "1_000 2\n", "0 1 2\nx y\n", "0 1\n0 1 2 3 4\n", "3 4\n1 2 -1\n",
    "0 ١\n", "0 1 1 \n", "123456789012345678901234 5\n5 6\n", "99999999999999999 3\n",
    "0 1\n\n# c\n2 3 0.25\n", "1 2\n2 1\n1 1\n", "5 5 3.5\n", "0 1 1e-5\n0 2 123456.789\n0 3 0.1\n",
    "0 1 1\n" * 3, "0 1 nan(1)\n", "0 1 -inf\n", "0 1 +\n", "0 1 -\n", "- 1\n", "+ 1\n", "0 1 \x00\n",
    "﻿0 1\n", "0 1 3.4028235e38\n", "0 1 1e39\n", "0 1 1.0000000001\n",
]

HAND_MM = [
    "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\n",
    "%%MatrixMarket matrix coordinate real general\n% weights below\n2 2 2\n1 2 2.0\n2 1 3.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix array real general\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n2 3 1\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 3\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n0 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n",
    "not a header\n1 2\n",
    "", "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 2 1\n",
    "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 2 1\n",
    "%%MATRIXMARKET MATRIX COORDINATE REAL SYMMETRIC\n2 2 1\n2 1 0.5\n",
    "%%MatrixMarket matrix coordinate real general\n% c\n\n% d\n3 3 3\n1 2 1\n% mid\n2 3 2\n\n3 1 4\n",
    "%%MatrixMarket matrix coordinate real general\n",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 x\n",
    "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "%%MatrixMarket matrix coordinate real general\n-1 -1 0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3 4\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 a 3\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 -3\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 q\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 inf\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1\n2 1 1\n",
    "%%MatrixMarket matrix coordinate pattern general\r\n3 3 2\r\n1 2\r\n2 3",
    "%%MatrixMarket matrix coordinate pattern general\r4 4 1\r4 4\r",
    "%%MatrixMarket matrix coordinate pattern general extra\n2 2 1\n1 2\n",
    "%%MatrixMarket tensor coordinate pattern general\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\n2 1 x\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1_0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 ٢\n",
    "%%MatrixMarket matrix coordinate pattern general\n5 5 1\n+5 +0005\n",
]


def rand_el(rng):
    n = int(rng.integers(1, 40))
    ids = np.arange(n)
    if rng.random() < 0.3:  # sparse ids -> remap
        ids = rng.choice(10 ** int(rng.integers(2, 12)), n, replace=False)
    lines = []
    for _ in range(int(rng.integers(1, 4 * n + 2))):
        i, j = ids[rng.integers(0, n)], ids[rng.integers(0, n)]
        sep = [" ", "\t", "  ", " \t "][int(rng.integers(0, 4))]
        parts = [str(i), str(j)]
        r = rng.random()
        if r < 0.5:
            parts.append(repr(float(rng.choice([0.5, 1.0, 2.0, 0.1, 3.25, 1e-3, 7.0]))))
        elif r < 0.6:
            parts.append(f"{rng.random() * 10:.9g}")
        line = sep.join(parts)
        if rng.random() < 0.1:
            line = "  " + line + " \t"
        lines.append(line)
        if rng.random() < 0.05:
            lines.append("# comment " + str(rng.integers(0, 99)))
        if rng.random() < 0.05:
            lines.append("")
    end = ["\n", "\r\n", "\r"][int(rng.integers(0, 3))]
    text = end.join(lines)
    if rng.random() < 0.7:
        text += end
    if rng.random() < 0.03:  # one malformed line somewhere
        k = int(rng.integers(0, len(lines)))
        bad = ["1", "x 2", "1 2 -1", "1 2 3 4", "-3 1", "1 2 zero"][int(rng.integers(0, 6))]
        lines[k] = bad
        text = end.join(lines) + end
    return text


def rand_mm(rng):
    n = int(rng.integers(1, 30))
    real = rng.random() < 0.5
    sym = "symmetric" if rng.random() < 0.5 else "general"
    ent = []
    for _ in range(int(rng.integers(1, 3 * n + 2))):
        i, j = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
        ent.append(f"{i} {j} {float(rng.choice([0.5, 1.0, 2.5, 4.0]))!r}" if real else f"{i} {j}")
    head = f"%%MatrixMarket matrix coordinate {'real' if real else 'pattern'} {sym}\n"
    if rng.random() < 0.3:
        head += "% generated\n"
    return head + f"{n} {n} {len(ent)}\n" + "\n".join(ent) + "\n"


def run_case(path, text, fmt):
    with open(path, "w", newline="") as f:
        f.write(text)
    case = {"name": os.path.basename(path), "text": text, "fmt": fmt}
    try:
        with open(path, "r") as f:
            if fmt == "edge-list":
                src, dst, w = refgraph._parse_edge_list(f, path)
                src, dst, n, mapping = refgraph._remap_ids(src, dst)
            else:
                n, src, dst, w = refgraph._parse_matrix_market(f, path)
                mapping = None
        g, m2 = load_graph(path, fmt, return_mapping=True)
        case.update(ok=True, n=int(n), src=[int(x) for x in src], dst=[int(x) for x in dst],
                    w=[float(x) for x in w],
                    mapping=None if m2 is None else [[int(k), int(v)] for k, v in m2.items()],
                    offsets=g.offsets.tolist(), targets=g.targets.tolist(), weights=[float(x) for x in g.weights])
        e, mm = io.StringIO(), io.StringIO()
        write_edgelist(g, e)
        write_matrix_market(g, mm)
        case.update(edgelist=e.getvalue(), mm=mm.getvalue())
        assert mapping is None or len(mapping) == n
    except GraphLoadError as exc:
        case.update(ok=False, error=str(exc))
    except ValueError as exc:  # e.g. UnicodeDecodeError is a ValueError
        case.update(ok=False, error="ValueError:" + type(exc).__name__)
    return case


def main():
    tmp = "/tmp/slpa_io_golden"
    os.makedirs(tmp, exist_ok=True)
    cases = []
    for k, t in enumerate(HAND_EL):
        cases.append(run_case(os.path.join(tmp, f"h{k}.el"), t, "edge-list"))
    for k, t in enumerate(HAND_MM):
        cases.append(run_case(os.path.join(tmp, f"m{k}.mtx"), t, "matrix-market"))
    rng = np.random.default_rng(2411)
    for k in range(150):
        cases.append(run_case(os.path.join(tmp, f"r{k}.el"), rand_el(rng), "edge-list"))
    for k in range(60):
        cases.append(run_case(os.path.join(tmp, f"q{k}.mtx"), rand_mm(rng), "matrix-market"))
    for c in cases:  # the path in messages is the test's own temp path
        if not c["ok"]:
            c["error"] = c["error"].replace(tmp + "/", "{dir}/")
    with open(os.path.join(HERE, "golden_io.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(len(cases), "cases;", sum(c["ok"] for c in cases), "loaded")


if __name__ == "__main__":
    main()
