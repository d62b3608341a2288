"""Golden fixtures for the CLI, made by running the
REFERENCE's own command line (sketchlpa/cli.py:61-311) in-process.

    python tests/golden/make_cli_golden.py

Writes tests/golden/golden_cli.json: input files, argv, exit code, stdout,
first stderr line and any written output file for run / bench / convert.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True

from sketchlpa import build_graph, write_edgelist  # noqa: E402
from sketchlpa.cli import main  # noqa: E402

TMP = "/tmp/slpa_cli_golden"


def files():
    out = {
        "triangle.el": "0 1\n1 2\n0 2\n",
        "cliques.el": "\n".join([f"{a} {b} 1" for a in range(4) for b in range(a + 1, 4)] +
                                [f"{a} {b} 1" for a in range(4, 8) for b in range(a + 1, 8)]) + "\n",
        "g.mtx": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\n",
        "bad.el": "0 zero\n",
        "weighted.mtx": "%%MatrixMarket matrix coordinate real general\n5 5 6\n1 2 0.5\n2 3 1.5\n3 1 2\n4 5 3\n"
                        "5 1 0.25\n2 2 1\n",
    }
    rng = np.random.default_rng(501)
    for name, n, p in (("rand40.el", 40, 0.15), ("rand300.el", 300, 0.04), ("hub.el", 400, 0.0)):
        edges = []
        for i in range(n):
            for j in range(i + 1, n):
                if rng.random() < p:
                    edges.append((i, j, float(rng.choice([0.5, 1.0, 2.0]))))
        if name == "hub.el":  # a high-degree vertex (chunked path) plus a ring
            edges = [(0, j, 1.0) for j in range(1, n)] + [(j, j % (n - 1) + 1, 1.0) for j in range(1, n)]
        g = build_graph(n, edges)
        buf = io.StringIO()
        write_edgelist(g, buf)
        out[name] = buf.getvalue()
    return out


CMDS = [
    ["run", "triangle.el", "--variant", "exact", "--report", "json"],
    ["run", "triangle.el", "--report", "json"],
    ["run", "triangle.el", "--report", "text"],
    ["run", "triangle.el", "--report", "csv"],
    ["run", "triangle.el", "--variant", "mg", "--k", "4", "--rho", "3", "--tau", "0.2", "--max-iters", "7",
     "--degree-threshold", "64", "--groups", "16", "--scan", "double", "--report", "json"],
    ["run", "triangle.el", "--variant", "exact", "--out-labels", "{tmp}/labels.tsv"],
    ["run", "rand300.el", "--report", "json", "--seed-order", "shuffled:7"],
    ["run", "rand300.el", "--report", "json", "--variant", "bm"],
    ["run", "rand300.el", "--report", "csv", "--scan", "double"],
    ["run", "hub.el", "--report", "json"],
    ["run", "hub.el", "--report", "json", "--variant", "bm", "--groups", "7"],
    ["run", "hub.el", "--report", "json", "--variant", "exact"],
    ["run", "g.mtx", "--format", "mm", "--report", "json"],
    ["run", "weighted.mtx", "--report", "text", "--variant", "exact"],
    ["run", "triangle.el", "--tau", "1.5"],
    ["run", "triangle.el", "--seed-order", "sideways"],
    ["run", "triangle.el", "--variant", "fast"],
    ["run", "absent.el"],
    ["run", "bad.el"],
    ["bench", "rand40.el", "--variants", "exact,mg", "--repeats", "3"],
    ["bench", "cliques.el", "--variants", "exact,mg", "--repeats", "1"],
    ["bench", "rand40.el", "--variants", "mg,bm", "--repeats", "1"],
    ["bench", "rand300.el", "--repeats", "2", "--report", "csv"],
    ["bench", "rand40.el", "--repeats", "0"],
    ["bench", "rand40.el", "--variants", ","],
    ["bench", "absent.el"],
    ["convert", "weighted.mtx", "--to", "edgelist"],
    ["convert", "rand40.el", "--to", "mm"],
    ["convert", "g.mtx", "--to", "edgelist", "--out", "{tmp}/out.el"],
    ["convert", "bad.el", "--to", "mm"],
]


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = main(argv)
        except SystemExit as exc:
            code = exc.code
    return code, out.getvalue(), err.getvalue()


def main_():
    os.makedirs(TMP, exist_ok=True)
    fs = files()
    for name, text in fs.items():
        with open(os.path.join(TMP, name), "w") as f:
            f.write(text)
    cases = []
    for cmd in CMDS:
        argv = [a.replace("{tmp}", TMP) for a in cmd]
        argv = [os.path.join(TMP, a) if a in fs or a == "absent.el" else a for a in argv]
        code, out, err = run(argv)
        written = None
        for a in cmd:
            if a.startswith("{tmp}/"):
                with open(a.replace("{tmp}", TMP)) as f:
                    written = f.read()
        cases.append({"argv": cmd, "code": code, "stdout": out.replace(TMP + "/", "{tmp}/"),
                      "stderr": err.replace(TMP + "/", "{tmp}/").strip().split("\n")[0] if err else "",
                      "written": written})
    with open(os.path.join(HERE, "golden_cli.json"), "w") as f:
        json.dump({"files": fs, "cases": cases}, f, indent=0)
    print(len(cases), "cli cases")


if __name__ == "__main__":
    main_()
