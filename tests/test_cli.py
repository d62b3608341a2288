"""CLI parity: paper_2411_19901_b200.cli against the
reference's own command line on the same files (golden_cli.json, made by
tests/golden/make_cli_golden.py from sketchlpa/cli.py).

Exit codes, stderr messages, report keys / values and writer output must
match; wall-clock fields are dropped and modularity compares within 1e-12
(device float64 tallies vs np.bincount summation order, metrics.py:45-48).
Usage / configuration errors are checked on the CPU (they never reach the
device); everything that loads a graph is a GPU test.
"""

import contextlib
import csv
import io
import json
import math
import os

import pytest

with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_cli.json")) as _f:
    GOLD = json.load(_f)
WALL = {"wall_time_ms", "mean_wall_time_ms", "wall_times_ms"}
FLOATS = {"modularity", "mean_modularity", "modularity_ratio_vs_exact"}


def run_cli(argv):
    from paper_2411_19901_b200.cli import main
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = main(argv)
        except SystemExit as exc:
            code = exc.code
    return code, out.getvalue(), err.getvalue()


def close(a, b):
    if a is None or b is None:
        return a is b
    return math.isclose(float(a), float(b), rel_tol=1e-12, abs_tol=1e-12)


def same_json(a, b):
    if isinstance(a, dict):
        assert set(a) == set(b)
        for k in a:
            if k in WALL:
                continue
            if k in FLOATS:
                assert close(a[k], b[k]), (k, a[k], b[k])
            elif k == "modularities":
                assert all(close(x, y) for x, y in zip(a[k], b[k])) and len(a[k]) == len(b[k])
            else:
                same_json(a[k], b[k])
    elif isinstance(a, list):
        assert len(a) == len(b)
        for x, y in zip(a, b):
            same_json(x, y)
    else:
        assert a == b and type(a) is type(b), (a, b)


def same_csv(a, b):
    ra, rb = list(csv.DictReader(io.StringIO(a))), list(csv.DictReader(io.StringIO(b)))
    assert len(ra) == len(rb)
    for x, y in zip(ra, rb):
        assert list(x) == list(y)
        for k in x:
            if k in WALL:
                continue
            if k in FLOATS:
                assert close(x[k] or None, y[k] or None), k
            elif k == "modularities":
                assert all(close(p, q) for p, q in zip(x[k].split(";"), y[k].split(";")))
            else:
                assert x[k] == y[k], k


def same_text(a, b):
    la, lb = a.splitlines(), b.splitlines()
    assert len(la) == len(lb)
    for x, y in zip(la, lb):
        if x.startswith("wall_time_ms:"):
            assert y.startswith("wall_time_ms:")
        elif x.startswith("modularity:"):
            assert close(x.split(": ")[1], y.split(": ")[1])
        else:
            assert x == y


def _materialise(tmp_path, case):
    for name, text in GOLD["files"].items():
        (tmp_path / name).write_text(text)
    argv = [a.replace("{tmp}", str(tmp_path)) for a in case["argv"]]
    return [str(tmp_path / a) if a in GOLD["files"] or a == "absent.el" else a for a in argv]


def _check(tmp_path, case):
    code, out, err = run_cli(_materialise(tmp_path, case))
    assert code == case["code"]
    want_err = case["stderr"].replace("{tmp}", str(tmp_path))
    assert (err.strip().split("\n")[0] if err else "") == want_err
    gold = case["stdout"].replace("{tmp}/", str(tmp_path) + "/")
    argv = case["argv"]
    if argv[0] == "convert" or not gold:
        assert out == gold
    elif "--report" in argv and argv[argv.index("--report") + 1] == "csv":
        same_csv(out, gold)
    elif argv[0] == "bench" or ("--report" in argv and argv[argv.index("--report") + 1] == "json"):
        same_json(json.loads(out), json.loads(gold))
    else:
        same_text(out, gold)
    if case["written"] is not None:
        path = next(a for a in case["argv"] if a.startswith("{tmp}/")).replace("{tmp}", str(tmp_path))
        with open(path) as f:
            assert f.read() == case["written"]


USAGE = [c for c in GOLD["cases"] if c["code"] == 1]
DEVICE = [c for c in GOLD["cases"] if c["code"] != 1]


@pytest.mark.parametrize("case", USAGE, ids=[" ".join(c["argv"]) for c in USAGE])
def test_cli_usage_errors(tmp_path, case):
    _check(tmp_path, case)


@pytest.mark.gpu
@pytest.mark.parametrize("case", DEVICE, ids=[" ".join(c["argv"]) for c in DEVICE])
def test_cli_matches_reference(tmp_path, case):
    _check(tmp_path, case)


@pytest.mark.gpu
def test_cli_module_entry_point(tmp_path):
    import subprocess
    import sys
    p = tmp_path / "t.el"
    p.write_text("0 1\n1 2\n0 2\n")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "paper_2411_19901_b200", "run", str(p), "--report", "json"],
                       capture_output=True, text=True, cwd=repo)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["num_communities"] == 1
