"""Every execution path against the oracle, bit-exact.

The degree classes (lane-per-vertex, chunked lane-per-vertex, warp-per-vertex,
giant gather+replay) are execution splits chosen by env thresholds
(SLPA_HI_SPLIT, SLPA_GIANT, read once per process), so each combination runs
in its own subprocess on graphs small enough for the oracle.  Also covers the
deferral schedules (SLPA_DEFER) and the fp64 fallback of integer sketches.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2411_19901_b200 as slpa
from oracle.oracle import get_oracle
from golden_io import GoldenGraph
orc = get_oracle()
eng = slpa.Engine(0)
out = []
for scale, seed in ((13, 5), (15, 6)):
    eng.gen_rmat(scale, seed=seed, permute=True)
    g = GoldenGraph(*eng.download())
    for kw in (dict(), dict(variant="bm"), dict(scan_mode="double"), dict(partial_groups=40),
               dict(sketch_slots=4, degree_threshold=64, partial_groups=16)):
        cfg = slpa.LpaConfig(**kw)
        ref = orc.lpa_run(g, cfg)
        labels, iters, delta, conv = eng.run(cfg)
        ok = (iters, delta, conv) == (ref.iterations, ref.delta_history, ref.converged) and np.array_equal(labels, ref.labels)
        out.append([scale, kw, bool(ok)])
    cfg = slpa.LpaConfig(worker_count=1)
    labels, iters, delta, conv = eng.run(cfg)
    out.append([scale, "async", bool(labels.min() >= 0 and labels.max() < g.num_vertices)])
print(json.dumps(out))
'''

ENVS = [
    {"SLPA_GIANT": "300"},
    {"SLPA_GIANT": "300", "SLPA_DEFER": "0"},
    {"SLPA_GIANT": "300", "SLPA_DEFER": "1"},
    {"SLPA_HI_SPLIT": "400", "SLPA_GIANT": "1500"},
    {"SLPA_HI_SPLIT": "100000"},
    {"SLPA_FORCE_FP64": "1", "SLPA_GIANT": "300"},
    {"SLPA_HI_GRP": "0", "SLPA_GIANT": "300"},
    {"SLPA_GIANT_GRP": "0", "SLPA_GIANT": "300"},
    {"SLPA_GIANT": "128"},
    {"SLPA_GIANT": "5000"},
    {"SLPA_GIANT": "300", "SLPA_HI_SMALL": "0"},
    {"SLPA_L2_PERSIST_MB": "40"},
    {"SLPA_SCAN": "0", "SLPA_GIANT": "300"},
    {"SLPA_DEFER_MIN": "0", "SLPA_GIANT": "300"},
    {"SLPA_DEFER_MIN": "50", "SLPA_GIANT": "300"},
    {"SLPA_GIANT_ASYNC": "0", "SLPA_GIANT": "300"},
    {"SLPA_ASYNC_SPLIT": "0", "SLPA_GIANT": "300"},
    {"SLPA_HI_SMALL": "0", "SLPA_GIANT": "300"},
    {"SLPA_HI_SMALL": "100000000"},
    {"SLPA_LO_SMALL": "0"},
    {"SLPA_R0_COMPACT": "0", "SLPA_GIANT": "300"},
    {"SLPA_COMMIT_POS": "0", "SLPA_SCAN_SORT_MIN": "0"},
    {"SLPA_LO_SMALL": "100000000", "SLPA_GIANT": "300"},
    {"SLPA_GIANT": "1000", "SLPA_HI_SPLIT": "300"},
    {"SLPA_HI_SLICE": "1000", "SLPA_GIANT": "300"},
]


@pytest.mark.parametrize("env", ENVS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_execution_paths_bit_exact(env):
    full = dict(os.environ)
    full.update(env)
    full["PYTHONPATH"] = os.pathsep.join([REPO, os.path.join(REPO, "tests"), full.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-c", SCRIPT, REPO], env=full, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    bad = [x for x in res if not x[2]]
    assert not bad, bad


RANGED = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2411_19901_b200 as slpa
eng = slpa.Engine(0)
out = {}
for scale, ef in ((9, 16), (13, 16), (14, 3)):
    eng.gen_rmat(scale, edge_factor=ef, seed=scale)
    off, tgt, w = eng.download()
    eng.validate()
    lab, iters, delta, conv = eng.run(slpa.LpaConfig())
    out[str(scale)] = [np.asarray(off).tolist(), np.asarray(tgt).tolist(), np.asarray(w).tolist(),
                       np.asarray(lab).tolist(), iters, delta]
print(json.dumps(out))
'''


def test_ranged_rmat_generator_matches_one_shot():
    """The range-by-range RMAT assembly (used above 2^29 edges, SURVEY C5 on
    one GPU) builds the same CSR as the one-shot assembly; forced here with
    SLPA_GEN_RANGES at small scales (including more ranges than rows hold)."""
    res = []
    for ranges in (None, "3", "7"):
        full = dict(os.environ)
        full.pop("SLPA_GEN_RANGES", None)
        if ranges:
            full["SLPA_GEN_RANGES"] = ranges
        full["PYTHONPATH"] = os.pathsep.join([REPO, full.get("PYTHONPATH", "")])
        r = subprocess.run([sys.executable, "-c", RANGED, REPO], env=full, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[1] == res[0]
    assert res[2] == res[0]
