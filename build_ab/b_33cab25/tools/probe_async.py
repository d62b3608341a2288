"""Async-schedule probe: community count / modularity of the async GPU mode
against the sequential oracle, and its run time (SLPA_ASYNC_WAVE from env)."""
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]
import paper_2411_19901_b200 as slpa  # noqa: E402
from golden_io import Golden, GoldenGraph  # noqa: E402
from oracle.oracle import get_oracle  # noqa: E402

orc = get_oracle()
F = os.environ.get("SLPA_ASYNC_WAVE", "default")


def one(name, g, eng, var, refcache={}):
    cfg = slpa.LpaConfig(variant=var)
    key = (name, var)
    if key not in refcache:
        ref = orc.lpa_run(g, cfg)
        refcache[key] = (orc.modularity(g, ref.labels), np.unique(ref.labels).size)
    q_ref, c_ref = refcache[key]
    c2 = slpa.LpaConfig(variant=var, worker_count=1)
    eng.run(c2)
    import torch
    t = time.perf_counter()
    a = eng.run(c2)
    dt = time.perf_counter() - t
    q = eng.tally(a[0], want_arrays=False)[0]
    nc = np.unique(a[0]).size
    print(f"F={F} {name:7s} {var} it {a[1]:2d} dQ {q - q_ref:+.4f} comm {nc}/{c_ref} ratio {nc / c_ref:.3f} "
          f"{dt * 1e3:.1f} ms", flush=True)


eng = slpa.Engine(0)
gd = Golden()
c1 = gd.graph("c1:mg")
eng.upload(c1)
one("C1", c1, eng, "mg")
one("C1", c1, eng, "bm")
for s in [16, 20, 24]:
    eng.gen_rmat(s, seed=2411, permute=True)
    g = GoldenGraph(*eng.download())
    one(f"rmat{s}", g, eng, "mg")
    if s < 24:
        one(f"rmat{s}", g, eng, "bm")
eng.gen_grid(2000, 2000, permute=True)
g = GoldenGraph(*eng.download())
one("grid2k", g, eng, "mg")
one("grid2k", g, eng, "bm")
