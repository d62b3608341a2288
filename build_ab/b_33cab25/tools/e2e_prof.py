"""Breakdown of the end-to-end lpa_run path (host graph in pinned memory):
upload (H2D + validation + symmetry/int checks), run (bins + sweeps + D2H).

    python tools/e2e_prof.py --scale 24
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_19901_b200 as slpa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
eng = slpa.Engine(0)
eng.gen_rmat(a.scale, seed=2411, permute=True)
off, tgt, w = eng.download()
po = torch.empty(off.size, dtype=torch.int64, pin_memory=True).numpy()
pt = torch.empty(tgt.size, dtype=torch.int32, pin_memory=True).numpy()
pw = torch.empty(w.size, dtype=torch.float32, pin_memory=True).numpy()
po[:], pt[:], pw[:] = off, tgt, w
g = slpa.Graph(po, pt, pw)
cfg = slpa.LpaConfig()
e2 = slpa.Engine(0)
for r in range(a.reps):
    t0 = time.perf_counter()
    e2.upload(g)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    labels, iters, hist, conv = e2.run(cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = e2.stats()
    print(f"rep {r}: upload {1e3*(t1-t0):.1f} ms  run+D2H {1e3*(t2-t1):.1f} ms (device {st['device_ms']:.1f})  "
          f"H2D GB {(po.nbytes+pt.nbytes+pw.nbytes)/1e9:.2f}")
