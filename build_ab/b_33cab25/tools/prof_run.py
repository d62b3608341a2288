"""One lpa_run on a device-generated graph -- the command ncu captures.

    python tools/prof_run.py --scale 22 [--variant mg|bm] [--mode det|async] [--runs 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2411_19901_b200 as slpa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--graph", default="rmat", choices=["rmat", "grid", "kmer"])
ap.add_argument("--variant", default="mg")
ap.add_argument("--mode", default="det")
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--range", action="store_true",
                help="cudaProfilerStart/Stop around the LAST run only (ncu --profile-from-start off)")
a = ap.parse_args()
eng = slpa.Engine(0)
if a.graph == "rmat":
    eng.gen_rmat(a.scale, seed=2411, permute=True)
elif a.graph == "grid":
    side = int(round((1 << a.scale) ** 0.5))
    eng.gen_grid(side, side, permute=True)
else:
    eng.gen_kmer(1 << a.scale, seed=3)
off, _, _ = eng.download() if a.profile else (None, None, None)
if off is not None:
    deg = np.diff(off)
    print("n", eng.n, "m", eng.m, "max_deg", int(deg.max()), "deg>=128:", int((deg >= 128).sum()),
          "arcs in hi:", int(deg[deg >= 128].sum()))
cfg = slpa.LpaConfig(variant=a.variant, worker_count=0 if a.mode == "det" else 1)
eng.set_profiling(a.profile)
rt = None
if a.range:
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if rt is None:
        import torch
        rt = torch.cuda.cudart()
for r in range(a.runs):
    t0 = time.perf_counter()
    if rt is not None and r == a.runs - 1:
        rt.cudaProfilerStart()
    labels, iters, delta, conv = eng.run(cfg, fetch_labels=False)
    if rt is not None and r == a.runs - 1:
        rt.cudaProfilerStop()
    st = eng.stats()
    print(f"run {r}: iters {iters} delta {delta} device_ms {st['device_ms']:.2f} wall {1e3*(time.perf_counter()-t0):.1f}")
if a.profile:
    for k, v in eng.profile().items():
        print(k, v)
