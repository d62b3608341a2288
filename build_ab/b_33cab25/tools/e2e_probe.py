"""Phases of the end-to-end path: upload from pinned host memory, run, labels back (SLPA_TRACE=1 for the
library's own phase split)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2411_19901_b200 as slpa
eng = slpa.Engine(0)
eng.gen_rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 24, seed=2411, permute=True)
off, tgt, w = eng.download()
po = torch.empty(off.size, dtype=torch.int64, pin_memory=True).numpy(); po[:] = off
pt = torch.empty(tgt.size, dtype=torch.int32, pin_memory=True).numpy(); pt[:] = tgt
pw = torch.empty(w.size, dtype=torch.float32, pin_memory=True).numpy(); pw[:] = w
g = slpa.Graph(po, pt, pw)
e2 = slpa.Engine(0)
cfg = slpa.LpaConfig()
for r in range(3):
    t0 = time.perf_counter(); e2.upload(g); t1 = time.perf_counter()
    lab, it, d, c = e2.run(cfg); t2 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms ({(po.nbytes+pt.nbytes+pw.nbytes)/(t1-t0)/1e9:.1f} GB/s)  run+labels {1e3*(t2-t1):.1f} ms  device {e2.stats()['device_ms']:.1f}", flush=True)
