"""Round-2 probe (GPU box): async acceptance numbers and full-size oracle timings.

    python tools/probe_r2.py [--big]
"""
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


def ncomm(labels):
    return int(np.unique(labels).size)


def compare(name, g, eng, variants=("mg",), workers=(1,)):
    for var in variants:
        cfg = slpa.LpaConfig(variant=var)
        t = time.perf_counter()
        ref = orc.lpa_run(g, cfg)
        t_ref = time.perf_counter() - t
        q_ref = orc.modularity(g, ref.labels)
        det = eng.run(cfg)
        ok = np.array_equal(det[0], ref.labels) and det[2] == ref.delta_history
        print(f"{name} {var} oracle {t_ref:.2f}s iters {ref.iterations} Q {q_ref:.4f} comm {ncomm(ref.labels)} det_equal {ok}",
              flush=True)
        for wc in workers:
            c2 = slpa.LpaConfig(variant=var, worker_count=wc)
            a = eng.run(c2)
            q = eng.tally(a[0], want_arrays=False)[0]
            nc = ncomm(a[0])
            print(f"   async wc={wc}: iters {a[1]} Q {q:.4f} dQ {q - q_ref:+.4f} comm {nc} ratio {nc / ncomm(ref.labels):.3f}",
                  flush=True)


def main():
    big = "--big" in sys.argv
    gd = Golden()
    c1 = gd.graph("c1:mg")
    eng = slpa.Engine(0)
    eng.upload(c1)
    compare("C1", c1, eng, variants=("mg", "bm"), workers=(1, 8, 64))
    for s in (16, 20) + ((24,) if big else ()):
        eng.gen_rmat(s, seed=2411, permute=True)
        g = GoldenGraph(*eng.download())
        compare(f"rmat{s}", g, eng, workers=(1,))
    if big:
        eng.gen_grid(4899, 4899, permute=True)
        g = GoldenGraph(*eng.download())
        compare("grid", g, eng, variants=("mg", "bm"))
        eng.gen_kmer(200_000_000, seed=3)
        g = GoldenGraph(*eng.download())
        del g
    eng.close()


if __name__ == "__main__":
    main()
