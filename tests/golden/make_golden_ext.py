"""Extra golden fixtures from the Python REFERENCE (round 2): the rest of the
drop-in's input domain.

    python tests/golden/make_golden_ext.py

* sketch_slots beyond the register / warp sketches (k = 40, 100, 257) with
  chunked high-degree rows, double scan and shared sketch (sketch.py:34-39
  accepts any k >= 1);
* the exact variant on hub graphs (degrees in the hundreds) with dyadic and
  non-dyadic float32 / float64 weights (lpa.py:92-107, np.bincount order);
* lpa_move on caller labels that include negative values (lpa.py:227-259
  takes any int32 labels);
* an iteration hook that MUTATES the live labels array (lpa.py:271-273,
  :297-298: the hook receives the live array, later sweeps see the edit).

Writes tests/golden/golden_ext.npz and merges its cases into
golden_index.json (the other groups are left untouched).  Imports the
reference from /root/reference (build container only).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (reference import + helpers)
from sketchlpa import LpaConfig, build_graph, lpa_run  # noqa: E402


def mutating_hook_case(st, name, g, cfg, graph_name):
    """lpa_run with a hook that overwrites the live labels after sweep 0."""
    hist = []

    def hook(it, pickless, labels):
        if it == 0:
            labels[::7] = labels[0]  # an instrumentation hook that edits the live array
        hist.append(labels.copy())

    t0 = time.perf_counter()
    res = lpa_run(g, cfg, iteration_hook=hook)
    dt = time.perf_counter() - t0
    st.put("ext", name, "labels", res.labels.astype(np.int32))
    st.put("ext", name, "label_hist", np.stack(hist).astype(np.int32))
    st.index[name] = {"group": "ext", "graph": graph_name, "kind": "run_mutating_hook", "n": int(g.num_vertices),
                      "m": int(g.num_arcs), "cfg": mg.cfg_dict(cfg), "has_order": False, "has_hist": True,
                      "iterations": res.iterations, "delta_history": [int(x) for x in res.delta_history],
                      "converged": bool(res.converged), "aux_bytes": int(res.aux_bytes), "ref_seconds": dt,
                      "hook": "it == 0: labels[::7] = labels[0]"}


def main():
    st = mg.Store()
    rng = np.random.default_rng(20261017)
    graphs = {}
    for r in range(4):  # hub graphs: a few vertices of degree 150-700, chunked rows
        n = int(rng.integers(200, 500))
        m = int(rng.integers(6 * n, 12 * n))
        hubs = rng.integers(0, n, 3)
        src = np.concatenate([rng.integers(0, n, m), np.repeat(hubs, 220)])
        dst = np.concatenate([rng.integers(0, n, m), rng.integers(0, n, 660)])
        w = rng.choice(np.array([0.5, 1.0, 2.0]), src.size)
        graphs[f"xhub{r}"] = build_graph(n, list(zip(src.tolist(), dst.tolist(), w.tolist())))
    for r in range(2):  # non-dyadic weights, float32 and float64
        n = int(rng.integers(150, 300))
        m = 10 * n
        hubs = rng.integers(0, n, 2)
        src = np.concatenate([rng.integers(0, n, m), np.repeat(hubs, 200)])
        dst = np.concatenate([rng.integers(0, n, m), rng.integers(0, n, 400)])
        w = rng.uniform(0.01, 3.0, src.size)
        for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
            graphs[f"xreal{r}_{tag}"] = build_graph(n, list(zip(src.tolist(), dst.tolist(), w.tolist())),
                                                    weight_dtype=dt)
    configs = {
        "mg_k40": LpaConfig(sketch_slots=40),
        "mg_k40_double": LpaConfig(sketch_slots=40, scan_mode="double"),
        "mg_k100": LpaConfig(sketch_slots=100),
        "mg_k100_t16p8": LpaConfig(sketch_slots=100, degree_threshold=16, partial_groups=8),
        "mg_k257_shared": LpaConfig(sketch_slots=257, shared_sketch=True),
        "mg_k70_shared_double": LpaConfig(sketch_slots=70, shared_sketch=True, scan_mode="double"),
        "exact": LpaConfig(variant="exact"),
        "mg": LpaConfig(),
    }
    for gname, g in graphs.items():
        st.graph("ext", gname, g)
        for cname, cfg in configs.items():
            if gname.startswith("xreal") and cname not in ("exact", "mg_k40", "mg_k100"):
                continue
            mg.run_case(st, "ext", f"{gname}:{cname}", g, cfg, graph_name=gname)
    # lpa_move on negative (and mixed-sign) caller labels
    for gname in ("xhub0", "xhub1", "xreal0_f32"):
        g = graphs[gname]
        n = g.num_vertices
        for t, pickless in enumerate((False, True, False)):
            if t < 2:
                labels = rng.integers(-n, n, n).astype(np.int32)
            else:
                labels = (-rng.integers(1, 2 ** 31 - 1, n)).astype(np.int32)  # all negative, large magnitude
            flags = rng.random(n) < 0.8
            for cname, cfg in (("mg", LpaConfig()), ("bm", LpaConfig(variant="bm")),
                               ("mg_hi_t2p3k3", LpaConfig(degree_threshold=2, partial_groups=3, sketch_slots=3)),
                               ("mg_k40", LpaConfig(sketch_slots=40))):
                mg.move_case(st, "ext", f"{gname}:negmove{t}:{cname}", g, cfg, labels, flags, pickless,
                             graph_name=gname)
            # the exact variant's np.bincount rejects negative labels: the reference raises
            name = f"{gname}:negmove{t}:exact"
            try:
                mg.move_case(st, "ext", name, g, LpaConfig(variant="exact"), labels, flags, pickless,
                             graph_name=gname)
            except ValueError as e:
                st.put("ext", name, "in_labels", labels.astype(np.int32))
                st.put("ext", name, "in_flags", flags.astype(np.uint8))
                st.index[name] = {"group": "ext", "graph": gname, "kind": "move_raises", "n": int(n),
                                  "m": int(g.num_arcs), "cfg": mg.cfg_dict(LpaConfig(variant="exact")),
                                  "pickless": bool(pickless), "has_order": False, "error": type(e).__name__,
                                  "message": str(e)}
    # a hook that edits the live labels
    for gname in ("xhub0", "xhub2"):
        for cname in ("mg", "exact"):
            mutating_hook_case(st, f"{gname}:mutating_hook:{cname}", graphs[gname], configs[cname], gname)

    np.savez_compressed(os.path.join(HERE, "golden_ext.npz"), **st.groups["ext"])
    with open(os.path.join(HERE, "golden_index.json")) as f:
        index = json.load(f)
    index = {k: v for k, v in index.items() if v.get("group") != "ext"}
    index.update(st.index)
    with open(os.path.join(HERE, "golden_index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print(f"ext cases: {len(st.index)}")


if __name__ == "__main__":
    main()
