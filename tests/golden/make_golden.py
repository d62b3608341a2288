"""Generate the golden parity fixtures by running the Python REFERENCE.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``sketchlpa`` from /root/reference/pkg/src and the reference's
own test generators from /root/reference/pkg/tests/conftest.py, builds the
cases listed below, runs the reference (``lpa_run`` with an iteration hook
capturing every sweep's labels, ``lpa_move`` on arbitrary label/flag states,
``modularity`` / ``community_stats``) and writes small compressed fixtures:

    tests/golden/golden_<group>.npz   arrays, keys "<case>/<field>"
    tests/golden/golden_index.json    per-case config and scalar results

Nothing at test time reads /root/reference; the fixtures travel instead.
"""

from __future__ import annotations

import importlib.util
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)
sys.dont_write_bytecode = True

import sketchlpa  # noqa: E402
from sketchlpa import Graph, LpaConfig, build_graph, community_stats, lpa_move, lpa_run, modularity  # noqa: E402

spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(REF_TESTS, "conftest.py"))
ref_conftest = importlib.util.module_from_spec(spec)
spec.loader.exec_module(ref_conftest)

from oracle.oracle import get_oracle  # noqa: E402  (generators only)

CFG_FIELDS = ("variant", "scan_mode", "sketch_slots", "pickless_gap", "tolerance", "max_iterations",
              "degree_threshold", "partial_groups", "worker_count", "shared_sketch")


class Store:
    def __init__(self):
        self.groups: dict[str, dict[str, np.ndarray]] = {}
        self.index: dict[str, dict] = {}

    def graph(self, group, name, g):
        arrs = self.groups.setdefault(group, {})
        arrs[f"{name}/offsets"] = np.asarray(g.offsets, dtype=np.int64)
        arrs[f"{name}/targets"] = np.asarray(g.targets, dtype=np.int32)
        arrs[f"{name}/weights"] = np.asarray(g.weights)

    def put(self, group, name, key, arr):
        self.groups.setdefault(group, {})[f"{name}/{key}"] = np.asarray(arr)

    def write(self):
        for group, arrs in self.groups.items():
            np.savez_compressed(os.path.join(HERE, f"golden_{group}.npz"), **arrs)
        with open(os.path.join(HERE, "golden_index.json"), "w") as f:
            json.dump(self.index, f, indent=1, sort_keys=True)


def cfg_dict(cfg):
    return {k: getattr(cfg, k) for k in CFG_FIELDS}


def run_case(st: Store, group, name, g, cfg, order=None, graph_name=None, keep_hist=True):
    """Record lpa_run outputs for (g, cfg)."""
    hist = []
    hooks = []

    def hook(it, pickless, labels):
        hooks.append((it, bool(pickless)))
        if keep_hist:
            hist.append(labels.copy())

    t0 = time.perf_counter()
    res = lpa_run(g, cfg, order=order, iteration_hook=hook)
    dt = time.perf_counter() - t0
    gname = graph_name or name
    if graph_name is None:
        st.graph(group, name, g)
    st.put(group, name, "labels", res.labels.astype(np.int32))
    if keep_hist:
        st.put(group, name, "label_hist", np.stack(hist).astype(np.int32))
    if order is not None:
        st.put(group, name, "order", np.asarray(order, dtype=np.int64))
    stats = community_stats(g, res.labels)
    try:
        q = modularity(g, res.labels)
    except ValueError:
        q = None
    st.index[name] = {
        "group": group,
        "graph": gname,
        "kind": "run",
        "n": int(g.num_vertices),
        "m": int(g.num_arcs),
        "cfg": cfg_dict(cfg),
        "has_order": order is not None,
        "has_hist": keep_hist,
        "iterations": res.iterations,
        "delta_history": [int(x) for x in res.delta_history],
        "converged": bool(res.converged),
        "aux_bytes": int(res.aux_bytes),
        "modularity": q,
        "num_communities": int(stats.num_communities),
        "hook_calls": hooks,
        "ref_seconds": dt,
    }
    return res


def move_case(st: Store, group, name, g, cfg, labels, unprocessed, pickless, order=None, graph_name=None):
    lab = labels.astype(np.int32).copy()
    fl = unprocessed.astype(bool).copy()
    delta = lpa_move(g, lab, fl, cfg, pickless, order)
    if graph_name is None:
        st.graph(group, name, g)
    st.put(group, name, "in_labels", labels.astype(np.int32))
    st.put(group, name, "in_flags", unprocessed.astype(np.uint8))
    st.put(group, name, "out_labels", lab)
    st.put(group, name, "out_flags", fl.astype(np.uint8))
    if order is not None:
        st.put(group, name, "order", np.asarray(order, dtype=np.int64))
    st.index[name] = {"group": group, "graph": graph_name or name, "kind": "move", "n": int(g.num_vertices),
                      "m": int(g.num_arcs), "cfg": cfg_dict(cfg), "pickless": bool(pickless),
                      "has_order": order is not None, "delta": int(delta)}


def metric_case(st: Store, group, name, g, labels, graph_name=None):
    if graph_name is None:
        st.graph(group, name, g)
    st.put(group, name, "labels", labels.astype(np.int32))
    stats = community_stats(g, labels)
    st.put(group, name, "sizes", stats.sizes.astype(np.int64))
    st.put(group, name, "internal", stats.internal_weight.astype(np.float64))
    st.put(group, name, "incident", stats.incident_weight.astype(np.float64))
    try:
        q = modularity(g, labels)
    except ValueError:
        q = None
    st.index[name] = {"group": group, "graph": graph_name or name, "kind": "metric", "n": int(g.num_vertices),
                      "m": int(g.num_arcs), "modularity": q, "num_communities": int(stats.num_communities)}


def to_ref(hg):
    return Graph(hg.offsets, hg.targets, hg.weights)


def sbm_c1(seed=2411, blocks=100, size=100, p_in=0.3, p_out=0.00104):
    """conftest.planted_partition_graph (conftest.py:91-100), row-chunked so
    the 10k x 10k draw stays small; the PCG64 stream is identical."""
    rng = np.random.default_rng(seed)
    n = blocks * size
    member = np.repeat(np.arange(blocks), size)
    src_all, dst_all = [], []
    step = 500
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        draw = rng.random((r1 - r0, n))
        same = member[r0:r1, None] == member[None, :]
        prob = np.where(same, p_in, p_out)
        hit = draw < prob
        hit &= np.arange(n)[None, :] > np.arange(r0, r1)[:, None]
        s, d = np.nonzero(hit)
        src_all.append(s + r0)
        dst_all.append(d)
    src = np.concatenate(src_all)
    dst = np.concatenate(dst_all)
    return build_graph(n, list(zip(src.tolist(), dst.tolist())))


def main():
    st = Store()
    orc = get_oracle()
    C = ref_conftest

    # ---------------------------------------------------------- hand cases
    hand = {
        "star3": C.star_graph(3),
        "two_cliques": C.two_cliques_graph(),
        "barbell": C.barbell_graph(),
        "path3": C.path_graph(3),
        "path12": C.path_graph(12),
        "triangle": C.triangle_graph(),
        "triangle_w": C.triangle_graph(2.0, 0.5, 1.0),
        "isolated1": build_graph(1, []),
        "empty3": build_graph(3, []),
        "selfloop": build_graph(2, [(0, 0, 3.0), (0, 1)]),
        "selfloops_mix": build_graph(5, [(0, 0, 3.0), (0, 1), (1, 1), (1, 2, 2.0), (2, 3), (3, 3, 0.5), (3, 4)]),
        "star256": C.star_graph(256),
        "star300_loop": build_graph(301, [(0, i) for i in range(1, 301)] + [(0, 0, 5.0)]),
    }
    for gname, g in hand.items():
        st.graph("hand", gname, g)
        for variant in ("exact", "bm", "mg"):
            run_case(st, "hand", f"{gname}:{variant}", g, LpaConfig(variant=variant), graph_name=gname)
        run_case(st, "hand", f"{gname}:mg_double", g, LpaConfig(variant="mg", scan_mode="double"), graph_name=gname)
    run_case(st, "hand", "star3:exact_1it", hand["star3"], LpaConfig(variant="exact", max_iterations=1), graph_name="star3")
    run_case(st, "hand", "star3:mg_1it", hand["star3"], LpaConfig(variant="mg", max_iterations=1), graph_name="star3")

    # ----------------------------------------------- random graph variants
    rng = np.random.default_rng(20241119)
    configs = {
        "mg": LpaConfig(),
        "bm": LpaConfig(variant="bm"),
        "exact": LpaConfig(variant="exact"),
        "mg_double": LpaConfig(scan_mode="double"),
        "mg_k3": LpaConfig(sketch_slots=3),
        "mg_k1": LpaConfig(sketch_slots=1),
        "mg_k3_double": LpaConfig(sketch_slots=3, scan_mode="double"),
        "mg_hi_t2p3k3": LpaConfig(degree_threshold=2, partial_groups=3, sketch_slots=3),
        "mg_hi_t2p3k3_double": LpaConfig(degree_threshold=2, partial_groups=3, sketch_slots=3, scan_mode="double"),
        "mg_hi_t4p40": LpaConfig(degree_threshold=4, partial_groups=40),
        "mg_hi_t3p32k4": LpaConfig(degree_threshold=3, partial_groups=32, sketch_slots=4),
        "mg_shared_t2k4": LpaConfig(degree_threshold=2, sketch_slots=4, shared_sketch=True),
        "mg_k16": LpaConfig(sketch_slots=16),
        "mg_k5_hi_t5p7": LpaConfig(sketch_slots=5, degree_threshold=5, partial_groups=7),
        "bm_hi_t2p3": LpaConfig(variant="bm", degree_threshold=2, partial_groups=3),
        "bm_hi_t3p33": LpaConfig(variant="bm", degree_threshold=3, partial_groups=33),
        "mg_gap1": LpaConfig(pickless_gap=1),
        "mg_gap2_tol02": LpaConfig(pickless_gap=2, tolerance=0.2),
        "mg_it5": LpaConfig(max_iterations=5),
        "exact_hi_t2": LpaConfig(variant="exact", degree_threshold=2),
    }
    for r in range(24):
        g = C.random_graph(rng, max_vertices=64, self_loops=(r % 3 != 0))
        gname = f"rand{r}"
        st.graph("rand", gname, g)
        for cname, cfg in configs.items():
            run_case(st, "rand", f"{gname}:{cname}", g, cfg, graph_name=gname)
        if r < 8:
            order = rng.permutation(g.num_vertices)
            for cname in ("mg", "bm", "mg_hi_t2p3k3", "exact"):
                run_case(st, "rand", f"{gname}:{cname}:order", g, configs[cname], order=order, graph_name=gname)
        # lpa_move on arbitrary states
        n = g.num_vertices
        for t, pickless in enumerate((False, True)):
            labels = rng.integers(0, n, n).astype(np.int32)
            flags = rng.random(n) < 0.7
            for cname in ("mg", "bm", "mg_hi_t2p3k3", "exact"):
                move_case(st, "rand", f"{gname}:move{t}:{cname}", g, configs[cname], labels, flags, pickless,
                          graph_name=gname)
        labels = rng.integers(0, n, n).astype(np.int32)
        metric_case(st, "rand", f"{gname}:metric", g, labels, graph_name=gname)

    # larger random multigraphs with high-degree vertices and default config
    for r in range(6):
        n = int(rng.integers(200, 600))
        m = int(rng.integers(8 * n, 20 * n))
        hubs = rng.integers(0, n, 4)
        src = np.concatenate([rng.integers(0, n, m), np.repeat(hubs, 150)])
        dst = np.concatenate([rng.integers(0, n, m), rng.integers(0, n, 600)])
        w = rng.choice(np.array([0.5, 1.0, 2.0]), src.size)
        g = build_graph(n, list(zip(src.tolist(), dst.tolist(), w.tolist())))
        gname = f"hub{r}"
        st.graph("rand", gname, g)
        for cname in ("mg", "bm", "mg_double", "exact", "mg_shared_t2k4"):
            cfg = configs[cname] if cname != "mg_shared_t2k4" else LpaConfig(shared_sketch=True)
            run_case(st, "rand", f"{gname}:{cname}", g, cfg, graph_name=gname)

    # non-dyadic float32 weights and float64 weights
    for r in range(4):
        n = int(rng.integers(50, 300))
        m = 6 * n
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        w = rng.uniform(0.01, 3.0, m)
        for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
            g = build_graph(n, list(zip(src.tolist(), dst.tolist(), w.tolist())), weight_dtype=dt)
            gname = f"realw{r}_{tag}"
            st.graph("rand", gname, g)
            for cname in ("mg", "bm", "mg_double", "mg_hi_t3p32k4", "exact"):
                run_case(st, "rand", f"{gname}:{cname}", g, configs[cname], graph_name=gname)

    # degree-capped graphs: mg single == exact (test_lpa.py:384-391)
    for r in range(10):
        g = C.degree_capped_graph(rng, cap=8)
        gname = f"cap{r}"
        st.graph("rand", gname, g)
        for cname in ("mg", "exact"):
            run_case(st, "rand", f"{gname}:{cname}", g, configs[cname], graph_name=gname)

    # asymmetric CSR built directly (Graph accepts it; marks follow out-arcs)
    for r in range(4):
        n = int(rng.integers(20, 80))
        deg = rng.integers(0, 12, n)
        offsets = np.zeros(n + 1, dtype=np.int64)
        offsets[1:] = np.cumsum(deg)
        targets = rng.integers(0, n, int(offsets[-1])).astype(np.int32)
        weights = rng.choice(np.array([0.5, 1.0, 2.0], dtype=np.float32), int(offsets[-1]))
        g = Graph(offsets, targets, weights)
        gname = f"asym{r}"
        st.graph("rand", gname, g)
        for cname in ("mg", "bm", "mg_hi_t2p3k3", "exact"):
            run_case(st, "rand", f"{gname}:{cname}", g, configs[cname], graph_name=gname)

    # ----------------------------------------------- planted partitions
    prng = np.random.default_rng(1234)
    for r in range(6):
        g = C.planted_partition_graph(prng)
        gname = f"pp{r}"
        st.graph("pp", gname, g)
        for cname in ("mg", "bm", "exact", "mg_double"):
            run_case(st, "pp", f"{gname}:{cname}", g, configs[cname], graph_name=gname)

    # ----------------------------------------------- C1 SBM (BASELINE configs[0])
    g = sbm_c1()
    st.graph("sbm", "c1", g)
    for cname in ("mg", "bm"):
        run_case(st, "sbm", f"c1:{cname}", g, configs[cname], graph_name="c1")

    # ----------------------------------------------- synthetic shapes (oracle generators)
    shapes = {
        "rmat10": orc.rmat(10, seed=11, permute=False),
        "rmat12p": orc.rmat(12, seed=12, permute=True),
        "rmat14p": orc.rmat(14, seed=14, permute=True),
        "grid40p": orc.grid(40, 40, permute=True),
        "grid25": orc.grid(25, 25, permute=False),
        "kmer5k": orc.kmer(5000, seed=3),
    }
    for gname, hg in shapes.items():
        g = to_ref(hg)
        st.graph("shape", gname, g)
        for cname in ("mg", "bm"):
            run_case(st, "shape", f"{gname}:{cname}", g, configs[cname], graph_name=gname,
                     keep_hist=g.num_vertices <= 20000)
        if gname in ("rmat10", "rmat12p", "grid40p"):
            run_case(st, "shape", f"{gname}:mg_double", g, configs["mg_double"], graph_name=gname)
            order = np.random.default_rng(5).permutation(g.num_vertices)
            run_case(st, "shape", f"{gname}:mg:order", g, configs["mg"], order=order, graph_name=gname)
        labels = np.random.default_rng(9).integers(0, g.num_vertices, g.num_vertices).astype(np.int32)
        metric_case(st, "shape", f"{gname}:metric", g, labels, graph_name=gname)

    st.write()
    total = sum(os.path.getsize(os.path.join(HERE, f"golden_{k}.npz")) for k in st.groups)
    print(f"wrote {len(st.index)} cases, {total / 1e6:.2f} MB, sketchlpa {sketchlpa.__version__}")


if __name__ == "__main__":
    main()
