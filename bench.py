#!/usr/bin/env python
"""Benchmark: LPA edges/s (|E| * iterations / s) -- BASELINE.json metric.

Workload (BASELINE.json configs[1]): nuMG8-LPA, deterministic mode (bit-exact
with the reference's sequential sweep), on RMAT scale 24, edge factor 16,
(A,B,C,D) = (.57,.19,.19,.05), seeded vertex permutation, duplicates merged
(synthetic).  One *step* = one full lpa_run (all iterations to
convergence) from fresh labels.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

* value  : device-resident graph, CUDA-event time of each run on the engine's
           stream (host syncs between rounds included), max over ranks.
* e2e    : same metric through the public API ``lpa_run(graph, cfg)`` with
           the graph in pinned HOST memory: H2D upload + validation + binning
           + run + D2H labels inside the timed region.
* roofline: dominant kernel family from the engine's profiling mode (CUDA
           events around each launch on its stream): algorithmic bytes
           (18 B per evaluated vertex + 12 B per scanned arc) /
           device time, against MEASURED_PEAKS.json hbm_gbs; `traffic` from
           an ncu capture of one run (profiles/ncu_traffic.json) on the same
           launch basis; `run_frac` = the whole run's algorithmic bytes
           (first evaluations only) over its device time.
* parity / quality: the GPU result checked against a complete sequential
           lpa_run of the oracle port on the same graph (labels, delta
           history, iterations), modularity and community count of both.
* cpu_baseline: that oracle run's time (1 thread; the algorithm is
           sequential), plus the Python reference itself (baseline/_ref):
           a full C1 run and a bounded sweep-0 prefix of the bench graph.
* --impl reference: complete oracle-port lpa_run's of the same workload on
           the host (time-budgeted, --ref-budget), the same unit of work.
* N > 1  : one RMAT graph of scale --scale + log2(N) partitioned by contiguous
           vertex ranges; deterministic mode (default): speculative rounds
           across ranks, NCCL all-gather of the owned label words + MAX-reduce
           of the dirty marks per round (bit-identical to 1 GPU); --mode
           async: the asynchronous partitioned sweep.  Scaling "weak".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from types import SimpleNamespace

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "LPA edges/s (|E|*iters/s)"
UNIT = "arcs*iters/s"
SEED = 2411
ALG_BYTES_PER_VERTEX = 18
ALG_BYTES_PER_ARC = 12
# kernel families for the roofline (engine profiling classes they sum)
FAMILIES = {
    "eval_hi": ("eval_hi_r0", "eval_hi_rk", "eval_mid_r0", "eval_mid_rk"),  # deg >= D_H (k_mg_hi_*, k_bm_hi_*)
    "eval_lo": ("eval_lo_r0", "eval_lo_rk"),                                # deg < D_H (k_lane_direct, k_lo_warp)
    "eval_giant": ("eval_giant",),                                          # deg >= 32768 (gather + block replay)
}


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("SLPA_BENCH_SHARE_GPU"):  # test harness: every rank on GPU 0 (gloo)
        local = 0
    return world, rank, local


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_full_runs(host_graph, cfg, budget_s, max_runs):
    """Complete sequential lpa_run's of the CPU oracle (oracle/lpa_oracle.c,
    the C restatement of lpa.py:262-308, pinned to the reference's golden
    vectors) on the bench graph, 1 host thread, until `budget_s` is spent
    (at least one run).  Returns (runs, result of the last run)."""
    from oracle.oracle import get_oracle
    orc = get_oracle()
    runs, res, spent = [], None, 0.0
    while len(runs) < max(1, max_runs) and (not runs or spent + runs[-1][0] <= budget_s):
        t0 = time.perf_counter()
        res = orc.lpa_run(host_graph, cfg)
        dt = time.perf_counter() - t0
        spent += dt
        runs.append((dt, res.iterations))
    return runs, res


def python_reference_sample(host_graph, variant, seconds):
    """The Python reference itself (baseline/_ref: sketchlpa 0.1.0, pip-
    installed by tools/install_reference.sh) on the host, BASELINE.md §2:
    a complete lpa_run on C1 (tests/golden c1) and -- C2 takes ~50 min in
    Python -- sweep 0 of the bench graph over a vertex prefix of about
    `seconds` through the reference's own sweep (lpa._process_vertices,
    lpa.py:204-224).  perf_counter around the call as cli.py:182-184."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "sketchlpa")):
        return {"unavailable": "baseline/_ref not installed (tools/install_reference.sh)"}
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import sketchlpa
    from sketchlpa import lpa as ref_lpa
    out = {"impl": "sketchlpa 0.1.0 (Python, pure numpy/loops)", "cores": 1}
    gold = os.path.join(REPO, "tests", "golden", "golden_sbm.npz")
    if os.path.exists(gold):
        z = np.load(gold)
        g1 = sketchlpa.Graph(z["c1/offsets"], z["c1/targets"], z["c1/weights"])
        t0 = time.perf_counter()
        r1 = sketchlpa.lpa_run(g1, sketchlpa.LpaConfig(variant=variant))
        dt = time.perf_counter() - t0
        out["c1_full_run"] = {"seconds": dt, "iterations": r1.iterations,
                              "value": g1.num_arcs * r1.iterations / dt, "unit": UNIT,
                              "modularity": float(sketchlpa.modularity(g1, r1.labels)),
                              "num_communities": int(sketchlpa.community_stats(g1, r1.labels).num_communities)}
    g = sketchlpa.Graph(host_graph.offsets, host_graph.targets, host_graph.weights)
    cfg = sketchlpa.LpaConfig(variant=variant)
    n = g.num_vertices
    labels = np.arange(n, dtype=np.int32)
    unprocessed = np.ones(n, dtype=bool)
    sel = ref_lpa._make_selector(g, labels, cfg)
    pos, arcs, spent, chunk = 0, 0, 0.0, 2048
    while spent < seconds and pos < n:
        hi = min(n, pos + chunk)
        t0 = time.perf_counter()
        ref_lpa._process_vertices(g, labels, unprocessed, sel, True, range(pos, hi))
        spent += time.perf_counter() - t0
        arcs += int(g.offsets[hi] - g.offsets[pos])
        pos = hi
        chunk = min(chunk * 2, 65536)
    out["bench_graph_sweep0_prefix"] = {"vertices": pos, "arcs": arcs, "seconds": spent, "value": arcs / spent,
                                        "unit": "arcs/s (sweep 0, pick-less; every vertex active)"}
    return out


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's CPU implementation of the path on
    this host.  The reference is Python and cannot be compiled, so per the
    tier rules the arm is the oracle port (oracle/lpa_oracle.c, the C
    restatement, pinned to the reference's golden vectors): COMPLETE
    lpa_run's of the same graph and config as the GPU arm -- the same unit
    of work, |E| x iterations / wall -- 1 host thread (the deterministic
    algorithm is sequential).  Steps are time-budgeted (--ref-budget); the
    line says how many ran.  The Python reference itself is timed beside it
    (python_reference)."""
    if rank != 0:
        return
    import paper_2411_19901_b200 as slpa
    from oracle.oracle import get_oracle
    orc = get_oracle()
    t0 = time.perf_counter()
    if args.graph == "grid":
        g = orc.grid(4899, 4899, permute=True)
    elif args.graph == "kmer":
        g = orc.kmer(200_000_000, seed=3)
    else:
        g = orc.rmat(args.scale, seed=SEED, permute=True)
    gen_s = time.perf_counter() - t0
    cfg = slpa.LpaConfig(variant=args.variant)
    runs, res = oracle_full_runs(g, cfg, args.ref_budget, args.steps)
    secs = [r[0] for r in runs]
    value = g.num_arcs * sum(r[1] for r in runs) / sum(secs)
    sample = (f"{len(runs)} complete sequential lpa_run(s) (oracle port, deterministic, {res.iterations} "
              f"iterations each) on {args.graph} n={g.num_vertices} m={g.num_arcs}; "
              f"graph generated on the CPU in {gen_s:.0f} s (outside the timing)")
    pyref = python_reference_sample(g, args.variant, args.py_seconds) if args.py_seconds > 0 else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(runs), "steps_requested": args.steps, "warmup": 0, "warmup_requested": args.warmup,
        "ms_per_step": 1000.0 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, g.num_vertices, g.num_arcs, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample,
                         "host_cpus": os.cpu_count(), "cpu_model": cpu_model(), "python_reference": pyref},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {"iterations": res.iterations, "delta_history": res.delta_history,
                   "num_communities": int(np.unique(res.labels).size)},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n, m, world):
    if getattr(args, "graph", "rmat") != "rmat":
        name = {"grid": "4899x4899 4-neighbour grid, unit weights, permuted ids (configs[2])",
                "kmer": "k-mer-like chain graph, 2e8 vertices, links kept w.p. 0.95 + n/20 chords, permuted ids (configs[3])"}
        vname = {"mg": "MG8", "bm": "BM", "exact": "exact"}[args.variant]
        return {"workload": f"nu{vname}-LPA {args.graph} ({name[args.graph]})",
                "graph": name[args.graph], "vertices": n, "arcs": m, "variant": args.variant,
                "mode": "deterministic (bit-exact sequential)" if args.mode == "det" else "async",
                "parallelism": "single GPU", "l2_policy": "inputs larger than L2"}
    return {
        "workload": (f"nuMG8-LPA RMAT s{args.scale} ef16 " + ("(configs[1])" if args.scale == 24 else
                     "(configs[4]'s graph on one GPU)" if args.scale == 27 else "")).strip() if args.variant == "mg"
        else f"nu{'BM' if args.variant == 'bm' else 'exact'}-LPA RMAT s{args.scale} ef16",
        "graph": f"RMAT scale {args.scale}, edge factor 16, A/B/C/D .57/.19/.19/.05, permuted ids, "
                 f"self-loops dropped, duplicates merged (seed {SEED})",
        "vertices": n, "arcs": m, "variant": args.variant,
        "mode": "deterministic (bit-exact sequential)" if args.mode == "det" else "async",
        "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
        "l2_policy": f"inputs larger than L2 (CSR ~{(8 * (n + 1) + 8 * m) / 1e9:.1f} GB >> 126 MB L2)",
    }


def run_partitioned(args, world, rank, local, dist):
    """N > 1: one graph partitioned by contiguous vertex ranges, the
    asynchronous partitioned sweep with an NCCL label all-gather and flag
    max-reduction per sweep (paper_2411_19901_b200/distributed.py).  Weak
    scaling: RMAT scale = --scale + log2(N) (N=8: scale 27)."""
    import math
    import torch
    import paper_2411_19901_b200 as slpa
    from paper_2411_19901_b200.distributed import lpa_run_partitioned, partition_ranges
    scale = args.scale + int(round(math.log2(world)))
    n = 1 << scale
    eng = slpa.Engine(local)
    ranges = eng.rmat_cuts(scale, world, seed=SEED, permute=True)  # arc-balanced contiguous ranges
    eng.part_gen_rmat(scale, *ranges[rank], seed=SEED, permute=True)
    cfg = slpa.LpaConfig(variant=args.variant, worker_count=0 if args.mode == "det" else 1)
    dev = torch.device(f"cuda:{local}")
    m_local = torch.tensor([eng.m], dtype=torch.int64, device=dev)
    dist.all_reduce(m_local)
    m = int(m_local.item())

    def barrier():
        torch.cuda.synchronize(local)
        dist.barrier()

    for _ in range(args.warmup):
        lpa_run_partitioned(eng, cfg, ranges)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters_all, xstats = [], []
    ev0.record()
    for _ in range(args.steps):
        res = lpa_run_partitioned(eng, cfg, ranges)
        iters_all.append(res.iterations)
        xstats.append((res.rounds, res.sparse_rounds, res.exchange_bytes))
    ev1.record()
    barrier()
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1000.0], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_s = float(t.item())
    value = float(m) * sum(iters_all) / t_s
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * t_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"nuMG8-LPA RMAT s{scale} ef16 partitioned over {world} GPUs",
                       "graph": f"RMAT scale {scale} (= {args.scale} + log2 N), edge factor 16, permuted, seed {SEED}",
                       "vertices": n, "arcs": m, "variant": args.variant,
                       "mode": ("deterministic (bit-exact sequential; speculative rounds with a per-round "
                                "label all-gather + dirty-mark max-reduce)") if args.mode == "det"
                               else "async (partitioned)",
                       "parallelism": f"{world} contiguous arc-balanced vertex ranges, NCCL label all-gather + "
                                      f"flag max-reduce on the library stream",
                       "ranges": ranges,
                       "l2_policy": "inputs larger than L2"},
            "iterations_per_step": iters_all,
            "exchange": {"rounds_per_step": xstats[-1][0], "sparse_rounds_per_step": xstats[-1][1],
                         "rank0_bytes_per_step": xstats[-1][2],
                         "dense_bytes_per_round": 4 * (ranges[0][1] - ranges[0][0]) + n},
            "gpu_launches": None, "e2e": None, "roofline": None,
            "cpu_baseline": None, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--graph", default="rmat", choices=["rmat", "grid", "kmer"],
                    help="rmat: configs[1] (default); grid: configs[2] 4899^2 grid; kmer: configs[3] 2e8-vertex k-mer-like")
    ap.add_argument("--variant", default="mg", choices=["mg", "bm", "exact"])
    ap.add_argument("--mode", default="det", choices=["det", "async"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="reference arm: CPU seconds of complete oracle runs (at least one run)")
    ap.add_argument("--py-seconds", type=float, default=10.0,
                    help="Python reference sample (baseline/_ref) beside the CPU numbers; 0 = skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (graphs beyond host RAM)")
    args = ap.parse_args()
    world, rank, local = dist_env()

    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        # NCCL between GPUs; SLPA_BENCH_BACKEND=gloo lets tests run the same
        # path with several ranks on one device
        dist.init_process_group(os.environ.get("SLPA_BENCH_BACKEND", "nccl"))

    import paper_2411_19901_b200 as slpa
    if world > 1:
        run_partitioned(args, world, rank, local, dist)
        return
    eng = slpa.Engine(local)
    if args.graph == "grid":
        eng.gen_grid(4899, 4899, permute=True)
    elif args.graph == "kmer":
        eng.gen_kmer(200_000_000, seed=3)
    else:
        eng.gen_rmat(args.scale, seed=SEED, permute=True)
    n, m = eng.n, eng.m
    cfg = slpa.LpaConfig(variant=args.variant, worker_count=0 if args.mode == "det" else 1)

    def barrier():
        torch.cuda.synchronize(local)
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        eng.run(cfg, fetch_labels=False)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t_dev, iters_all, launches = 0.0, [], 0
    stats_sum = {"first_evals": 0, "first_arcs": 0, "vertex_evals": 0, "arc_reads": 0, "rounds": 0}
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        _, iters, delta, conv = eng.run(cfg, fetch_labels=False)
        st = eng.stats()
        t_dev += st["device_ms"]
        iters_all.append(iters)
        launches += st["kernel_launches"]
        for k in stats_sum:
            stats_sum[k] += st[k]
    barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    stats_last = eng.stats()
    arcs_done = float(m) * float(sum(iters_all))
    t_s = t_dev / 1000.0
    if dist is not None:
        tt = torch.tensor([t_s, arcs_done], dtype=torch.float64, device=f"cuda:{local}")
        t_max = tt[:1].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        work = tt[1:].clone()
        dist.all_reduce(work, op=dist.ReduceOp.SUM)
        t_s, arcs_done = float(t_max.item()), float(work.item())
    value = arcs_done / t_s

    # ---- roofline (profiling pass, outside the timed region)
    eng.set_profiling(True)
    eng.run(cfg, fetch_labels=False)
    prof = eng.profile()
    st_prof = eng.stats()  # profiling run: first_evals / first_arcs = the sequential sweeps' processed set
    eng.set_profiling(False)
    fams = {}
    for fam, members in FAMILIES.items():
        fams[fam] = {k: sum(prof[c][k] for c in members) for k in ("launches", "ms", "evals", "arcs")}
    dom_name, dom = max(fams.items(), key=lambda kv: kv[1]["ms"])
    alg_bytes = ALG_BYTES_PER_VERTEX * dom["evals"] + ALG_BYTES_PER_ARC * dom["arcs"]
    achieved = alg_bytes / (dom["ms"] / 1000.0) / 1e9 if dom["ms"] > 0 else 0.0
    peak, peak_src = peaks()
    total_ms = sum(v["ms"] for v in prof.values())
    traffic, traffic_run, sectors_per_request = None, None, None
    tfile = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):  # tools/ncu_traffic.py over an ncu capture of ONE lpa_run of this workload
        with open(tfile) as f:
            tj = json.load(f)
        if (tj.get("scale") == args.scale and tj.get("variant") == args.variant and tj.get("mode") == args.mode
                and tj.get("graph", "rmat") == args.graph and tj.get("basis") == "one lpa_run"):
            c = tj.get("families", {}).get(dom_name)
            if c and dom["launches"]:
                traffic_run = c["dram_bytes_per_run"]
                traffic = traffic_run / dom["launches"]  # same launch count as alg_bytes_per_launch
                sectors_per_request = c.get("ld_sectors_per_request")
    # run level: bytes of the vertices each sweep processes
    # (first evaluation only: re-evaluations are overhead) over the whole run
    run_alg = ALG_BYTES_PER_VERTEX * st_prof["first_evals"] + ALG_BYTES_PER_ARC * st_prof["first_arcs"]
    run_achieved = run_alg / (t_s / args.steps) / 1e9

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    e2e_labels = None
    host_graph = None
    int_path = False
    if (rank == 0 or world > 1) and not args.no_e2e:
        off, tgt, w = eng.download()
        # the device's exactness test for integer sketch values (slpa_graph.cu)
        nz = np.diff(off) > 0  # reduceat needs in-range starts: non-empty rows only
        wdeg = np.add.reduceat(w.astype(np.float64), off[:-1][nz]) if w.size else np.zeros(0)
        int_path = bool(np.all(w == np.floor(w)) and (wdeg.max(initial=0) < 2.0 ** 31))
        pin_off = torch.empty(off.size, dtype=torch.int64, pin_memory=True).numpy()
        pin_tgt = torch.empty(tgt.size, dtype=torch.int32, pin_memory=True).numpy()
        pin_w = torch.empty(w.size, dtype=torch.float32, pin_memory=True).numpy()
        pin_off[:] = off
        pin_tgt[:] = tgt
        pin_w[:] = w
        del off, tgt, w
        host_graph = slpa.Graph(pin_off, pin_tgt, pin_w)
        e2e_steps = args.e2e_steps or max(2, min(args.steps, 5))
        eng2 = slpa.Engine(local)
        res = slpa.lpa_run(host_graph, cfg, engine=eng2)  # warm-up (allocations)
        barrier()
        t0 = time.perf_counter()
        e2e_iters = 0
        for _ in range(e2e_steps):
            res = slpa.lpa_run(host_graph, cfg, engine=eng2)
            e2e_iters += res.iterations
        e2e_t = time.perf_counter() - t0
        eng2.close()
        h2d = pin_off.nbytes + pin_tgt.nbytes + pin_w.nbytes
        d2h = n * 4 + cfg.max_iterations * 8
        e2e_val = float(m) * e2e_iters / e2e_t
        if dist is not None:
            tt = torch.tensor([e2e_t, float(m) * e2e_iters], dtype=torch.float64, device=f"cuda:{local}")
            a = tt[:1].clone()
            dist.all_reduce(a, op=dist.ReduceOp.MAX)
            b = tt[1:].clone()
            dist.all_reduce(b, op=dist.ReduceOp.SUM)
            e2e_val = float(b.item()) / float(a.item())
        e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": e2e_steps, "s_per_step": e2e_t / e2e_steps}
        e2e_labels = res.labels

    cpu, parity, quality = None, None, None
    if rank == 0 and world == 1 and host_graph is not None:
        # the GPU result of this workload, checked against the reference's
        # sequential algorithm (oracle port) on the same graph: labels,
        # delta history, iterations; quality (Q, |communities|) beside it
        labels_gpu, it_gpu, delta_gpu, conv_gpu = eng.run(cfg)
        q_gpu, nc_gpu = eng.tally(labels_gpu, want_arrays=False)[:2]
        quality = {"gpu": {"modularity": q_gpu, "num_communities": int(nc_gpu), "iterations": it_gpu,
                           "delta_history": delta_gpu}}
        if not args.no_cpu_baseline:
            from oracle.oracle import get_oracle
            runs, ref = oracle_full_runs(host_graph, slpa.LpaConfig(variant=args.variant), 0.0, 1)
            q_ref = get_oracle().modularity(host_graph, ref.labels)
            nc_ref = int(np.unique(ref.labels).size)
            quality["cpu_reference"] = {"modularity": q_ref, "num_communities": nc_ref,
                                        "iterations": ref.iterations, "delta_history": ref.delta_history}
            if args.mode == "det":
                parity = {"vs": "oracle port: complete sequential lpa_run on the same graph",
                          "labels_equal": bool(np.array_equal(labels_gpu, ref.labels)),
                          "e2e_labels_equal": bool(np.array_equal(e2e_labels, ref.labels)),
                          "delta_history_equal": delta_gpu == ref.delta_history,
                          "iterations_equal": it_gpu == ref.iterations, "converged_equal": conv_gpu == ref.converged}
            else:
                parity = {"vs": "sequential oracle (async acceptance: |dQ| <= 0.01, communities within 5%)",
                          "dQ": q_gpu - q_ref, "communities_ratio": nc_gpu / max(1, nc_ref)}
            cpu = {"value": float(m) * ref.iterations / runs[0][0], "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"one complete sequential lpa_run (oracle port, {ref.iterations} iterations) on the "
                             f"bench graph: {runs[0][0]:.1f} s",
                   "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}
            if args.py_seconds > 0:
                cpu["python_reference"] = python_reference_sample(host_graph, args.variant, args.py_seconds)

    if rank == 0:
        dev_b, graph_b = stats_last["device_bytes"], stats_last["graph_bytes"]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * t_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32" if int_path else "f64",
            "dtype_note": ("u32: sketch / vote values in uint32, exact (bit-identical to the reference's "
                           "binary64) because every weight is integral and every weighted degree < 2^31, checked "
                           "on the device at upload; otherwise the binary64 kernels run"),
            "data": "synthetic",
            "config": workload_config(args, n, m, world),
            "iterations_per_step": iters_all,
            "wall_s_timed": wall,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": dom_name,
                         "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes / max(dom["launches"], 1),
                         "launches_per_run": dom["launches"],
                         "alg_bytes_per_run": alg_bytes, "traffic_per_run": traffic_run,
                         "traffic_over_alg": (traffic_run / alg_bytes) if traffic_run and alg_bytes else None,
                         "ld_sectors_per_request": sectors_per_request,
                         "ms_per_launch": dom["ms"] / max(dom["launches"], 1),
                         "share_of_step": dom["ms"] / total_ms if total_ms else None,
                         "run_alg_bytes": run_alg, "run_achieved": run_achieved, "run_frac": run_achieved / peak,
                         "run_processed_vertices": st_prof["first_evals"], "run_processed_arcs": st_prof["first_arcs"],
                         "basis": ("per launch: the family's algorithmic bytes (18 B per evaluated vertex + 12 B "
                                   "per scanned arc, re-evaluations included) and its ncu DRAM bytes over ONE "
                                   "lpa_run, both divided by the same kernel-launch count; run_frac: 18 B per "
                                   "vertex the sequential sweeps process + 12 B per arc of it (each sweep's "
                                   "processed set, counted on the device from the turn bits of the final "
                                   "evaluations), over the whole run's device time"),
                         "families": fams, "profile": prof},
            "memory": {"device_bytes": dev_b, "graph_bytes": graph_b,
                       "device_bytes_per_vertex": dev_b / max(n, 1), "device_bytes_per_arc": dev_b / max(m, 1),
                       "engine_bytes_per_vertex": (dev_b - graph_b) / max(n, 1),
                       "reference_model_aux_bytes": slpa.aux_memory_estimate(
                           SimpleNamespace(num_vertices=n, weights=np.zeros(0, eng.weights_dtype)), cfg)},
            "quality": quality,
            "parity": parity,
            "cpu_baseline": cpu,
            "clocks": clk,
            "run_stats": {k: v / args.steps for k, v in stats_sum.items()},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
