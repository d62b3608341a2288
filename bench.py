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
* roofline: dominant kernel class from the engine's profiling mode (CUDA
           events around each launch on its stream): algorithmic bytes
           (18 B per evaluated vertex + 12 B per scanned arc) /
           device time, against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline: the CPU oracle (C restatement of the reference) on this
           host, 1 thread, a bounded prefix of sweep 0 on the same graph.
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

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "LPA edges/s (|E|*iters/s)"
UNIT = "arcs*iters/s"
SEED = 2411
ALG_BYTES_PER_VERTEX = 18
ALG_BYTES_PER_ARC = 12


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


def cpu_baseline_sample(host_graph, variant, seconds):
    """The oracle's sequential sweep 0 over a growing vertex prefix for about
    `seconds` of CPU time; returns (arcs/s, sample description)."""
    from oracle.oracle import get_oracle
    import paper_2411_19901_b200 as slpa
    orc = get_oracle()
    cfg = slpa.LpaConfig(variant=variant)
    n = host_graph.num_vertices
    labels = np.arange(n, dtype=np.int32)
    flags = np.ones(n, dtype=np.uint8)
    off = host_graph.offsets
    pos, arcs, t_total = 0, 0, 0.0
    chunk = 4096
    while t_total < seconds and pos < n:
        hi = min(n, pos + chunk)
        t0 = time.perf_counter()
        orc.lpa_move_range(host_graph, labels, flags, cfg, True, pos, hi)
        t_total += time.perf_counter() - t0
        arcs += int(off[hi] - off[pos])
        pos = hi
        chunk = min(chunk * 2, 1 << 20)
    return arcs / t_total, f"sweep 0 (pick-less) over vertices [0, {pos}) of {n}: {arcs} arcs in {t_total:.1f} s"


def run_reference_arm(args, world, rank):
    """--impl reference: the CPU oracle (restatement of the reference's
    sequential LPA), 1 host thread, bounded samples of the same workload."""
    if rank != 0:
        return
    from oracle.oracle import get_oracle
    import paper_2411_19901_b200 as slpa
    orc = get_oracle()
    t0 = time.perf_counter()
    g = orc.rmat(args.scale, seed=SEED, permute=True)
    gen_s = time.perf_counter() - t0
    cfg = slpa.LpaConfig(variant=args.variant)
    n = g.num_vertices
    vals = []
    samples = []
    for step in range(args.warmup + args.steps):
        labels = np.arange(n, dtype=np.int32)
        flags = np.ones(n, dtype=np.uint8)
        lo = (step * 131071) % max(n - 200000, 1)
        hi = min(n, lo + args.ref_prefix)
        t0 = time.perf_counter()
        orc.lpa_move_range(g, labels, flags, cfg, True, lo, hi)
        dt = time.perf_counter() - t0
        arcs = int(g.offsets[hi] - g.offsets[lo])
        if step >= args.warmup:
            vals.append(arcs / dt)
            samples.append((lo, hi, arcs, dt))
    value = float(np.median(vals))
    sample = (f"sweep-0 vertex ranges of {args.ref_prefix} vertices (first [{samples[0][0]},{samples[0][1]})), "
              f"RMAT s{args.scale} ef16, {g.num_arcs} arcs; graph generated on CPU in {gen_s:.0f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * float(np.mean([s[3] for s in samples])),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, g.num_vertices, g.num_arcs, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n, m, world):
    if getattr(args, "graph", "rmat") != "rmat":
        name = {"grid": "4899x4899 4-neighbour grid, unit weights, permuted ids (configs[2])",
                "kmer": "k-mer-like chain graph, 2e8 vertices, links kept w.p. 0.95 + n/20 chords, permuted ids (configs[3])"}
        return {"workload": f"nu{'MG8' if args.variant == 'mg' else 'BM'}-LPA {args.graph} ({name[args.graph]})",
                "graph": name[args.graph], "vertices": n, "arcs": m, "variant": args.variant,
                "mode": "deterministic (bit-exact sequential)" if args.mode == "det" else "async",
                "parallelism": "single GPU", "l2_policy": "inputs larger than L2"}
    return {
        "workload": f"nuMG8-LPA RMAT s{args.scale} ef16 (configs[1])" if args.variant == "mg"
        else f"nuBM-LPA RMAT s{args.scale} ef16",
        "graph": f"RMAT scale {args.scale}, edge factor 16, A/B/C/D .57/.19/.19/.05, permuted ids, "
                 f"self-loops dropped, duplicates merged (seed {SEED})",
        "vertices": n, "arcs": m, "variant": args.variant,
        "mode": "deterministic (bit-exact sequential)" if args.mode == "det" else "async",
        "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
        "l2_policy": "inputs larger than L2 (CSR ~4.3 GB >> 126 MB L2)",
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
    ranges = partition_ranges(n, world)
    eng = slpa.Engine(local)
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
    iters_all = []
    ev0.record()
    for _ in range(args.steps):
        res = lpa_run_partitioned(eng, cfg, ranges)
        iters_all.append(res.iterations)
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
                       "parallelism": f"{world} contiguous vertex ranges, NCCL label all-gather + flag max-reduce",
                       "l2_policy": "inputs larger than L2"},
            "iterations_per_step": iters_all, "gpu_launches": None, "e2e": None, "roofline": None,
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
    ap.add_argument("--variant", default="mg", choices=["mg", "bm"])
    ap.add_argument("--mode", default="det", choices=["det", "async"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-prefix", type=int, default=400000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        _, iters, delta, conv = eng.run(cfg, fetch_labels=False)
        st = eng.stats()
        t_dev += st["device_ms"]
        iters_all.append(iters)
        launches += st["kernel_launches"]
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
    eng.set_profiling(False)
    dom_name, dom = max(((k, v) for k, v in prof.items() if k.startswith("eval")), key=lambda kv: kv[1]["ms"])
    alg_bytes = ALG_BYTES_PER_VERTEX * dom["evals"] + ALG_BYTES_PER_ARC * dom["arcs"]
    achieved = alg_bytes / (dom["ms"] / 1000.0) / 1e9 if dom["ms"] > 0 else 0.0
    peak, peak_src = peaks()
    total_ms = sum(v["ms"] for v in prof.values())
    traffic = None
    tfile = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):  # written by tools/ncu_traffic.py from an ncu capture of the same workload
        with open(tfile) as f:
            tj = json.load(f)
        if (tj.get("scale") == args.scale and tj.get("variant") == args.variant and tj.get("mode") == args.mode
                and tj.get("graph", "rmat") == args.graph):
            c = tj.get("classes", {}).get(dom_name)
            traffic = c.get("dram_bytes_per_launch") if c else None

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    host_graph = None
    if rank == 0 or world > 1:
        off, tgt, w = eng.download()
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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and host_graph is not None:
        v, sample = cpu_baseline_sample(host_graph, args.variant, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample,
               "host_cpus": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * t_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, n, m, world),
            "iterations_per_step": iters_all,
            "wall_s_timed": wall,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": dom_name,
                         "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes / max(dom["launches"], 1),
                         "ms_per_launch": dom["ms"] / max(dom["launches"], 1),
                         "share_of_step": dom["ms"] / total_ms if total_ms else None,
                         "profile": prof},
            "cpu_baseline": cpu,
            "clocks": clk,
            "run_stats": {k: stats_last[k] for k in ("rounds", "vertex_evals", "arc_reads", "first_evals",
                                                     "first_arcs", "device_bytes", "graph_bytes")},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
