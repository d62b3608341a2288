"""Multi-GPU driver (paper_2411_19901_b200/distributed.py).

CPU (gloo, world_size 2): the exchange/driver logic is exercised with a mock
engine whose part_sweep is a sequential CPU restatement of the partitioned
asynchronous sweep (each rank visits its owned vertices in order, reading its
own replica).  With that schedule the distributed run is deterministic, so it
must equal a single-process simulation of the same exchange protocol.

GPU: two processes share one B200 (gloo over CUDA tensors -- NCCL needs one
GPU per rank) and run the real CUDA partitioned sweep end to end.
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class MockEngine:
    """CPU stand-in for Engine.part_* (test-only; uses the oracle selector)."""

    def __init__(self, g, vb, ve, oracle):
        self.g, self.n, self.v_begin, self.v_end, self.oracle = g, g.num_vertices, vb, ve, oracle

    def part_begin(self, cfg):
        import torch
        self.lab = torch.arange(self.n, dtype=torch.int32)
        self.fl = torch.zeros(self.n, dtype=torch.uint8)
        self.fl[self.v_begin:self.v_end] = 1

    def part_buffers(self):
        return self.lab, self.fl

    def part_sweep(self, cfg, pickless):
        return sweep_range(self.g, self.lab.numpy(), self.fl.numpy(), self.v_begin, self.v_end, cfg, pickless,
                           self.oracle)

    def part_end_exchange(self):
        self.fl[: self.v_begin] = 0
        self.fl[self.v_end:] = 0


def sweep_range(g, lab, fl, vb, ve, cfg, pickless, oracle):
    changed = 0
    for v in range(vb, ve):
        if not fl[v]:
            continue
        fl[v] = 0
        cand = oracle.select(g, lab, v, cfg)
        if cand != lab[v] and (not pickless or cand < lab[v]):
            lab[v] = cand
            changed += 1
            fl[g.targets[g.offsets[v]:g.offsets[v + 1]]] = 1
    return changed


def simulate(g, cfg, ranges, oracle):
    """Single-process model of lpa_run_partitioned's exchange protocol."""
    n = g.num_vertices
    labs = [np.arange(n, dtype=np.int32) for _ in ranges]
    fls = []
    for b, e in ranges:
        f = np.zeros(n, dtype=np.uint8)
        f[b:e] = 1
        fls.append(f)
    hist, conv = [], False
    for it in range(cfg.max_iterations):
        pickless = it % cfg.pickless_gap == 0
        delta = sum(sweep_range(g, labs[r], fls[r], b, e, cfg, pickless, oracle) for r, (b, e) in enumerate(ranges))
        merged = np.concatenate([labs[r][b:e] for r, (b, e) in enumerate(ranges)])
        fmax = np.max(np.stack(fls), axis=0)
        for r, (b, e) in enumerate(ranges):
            labs[r][:] = merged
            fls[r][:] = 0
            fls[r][b:e] = fmax[b:e]
        hist.append(delta)
        if not pickless and delta / n < cfg.tolerance:
            conv = True
            break
    return labs[0], hist, conv


def _worker(rank, world, port, payload, out):
    import torch.distributed as dist
    from oracle.oracle import HostGraph, get_oracle
    from paper_2411_19901_b200 import LpaConfig
    from paper_2411_19901_b200.distributed import lpa_run_partitioned
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = HostGraph(*payload["graph"])
    cfg = LpaConfig(**payload["cfg"])
    ranges = payload["ranges"]
    eng = MockEngine(g, ranges[rank][0], ranges[rank][1], get_oracle())
    res = lpa_run_partitioned(eng, cfg, ranges)
    out[rank] = (eng.lab.numpy().copy(), res.delta_history, res.converged)
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["mg", "bm"])
def test_gloo_two_ranks_match_protocol_simulation(oracle, variant):
    import torch.multiprocessing as mp
    from paper_2411_19901_b200 import LpaConfig
    from paper_2411_19901_b200.distributed import partition_ranges
    g = oracle.rmat(9, seed=31, permute=True)
    cfg = LpaConfig(variant=variant, worker_count=2)
    ranges = partition_ranges(g.num_vertices, 2, np.diff(g.offsets))
    payload = {"graph": (g.offsets, g.targets, g.weights), "cfg": cfg.__dict__, "ranges": ranges}
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), payload, out), nprocs=2, join=True)
    lab_ref, hist_ref, conv_ref = simulate(g, cfg, ranges, oracle)
    for r in range(2):
        lab, hist, conv = out[r]
        assert hist == hist_ref
        assert conv == conv_ref
        np.testing.assert_array_equal(lab, lab_ref)


def test_partition_ranges():
    from paper_2411_19901_b200.distributed import partition_ranges
    assert partition_ranges(10, 3) == [(0, 4), (4, 8), (8, 10)]
    deg = np.array([100, 1, 1, 1, 1, 1, 1, 100])
    r = partition_ranges(8, 2, deg)
    assert r[0][0] == 0 and r[-1][1] == 8 and r[0][1] == r[1][0]
    assert 1 <= r[0][1] <= 7
    for world in (1, 2, 4, 8):
        rs = partition_ranges(1000, world, np.ones(1000))
        assert rs[0][0] == 0 and rs[-1][1] == 1000
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))


# ---------------------------------------------------------------- GPU, real kernels
def _gpu_worker(rank, world, port, scale, out):
    import torch.distributed as dist
    import paper_2411_19901_b200 as slpa
    from paper_2411_19901_b200.distributed import lpa_run_partitioned, modularity_partitioned, partition_ranges
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1 << scale
    ranges = partition_ranges(n, world)
    eng = slpa.Engine(0)
    eng.part_gen_rmat(scale, *ranges[rank], seed=77, permute=True)
    cfg = slpa.LpaConfig(worker_count=1)
    res = lpa_run_partitioned(eng, cfg, ranges)
    q = modularity_partitioned(eng, ranges)
    lab, _ = eng.part_buffers()
    out[rank] = (lab.cpu().numpy(), res.delta_history, res.converged, q, eng.m)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_two_ranks_one_device(oracle):
    import torch.multiprocessing as mp
    scale = 15
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(2, _free_port(), scale, out), nprocs=2, join=True)
    g = oracle.rmat(scale, seed=77, permute=True)
    lab0, hist0, conv0, q0, m0 = out[0]
    lab1, hist1, conv1, q1, m1 = out[1]
    assert m0 + m1 == g.num_arcs  # the two row blocks partition the arcs
    np.testing.assert_array_equal(lab0, lab1)  # replicas agree after the last exchange
    assert hist0 == hist1 and conv0 == conv1
    assert q0 == pytest.approx(q1, abs=1e-12)
    assert q0 == pytest.approx(oracle.modularity(g, lab0), abs=1e-9)  # partitioned tally == oracle tally
    ref = oracle.lpa_run(g, type("C", (), dict(variant="mg", scan_mode="single", sketch_slots=8, pickless_gap=8,
                                               tolerance=0.05, max_iterations=20, degree_threshold=128,
                                               partial_groups=32, shared_sketch=False))())
    q_ref = oracle.modularity(g, ref.labels)
    assert q0 >= q_ref - 0.01, (q0, q_ref)


# ---------------------------------------------------------------- deterministic partitioned sweep (§8 e3)
CHG = np.uint32(0x80000000)
LMASK = np.uint32(0x7FFFFFFF)


class MockDetEngine(MockEngine):
    """CPU stand-in for the deterministic Engine.part_det_* protocol: each
    round evaluates the owned flagged (round 0) or dirty vertices against the
    speculative label words (lower neighbours: L1, higher: L0) and marks the
    higher-positioned dependants of any vertex whose word moves -- the
    speculative-round scheme of DESIGN.md §3, restated on the CPU."""

    def part_begin(self, cfg):
        import torch
        super().part_begin(cfg)
        self.lab_new = torch.arange(self.n, dtype=torch.int32)
        self.lab_sent = np.arange(self.n, dtype=np.uint32)
        self.dirty = torch.zeros(self.n, dtype=torch.uint8)
        self.fnext = np.zeros(self.n, dtype=np.uint8)

    def part_det_buffers(self):
        return self.lab_new, self.dirty

    # sparse round exchange (libslpa_b200 slpa_part_det_collect / _apply / _dense)
    def part_det_collect(self):
        import torch
        L1 = self.lab_new.numpy().view(np.uint32)
        d = self.dirty.numpy()
        own = np.arange(self.v_begin, self.v_end)
        moved = own[L1[own] != self.lab_sent[own]]
        self.lab_sent[moved] = L1[moved]
        mask = np.ones(self.n, dtype=bool)
        mask[self.v_begin:self.v_end] = False
        marks = np.flatnonzero((d != 0) & mask)
        words = np.stack([moved.astype(np.int64), L1[moved].astype(np.int64)], axis=1).reshape(-1)
        lst = np.concatenate([words, marks]).astype(np.uint32).view(np.int32)
        return (torch.from_numpy(lst.copy()) if lst.size else None), int(moved.size), int(marks.size)

    def part_det_apply(self, recv, stride, counts, world, rank):
        L1 = self.lab_new.numpy().view(np.uint32)
        d = self.dirty.numpy()
        d[: self.v_begin] = 0
        d[self.v_end:] = 0
        r_all = recv.numpy()
        for r in range(world):
            if r == rank:
                continue
            nw, nm = int(counts[2 * r]), int(counts[2 * r + 1])
            lst = r_all[r * stride: r * stride + 2 * nw + nm]
            ids = lst[0:2 * nw:2]
            L1[ids] = lst[1:2 * nw:2].view(np.uint32)
            t = lst[2 * nw:]
            t = t[(t >= self.v_begin) & (t < self.v_end)]
            d[t] = 1
        return int(d[self.v_begin:self.v_end].astype(np.int64).sum())

    def part_det_dense(self):
        pass

    def part_arc_hash(self):
        """Additive forward / reverse arc sums of the owned rows (the
        library's k_arc_checks hashes, restated with a simpler mix)."""
        g = self.g
        mask = np.uint64((1 << 64) - 1)
        f = r = np.uint64(0)
        for v in range(self.v_begin, self.v_end):
            for t in g.targets[g.offsets[v]:g.offsets[v + 1]]:
                f = (f + np.uint64((v * 1000003 + int(t)) * 2654435761 % (1 << 61))) & mask
                r = (r + np.uint64((int(t) * 1000003 + v) * 2654435761 % (1 << 61))) & mask
        return np.array([f, r, f, r], dtype=np.uint64)

    def part_set_symmetric(self, symmetric):
        self.symmetric = symmetric

    def part_det_round(self, cfg, pickless, rnd):
        g = self.g
        L0 = self.lab.numpy()
        L1 = self.lab_new.numpy().view(np.uint32)
        F0 = self.fl.numpy()
        d = self.dirty.numpy()
        if rnd == 0:
            self.fnext[:] = 0
            work = [v for v in range(self.v_begin, self.v_end) if F0[v] and g.degree(v) > 0]
        else:
            work = [v for v in range(self.v_begin, self.v_end) if d[v]]
        marks = np.zeros(self.n, dtype=np.uint8)
        for v in work:
            nb = g.targets[g.offsets[v]:g.offsets[v + 1]]
            view = L0.copy()
            view[:v] = (L1[:v] & LMASK).astype(np.int32)
            cand = self.oracle.select(g, view, v, cfg)
            cur = int(L0[v])
            lower_changed = bool(np.any((L1[nb[nb < v]] & CHG) != 0))
            turn = bool(F0[v]) or lower_changed
            chg = turn and cand != cur and (not pickless or cand < cur)
            word = np.uint32(cand) | CHG if chg else np.uint32(cur)
            if word != L1[v]:
                L1[v] = word
                marks[nb[nb > v]] = 1
        d[:] = marks

    def part_det_import(self):
        return int(self.dirty.numpy().astype(np.int64).sum())

    def part_det_commit(self, cfg):
        g = self.g
        L0 = self.lab.numpy()
        L1 = self.lab_new.numpy().view(np.uint32)
        delta = 0
        for v in range(self.v_begin, self.v_end):
            if L1[v] & CHG:
                delta += 1
                nb = g.targets[g.offsets[v]:g.offsets[v + 1]]
                self.fnext[nb[nb <= v]] = 1
        moved = (L1 & CHG) != 0
        L0[moved] = (L1[moved] & LMASK).astype(np.int32)
        L1[moved] &= LMASK
        self.lab_sent[:] = L1
        self.fl.numpy()[:] = self.fnext
        return delta


def _det_worker(rank, world, port, payload, out):
    import torch.distributed as dist
    from oracle.oracle import HostGraph, get_oracle
    from paper_2411_19901_b200 import LpaConfig
    from paper_2411_19901_b200.distributed import lpa_run_partitioned
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = HostGraph(*payload["graph"])
    cfg = LpaConfig(**payload["cfg"])
    ranges = payload["ranges"]
    eng = MockDetEngine(g, ranges[rank][0], ranges[rank][1], get_oracle())
    res = lpa_run_partitioned(eng, cfg, ranges, exchange=payload.get("exchange", "auto"))
    out[rank] = (eng.lab.numpy().copy(), res.delta_history, res.converged)
    dist.destroy_process_group()


@pytest.mark.parametrize("variant,world,exchange", [("mg", 2, "auto"), ("bm", 2, "sparse"), ("mg", 3, "sparse"),
                                                     ("mg", 3, "dense")])
def test_gloo_deterministic_partition_equals_sequential_reference(oracle, variant, world, exchange):
    """The deterministic partitioned protocol reproduces the sequential sweep
    (the oracle, pinned to the reference's golden vectors) bit for bit."""
    import torch.multiprocessing as mp
    from paper_2411_19901_b200 import LpaConfig
    from paper_2411_19901_b200.distributed import partition_ranges
    g = oracle.rmat(8, seed=33, permute=True)
    cfg = LpaConfig(variant=variant, degree_threshold=16, partial_groups=4)
    ranges = partition_ranges(g.num_vertices, world, np.diff(g.offsets))
    payload = {"graph": (g.offsets, g.targets, g.weights), "cfg": cfg.__dict__, "ranges": ranges,
               "exchange": exchange}
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_det_worker, args=(world, _free_port(), payload, out), nprocs=world, join=True)
    ref = oracle.lpa_run(g, cfg)
    for r in range(world):
        lab, hist, conv = out[r]
        assert hist == ref.delta_history
        assert conv == ref.converged
        np.testing.assert_array_equal(lab, ref.labels)


def _gpu_det_worker(rank, world, port, scale, variant, out, exchange="auto"):
    import torch.distributed as dist
    import paper_2411_19901_b200 as slpa
    from paper_2411_19901_b200.distributed import lpa_run_partitioned, partition_ranges
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = slpa.Engine(0)
    ranges = eng.rmat_cuts(scale, world, seed=78, permute=True)  # arc-balanced
    eng.part_gen_rmat(scale, *ranges[rank], seed=78, permute=True)
    cfg = slpa.LpaConfig(variant=variant)
    res = lpa_run_partitioned(eng, cfg, ranges, exchange=exchange)
    lab, _ = eng.part_buffers()
    out[rank] = (lab.cpu().numpy(), res.delta_history, res.converged, res.iterations)
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("variant,world,exchange", [("mg", 2, "auto"), ("bm", 2, "auto"), ("mg", 3, "auto"),
                                                     ("mg", 2, "sparse"), ("mg", 3, "dense")])
def test_gpu_deterministic_partition_bit_exact(oracle, variant, world, exchange):
    """Two / three processes share one B200 (gloo over CUDA tensors) and run
    the CUDA deterministic partitioned sweep: every replica equals the
    sequential reference (oracle) bit for bit."""
    import torch.multiprocessing as mp
    from paper_2411_19901_b200 import LpaConfig
    scale = 14
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_det_worker, args=(world, _free_port(), scale, variant, out, exchange), nprocs=world, join=True)
    g = oracle.rmat(scale, seed=78, permute=True)
    ref = oracle.lpa_run(g, LpaConfig(variant=variant))
    for r in range(world):
        lab, hist, conv, iters = out[r]
        assert hist == ref.delta_history
        assert (iters, conv) == (ref.iterations, ref.converged)
        np.testing.assert_array_equal(lab, ref.labels)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["det", "async"])
def test_bench_multi_rank_path(mode):
    """bench.py's N > 1 path end to end under torchrun: two ranks share one
    B200 over gloo (the driver's scaling run uses NCCL on N GPUs)."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SLPA_BENCH_BACKEND="gloo", SLPA_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(repo, "bench.py"), "--gpus", "2", "--scale",
           "15", "--steps", "2", "--warmup", "1", "--mode", mode]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=repo)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["vertices"] == 1 << 16


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_rmat_cuts_arc_balanced(oracle, world):
    """Engine.rmat_cuts: the device histogram of the RMAT edge stream gives the
    same cuts as numpy on the oracle's edge stream (multigraph degrees), and
    the ranges cover [0, n) with near-equal arc counts of the merged CSR."""
    import paper_2411_19901_b200 as slpa
    from oracle.oracle import rmat_thresholds
    scale = 14
    eng = slpa.Engine(0)
    ranges = eng.rmat_cuts(scale, world, seed=5, permute=True)
    n = 1 << scale
    ne = 16 << scale
    src = np.empty(ne, dtype=np.uint32)
    dst = np.empty(ne, dtype=np.uint32)
    ta, tab, tabc = rmat_thresholds(0.57, 0.19, 0.19)
    k = oracle.lib.orc_rmat_edges(scale, ne, ta, tab, tabc, 5, 1, 7, src.ctypes.data, dst.ctypes.data)
    deg = np.bincount(np.concatenate([src[:k], dst[:k]]).astype(np.int64), minlength=n)
    incl = np.cumsum(deg)
    want = [0] + [int(np.searchsorted(incl, int(incl[-1] * r / world), side="right")) for r in range(1, world)] + [n]
    want = np.maximum.accumulate(want)
    assert ranges == [(int(want[r]), int(want[r + 1])) for r in range(world)]
    g = oracle.rmat(scale, seed=5, permute=True)
    arcs = [int(g.offsets[e] - g.offsets[b]) for b, e in ranges]
    assert max(arcs) <= 1.05 * g.num_arcs / world


def _asym_worker(rank, world, port, out):
    import torch.distributed as dist
    import paper_2411_19901_b200 as slpa
    from paper_2411_19901_b200.distributed import lpa_run_partitioned
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 8
    ranges = [(0, 4), (4, 8)]
    b, e = ranges[rank]
    # a directed ring: every arc's reverse is missing
    ro = np.arange(e - b + 1, dtype=np.int64)
    tg = np.array([(v + 1) % n for v in range(b, e)], dtype=np.int32)
    eng = slpa.Engine(0)
    eng.part_upload(n, b, e, ro, tg, np.ones(e - b, dtype=np.float32))
    try:
        lpa_run_partitioned(eng, slpa.LpaConfig(), ranges)
        out[rank] = "ran"
    except ValueError as ex:
        out[rank] = "ValueError: " + str(ex)
    res = lpa_run_partitioned(eng, slpa.LpaConfig(worker_count=1), ranges)  # the async sweep accepts it
    out[rank] = out[rank] + f" | async {res.iterations}"
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_partitioned_det_rejects_asymmetric():
    """the deterministic partitioned rounds need a symmetric graph;
    the ranks' combined arc hashes detect a directed one and the run refuses
    (the asynchronous sweep does not depend on symmetry)."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_asym_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert out[r].startswith("ValueError") and "symmetric" in out[r] and "| async" in out[r]
