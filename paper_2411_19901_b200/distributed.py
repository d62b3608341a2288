"""Multi-GPU label propagation: contiguous vertex ranges, one process (and
one Engine) per GPU, label / mark exchange over torch.distributed (NCCL on
GPUs; the exchange logic is backend-agnostic and is tested with gloo).

Asynchronous sweeps (worker_count > 0; the paper's multi-GPU model,
SURVEY §8(e2)), per sweep:

1. every rank sweeps its own rows in place (libslpa_b200 ``slpa_part_sweep``)
   reading its label replica -- remote labels are one exchange old;
2. each owned label range is broadcast from its owner into every replica,
   in place;
3. the flag arrays are max-reduced: a rank's remote entries carry the
   "neighbour changed" marks of lpa.py:223 for vertices other ranks own;
   ``slpa_part_end_exchange`` then clears the remote entries;
4. delta (changed vertices) is summed; the convergence test is lpa.py:299.

Deterministic sweeps (worker_count == 0) run the speculative
rounds of the single-GPU engine across ranks: per round every
rank evaluates its owned flagged / dirty vertices, then publishes the owned
speculative label words (lab_new, bit 31 = changed) that moved and the dirty
marks it set on other ranks' vertices -- as changed-only lists when they are
short (most rounds), else densely (the owned ranges broadcast in place, the
marks MAX-reduced as bytes); the sweep ends when no mark is set anywhere.  Stale remote reads are re-evaluated through the marks like any
other speculation, so labels, delta history and iteration count are
bit-identical to the sequential reference (lpa.py:204-224).

The collectives operate on zero-copy torch views of the library's device
buffers (``Engine.part_buffers``); torch is the plumbing, the sweep is the
library's CUDA code.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def partition_ranges(n: int, world: int, degrees=None):
    """Contiguous [begin, end) vertex ranges.  Balanced by arc count when
    per-vertex degrees are given, else by vertex count."""
    if world <= 0:
        raise ValueError("world must be positive")
    if degrees is None:
        step = -(-n // world)
        return [(min(n, r * step), min(n, (r + 1) * step)) for r in range(world)]
    cum = np.concatenate([[0], np.cumsum(np.asarray(degrees, dtype=np.int64))])
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


class Exchange:
    """Label exchange + flag max-reduction over torch.distributed."""

    def __init__(self, ranges, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.ranges = ranges
        self.world = len(ranges)
        self.rank = dist.get_rank(group)

    def labels(self, lab):
        """Every rank's owned range of `lab` into every replica, in place: one
        broadcast per rank from the owner, straight out of and into the label
        array (no staging copies; the ranges need not be equal)."""
        for r, (rb, re) in enumerate(self.ranges):
            if re > rb:
                src = r if self.group is None else self.dist.get_global_rank(self.group, r)
                self.dist.broadcast(lab[rb:re], src=src, group=self.group)

    def flags(self, fl):
        self.dist.all_reduce(fl, op=self.dist.ReduceOp.MAX, group=self.group)

    def sum(self, x: int, device) -> int:
        import torch
        t = torch.tensor([int(x)], dtype=torch.int64, device=device)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def sum_f64(self, x: float, device) -> float:
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())


@dataclass
class PartitionedResult:
    iterations: int
    delta_history: list = field(default_factory=list)
    converged: bool = False
    rounds: int = 0                  # deterministic: speculative rounds over all sweeps
    sparse_rounds: int = 0           #   of which exchanged changed-only lists
    exchange_bytes: int = 0          #   bytes this rank contributed to the round exchanges


def _sync(t):
    if getattr(t, "is_cuda", False):
        import torch
        torch.cuda.current_stream(t.device).synchronize()


class _OnLibraryStream:
    """Run torch work (the collectives and their staging copies) on the
    library's own CUDA stream: the exchange is ordered after the sweep's
    kernels and before the next library call on the device, with no host
    synchronisation in between (NCCL's internal stream joins the current
    stream through events)."""

    def __init__(self, engine, device):
        import torch
        self.torch = torch
        self.device = device
        self.ext = torch.cuda.ExternalStream(engine.stream(), device=device) if device.type == "cuda" else None
        self.ctx = None

    def __enter__(self):
        if self.ext is not None:
            self.ctx = self.torch.cuda.stream(self.ext)
            self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)
        return False


def confirm_symmetric(engine, group=None) -> bool:
    """Combine the ranks' arc hashes: the partitioned graph is
    symmetric iff the global forward and reverse sums agree; the library is
    told the answer (its deterministic rounds require a symmetric graph)."""
    import torch
    import torch.distributed as dist
    h = engine.part_arc_hash().view(np.int64)  # two's complement: sums wrap mod 2^64 on every backend
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor(h.copy(), dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    v = t.cpu().numpy()
    sym = bool(v[0] == v[1] and v[2] == v[3])
    engine.part_set_symmetric(sym)
    return sym


def _det_round_exchange(engine, ex, lab_new, dirty, on_lib, mode, stats=None) -> int:
    """One round's exchange; returns the global dirty-vertex count.

    sparse: every rank publishes the owned label words that moved since its
    last exchange and the marks it set on remote vertices (one all-gather of
    padded int32 lists); dense: the owned ranges of the label words are
    broadcast in place and the dirty marks MAX-reduced as bytes.  "auto" picks the
    sparse exchange unless the longest list would move more bytes than the
    dense one -- decided from the all-gathered counts, so every rank agrees."""
    import torch
    lst, nw, nm = engine.part_det_collect()
    dev = lab_new.device
    counts = torch.tensor([nw, nm], dtype=torch.int64, device=dev)
    allc = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(ex.world)]
    ex.dist.all_gather(allc, counts, group=ex.group)
    cnt = torch.stack(allc).cpu().numpy().reshape(-1)
    longest = int(max(2 * cnt[2 * r] + cnt[2 * r + 1] for r in range(ex.world)))
    n = lab_new.numel()
    sparse = mode == "sparse" or (mode == "auto" and longest * 4 * ex.world < 5 * n)
    if stats is not None:
        stats["rounds"] += 1
        stats["sparse_rounds"] += int(sparse)
        b, e = ex.ranges[ex.rank]
        stats["bytes"] += 4 * longest if sparse else 4 * (e - b) + n
    if sparse:
        stride = max(longest, 1)
        with on_lib:
            send = torch.zeros(stride, dtype=torch.int32, device=dev)
            if lst is not None:
                send[: lst.numel()].copy_(lst)
            parts = [torch.empty(stride, dtype=torch.int32, device=dev) for _ in range(ex.world)]
            ex.dist.all_gather(parts, send, group=ex.group)
            recv = torch.cat(parts)
        local = engine.part_det_apply(recv, stride, cnt, ex.world, ex.rank)
        return ex.sum(local, dev)
    engine.part_det_dense()
    with on_lib:  # the exchange follows the round's kernels on the library stream
        ex.labels(lab_new)
        ex.flags(dirty)
    return engine.part_det_import()  # global count (identical on every rank)


def _det_sweep(engine, cfg, pickless, ex, lab_new, dirty, mode="auto", stats=None) -> int:
    """One deterministic partitioned sweep: speculative rounds until no rank
    holds a dirty vertex, then the commit.  Returns the
    rank-local count of changed owned vertices."""
    rnd = 0
    on_lib = _OnLibraryStream(engine, lab_new.device)
    while True:
        engine.part_det_round(cfg, pickless, rnd)  # kernels queued on the library stream
        if _det_round_exchange(engine, ex, lab_new, dirty, on_lib, mode, stats) == 0:
            break
        rnd += 1
    return engine.part_det_commit(cfg)


def lpa_run_partitioned(engine, cfg, ranges, group=None, iteration_hook=None, exchange="auto") -> PartitionedResult:
    """lpa_run (lpa.py:262-308) over the ranks of `group`; `engine` holds this
    rank's rows (Engine.part_gen_rmat / part_upload).  worker_count > 0: the
    asynchronous partitioned sweep; worker_count == 0: the deterministic one
    (bit-identical to the sequential reference)."""
    cfg.validate()
    ex = Exchange(ranges, group)
    n = engine.n
    det = cfg.worker_count == 0
    if det and not confirm_symmetric(engine, group):
        raise ValueError("the partitioned deterministic sweep needs a symmetric graph "
                         "(every arc's reverse present with the same weight); use worker_count > 0")
    engine.part_begin(cfg)
    lab, fl = engine.part_buffers()
    on_lib = _OnLibraryStream(engine, lab.device)
    if det:
        lab_new, dirty = engine.part_det_buffers()
    history = []
    stats = {"rounds": 0, "sparse_rounds": 0, "bytes": 0}
    converged = False
    for it in range(cfg.max_iterations):
        pickless = (it % cfg.pickless_gap) == 0
        if det:
            local = _det_sweep(engine, cfg, pickless, ex, lab_new, dirty, exchange, stats)
        else:
            local = engine.part_sweep(cfg, pickless)
        with on_lib:
            if not det:
                ex.labels(lab)
            ex.flags(fl)
        engine.part_end_exchange()  # library stream: after the exchange
        delta = ex.sum(local, lab.device)
        history.append(delta)
        if iteration_hook is not None:
            iteration_hook(it, pickless, lab)
        if not pickless and (delta / n if n else 0.0) < cfg.tolerance:
            converged = True
            break
    return PartitionedResult(len(history), history, converged, stats["rounds"], stats["sparse_rounds"], stats["bytes"])


def modularity_partitioned(engine, ranges, group=None) -> float:
    """metrics.py:63-74 over a partition: rank-local tallies, incident
    all-reduced, internal weight summed."""
    ex = Exchange(ranges, group)
    internal, incident, _sizes = engine.part_tally()
    ex.dist.all_reduce(incident, group=group)
    total_internal = ex.sum_f64(internal, incident.device)
    return engine.part_modularity(total_internal)
