"""Drop-in for the reference engine (sketchlpa/lpa.py) on the B200.

Same names, fields, defaults, validation and return types as the
reference's ``LpaConfig`` / ``LpaResult`` / ``lpa_run`` / ``lpa_move`` /
``aux_memory_estimate`` (lpa.py:44-89, :227-333).  The work runs in
libslpa_b200.so:

* ``worker_count == 0`` (default): the deterministic GPU sweep, bit-identical
  to the reference's sequential sweep -- labels after every iteration,
  ``delta_history``, ``iterations`` and ``converged``.
* ``worker_count > 0``: the asynchronous in-place GPU sweep (the paper's
  execution model; the reference's threaded mode is its CPU analogue).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .engine import default_engine

VARIANTS = ("exact", "bm", "mg")
SCAN_MODES = ("single", "double")

_LABEL_BYTES = 4
_FLAG_BYTES = 1
_KEY_BYTES = 4


@dataclass
class LpaConfig:
    """lpa.py:44-80 -- identical fields, defaults and validation."""

    variant: str = "mg"
    scan_mode: str = "single"
    sketch_slots: int = 8
    pickless_gap: int = 8
    tolerance: float = 0.05
    max_iterations: int = 20
    degree_threshold: int = 128
    partial_groups: int = 32
    worker_count: int = 0
    shared_sketch: bool = False

    def validate(self) -> None:
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}")
        if self.scan_mode not in SCAN_MODES:
            raise ValueError(f"scan_mode must be one of {SCAN_MODES}")
        if self.sketch_slots < 1:
            raise ValueError("sketch_slots must be at least 1")
        if self.pickless_gap < 1:
            raise ValueError("pickless_gap must be at least 1")
        if not (0 < self.tolerance <= 1):
            raise ValueError("tolerance must be in (0, 1]")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.degree_threshold < 1:
            raise ValueError("degree_threshold must be at least 1")
        if self.partial_groups < 1:
            raise ValueError("partial_groups must be at least 1")
        if self.worker_count < 0:
            raise ValueError("worker_count must be non-negative")


@dataclass
class LpaResult:
    """lpa.py:83-89."""

    labels: np.ndarray
    iterations: int
    delta_history: list[int] = field(default_factory=list)
    converged: bool = False
    aux_bytes: int = 0


def _check_order(order, n):
    """lpa.py:283-288."""
    order = np.asarray(order, dtype=np.int64)
    check = np.zeros(n, dtype=bool)
    if order.size and (order.min() < 0 or order.max() >= n):
        raise ValueError("order must be a permutation of all vertex ids")
    check[order] = True
    if order.size != n or not check.all():
        raise ValueError("order must be a permutation of all vertex ids")
    return order


def lpa_run(g, cfg: LpaConfig = None, *, order=None, iteration_hook=None, engine=None) -> LpaResult:
    """Run label propagation to convergence or the iteration cap (lpa.py:262-308).

    ``iteration_hook(iteration, pickless, labels)`` is called after every
    sweep with a host copy of the labels.  ``engine`` optionally supplies a
    resident-graph :class:`Engine` (default: a cached per-thread one; the
    graph is uploaded on every call, like the reference reads its Graph).
    """
    if cfg is None:
        cfg = LpaConfig()
    cfg.validate()
    n = int(g.num_vertices)
    if order is not None:
        order = _check_order(order, n)
    eng = engine or default_engine()
    eng.upload(g, order=order)
    labels, iters, history, converged = eng.run(cfg, hook=iteration_hook)
    return LpaResult(
        labels=labels,
        iterations=iters,
        delta_history=history,
        converged=converged,
        aux_bytes=aux_memory_estimate(g, cfg),
    )


def lpa_move(g, labels, unprocessed, cfg: LpaConfig, pickless: bool, order=None, *, engine=None) -> int:
    """One propagation sweep on caller state (lpa.py:227-259).

    Mutates ``labels`` (int32) and ``unprocessed`` (bool) in place and
    returns the number of vertices that changed.
    """
    n = int(g.num_vertices)
    if order is not None:
        order = _check_order(order, n)
    eng = engine or default_engine()
    eng.upload(g, order=order)
    return eng.move(cfg, labels, unprocessed, pickless)


def aux_memory_estimate(g, cfg: LpaConfig) -> int:
    """lpa.py:311-333 -- the reference's deterministic model (not the
    measured device footprint; see Engine.stats()['device_bytes'])."""
    cfg.validate()
    n = g.num_vertices
    value_bytes = np.dtype(g.weights.dtype).itemsize
    workers = max(cfg.worker_count, 1)
    base = n * (_LABEL_BYTES + _FLAG_BYTES)
    if cfg.variant == "exact":
        per_worker = n * (_KEY_BYTES + value_bytes)
    elif cfg.variant == "mg":
        per_worker = cfg.partial_groups * cfg.sketch_slots * (_KEY_BYTES + value_bytes)
    else:
        per_worker = cfg.partial_groups * (_KEY_BYTES + value_bytes)
    return base + workers * per_worker
