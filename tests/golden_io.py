"""Access to the committed golden fixtures (tests/golden/, produced by
make_golden.py from the Python reference)."""

import json
import os
from types import SimpleNamespace

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class GoldenGraph:
    __slots__ = ("num_vertices", "num_arcs", "offsets", "targets", "weights")

    def __init__(self, offsets, targets, weights):
        self.offsets = offsets
        self.targets = targets
        self.weights = weights
        self.num_vertices = int(offsets.size - 1)
        self.num_arcs = int(targets.size)

    def degree(self, i):
        return int(self.offsets[i + 1] - self.offsets[i])


class Golden:
    def __init__(self):
        with open(os.path.join(HERE, "golden_index.json")) as f:
            self.index = json.load(f)
        self._npz = {}
        self._graphs = {}

    def _arr(self, group):
        if group not in self._npz:
            self._npz[group] = np.load(os.path.join(HERE, f"golden_{group}.npz"))
        return self._npz[group]

    def names(self, kind=None, group=None):
        return sorted(k for k, v in self.index.items()
                      if (kind is None or v["kind"] == kind) and (group is None or v["group"] == group))

    def graph(self, name):
        meta = self.index[name]
        key = (meta["group"], meta["graph"])
        if key not in self._graphs:
            a = self._arr(meta["group"])
            gname = meta["graph"]
            self._graphs[key] = GoldenGraph(a[f"{gname}/offsets"], a[f"{gname}/targets"], a[f"{gname}/weights"])
        return self._graphs[key]

    def get(self, name, field):
        meta = self.index[name]
        a = self._arr(meta["group"])
        k = f"{name}/{field}"
        return a[k] if k in a.files else None

    def cfg(self, name, cls=None):
        d = dict(self.index[name]["cfg"])
        if cls is None:
            return SimpleNamespace(**d)
        return cls(**d)

    def meta(self, name):
        return self.index[name]
