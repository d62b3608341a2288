"""Patch the reference package's own entry points onto the B200 engine
(INTEGRATION.md §2 applied for real).

    import sketchlpa
    from paper_2411_19901_b200.integration import install
    install(sketchlpa)          # sketchlpa.lpa_run & co. now run on the B200

Every caller of the reference -- ``cli._cmd_run`` / ``_cmd_bench``
(cli.py:183, :236), the demos, the reference's own test-suite -- then goes
through the drop-in without a code change.  The wrappers keep the
reference's types: results come back as ``sketchlpa.LpaResult`` /
``sketchlpa.CommunityStats`` and graphs as ``sketchlpa.Graph``.

Replaced (module attribute and every ``from .x import name`` copy):

  lpa.lpa_run, lpa.lpa_move                       lpa.py:227-308
  metrics.modularity, metrics.community_stats     metrics.py:52-74
  graph.load_graph, graph.build_graph             graph.py:142-162, :310-349
  graph.write_edgelist, graph.write_matrix_market graph.py:352-375
  graph.validate_graph                            graph.py:378-403

The selectors, sketches and ``aux_memory_estimate`` stay the reference's
(per-vertex Python helpers the GPU path does not call).
"""

from __future__ import annotations

import sys

import numpy as np

from . import graph as _g
from . import graph_io as _io
from . import lpa as _lpa
from . import metrics as _m

_ORIGINALS = {}


def _wrap(ref):
    Graph = ref.graph.Graph

    def as_ref_graph(g):
        return Graph(g.offsets, g.targets, g.weights)

    def lpa_run(g, cfg=None, *, order=None, iteration_hook=None):
        if cfg is None:
            cfg = ref.lpa.LpaConfig()
        r = _lpa.lpa_run(g, cfg, order=order, iteration_hook=iteration_hook)
        return ref.lpa.LpaResult(labels=r.labels, iterations=r.iterations, delta_history=r.delta_history,
                                 converged=r.converged, aux_bytes=ref.lpa.aux_memory_estimate(g, cfg))

    def lpa_move(g, labels, unprocessed, cfg, pickless, order=None):
        return _lpa.lpa_move(g, labels, unprocessed, cfg, pickless, order=order)

    def community_stats(g, labels):
        s = _m.community_stats(g, labels)
        return ref.metrics.CommunityStats(num_communities=s.num_communities, sizes=s.sizes,
                                          internal_weight=s.internal_weight, incident_weight=s.incident_weight)

    def modularity(g, labels):
        return _m.modularity(g, labels)

    def build_graph(num_vertices, edges, weight_dtype=np.float32):
        return as_ref_graph(_g.build_graph(num_vertices, edges, weight_dtype))

    def load_graph(path, fmt=None, *, weight_dtype=np.float32, return_mapping=False):
        try:
            out = _io.load_graph(path, fmt, weight_dtype=weight_dtype, return_mapping=return_mapping)
        except _g.GraphLoadError as exc:  # the reference's exception type
            raise ref.graph.GraphLoadError(str(exc)) from None
        if return_mapping:
            return as_ref_graph(out[0]), out[1]
        return as_ref_graph(out)

    return {
        ("lpa", "lpa_run"): lpa_run,
        ("lpa", "lpa_move"): lpa_move,
        ("metrics", "community_stats"): community_stats,
        ("metrics", "modularity"): modularity,
        ("graph", "build_graph"): build_graph,
        ("graph", "load_graph"): load_graph,
        ("graph", "write_edgelist"): _io.write_edgelist,
        ("graph", "write_matrix_market"): _io.write_matrix_market,
        ("graph", "validate_graph"): _io.validate_graph,
    }


def install(ref) -> None:
    """Point ``ref`` (the imported ``sketchlpa`` package) at the B200 engine."""
    import importlib
    for sub in ("lpa", "metrics", "graph", "cli"):
        importlib.import_module(f"{ref.__name__}.{sub}")
    repl = _wrap(ref)
    mods = [m for name, m in list(sys.modules.items())
            if m is not None and (name == ref.__name__ or name.startswith(ref.__name__ + "."))]
    for (home, name), fn in repl.items():
        orig = getattr(getattr(ref, home), name)
        _ORIGINALS.setdefault((ref.__name__, home, name), orig)
        for mod in mods:  # the defining module and every module that imported the name
            if getattr(mod, name, None) is orig:
                setattr(mod, name, fn)


def uninstall(ref) -> None:
    import importlib
    for (pkg, home, name), orig in list(_ORIGINALS.items()):
        if pkg != ref.__name__:
            continue
        cur = getattr(importlib.import_module(f"{pkg}.{home}"), name)
        for mod_name, mod in list(sys.modules.items()):
            if mod is not None and (mod_name == pkg or mod_name.startswith(pkg + ".")) and \
                    getattr(mod, name, None) is cur:
                setattr(mod, name, orig)
        del _ORIGINALS[(pkg, home, name)]
