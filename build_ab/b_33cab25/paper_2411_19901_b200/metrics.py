"""Drop-in for sketchlpa/metrics.py: modularity and community tallies,
computed by the device tally kernel (slpa_metrics.cu)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import default_engine


@dataclass
class CommunityStats:
    """metrics.py:18-31."""

    num_communities: int
    sizes: np.ndarray
    internal_weight: np.ndarray
    incident_weight: np.ndarray


def _labels_checked(g, labels):
    labels = np.asarray(labels)
    if labels.shape != (g.num_vertices,):  # metrics.py:36-37
        raise ValueError("labels must have one entry per vertex")
    n = g.num_vertices
    if labels.size and (labels.min() < 0 or labels.max() >= n):  # metrics.py:39-40
        raise ValueError("label out of range")
    return np.ascontiguousarray(labels, dtype=np.int32)


def community_stats(g, labels, *, engine=None) -> CommunityStats:
    """metrics.py:52-60."""
    labels = _labels_checked(g, labels)
    eng = engine or default_engine()
    eng.upload(g)
    _, nc, sizes, internal, incident = eng.tally(labels, want_arrays=True)
    return CommunityStats(num_communities=int(nc), sizes=sizes, internal_weight=internal,
                          incident_weight=incident)


def modularity(g, labels, *, engine=None) -> float:
    """metrics.py:63-74; ValueError on a graph with no arc weight."""
    labels = _labels_checked(g, labels)
    eng = engine or default_engine()
    eng.upload(g)
    q, _, _, _, _ = eng.tally(labels, want_arrays=False)
    if q is None:
        raise ValueError("modularity is undefined on a graph with no edges")
    return float(q)
