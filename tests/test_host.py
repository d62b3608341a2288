"""CPU-only checks of the host side: the C ABI library loads and exports
every symbol include/slpa.h declares, the Python mirror of LpaConfig /
aux_memory_estimate matches the reference, and the product fails loudly
(no CPU fallback) when no GPU is present."""

import ctypes
import os
import re

import numpy as np
import pytest

from golden_io import Golden

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "slpa.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(slpa_[a-z0-9_]+)\s*\(", src)) - {"slpa_hook_fn"})


@pytest.fixture(scope="module")
def lib():
    from paper_2411_19901_b200.build import build
    from paper_2411_19901_b200 import _lib
    build()
    return _lib.load_library()


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_python_signatures_cover_header(lib):
    from paper_2411_19901_b200._lib import SIGNATURES
    assert set(header_symbols()) == set(SIGNATURES)


def test_library_is_sm100a(lib):
    from paper_2411_19901_b200._lib import LIB_PATH
    out = os.popen(f"cuobjdump --list-elf {LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_version_string(lib):
    assert b"sm_100a" in lib.slpa_version()


def test_aux_memory_c_abi_matches_reference_formula(lib):
    from paper_2411_19901_b200._lib import SlpaConfig
    for variant, expect in ((2, 2088), (1, 296), (0, 104)):  # test_lpa.py:434-438 (two 4-cliques)
        c = SlpaConfig(variant, 0, 8, 8, 0.05, 20, 128, 32, 0, 0)
        assert lib.slpa_aux_memory_estimate(8, 4, ctypes.byref(c)) == expect


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly(lib):
    import paper_2411_19901_b200 as slpa
    with pytest.raises(RuntimeError):
        slpa.Engine(0)


class TestConfig:
    """test_lpa.py:48-77 restated against the drop-in."""

    def test_defaults(self):
        from paper_2411_19901_b200 import LpaConfig
        cfg = LpaConfig()
        assert (cfg.variant, cfg.scan_mode, cfg.sketch_slots, cfg.pickless_gap, cfg.tolerance,
                cfg.max_iterations, cfg.degree_threshold, cfg.partial_groups, cfg.worker_count,
                cfg.shared_sketch) == ("mg", "single", 8, 8, 0.05, 20, 128, 32, 0, False)

    @pytest.mark.parametrize("field,value", [
        ("variant", "fast"), ("scan_mode", "triple"), ("sketch_slots", 0), ("pickless_gap", 0),
        ("tolerance", 0.0), ("tolerance", 1.5), ("max_iterations", 0), ("degree_threshold", 0),
        ("partial_groups", 0), ("worker_count", -1)])
    def test_validation_rejects_bad_fields(self, field, value):
        from paper_2411_19901_b200 import LpaConfig
        with pytest.raises(ValueError):
            LpaConfig(**{field: value}).validate()


def test_aux_memory_matches_golden():
    from paper_2411_19901_b200 import LpaConfig, aux_memory_estimate
    G = Golden()
    for name in G.names("run")[:200]:
        g = G.graph(name)
        cfg = G.cfg(name, LpaConfig)
        assert aux_memory_estimate(g, cfg) == G.meta(name)["aux_bytes"]


def test_graph_container_validation():
    from paper_2411_19901_b200 import Graph
    g = Graph([0, 1, 2], [1, 0], np.array([1.0, 1.0], dtype=np.float32))
    assert g.num_vertices == 2 and g.num_arcs == 2
    assert not g.offsets.flags.writeable
    with pytest.raises(ValueError):
        Graph([1, 2], [0], [1.0])
    with pytest.raises(ValueError):
        Graph([0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        Graph([0, 1], [5], [1.0])
    with pytest.raises(ValueError):
        Graph([0, 1], [0], [0.0])


def test_oracle_verify_sweep_detects_corruption(oracle):
    g = oracle.rmat(11, seed=5)
    from types import SimpleNamespace
    cfg = SimpleNamespace(variant="mg", scan_mode="single", sketch_slots=8, pickless_gap=8, tolerance=0.05,
                          max_iterations=20, degree_threshold=128, partial_groups=32, worker_count=0,
                          shared_sketch=False)
    n = g.num_vertices
    L = np.arange(n, dtype=np.int32)
    F = np.ones(n, dtype=np.uint8)
    for it in range(3):
        L0, F0 = L.copy(), F.copy()
        oracle.lpa_move(g, L, F, cfg, it == 0)
        bad, first = oracle.verify_sweep(g, L0, F0, L, F, cfg, it == 0)
        assert bad == 0
    L0, F0 = L.copy(), F.copy()
    oracle.lpa_move(g, L, F, cfg, False)
    changed = np.flatnonzero(L != L0)
    if changed.size:
        L2 = L.copy()
        v = changed[0]
        L2[v] = L0[v]
        bad, first = oracle.verify_sweep(g, L0, F0, L2, F, cfg, False)
        assert bad >= 1
