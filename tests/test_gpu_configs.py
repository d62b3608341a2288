"""BASELINE configs[2] and configs[3] at full size, through the same
size-independent checks as tests/test_gpu_scale.py (configs[1]):

* configs[2]: nuBM-LPA and nuMG8-LPA on a 4899 x 4899 4-neighbour grid
  (24,000,201 vertices, degree <= 4, permuted ids) -- the low-degree
  lane-per-vertex path only;
* configs[3]: nuMG8-LPA on a k-mer-like graph of 200,000,000 vertices
  (average degree ~2) -- the memory-footprint stress case.

Each GPU sweep is checked vertex by vertex (oracle.verify_sweep on an exact
prefix plus random samples: v's output depends only on the end-of-sweep
labels of lower vertices and the start-of-sweep labels of higher ones), and
the deterministic lpa_run must reproduce the verified sweeps.  Peak device
memory per vertex is recorded against the reference's O(|V|) model.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _verify_sweeps(slpa, eng, g, oracle, cfg, sweeps=2, seed=3):
    n = g.num_vertices
    rng = np.random.default_rng(seed)
    labels = np.arange(n, dtype=np.int32)
    flags = np.ones(n, dtype=bool)
    deltas = []
    for it in range(sweeps):
        pickless = it % cfg.pickless_gap == 0
        L0, F0 = labels.copy(), flags.copy()
        d = eng.move(cfg, labels, flags, pickless)
        deltas.append(d)
        assert d == int(np.count_nonzero(labels != L0))
        sample = np.concatenate([np.arange(min(n, 20000)), rng.integers(0, n, 200000)])
        bad, first = oracle.verify_sweep(g, L0, F0, labels, flags, cfg, pickless, sample)
        assert bad == 0, f"sweep {it}: {bad} mismatching vertices, first {first}"
    out, iters, delta, conv = eng.run(cfg)
    assert delta[:sweeps] == deltas
    return out, iters, delta


@pytest.mark.parametrize("variant", ["bm", "mg"])
def test_config2_grid_full_size(oracle, variant):
    import paper_2411_19901_b200 as slpa
    from golden_io import GoldenGraph
    eng = slpa.Engine(0)
    eng.gen_grid(4899, 4899, permute=True)
    assert eng.n == 24_000_201
    g = GoldenGraph(*eng.download())
    assert int(np.diff(g.offsets).max()) <= 4
    out, iters, delta = _verify_sweeps(slpa, eng, g, oracle, slpa.LpaConfig(variant=variant))
    q = eng.tally(out, want_arrays=False)[0]
    assert q == pytest.approx(oracle.modularity(g, out), abs=1e-9)
    eng.close()


def test_config3_kmer_200m(oracle):
    import paper_2411_19901_b200 as slpa
    from golden_io import GoldenGraph
    eng = slpa.Engine(0)
    eng.gen_kmer(200_000_000, seed=3)
    assert eng.n == 200_000_000
    g = GoldenGraph(*eng.download())
    cfg = slpa.LpaConfig()
    out, iters, delta = _verify_sweeps(slpa, eng, g, oracle, cfg, sweeps=2)
    st = eng.stats()
    # engine state beyond the CSR stays O(|V|): a few tens of bytes per vertex
    assert (st["device_bytes"] - st["graph_bytes"]) / eng.n < 64
    eng.close()
