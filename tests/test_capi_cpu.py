"""CPU suite for the product library: it loads without a GPU, exports every
symbol the C header declares, and its host helpers agree with the oracle."""
import os
import re

import numpy as np
import pytest

from tests.oracle_adapter import O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
am = pytest.importorskip("paper_2004_00540_b200")


def declared_symbols():
    with open(os.path.join(ROOT, "include", "actmap_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(am_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = am.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_generators_match_oracle():
    for (w, h, d, s) in [(64, 64, 0.3, 42), (100, 37, 0.45, 1), (5, 5, 0.0, 3), (333, 222, 0.4, 4)]:
        assert np.array_equal(am.random_maze(w, h, d, s), O.random_maze(w, h, d, s))
    for (w, h) in [(5, 5), (2, 2), (9, 9), (12, 7), (7, 12)]:
        assert np.array_equal(am.comb_maze(w, h), O.comb_maze(w, h))
    with pytest.raises(am.InvalidInputError):
        am.random_maze(10, 10, 1.0, 0)
    with pytest.raises(am.InvalidInputError):
        am.comb_maze(1, 5)


def test_straighten_and_metrics_match_oracle():
    rng = np.random.default_rng(1)
    occ = (rng.random((80, 80)) < 0.3).astype(np.uint8)
    for _ in range(100):
        p = [(40, 40)]
        for _ in range(60):
            dr, dc = rng.integers(-1, 2, 2)
            if dr == 0 and dc == 0:
                dr = 1
            p.append((min(79, max(0, p[-1][0] + dr)), min(79, max(0, p[-1][1] + dc))))
        p = np.array(p, np.uint32)
        assert np.array_equal(am.straighten(p), O.straighten(p))
        for rule in (am.STRICT, am.PERMISSIVE):
            assert np.array_equal(am.straighten(p, occ, rule), O.straighten(p, occ, rule))
        assert am.path_metrics(p) == O.path_metrics(p)


def test_layer_bound_host():
    for w, h in [(9, 9), (1, 1), (1000, 1000), (23170, 23170), (7, 300)]:
        assert am.layer_bound(w, h) == O.layer_bound(w, h)


def test_workload_generators_match_oracle():
    """am_kruskal_maze / am_city_grid (C2 / C3 workloads) reproduce the oracle's generators exactly."""
    for w, h, s in [(41, 31, 2), (512, 300, 7), (3, 3, 1), (1025, 77, 11)]:
        assert np.array_equal(am.kruskal_maze(w, h, s), O.kruskal_maze(w, h, s)), (w, h, s)
    for w, h, s in [(300, 500, 3), (1000, 700, 9), (5, 5, 1)]:
        assert np.array_equal(am.city_grid(w, h, s), O.city_grid(w, h, s)), (w, h, s)
    with pytest.raises(am.InvalidInputError):
        am.kruskal_maze(2, 10, 0)
