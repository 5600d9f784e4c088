"""CPU suite: pin the oracle against the SPEC worked examples and the
closed-form law (independent BFS), before it is trusted as the GPU checker."""
import numpy as np
import pytest

from tests.kat_runner import load_kats, run_kat
from tests.oracle_adapter import O, OracleImpl

IMPL = OracleImpl()


@pytest.mark.parametrize("kat", load_kats(), ids=lambda k: k["name"])
def test_spec_kat(kat):
    assert run_kat(IMPL, kat) in (None, "skip")


def expected_auto(occ, sm, cap):
    """P3 outcome predicted from BFS alone (independent of the stencil)."""
    hops = O.bfs_multi_source(occ, sm)
    free = occ == 0
    reach = hops != O.UNREACH
    maxd = int(hops[reach].max())
    unreachable_free = int((free & ~reach).sum())
    if unreachable_free == 0:
        lu, cause = max(1, maxd), O.FILLED
    else:
        lu, cause = maxd + 1, O.STALLED
    if lu > cap:
        lu, cause = cap, (O.FILLED if (unreachable_free == 0 and maxd <= cap) else O.CAP)
    return lu, cause


def suite(n_seeds, sizes, densities, nsrc_list):
    for seed in range(n_seeds):
        for n in sizes:
            for dens in densities:
                for ns in nsrc_list:
                    yield seed, n, dens, ns


@pytest.mark.parametrize("n", [32, 64])
def test_activity_law_random_suite(n):
    """SPEC.md:498 (acceptance 1, reduced seed count for the CPU suite)."""
    for seed, _, dens, ns in suite(6, [n], [0.0, 0.1, 0.3, 0.45], [1, 3, 9]):
        occ = O.random_maze(n, n, dens, 1000 + seed)
        src = O.sample_free_cells(occ, ns, seed)
        sm = O.source_mask(occ, src)
        hops = O.bfs_multi_source(occ, sm)
        for L in (1, n // 2, n, 2 * n):
            m = O.propagate(occ, sm, L)
            bad, _ = O.check_activity(occ, m, hops, L)
            assert bad == 0, (seed, n, dens, ns, L)


def test_mode_and_sentinel_equivalence():
    """SPEC.md:499 (acceptance 2): batched == iterative == reference, elementwise."""
    for seed in range(5):
        occ = O.random_maze(48, 40, 0.3, seed)
        sm = O.source_mask(occ, O.sample_free_cells(occ, 3, seed))
        for L in (1, 7, 64):
            a = O.propagate(occ, sm, L, O.BATCHED)
            b = O.propagate(occ, sm, L, O.ITERATIVE)
            c = O.propagate_reference(occ, sm, L)
            d = O.propagate(occ, sm, L, O.BATCHED, threads=4)
            assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)


def test_auto_matches_bfs_prediction():
    for seed in range(20):
        n = 24 + seed
        occ = O.random_maze(n, n + 3, [0.0, 0.3, 0.45, 0.55][seed % 4], seed)
        sm = O.source_mask(occ, O.sample_free_cells(occ, 1 + seed % 4, seed))
        for cap in (1, 5, 10_000):
            _, lu, cause = O.propagate_auto(occ, sm, cap)
            assert (lu, cause) == expected_auto(occ, sm, cap), (seed, cap)


def test_comb_maze_auto_equals_eccentricity():
    """SPEC.md:131,503(c): comb maze L_used equals the BFS eccentricity of the source."""
    for w, h in [(9, 9), (5, 5), (12, 7), (7, 12), (2, 2)]:
        occ = O.comb_maze(w, h)
        src = np.array([[0, w - 1]] if w >= h else [[h - 1, 0]], np.uint32)
        sm = O.source_mask(occ, src)
        hops = O.bfs_multi_source(occ, sm)
        ecc = int(hops[hops != O.UNREACH].max())
        _, lu, cause = O.propagate_auto(occ, sm, 10_000)
        assert cause == O.FILLED and lu == max(1, ecc)
        worst, _, _ = O.layer_bound(w, h)
        assert ecc <= worst  # relationship recorded, not equality


def test_paths_step_optimal_and_straighten_noop():
    """SPEC.md:500 (acceptance 3) on a reduced set; pins P1/P1'."""
    for seed in range(10):
        occ = O.random_maze(64, 64, 0.3, 77 + seed)
        src = O.sample_free_cells(occ, 2, seed)
        sm = O.source_mask(occ, src)
        m, lu, _ = O.propagate_auto(occ, sm, 512)
        hops = O.bfs_multi_source(occ, sm)
        tg = O.sample_free_cells(occ, 12, 500 + seed, exclude=sm)
        for t in tg:
            d = hops[t[0], t[1]]
            for s in range(5):
                st, p = O.reconstruct_simple(occ, sm, m, t, s)
                if d == O.UNREACH:
                    assert st == O.EUNCOVERED
                    continue
                assert st == O.OK and len(p) - 1 == d
                assert sm[p[-1][0], p[-1][1]] == 1
            st, p = O.reconstruct_euclidean(occ, sm, m, t)
            if d == O.UNREACH:
                assert st == O.EUNCOVERED
                continue
            assert st == O.OK and len(p) - 1 == d
            assert np.array_equal(O.straighten(p), p)
            assert np.array_equal(O.straighten(p, occ), p)
            diffs = np.abs(np.diff(p.astype(np.int64), axis=0))
            assert (diffs.max(axis=1) == 1).all()


def test_straighten_idempotent_and_strict_rule():
    rng = np.random.default_rng(3)
    for _ in range(50):
        # random unit-Chebyshev walk
        p = [(50, 50)]
        for _ in range(40):
            dr, dc = rng.integers(-1, 2, 2)
            if dr == 0 and dc == 0:
                dc = 1
            p.append((p[-1][0] + dr, p[-1][1] + dc))
        p = np.array(p, np.uint32)
        s1 = O.straighten(p)
        assert np.array_equal(O.straighten(s1), s1)
    # strict rule blocks squeezing between two diagonal obstacles
    occ = np.zeros((3, 3), np.uint8)
    occ[0, 1] = 1
    occ[1, 0] = 1
    path = np.array([[1, 0], [0, 0], [0, 1]], np.uint32)  # geometry only
    assert len(O.straighten(path)) == 2
    path2 = np.array([[0, 0], [1, 1]], np.uint32)
    assert len(O.straighten(path2, occ, O.STRICT)) == 2


def test_nearest_source_multi():
    """SPEC.md:502 (acceptance 5): >=30 sources, >=8 targets -> reached source is hop-nearest."""
    occ = O.random_maze(96, 96, 0.25, 5)
    src = O.sample_free_cells(occ, 30, 11)
    sm = O.source_mask(occ, src)
    m, _, _ = O.propagate_auto(occ, sm, 1000)
    hops = O.bfs_multi_source(occ, sm)
    tg = O.sample_free_cells(occ, 8, 12, exclude=sm)
    for t in tg:
        if hops[t[0], t[1]] == O.UNREACH:
            continue
        st, p = O.reconstruct_euclidean(occ, sm, m, t)
        assert st == O.OK
        d_from_t = O.bfs_from(occ, int(t[0]), int(t[1]))
        reached = p[-1]
        assert d_from_t[reached[0], reached[1]] == hops[t[0], t[1]]


def test_generators_deterministic():
    a = O.kruskal_maze(65, 65, 2)
    assert np.array_equal(a, O.kruskal_maze(65, 65, 2))
    # perfect maze: corridor cells form one 4-connected tree -> all reachable
    sm = np.zeros_like(a)
    sm[1, 1] = 1
    hops = O.bfs_multi_source(a, sm)
    assert ((a == 0) <= (hops != O.UNREACH)).all()
    c = O.city_grid(300, 200, 3)
    assert 0.2 < c.mean() < 0.9
