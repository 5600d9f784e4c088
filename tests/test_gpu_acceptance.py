"""The reference's acceptance matrix run through the device path.

1. Activity law: >= 50 seeds x grids {32^2, 64^2, 128^2} x densities {0, 0.1, 0.3, 0.45}
   x L in {1, n/2, n, 2n} x source counts {1, 3, 9}: check_activity (oracle.hpp) against
   an independent CPU BFS reports zero violations of value(c) = max(0, L+1-d_BFS8(c)) on the DEVICE map.
2. Kernel equivalence: propagate batched, propagate iterative, propagate_reference and the
   small-grid batch entry point are elementwise identical on the same suite.
3. Step-optimality: reconstruct_simple steps == BFS hops for every covered cell of 100 random
   64x64 mazes, tie seeds 0..4 (the device walks every covered free cell).
5. Multi-source nearest assignment: >= 30 sources, >= 8 targets, every path ends at a
   geodesically nearest source.
6. Auto-L: (a) empty n x n, centre source -> floor(n/2), filled; (c) comb maze -> BFS
   eccentricity of the source.
"""
import os

import numpy as np
import pytest

from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = pytest.mark.gpu
SEEDS = int(os.environ.get("AM_ACCEPT_SEEDS", "50"))


@pytest.mark.parametrize("n", [32, 64, 128])
@pytest.mark.parametrize("density", [0.0, 0.1, 0.3, 0.45])
def test_acceptance_1_2_activity_law_and_kernel_equivalence(n, density):
    ctx = am.Context(0)
    Ls = sorted({1, n // 2, n, 2 * n})
    checked = 0
    for ns in (1, 3, 9):
        occs, srcs = [], []
        for seed in range(SEEDS):
            occ = O.random_maze(n, n, density, 10_000 * ns + 100 * seed + int(density * 100) + n)
            src = O.sample_free_cells(occ, ns, seed)
            occs.append(occ)
            srcs.append(src)
        batch = am.Batch(np.stack(occs), srcs, ctx)
        for seed, (occ, src) in enumerate(zip(occs, srcs)):
            sm = O.source_mask(occ, src)
            hops = O.bfs_multi_source(occ, sm)
            g = am.Grid(occ, src, ctx)
            for L in Ls:
                r = g.propagate(L)
                assert r.layers_used == L
                vals = g.activity()
                bad, where = O.check_activity(occ, vals, hops, L)
                assert bad == 0, (n, density, ns, seed, L, where)
                g.propagate(L, am.ITERATIVE)
                assert np.array_equal(g.activity(), vals), ("iterative", n, density, ns, seed, L)
                assert np.array_equal(am.propagate_reference(occ, src, L, ctx=ctx), vals), \
                    ("reference", n, density, ns, seed, L)
                checked += 1
            g.close()
        for L in Ls:
            used, _, _ = batch.propagate(layers=L)
            maps = batch.activity()
            assert (used == L).all()
            for seed, (occ, src) in enumerate(zip(occs, srcs)):
                sm = O.source_mask(occ, src)
                bad, where = O.check_activity(occ, maps[seed], O.bfs_multi_source(occ, sm), L)
                assert bad == 0, ("batch", n, density, ns, seed, L, where)
        batch.close()
    assert checked == 3 * SEEDS * len(Ls)
    ctx.close()


def test_acceptance_3_step_optimality():
    ctx = am.Context(0)
    walked = 0
    for m in range(100):
        occ = O.random_maze(64, 64, 0.3, 300 + m)
        src = O.sample_free_cells(occ, 1 + m % 3, m)
        sm = O.source_mask(occ, src)
        hops = O.bfs_multi_source(occ, sm)
        g = am.Grid(occ, src, ctx)
        r = g.propagate_auto(4 * 64 + 8)
        vals = g.activity()
        tg = np.argwhere((occ == 0) & (vals > 0)).astype(np.uint32)
        for seed in range(5):
            off, pts, st = g.trace(tg, am.SIMPLE, seed)
            assert (st == 0).all()
            steps = np.diff(off.astype(np.int64)) - 1
            assert np.array_equal(steps, hops[tg[:, 0], tg[:, 1]].astype(np.int64)), (m, seed)
            ends = pts[off[1:].astype(np.int64) - 1]
            assert sm[ends[:, 0], ends[:, 1]].all(), (m, seed)
            walked += len(tg)
        assert r.layers_used >= 1
        g.close()
    assert walked > 100 * 5 * 1000
    ctx.close()


def test_acceptance_5_multi_source_nearest():
    ctx = am.Context(0)
    for k in range(4):
        occ = O.random_maze(200, 160, 0.25, 900 + k)
        src = O.sample_free_cells(occ, 32 + k, 900 + k)
        sm = O.source_mask(occ, src)
        tg = O.sample_free_cells(occ, 12, 950 + k, exclude=sm)
        g = am.Grid(occ, src, ctx)
        g.propagate_auto(4 * 200)
        for method in (am.EUCLIDEAN, am.SIMPLE):
            for (st, pts), t in zip(g.paths(tg, method, 1), tg):
                if st != 0:
                    continue
                d_t = O.bfs_from(occ, int(t[0]), int(t[1]))
                d_near = min(int(d_t[s[0], s[1]]) for s in src)
                end = pts[-1]
                assert sm[end[0], end[1]] and int(d_t[end[0], end[1]]) == d_near, (k, tuple(t), method)
        g.close()
    ctx.close()


@pytest.mark.parametrize("n", [5, 9, 33])
def test_acceptance_6a_empty_grid_floor_half(n):
    occ = np.zeros((n, n), np.uint8)
    g = am.Grid(occ, np.array([[n // 2, n // 2]], np.uint32))
    r = g.propagate_auto(4 * n)
    assert (r.layers_used, r.cause) == (n // 2, am.FILLED)
    g.close()


@pytest.mark.parametrize("w,h", [(9, 9), (65, 33), (31, 200)])
def test_acceptance_6c_comb_maze_eccentricity(w, h):
    occ = O.comb_maze(w, h)
    s = (0, w - 1) if w >= h else (h - 1, 0)
    src = np.array([s], np.uint32)
    ecc = int(O.bfs_from(occ, *s)[occ == 0].max())
    g = am.Grid(occ, src)
    r = g.propagate_auto(w * h)
    assert (r.layers_used, r.cause) == (max(1, ecc), am.FILLED)
    g.close()
