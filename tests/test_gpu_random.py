"""Randomised differential suite: seeded random grids (shape, density, generator, sources, layer mode)
through the device path twice on the same grid, against the CPU oracle -- maps, layers_used / cause,
and the point sequences of sampled targets for both reconstruction methods, bit for bit."""
import os

import numpy as np
import pytest

from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = pytest.mark.gpu


def case(seed):
    rng = np.random.default_rng(seed)
    top = 2000 if seed % 16 == 0 else 600  # an occasional larger grid (several tile bands / chunks)
    w, h = int(rng.integers(1, top)), int(rng.integers(1, top))
    kind = int(rng.integers(0, 3))
    if kind == 0 or min(w, h) < 3:
        occ = O.random_maze(w, h, float(rng.choice([0.0, 0.1, 0.3, 0.45, 0.6])), seed)
    elif kind == 1:
        occ = O.kruskal_maze(w, h, seed)
    else:
        occ = O.city_grid(w, h, seed)
    free = int((occ == 0).sum())
    if free == 0:
        return None
    ns = int(min(free, rng.integers(1, 12)))
    src = O.sample_free_cells(occ, ns, seed)
    mode = int(rng.integers(0, 3))  # 0 auto, 1 fixed L, 2 auto with a small cap
    layers = int(rng.integers(1, 2 * max(w, h) + 3))
    cap = int(rng.integers(1, 40)) if mode == 2 else 4 * max(w, h) + 8
    return occ, src, mode, layers, cap, rng


@pytest.mark.parametrize("seed", range(int(os.environ.get("AM_RANDOM_CASES", "160"))))
def test_random_grid_matches_oracle(seed):
    c = case(1000 + seed)
    if c is None:
        pytest.skip("no free cell")
    occ, src, mode, layers, cap, rng = c
    sm = O.source_mask(occ, src)
    if mode == 1:
        ref = O.propagate(occ, sm, layers)
        want = (layers, am.FIXED)
    else:
        ref, rl, rc = O.propagate_auto(occ, sm, cap)
        want = (rl, rc)
    g = am.Grid(occ, src)
    for run in range(2):
        r = g.propagate(layers) if mode == 1 else g.propagate_auto(cap)
        got = (r.layers_used, r.cause if mode != 1 else am.FIXED)
        assert got == want, (seed, run, got, want)
        vals = g.activity()
        assert np.array_equal(vals, ref), (seed, run)
    cand = np.argwhere((occ == 0) & (ref > 0))
    if len(cand):
        pick = cand[rng.integers(0, len(cand), size=min(6, len(cand)))].astype(np.uint32)
        for method in (am.EUCLIDEAN, am.SIMPLE):
            res = g.paths(pick, method, seed=seed)
            for (st, pts), t in zip(res, pick):
                if method == am.EUCLIDEAN:
                    ost, opts = O.reconstruct_euclidean(occ, sm, ref, t)
                else:
                    ost, opts = O.reconstruct_simple(occ, sm, ref, t, seed)
                assert st == ost == 0, (seed, method, tuple(t))
                assert np.array_equal(pts, opts), (seed, method, tuple(t))
    g.close()


@pytest.mark.parametrize("seed", range(int(os.environ.get("AM_RANDOM_CASES", "160")) // 4))
def test_random_slabs_and_batches_match_oracle(seed):
    rng = np.random.default_rng(5000 + seed)
    w, h = int(rng.integers(8, 700)), int(rng.integers(40, 900))
    occ = O.random_maze(w, h, float(rng.choice([0.0, 0.2, 0.35, 0.5])), seed)
    if (occ == 0).sum() < 4:
        pytest.skip("too few free cells")
    src = O.sample_free_cells(occ, int(rng.integers(1, 6)), seed)
    sm = O.source_mask(occ, src)
    cap = 4 * max(w, h) + 8
    ref, rl, rc = O.propagate_auto(occ, sm, cap)
    # row slabs: random cut count, cuts from the library's rule or random (>= K rows each)
    n = int(rng.integers(2, 6))
    if h < 8 * n:
        n = 2
    cuts = sorted(set([0, h] + [int(x) for x in rng.choice(np.arange(8, h - 7), size=n - 1, replace=False)]))
    if any(b - a < 8 for a, b in zip(cuts, cuts[1:])):
        cuts = [0, h // 2, h]
    slabs = [am.Grid.slab(occ, src, a, b) for a, b in zip(cuts, cuts[1:])]
    full = am.Grid(occ, src)
    for run in range(2):
        r = am.slabs_propagate(slabs, 0, cap)
        assert (r.layers_used, r.cause) == (rl, rc), (seed, run, cuts)
        am.slabs_gather(slabs, full)
        assert np.array_equal(full.activity(), ref), (seed, run, cuts)
    for x in slabs + [full]:
        x.close()
    # small-maze batch of random size
    mw, mh, nb = int(rng.integers(4, 90)), int(rng.integers(4, 90)), int(rng.integers(1, 40))
    mazes = np.stack([O.random_maze(mw, mh, 0.3, 7000 + seed * 64 + i) for i in range(nb)])
    keep = [i for i in range(nb) if (mazes[i] == 0).sum() > 0]
    mazes = mazes[keep]
    if len(mazes) == 0:
        return
    msrc = [O.sample_free_cells(m, 1, seed + i) for i, m in enumerate(mazes)]
    b = am.Batch(mazes, msrc)
    used, cause, _ = b.propagate(auto_cap=512)
    maps = b.activity()
    for i, m in enumerate(mazes):
        mref, ml, mc = O.propagate_auto(m, O.source_mask(m, msrc[i]), 512)
        assert (int(used[i]), int(cause[i])) == (ml, mc), (seed, i)
        assert np.array_equal(maps[i], mref), (seed, i)
    b.close()
