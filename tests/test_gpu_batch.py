"""Small-grid batch path (config C5: many independent 256x256 mazes) vs the
oracle run maze by maze: per-maze map, layers_used, cause and paths."""
import numpy as np
import pytest

from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = pytest.mark.gpu


def make_batch(n, w, h, seed0, dens=0.3, ns=1):
    occ = np.stack([O.random_maze(w, h, dens, seed0 + i) for i in range(n)])
    src = [O.sample_free_cells(occ[i], ns, seed0 + i) for i in range(n)]
    return occ, src


def check(b, occ, src, cap, sample, method_seed=((am.EUCLIDEAN, 0), (am.SIMPLE, 2))):
    lu, cause, _ = b.propagate(auto_cap=cap)
    maps = b.activity()
    for i in sample:
        sm = O.source_mask(occ[i], src[i])
        ref, rl, rc = O.propagate_auto(occ[i], sm, cap)
        assert (lu[i], cause[i]) == (rl, rc), (i, lu[i], cause[i], rl, rc)
        assert np.array_equal(maps[i], ref), i
    tg = []
    for i in sample:
        sm = O.source_mask(occ[i], src[i])
        for t in O.sample_free_cells(occ[i], 8, 77 + i, exclude=sm):
            tg.append((i, t[0], t[1]))
    tg = np.array(tg, np.uint32)
    for method, seed in method_seed:
        off, pts, st = b.trace(tg, method, seed)
        for k, (i, r, c) in enumerate(tg):
            sm = O.source_mask(occ[i], src[i])
            if method == am.EUCLIDEAN:
                ost, opts = O.reconstruct_euclidean(occ[i], sm, maps[i], (r, c))
            else:
                ost, opts = O.reconstruct_simple(occ[i], sm, maps[i], (r, c), seed)
            assert st[k] == ost, (i, r, c)
            if ost == 0:
                assert np.array_equal(pts[off[k]:off[k + 1]], opts), (i, r, c, method)


def test_batch_small_mixed_outcomes():
    # densities up to 0.6 give stalled mazes next to filled ones; cap 40 leaves some capped
    occ = np.stack([O.random_maze(64, 48, d, 100 + i) for i, d in enumerate([0.0, 0.3, 0.45, 0.6] * 6)])
    src = [O.sample_free_cells(occ[i], 1 + i % 3, 100 + i) for i in range(len(occ))]
    b = am.Batch(occ, src)
    for cap in (40, 1000, 1):
        check(b, occ, src, cap, range(len(occ)))
    lu, cause, _ = b.propagate(layers=13)
    maps = b.activity()
    for i in range(len(occ)):
        assert lu[i] == 13 and np.array_equal(maps[i], O.propagate(occ[i], O.source_mask(occ[i], src[i]), 13))
    b.close()


def predicted_auto(occ, hops, cap):
    """propagate_auto's (L_used, cause) from the BFS alone (pin P3)."""
    reach = hops != O.UNREACH
    maxd = int(hops[reach].max())
    unreachable_free = bool(((occ == 0) & ~reach).any())
    lu, cause = (max(1, maxd), O.FILLED) if not unreachable_free else (maxd + 1, O.STALLED)
    if lu > cap:
        lu, cause = cap, (O.FILLED if (not unreachable_free and maxd <= cap) else O.CAP)
    return lu, cause


def c5_workload(n=4096):
    """config C5 exactly as bench.py runs it (bench.c5_workload): 256^2 random mazes (0.30, seeds 5000+i),
    1 source and 8 targets each"""
    import bench

    occ, src, tg, cap = bench.c5_workload(am, n)
    assert cap == 1024
    return occ, src, tg


def test_batch_c5_every_maze():
    """4096 x 256^2 (config C5): EVERY maze's map (closed-form law against a CPU BFS: all cells), L_used and
    cause (predicted from the BFS), and every one of the 32768 Euclidean paths against the oracle's
    reconstruction on the device map; a sample of mazes also against the oracle's full propagate_auto."""
    n, cap = 4096, 1024
    occ, src, tg = c5_workload(n)
    b = am.Batch(occ, src)
    lu, cause, _ = b.propagate(auto_cap=cap)
    maps = b.activity()
    for i in range(n):
        sm = O.source_mask(occ[i], src[i])
        hops = O.bfs_multi_source(occ[i], sm)
        assert (int(lu[i]), int(cause[i])) == predicted_auto(occ[i], hops, cap), i
        bad, where = O.check_activity(occ[i], maps[i], hops, int(lu[i]))
        assert bad == 0, (i, where)
    off, pts, st = b.trace(tg, am.EUCLIDEAN, 0)
    for k, (i, r, c) in enumerate(tg):
        sm = O.source_mask(occ[i], src[i])
        ost, opts = O.reconstruct_euclidean(occ[i], sm, maps[i], (r, c), cap=int(lu[i]) + 2)
        assert st[k] == ost, (i, r, c)
        if ost == 0:
            assert np.array_equal(pts[off[k]:off[k + 1]], opts), (i, r, c)
    check(b, occ, src, cap, list(range(0, n, 257)) + [n - 1])
    b.close()


def test_batch_rejects_bad_input():
    occ = np.zeros((2, 8, 8), np.uint8)
    with pytest.raises(am.InvalidInputError):
        am.Batch(occ, [np.zeros((0, 2), np.uint32), [[0, 0]]])
    occ[1, 0, 0] = 1
    with pytest.raises(am.InvalidInputError):
        am.Batch(occ, [[[1, 1]], [[0, 0]]])


@pytest.mark.parametrize("n,w,h,dens", [
    (7, 1000, 30, 0.3),   # 32 words per row: one warp per row group, 4 rows per thread
    (5, 20, 1000, 0.3),   # one word per row: 256 row groups, 4 rows per thread
    (3, 33, 257, 0.25),   # ragged words (33 columns) and rows
    (9, 256, 256, 0.0),   # empty mazes: filled at floor-ish eccentricity
    (4, 4, 4, 0.0),       # tiny mazes: 4 x 4
])
def test_batch_wave_shapes(n, w, h, dens):
    """K5 (k_batch_wave) across maze shapes: word columns 1..32, rows per thread 1..32, ragged edges."""
    occ = np.stack([O.random_maze(w, h, dens, 300 + i) for i in range(n)])
    src = [O.sample_free_cells(occ[i], 1 + i % 2, 300 + i) for i in range(n)]
    b = am.Batch(occ, src)
    cap = 4 * max(w, h) + 8
    check(b, occ, src, cap, range(n))
    lu, cause, _ = b.propagate(layers=max(1, min(w, h) // 2))
    maps = b.activity()
    for i in range(n):
        sm = O.source_mask(occ[i], src[i])
        assert np.array_equal(maps[i], O.propagate(occ[i], sm, int(lu[i]))), i
    b.close()


def test_batch_large_cap_takes_the_tile_path():
    """A cap past the 16-bit range falls back to the packed tile path (same results)."""
    occ = np.stack([O.random_maze(40, 30, 0.3, 900 + i) for i in range(6)])
    src = [O.sample_free_cells(occ[i], 1, 900 + i) for i in range(6)]
    b = am.Batch(occ, src)
    check(b, occ, src, 40000, range(6), method_seed=((am.EUCLIDEAN, 0),))
    b.close()
