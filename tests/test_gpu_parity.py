"""GPU parity suite: the CUDA path through the C ABI vs the CPU oracle, bit-exact.

Integer work, so the bar is exact equality of every activity value, of
layers_used / termination cause, and of every path point."""
import numpy as np
import pytest

from tests.kat_runner import load_kats, run_kat
from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def impl():
    from tests.product_adapter import ProductImpl

    return ProductImpl()


@pytest.mark.parametrize("kat", load_kats(), ids=lambda k: k["name"])
def test_spec_kat_on_device(impl, kat):
    assert run_kat(impl, kat) in (None, "skip")


SHAPES = [(1, 1), (1, 300), (300, 1), (7, 5), (37, 1000), (1000, 37), (241, 239), (255, 257), (513, 130),
          (129, 700), (2000, 64),
          # active-tile geometry edges: 112-column tile bands, 32-row chunks
          (112, 32), (113, 33), (224, 31), (225, 64), (336, 65), (111, 96)]


@pytest.mark.parametrize("w,h", SHAPES)
def test_fixed_layers_match_oracle(w, h):
    for seed, dens, ns in [(1, 0.0, 1), (2, 0.3, 3), (3, 0.45, 9)]:
        occ = O.random_maze(w, h, dens, seed)
        if (occ == 0).sum() < ns:
            continue
        src = O.sample_free_cells(occ, ns, seed)
        sm = O.source_mask(occ, src)
        for L in (1, 2, 7, 8, 9, 16, 17, 40, 2 * max(w, h) + 3):
            ref = O.propagate(occ, sm, L, threads=8)
            got = am.propagate(occ, src, L)
            assert np.array_equal(got, ref), (w, h, seed, L, np.argwhere(got != ref)[:5])


def test_iterative_mode_and_sentinel_kernel():
    occ = O.random_maze(300, 211, 0.3, 5)
    src = O.sample_free_cells(occ, 4, 5)
    sm = O.source_mask(occ, src)
    for L in (1, 9, 33):
        ref = O.propagate(occ, sm, L)
        assert np.array_equal(am.propagate(occ, src, L, mode=am.ITERATIVE), ref)
        assert np.array_equal(am.propagate_reference(occ, src, L), ref)


def test_propagate_layer_arbitrary_input():
    rng = np.random.default_rng(0)
    occ = O.random_maze(130, 77, 0.3, 9)
    src = O.sample_free_cells(occ, 3, 9)
    sm = O.source_mask(occ, src)
    a = rng.integers(0, 2**32, size=occ.shape, dtype=np.uint64).astype(np.uint32)
    a[occ != 0] = 0
    assert np.array_equal(am.propagate_layer(a, occ, src), O.propagate_layer(occ, sm, a))


@pytest.mark.parametrize("w,h", [(64, 64), (300, 200), (513, 257), (1000, 37), (37, 1000), (1024, 1024)])
def test_auto_matches_oracle(w, h):
    for seed, dens, ns in [(11, 0.0, 1), (12, 0.3, 1), (13, 0.45, 5), (14, 0.6, 2), (15, 0.3, 9)]:
        occ = O.random_maze(w, h, dens, seed)
        src = O.sample_free_cells(occ, ns, seed)
        sm = O.source_mask(occ, src)
        for cap in (1, 5, 8, 9, 37, 4 * max(w, h)):
            ref, rl, rc = O.propagate_auto(occ, sm, cap, threads=8)
            got, gl, gc = am.propagate_auto(occ, src, cap)
            assert (gl, gc) == (rl, rc), (w, h, seed, cap, gl, gc, rl, rc)
            assert np.array_equal(got, ref), (w, h, seed, cap)


def test_auto_all_sources_and_isolated_source():
    occ = np.zeros((20, 30), np.uint8)
    src = np.argwhere(occ == 0).astype(np.uint32)  # every free cell is a source
    got, gl, gc = am.propagate_auto(occ, src, 50)
    ref, rl, rc = O.propagate_auto(occ, O.source_mask(occ, src), 50)
    assert (gl, gc) == (rl, rc) == (1, O.FILLED) and np.array_equal(got, ref)
    occ = np.ones((9, 9), np.uint8)
    occ[4, 4] = 0
    occ[0, 0] = 0
    got, gl, gc = am.propagate_auto(occ, [[4, 4]], 50)
    ref, rl, rc = O.propagate_auto(occ, O.source_mask(occ, np.array([[4, 4]], np.uint32)), 50)
    assert (gl, gc) == (rl, rc) == (1, O.STALLED) and np.array_equal(got, ref)


def test_paths_match_oracle():
    occ = O.random_maze(700, 500, 0.3, 21)
    src = O.sample_free_cells(occ, 5, 21)
    sm = O.source_mask(occ, src)
    g = am.Grid(occ, src)
    r = g.propagate_auto(4 * 700)
    amap = g.activity()
    ref, rl, _ = O.propagate_auto(occ, sm, 4 * 700, threads=8)
    assert r.layers_used == rl and np.array_equal(amap, ref)
    tg = O.sample_free_cells(occ, 200, 22, exclude=sm)
    tg = np.concatenate([tg, src[:1], np.array([[0, 0], [499, 699]], np.uint32)])
    for method in (am.EUCLIDEAN, am.SIMPLE):
        for seed in ((0,) if method == am.EUCLIDEAN else (0, 1, 2, 3, 4)):
            res = g.paths(tg, method, seed)
            for (st, pts), t in zip(res, tg):
                if method == am.SIMPLE:
                    ost, opts = O.reconstruct_simple(occ, sm, ref, t, seed)
                else:
                    ost, opts = O.reconstruct_euclidean(occ, sm, ref, t)
                assert st == ost, (t, st, ost)
                if st == 0:
                    assert np.array_equal(pts, opts), (t, method, seed)
    g.close()


def test_path_errors():
    occ = np.zeros((9, 9), np.uint8)
    occ[2, 2] = 1
    g = am.Grid(occ, [[0, 0]])
    g.propagate(3)
    res = g.paths([[2, 2], [8, 8], [9, 0], [0, 0], [1, 1]], am.EUCLIDEAN)
    assert [s for s, _ in res] == [am.EINVAL, am.EUNCOVERED, am.EINVAL, am.OK, am.OK]
    assert res[3][1].tolist() == [[0, 0]]
    with pytest.raises(am.UncoveredTargetError):
        am.reconstruct_euclidean(am.propagate(occ, [[0, 0]], 1), occ, [[0, 0]], [8, 8])
    with pytest.raises(am.InvalidInputError):
        am.Grid(occ, [[2, 2]])
    with pytest.raises(am.InvalidInputError):
        am.Grid(occ, [[9, 9]])
    g.close()


def test_promotion_to_32bit_cells():
    """A serpentine longer than the 16-bit range: auto mode promotes mid-run, exactly."""
    occ = O.comb_maze(330, 200)  # corridor ~ 330*100 cells > 32767
    src = np.array([[0, 329]], np.uint32)
    sm = O.source_mask(occ, src)
    g = am.Grid(occ, src)
    r = g.propagate_auto(200_000)
    hops = O.bfs_multi_source(occ, sm)
    ecc = int(hops[hops != O.UNREACH].max())
    assert ecc > 32767 and r.cell_bits == 32
    assert (r.layers_used, r.cause) == (ecc, O.FILLED)
    vals = g.activity()
    bad, _ = O.check_activity(occ, vals, hops, r.layers_used)
    assert bad == 0
    # paths on the 32-bit map (the 32-bit walk), both methods, against the oracle on the downloaded map
    far = np.argwhere(hops == ecc)[:1]
    mid = np.argwhere((hops > 16000) & (hops < 16010))[:2]
    tg = np.concatenate([far, mid]).astype(np.uint32)
    for method in (am.EUCLIDEAN, am.SIMPLE):
        for (st, pts), t in zip(g.paths(tg, method, seed=5), tg):
            if method == am.EUCLIDEAN:
                ost, opts = O.reconstruct_euclidean(occ, sm, vals, t)
            else:
                ost, opts = O.reconstruct_simple(occ, sm, vals, t, 5)
            assert st == ost == 0 and np.array_equal(pts, opts), (method, tuple(t))
    # the next solve on the same grid starts over in 16-bit cells and promotes again
    r2 = g.propagate_auto(200_000)
    assert (r2.layers_used, r2.cause, r2.cell_bits) == (r.layers_used, r.cause, 32)
    assert np.array_equal(g.activity(), vals)
    # fixed L beyond 16 bits starts in 32-bit cells
    occ2 = O.random_maze(64, 48, 0.2, 3)
    src2 = O.sample_free_cells(occ2, 2, 3)
    L = 40_000
    assert np.array_equal(am.propagate(occ2, src2, L), O.propagate(occ2, O.source_mask(occ2, src2), L, threads=8))
    g.close()


def test_repeat_after_download_and_mixed_calls():
    """Download reuses the idle buffer as staging; the next solve must be unaffected."""
    occ = O.random_maze(777, 333, 0.3, 8)
    src = O.sample_free_cells(occ, 3, 8)
    sm = O.source_mask(occ, src)
    g = am.Grid(occ, src)
    ref, rl, rc = O.propagate_auto(occ, sm, 5000, threads=8)
    for _ in range(3):
        r = g.propagate_auto(5000)
        assert (r.layers_used, r.cause) == (rl, rc)
        assert np.array_equal(g.activity(), ref)
    g.propagate(20)
    assert np.array_equal(g.activity(), O.propagate(occ, sm, 20))
    g.close()


def test_repeated_runs_on_one_grid_are_identical():
    """Many propagate_auto calls on the same grid (as a planner session or the bench does): every run
    equals the oracle.  Regression: lag was once added to the junk low bits of wall / padding cells,
    which grew across runs until it carried into the flag bit (intermittent wrong maps / causes)."""
    occ = O.kruskal_maze(1024, 1024, 5)
    src = O.sample_free_cells(occ, 16, 5)
    sm = O.source_mask(occ, src)
    ref, rl, rc = O.propagate_auto(occ, sm, 20000)
    g = am.Grid(occ, src)
    for run in range(24):
        r = g.propagate_auto(20000)
        assert (r.layers_used, r.cause) == (rl, rc), run
        if run % 4 == 3:
            assert np.array_equal(g.activity(), ref), run
    g.close()


def test_repeated_runs_slabs_batch_dense_are_identical():
    """The same repeated-run check for in-process row slabs, the small-maze batch and the dense sweep."""
    occ = O.kruskal_maze(512, 640, 9)
    src = O.sample_free_cells(occ, 8, 9)
    sm = O.source_mask(occ, src)
    ref, rl, rc = O.propagate_auto(occ, sm, 8000)
    H = occ.shape[0]
    cuts = [0, 192, 448, H]
    slabs = [am.Grid.slab(occ, src, cuts[k], cuts[k + 1]) for k in range(3)]
    full = am.Grid(occ, src)
    dctx = am.Context(0, dense=True)
    gd = am.Grid(occ, src, dctx)
    mazes = np.stack([O.random_maze(64, 64, 0.3, 300 + i) for i in range(16)])
    msrc = [O.sample_free_cells(mazes[i], 1, 400 + i) for i in range(16)]
    bref = [O.propagate_auto(mazes[i], O.source_mask(mazes[i], msrc[i]), 1024) for i in range(16)]
    b = am.Batch(mazes, msrc)
    for run in range(12):
        r = am.slabs_propagate(slabs, 0, 8000)
        assert (r.layers_used, r.cause) == (rl, rc), ("slabs", run)
        rd = gd.propagate_auto(8000)
        assert (rd.layers_used, rd.cause) == (rl, rc), ("dense", run)
        used, cause, _ = b.propagate(auto_cap=1024)
        assert [(int(u), int(c)) for u, c in zip(used, cause)] == [(x[1], x[2]) for x in bref], ("batch", run)
        if run % 4 == 3:
            am.slabs_gather(slabs, full)
            assert np.array_equal(full.activity(), ref), ("slabs map", run)
            assert np.array_equal(gd.activity(), ref), ("dense map", run)
            maps = b.activity()
            for i in range(16):
                assert np.array_equal(maps[i], bref[i][0]), ("batch map", run, i)
    for x in slabs + [full, gd]:
        x.close()
    b.close()
    dctx.close()


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("w,h", [(1031, 1033), (2081, 515), (32, 40000), (1024, 1024)])
def test_packed_occupancy_upload(w, h, pinned, monkeypatch):
    """Grids of >= 2^20 cells cross PCIe packed to 1 bit per cell (upload.cu): any nonzero byte is an
    obstacle (grid.hpp:20), ragged row ends, chunk edges; maps equal the oracle's, and the library's H2D
    byte counter shows the packed size.  From pinned memory the first rows cross as raw bytes and are
    packed on the device beside the host workers (the split must not show in the maps; AM_RAW_SHARE is
    read per upload)."""
    monkeypatch.setenv("AM_RAW_SHARE", "20")
    rng = np.random.default_rng(w + h)
    occ = O.random_maze(w, h, 0.35, w)
    vals = rng.integers(1, 256, size=occ.shape, dtype=np.uint8)
    occ_multi = np.where(occ != 0, vals, 0).astype(np.uint8)  # obstacles as arbitrary nonzero bytes
    if pinned:
        import torch

        occ_multi = torch.from_numpy(occ_multi).pin_memory().numpy()
    src = O.sample_free_cells(occ, 5, 3)
    sm = O.source_mask(occ, src)
    ctx = am.Context(0)
    try:
        b0 = ctx.h2d_bytes()
        g = am.Grid(occ_multi, src, ctx)
        pw = (w + 31) // 32
        raw = h * 20 // 100 if pinned else 0
        assert ctx.h2d_bytes() - b0 == raw * w + (h - raw) * pw * 4 + src.nbytes
        for L in (5, 64):
            g.propagate(L)
            assert np.array_equal(g.activity(), O.propagate(occ, sm, L, threads=8)), (w, h, L)
        r = g.propagate_auto(4 * max(w, h))
        hops = O.bfs_multi_source(occ, sm)
        assert O.check_activity(occ, g.activity(), hops, r.layers_used)[0] == 0
        g.close()
    finally:
        ctx.close()


def test_map_stream_ordering():
    """The field of a bit-plane run is encoded on the context's map stream beside the path walkers; every
    reader joins it.  Interleave runs, walks and downloads on two grids of one context and check each map
    against the oracle (a missing join shows up as a stale or half-encoded field)."""
    ctx = am.Context(0)
    try:
        grids = []
        for seed, (w, h) in enumerate([(1500, 900), (700, 1300)]):
            occ = O.random_maze(w, h, 0.35, 40 + seed)
            src = O.sample_free_cells(occ, 4, 41 + seed)
            tgt = O.sample_free_cells(occ, 30, 42 + seed, exclude=src)
            grids.append((occ, src, O.source_mask(occ, src), tgt, am.Grid(occ, src, ctx)))
        for L in (9, 300, 64):
            for occ, src, sm, tgt, g in grids:
                g.propagate(L)
            for occ, src, sm, tgt, g in reversed(grids):
                g.trace(tgt, am.EUCLIDEAN)  # joins after its launch
            for occ, src, sm, tgt, g in grids:
                assert np.array_equal(g.activity(), O.propagate(occ, sm, L, threads=8)), L
        occ, src, sm, tgt, g = grids[0]
        r = g.propagate_auto(4000)
        r2 = g.propagate_auto(4000)  # the second run starts while the first run's encoding may be in flight
        assert (r.layers_used, r.cause) == (r2.layers_used, r2.cause)
        hops = O.bfs_multi_source(occ, sm)
        assert O.check_activity(occ, g.activity(), hops, r2.layers_used)[0] == 0
        for *_, g in grids:
            g.close()
    finally:
        ctx.close()


@pytest.mark.parametrize("run_max", ["off", "1", "12", "60", "400"])
def test_cluster_stretches_match_oracle(run_max, monkeypatch):
    """Light stretches (k_bits_run: one thread-block cluster runs block after block while few tiles are
    listed) entered from the start, left when the front grows, re-entered in the tail: forced thresholds
    (AM_BITS_RUN_MAX, read per run) give every transition pattern.  Fixed-L maps equal the oracle; auto
    runs match the BFS law and the BFS-predicted outcome (tests/test_gpu_scale.py)."""
    from tests.test_gpu_scale import predicted_auto

    if run_max == "off":
        monkeypatch.setenv("AM_BITS_RUN", "0")
    else:
        monkeypatch.setenv("AM_BITS_RUN_MAX", run_max)
    ctx = am.Context(0)
    try:
        for w, h, dens, ns, seed in [(2000, 1500, 0.3, 3, 61), (1500, 2100, 0.45, 40, 62), (4096, 300, 0.2, 1, 63)]:
            occ = O.random_maze(w, h, dens, seed)
            src = O.sample_free_cells(occ, ns, seed)
            sm = O.source_mask(occ, src)
            g = am.Grid(occ, src, ctx)
            for L in (16, 100, 333):
                g.propagate(L)
                assert np.array_equal(g.activity(), O.propagate(occ, sm, L, threads=8)), (w, h, L, run_max)
            hops = O.bfs_multi_source(occ, sm)
            for cap in (48, 4 * max(w, h)):
                r = g.propagate_auto(cap)
                assert (r.layers_used, r.cause) == predicted_auto(occ, hops, cap), (w, h, cap, run_max)
                assert O.check_activity(occ, g.activity(), hops, r.layers_used)[0] == 0, (w, h, cap, run_max)
            g.close()
    finally:
        ctx.close()


def test_cluster_stretch_thresholds_sweep(monkeypatch):
    """Many stretch thresholds on small grids whose propagation ends in light blocks: every entry / exit /
    re-entry point of the cluster stretches must give the BFS-predicted outcome and a law-abiding map
    (a stretch re-entered right at the fixed point must not see the previous stretch's fixed-point words)."""
    from tests.test_gpu_scale import predicted_auto

    ctx = am.Context(0)
    try:
        for seed in range(4):
            occ = O.random_maze(700, 500, 0.3 + 0.05 * seed, 70 + seed)
            src = O.sample_free_cells(occ, 1 + 3 * seed, 71 + seed)
            sm = O.source_mask(occ, src)
            hops = O.bfs_multi_source(occ, sm)
            want = predicted_auto(occ, hops, 4000)
            g = am.Grid(occ, src, ctx)
            for run_max in ("0", "1", "2", "3", "5", "8", "13", "21", "34", "55", "89"):
                monkeypatch.setenv("AM_BITS_RUN_MAX", run_max)
                r = g.propagate_auto(4000)
                assert (r.layers_used, r.cause) == want, (seed, run_max, r.layers_used, r.cause, want)
                assert O.check_activity(occ, g.activity(), hops, r.layers_used)[0] == 0, (seed, run_max)
            g.close()
    finally:
        ctx.close()
