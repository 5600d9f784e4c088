"""Row-slab decomposition on the device vs the oracle.

One GPU, n in-process slabs (the same halo-exchange / flag-reduction driver
the NCCL path uses; only the transport differs): the assembled map,
layers_used / cause and the paths traced on the gathered map must be
identical to the single-grid oracle results."""
import numpy as np
import pytest

from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = pytest.mark.gpu


def split(h, n):
    return [(h * r // n, h * (r + 1) // n) for r in range(n)]


def make_slabs(occ, src, n, ctx):
    return [am.Grid.slab(occ, src, a, b, ctx) for a, b in split(occ.shape[0], n)]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7])
def test_slabs_auto_match_oracle(n):
    ctx = am.default_context()
    for seed, (w, h), dens, ns in [(1, (300, 200), 0.3, 3), (2, (517, 611), 0.4, 5), (3, (64, 129), 0.0, 1),
                                   (4, (1000, 333), 0.55, 4)]:
        occ = O.random_maze(w, h, dens, seed)
        src = O.sample_free_cells(occ, ns, seed)
        sm = O.source_mask(occ, src)
        slabs = make_slabs(occ, src, n, ctx)
        for cap in (3, 9, 4 * max(w, h)):
            r = am.slabs_propagate(slabs, auto_cap=cap)
            ref, rl, rc = O.propagate_auto(occ, sm, cap, threads=8)
            assert (r.layers_used, r.cause) == (rl, rc), (n, seed, cap)
            got = np.concatenate([s.activity() for s in slabs])
            assert np.array_equal(got, ref), (n, seed, cap)
        for L in (1, 8, 17):
            am.slabs_propagate(slabs, layers=L)
            got = np.concatenate([s.activity() for s in slabs])
            assert np.array_equal(got, O.propagate(occ, sm, L)), (n, seed, L)
        for s in slabs:
            s.close()


def aligned_split(h, n, tile_rows=32):
    """am_comm_slab_rows' cuts: tile-chunk multiples, so the slabs run with active-tile skipping."""
    def cut(k):
        b = h * k // n
        if 0 < k < n and h >= 2 * tile_rows * n:
            b = (b + tile_rows // 2) // tile_rows * tile_rows
        return b
    return [(cut(r), cut(r + 1)) for r in range(n)]


@pytest.mark.parametrize("n", [2, 3, 5])
def test_tile_slabs_match_oracle_and_dense(n):
    """Slabs meeting at tile-chunk boundaries use active tiles with boundary-row exchange + halo scan."""
    ctx, dctx = am.default_context(), am.Context(0, dense=True)
    for seed, (w, h), dens, ns in [(5, (300, 400), 0.3, 4), (6, (517, 700), 0.45, 6), (7, (240, 320), 0.0, 2),
                                   (8, (1100, 1024), 0.4, 9)]:
        occ = O.random_maze(w, h, dens, seed)
        # sources right at the slab boundaries too
        cuts = [a for a, _ in aligned_split(h, n)][1:]
        src = np.concatenate([O.sample_free_cells(occ, ns, seed),
                              np.array([[c, x] for c in cuts for x in range(0, w, 97) if occ[c, x] == 0][:6],
                                       np.uint32).reshape(-1, 2)])
        src = np.unique(src, axis=0)
        sm = O.source_mask(occ, src)
        slabs = [am.Grid.slab(occ, src, a, b, ctx) for a, b in aligned_split(h, n)]
        dslabs = [am.Grid.slab(occ, src, a, b, dctx) for a, b in aligned_split(h, n)]
        for cap in (5, 8, 4 * max(w, h)):
            r = am.slabs_propagate(slabs, auto_cap=cap)
            assert r.block_launches == 0 or r.tiles_total > 0, "tile mode expected for aligned slabs"
            ref, rl, rc = O.propagate_auto(occ, sm, cap, threads=8)
            assert (r.layers_used, r.cause) == (rl, rc), (n, seed, cap)
            got = np.concatenate([s.activity() for s in slabs])
            assert np.array_equal(got, ref), (n, seed, cap)
            rd = am.slabs_propagate(dslabs, auto_cap=cap)
            assert rd.tiles_total == 0 and (rd.layers_used, rd.cause) == (rl, rc)
        for L in (8, 24, 3 * max(w, h) // 2):
            am.slabs_propagate(slabs, layers=L)
            got = np.concatenate([s.activity() for s in slabs])
            assert np.array_equal(got, O.propagate(occ, sm, L)), (n, seed, L)
        for s in slabs + dslabs:
            s.close()
    dctx.close()


def test_slabs_gather_then_trace():
    ctx = am.default_context()
    occ = O.random_maze(800, 600, 0.35, 11)
    src = O.sample_free_cells(occ, 6, 11)
    sm = O.source_mask(occ, src)
    slabs = make_slabs(occ, src, 4, ctx)
    r = am.slabs_propagate(slabs, auto_cap=3200)
    full = am.Grid(occ, src, ctx)
    am.slabs_gather(slabs, full)
    ref, rl, _ = O.propagate_auto(occ, sm, 3200, threads=8)
    assert r.layers_used == rl and np.array_equal(full.activity(), ref)
    tg = O.sample_free_cells(occ, 100, 12, exclude=sm)
    for (st, pts), t in zip(full.paths(tg, am.EUCLIDEAN), tg):
        ost, opts = O.reconstruct_euclidean(occ, sm, ref, t)
        assert st == ost and (st != 0 or np.array_equal(pts, opts))
    for s in slabs:
        s.close()
    full.close()


def test_slab_validation():
    ctx = am.default_context()
    occ = np.zeros((40, 50), np.uint8)
    with pytest.raises(am.InvalidInputError):
        am.Grid.slab(occ, [[0, 0]], 0, 4, ctx)  # fewer rows than the halo depth
    with pytest.raises(am.InvalidInputError):
        am.Grid.slab(occ, [[0, 0]], 10, 50, ctx)


def test_tile_slabs_promotion_to_32bit():
    """Tile-mode slabs across the 16 -> 32-bit promotion: boundary rows, halos and lags stay exact."""
    occ = O.comb_maze(330, 200)  # serpentine longer than the 16-bit range
    src = np.array([[0, 329]], np.uint32)
    sm = O.source_mask(occ, src)
    ctx = am.default_context()
    cuts = aligned_split(occ.shape[0], 2)
    assert cuts[0][1] % 32 == 0
    slabs = [am.Grid.slab(occ, src, a, b, ctx) for a, b in cuts]
    r = am.slabs_propagate(slabs, auto_cap=200_000)
    hops = O.bfs_multi_source(occ, sm)
    ecc = int(hops[hops != O.UNREACH].max())
    assert r.cell_bits == 32 and r.tiles_total > 0
    assert (r.layers_used, r.cause) == (ecc, O.FILLED)
    got = np.concatenate([s.activity() for s in slabs])
    bad, _ = O.check_activity(occ, got, hops, r.layers_used)
    assert bad == 0
    for s in slabs:
        s.close()
