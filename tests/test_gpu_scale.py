"""GPU parity at the BASELINE.json configuration sizes (SURVEY.md §8c big-grid
procedure): exact elementwise comparison with the oracle on a fixed-L slice,
the closed-form law against an independent CPU BFS at the fixed point, the
auto-L outcome predicted from the BFS, and every path point against the
oracle's reconstruction on the same map."""
import os

import numpy as np
import pytest

from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = os.cpu_count() or 1


def predicted_auto(occ, hops, cap):
    reach = hops != O.UNREACH
    maxd = int(hops[reach].max())
    unreachable_free = bool(((occ == 0) & ~reach).any())
    if not unreachable_free:
        lu, cause = max(1, maxd), O.FILLED
    else:
        lu, cause = maxd + 1, O.STALLED
    if lu > cap:
        lu, cause = cap, (O.FILLED if (not unreachable_free and maxd <= cap) else O.CAP)
    return lu, cause


def check_paths(g, occ, sm, amap, targets, hops, methods=((am.EUCLIDEAN, 0), (am.SIMPLE, 3))):
    cap = int(g.layers) + 2
    for method, seed in methods:
        res = g.paths(targets, method, seed)
        for (st, pts), t in zip(res, targets):
            if method == am.EUCLIDEAN:
                ost, opts = O.reconstruct_euclidean(occ, sm, amap, t, cap=cap)
            else:
                ost, opts = O.reconstruct_simple(occ, sm, amap, t, seed, cap=cap)
            assert st == ost, (tuple(t), st, ost)
            if st == 0:
                assert np.array_equal(pts, opts), (tuple(t), method)
                assert len(pts) - 1 == hops[t[0], t[1]]  # step-optimal


def run_config(occ, src, targets, cap, fixed_slice=None):
    sm = O.source_mask(occ, src)
    g = am.Grid(occ, src)
    if fixed_slice:
        g.propagate(fixed_slice)
        ref = O.propagate(occ, sm, fixed_slice, threads=THREADS)
        assert np.array_equal(g.activity(), ref), "fixed-L slice differs from the oracle"
        del ref
    r = g.propagate_auto(cap)
    amap = g.activity()
    hops = O.bfs_multi_source(occ, sm)
    assert (r.layers_used, r.cause) == predicted_auto(occ, hops, cap)
    bad, samples = O.check_activity(occ, amap, hops, r.layers_used)
    assert bad == 0, samples
    check_paths(g, occ, sm, amap, targets, hops)
    g.close()
    return r


def test_c2_kruskal_4096():
    occ = O.kruskal_maze(4096, 4096, 2)
    src = O.sample_free_cells(occ, 16, 2)
    sm = O.source_mask(occ, src)
    tg = O.sample_free_cells(occ, 16, 3, exclude=sm)
    worst, _, _ = O.layer_bound(4096, 4096)
    run_config(occ, src, tg, worst, fixed_slice=64)


def test_c3_city_16384():
    occ = O.city_grid(16384, 16384, 3)
    src = O.sample_free_cells(occ, 64, 3)
    sm = O.source_mask(occ, src)
    tg = O.sample_free_cells(occ, 1000, 4, exclude=sm)
    run_config(occ, src, tg, 4 * 16384)


def test_c4_dense_23170():
    """The exact instance bench.py times (its own grid, sources and 4096 targets)."""
    import bench

    n = 23170
    occ, src, tg = bench.make_workload(am.random_maze)
    assert np.array_equal(occ[:64], O.random_maze(n, n, 0.40, 4)[:64])
    r = run_config(occ, src, tg, bench.AUTO_CAP, fixed_slice=64)
    assert r.cell_bits == 16 and r.block_launches > 0


def test_device_trace_matches_host_trace():
    import torch

    occ = O.random_maze(3000, 2000, 0.35, 9)
    src = O.sample_free_cells(occ, 8, 9)
    sm = O.source_mask(occ, src)
    tg = O.sample_free_cells(occ, 300, 10, exclude=sm)
    g = am.Grid(occ, src)
    g.propagate_auto(12000)
    off, pts, st = g.trace(tg, am.EUCLIDEAN)
    dev = torch.device("cuda:0")
    d_t = torch.from_numpy(tg.astype(np.int32)).to(dev)
    d_off = torch.zeros(len(tg) + 1, dtype=torch.int64, device=dev)
    d_pts = torch.zeros(2 * int(off[-1]) + 2, dtype=torch.int32, device=dev)
    d_st = torch.zeros(len(tg), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    g.ctx.trace_device(g, d_t.data_ptr(), len(tg), am.EUCLIDEAN, 0, d_off.data_ptr(), d_pts.data_ptr(),
                       int(off[-1]), d_st.data_ptr())
    g.ctx.synchronize()
    assert np.array_equal(d_off.cpu().numpy().astype(np.uint64), off)
    assert np.array_equal(d_st.cpu().numpy(), st)
    got = d_pts.cpu().numpy().view(np.uint32)[: 2 * int(off[-1])].reshape(-1, 2)
    assert np.array_equal(got, pts)
    g.close()
