import numpy as np, sys
sys.path.insert(0, '.')
import paper_2004_00540_b200 as am
from tests.oracle_adapter import O
for (w, h) in [(1031, 1033), (33, 40000), (257, 129), (4100, 300)]:
    occ = O.random_maze(w, h, 0.35, w)
    src = O.sample_free_cells(occ, 5, 3)
    sm = O.source_mask(occ, src)
    ctx = am.Context(0)
    g = am.Grid(occ, src, ctx)
    r = g.propagate_auto(4 * max(w, h))
    tgt = O.sample_free_cells(occ, 40, 7)
    off, pts, st = g.trace(tgt, am.EUCLIDEAN)
    a = g.activity()
    hops = O.bfs_multi_source(occ, sm)
    bad = O.check_activity(occ, a, hops, r.layers_used)[0]
    g.propagate(37)
    b = g.activity()
    ok = np.array_equal(b, O.propagate(occ, sm, 37, threads=8))
    print(w, h, r.layers_used, bad, ok, int((st == 0).sum()), flush=True)
    g.close(); ctx.close()
