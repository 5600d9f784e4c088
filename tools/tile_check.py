"""Quick parity probe of the active-tile path: tile-mode maps vs dense-mode maps and the oracle.
  python tools/tile_check.py   (GPU box)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_00540_b200 as am  # noqa: E402
from oracle import oracle as orc  # noqa: E402

occ = orc.random_maze(700, 600, 0.35, 3)
src = orc.sample_free_cells(occ, 5, 11)
sm = np.zeros_like(occ)
sm[src[:, 0], src[:, 1]] = 1
tctx, dctx = am.Context(0), am.Context(0, dense=True)
gt, gd = am.Grid(occ, src, tctx), am.Grid(occ, src, dctx)
for L in (8, 16, 24, 40, 200):
    gt.propagate(L)
    gd.propagate(L)
    a, d = gt.activity(), gd.activity()
    ref = orc.propagate(occ, sm, L)
    bad = np.argwhere(a != ref)
    print(L, "tiles==oracle" if len(bad) == 0 else f"tiles DIFF {len(bad)} first {bad[:3].tolist()}",
          "dense==oracle" if np.array_equal(d, ref) else "dense DIFF")
ra, rd = gt.propagate_auto(4000), gd.propagate_auto(4000)
print("auto", ra.layers_used, rd.layers_used, np.array_equal(gt.activity(), gd.activity()))
os._exit(0)
