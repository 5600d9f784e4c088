"""C4 fixed point under the library at ACTMAP_LIB: L_used, cause and a digest of the full map, so A/B
kernel builds can be compared for bit-exact equality at full size.  Usage (GPU box):
  python tools/c4_hash.py
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402

occ, src, tgt = bench.make_workload(am.random_maze)
ctx = am.Context(0)
g = am.Grid(occ, src, ctx)
r = g.propagate_auto(bench.AUTO_CAP)
m = g.activity()
print("C4", r.layers_used, r.cause, r.tiles_processed, hashlib.md5(m.tobytes()).hexdigest())
os._exit(0)
