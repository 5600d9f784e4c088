"""C2 (4096^2 Kruskal maze, 16 sources) propagate time per library: ACTMAP_LIB=... python tools/c2_time.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402

occ = am.kruskal_maze(4096, 4096, 2)
src = bench.sample_points(occ, 16, 2)
ctx = am.Context(0)
g = am.Grid(occ, src, ctx)
g.propagate_auto(4096 * 4096)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    r = g.propagate_auto(4096 * 4096)
    ts.append(time.perf_counter() - t0)
print(f"C2 propagate {min(ts) * 1e3:.2f} ms, L_used {r.layers_used}, blocks {r.block_launches}, "
      f"{min(ts) * 1e6 / r.block_launches:.2f} us/block, tiles/block {r.tiles_processed / r.block_launches:.1f}")
os._exit(0)
