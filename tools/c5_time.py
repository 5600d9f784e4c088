"""C5 batch (4096 x 256^2 random mazes, 1 source + 8 targets each, cap 1024): propagate vs trace split.
  python tools/c5_time.py   (GPU box)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402

n = 4096
mazes = np.stack([am.random_maze(256, 256, 0.30, 5000 + i) for i in range(n)])
srcs = [bench.sample_points(mazes[i], 1, 5000 + i) for i in range(n)]
tg = np.concatenate([np.column_stack([np.full(8, i, np.uint32), bench.sample_points(mazes[i], 8, 9000 + i)])
                     for i in range(n)]).astype(np.uint32)
ctx = am.Context(0)
b = am.Batch(mazes, srcs, ctx)
import torch  # noqa: E402
h_pts = torch.empty((8 << 20, 2), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
for rep in range(3):
    t0 = time.perf_counter()
    used, cause, r = b.propagate(auto_cap=1024)
    t1 = time.perf_counter()
    off, pts, st = b.trace(tg, am.EUCLIDEAN, out=h_pts)
    t2 = time.perf_counter()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t3 = time.perf_counter()
    off, pts, st = b.trace(tg, am.EUCLIDEAN, out=h_pts)
    t4 = time.perf_counter()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
k = {}
for e in ev:
    k[e.name[:40]] = k.get(e.name[:40], 0) + e.device_time_total
print("trace call", round(1e3 * (t4 - t3), 2), "ms; device:", {a: round(v / 1e3, 3) for a, v in k.items()})
print(f"C5: propagate {1e3 * (t1 - t0):.2f} ms (global L {r.layers_computed}, blocks {r.block_launches}, "
      f"tiles/block {r.tiles_processed / max(r.block_launches, 1):.0f}, max L_used {int(np.max(used))}, "
      f"mean {float(np.mean(used)):.0f}), trace {1e3 * (t2 - t1):.2f} ms ({len(pts)} points)")
os._exit(0)
