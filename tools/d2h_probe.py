"""Full-map download paths on the C4 grid: raw pinned D2H vs am_activity_download (decode + chunked copy).
  python tools/d2h_probe.py   (GPU box)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


occ, src, _ = bench.make_workload(am.random_maze)
H, W = occ.shape
ctx = am.Context(0)
g = am.Grid(occ, src, ctx)
g.propagate_auto(bench.AUTO_CAP)
h_map = torch.empty((H, W), dtype=torch.int32, pin_memory=True)
d_map = torch.empty((H, W), dtype=torch.int32, device="cuda")
hm = h_map.numpy().view(np.uint32)
print(f"raw torch D2H 2.15 GB: {t(lambda: h_map.copy_(d_map, non_blocking=True)):.2f} ms")
half = H // 2
print(f"raw torch D2H 2 x 1.07 GB: {t(lambda: (h_map[:half].copy_(d_map[:half], non_blocking=True), h_map[half:].copy_(d_map[half:], non_blocking=True))):.2f} ms")
print(f"am_activity_download: {t(lambda: g.activity(out=hm)):.2f} ms")
print(f"am_activity_download_device (decode only): {t(lambda: (g.activity_to_device(d_map.data_ptr()), ctx.synchronize())):.2f} ms")
g.close()
ctx.close()
os._exit(0)
