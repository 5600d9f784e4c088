"""Wall-clock split of one end-to-end C4 solve through the C ABI (host buffers).

Prints the time of every public call of bench.py's e2e leg plus the raw pinned
PCIe copy bandwidth for the same byte counts, so the e2e number can be read
against what the link allows.  Usage (GPU box): python tools/e2e_breakdown.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    torch.cuda.set_device(0)
    occ, src, tgt = bench.make_workload(am.random_maze)
    H, W = occ.shape
    ctx = am.Context(0, timing=True)
    h_occ = torch.from_numpy(occ).pin_memory()
    h_map = torch.empty((H, W), dtype=torch.int32, pin_memory=True)
    d_occ = torch.empty_like(h_occ, device="cuda")
    d_map = torch.empty_like(h_map, device="cuda")
    for name, a, b in (("h2d occ", d_occ, h_occ), ("d2h map", h_map, d_map)):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.copy_(b, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"raw {name}: {b.numel() * b.element_size() / 1e6:.0f} MB in {dt * 1e3:.2f} ms "
              f"= {b.numel() * b.element_size() / dt / 1e9:.1f} GB/s")
    del d_occ, d_map
    hm = h_map.numpy().view(np.uint32)
    h_pts = torch.empty((16 << 20, 2), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    ho = h_occ.numpy()
    for rep in range(reps):
        t = [time.perf_counter()]
        g = am.Grid(ho, src, ctx)
        ctx.synchronize()
        t.append(time.perf_counter())
        g.propagate_auto(bench.AUTO_CAP)
        t.append(time.perf_counter())
        g.trace(tgt, am.EUCLIDEAN, out=h_pts)
        t.append(time.perf_counter())
        g.activity(out=hm)
        t.append(time.perf_counter())
        g.close()
        t.append(time.perf_counter())
        names = ("create", "propagate", "trace", "download", "close")
        parts = " ".join(f"{n}={(b - a) * 1e3:.1f}" for n, a, b in zip(names, t, t[1:]))
        print(f"rep {rep}: total={(t[-1] - t[0]) * 1e3:.1f} ms  {parts}  pool={ctx.pool_bytes()}")
    ctx.close()
    os._exit(0)


if __name__ == "__main__":
    main()
