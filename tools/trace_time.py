"""Path extraction timing on the C4 instance: am_trace_paths_device (counts + scan + walk) for both
methods, CUDA events on the library stream, median of 5; a digest of the points (compare builds).

  ACTMAP_LIB=build_ab/x.so python tools/trace_time.py
"""
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = am.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    occ, src, tgt = bench.make_workload(am.random_maze)
    g = am.Grid(occ, src, ctx)
    r = g.propagate_auto(bench.AUTO_CAP)
    n = len(tgt)
    dev = torch.device("cuda:0")
    d_tgt = torch.from_numpy(tgt.astype(np.int32)).to(dev)
    d_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    d_st = torch.zeros(n, dtype=torch.int32, device=dev)
    for method, name in ((am.EUCLIDEAN, "euclidean"), (am.SIMPLE, "simple")):
        off, st = g.path_counts(tgt, method, 3)
        total = int(off[-1])
        d_pts = torch.empty(2 * total, dtype=torch.int32, device=dev)
        times = []
        for _ in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.trace_device(g, d_tgt.data_ptr(), n, method, 3, d_off.data_ptr(), d_pts.data_ptr(), total,
                             d_st.data_ptr())
            b.record(stream)
            ctx.synchronize()
            times.append(a.elapsed_time(b))
        times = sorted(times[1:])
        pts = d_pts.cpu().numpy()
        print(f"{name}: {times[2]:.3f} ms (min {times[0]:.3f}) points={total} ok={int((d_st == 0).sum())}/{n} "
              f"digest={hashlib.sha1(pts.tobytes()).hexdigest()[:16]} L_used={r.layers_used}", flush=True)
    g.close()
    ctx.close()


if __name__ == "__main__":
    main()
