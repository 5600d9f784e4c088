"""Longest-path chain of the C4 walk: every target's path length (closed-form counts), then the time of
the longest path walked alone (one warp, no contention), the 64 longest together, and all 4096.
  python tools/walk_chain.py   (GPU box)"""
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
    off, st = g.path_counts(tgt, am.EUCLIDEAN, 0)
    lens = np.diff(off.astype(np.int64))
    order = np.argsort(-lens)
    print(f"L_used={r.layers_used} paths: max {lens.max()} mean {lens.mean():.0f} p99 {np.percentile(lens, 99):.0f} "
          f"sum {lens.sum()}", flush=True)
    dev = torch.device("cuda:0")
    for k in (1, 8, 64, 512, len(tgt)):
        sel = tgt[order[:k]]
        d_tgt = torch.from_numpy(sel.astype(np.int32)).to(dev)
        d_off = torch.zeros(k + 1, dtype=torch.int64, device=dev)
        d_st = torch.zeros(k, dtype=torch.int32, device=dev)
        total = int(lens[order[:k]].sum())
        d_pts = torch.empty(2 * total, dtype=torch.int32, device=dev)
        times = []
        for _ in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.trace_device(g, d_tgt.data_ptr(), k, am.EUCLIDEAN, 0, d_off.data_ptr(), d_pts.data_ptr(), total,
                             d_st.data_ptr())
            b.record(stream)
            ctx.synchronize()
            times.append(a.elapsed_time(b))
        t = sorted(times[1:])[1]
        print(f"{k:5d} longest targets: {t:.3f} ms, {1e6 * t / lens[order[0]]:.1f} ns per step of the longest "
              f"({lens[order[0]]} steps)", flush=True)
    g.close()
    ctx.close()


if __name__ == "__main__":
    main()
