"""Items per bit-plane block and where the time of a propagate_auto goes by block size: the listed tiles of
block b come from fixed-L runs (tiles_processed after 16 b layers), the per-block span from the device
timeline (end-to-end spacing of consecutive k_bits_tiles launches).  Tells how much of a solve is spent in
blocks with few tiles, which are latency-bound.  Usage (GPU box):  python tools/light_profile.py [c4|c2|c3]
"""
import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def spans(g, cap):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = g.propagate_auto(cap)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "t.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"
          and "bits_tiles" in e["name"]]
    ev.sort(key=lambda e: e["ts"])
    ends = [e["ts"] + e["dur"] for e in ev]
    return res, [ends[0] - ev[0]["ts"]] + [b - a for a, b in zip(ends, ends[1:])]


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c4"
    torch.cuda.set_device(0)
    if which == "c4":
        occ, src, _ = bench.make_workload(am.random_maze)
        cap = bench.AUTO_CAP
    else:
        occ, src, _, cap = getattr(bench, f"{which}_workload")(am)
    ctx = am.Context(0)
    g = am.Grid(occ, src, ctx)
    g.propagate_auto(cap)
    res, sp = spans(g, cap)
    nb = res.block_launches
    cum = [0]
    for b in range(1, nb + 1):
        cum.append(g.propagate(16 * b).tiles_processed)
    n = np.diff(np.array(cum))
    sp = np.array(sp[: len(n)])
    print(f"{which}: L_used {res.layers_used}, blocks {nb}, items {cum[-1]}, timeline {sp.sum() / 1e3:.2f} ms")
    edges = [0, 16, 64, 148, 256, 592, 1184, 2368, 1 << 30]
    for lo, hi in zip(edges, edges[1:]):
        m = (n > lo if lo else n >= 0) & (n <= hi)
        if m.any():
            print(f"  items ({lo:5d}, {hi:7d}]: blocks {int(m.sum()):4d}, span {sp[m].sum() / 1e3:6.3f} ms, "
                  f"mean {sp[m].mean():6.2f} us/block, mean items {n[m].mean():7.1f}")
    g.close()
    ctx.close()


if __name__ == "__main__":
    main()
