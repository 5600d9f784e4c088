"""Paper Appendix Table 1 on B200 (report.hpp:44-48 ModeComparison): a 2000x2000
grid, 2000 layers as one batched run vs 2000 single-layer iterations.

  python tools/mode_compare.py [reps]     (GPU box) -> one JSON line

Rows: batched (one am_propagate call: exact active-tile skipping, and the dense sweep), iterative
(am_propagate mode ITERATIVE: one launch + host-visible boundary per layer, map resident), and the
paper's recursive setting (am_propagate_layer on host buffers: every layer's map goes to the device
and back, "passing data between the CPU and GPU").  Medians of `reps` runs; bit-equality of the
three final maps is checked.
"""
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_00540_b200 as am  # noqa: E402

N, L = 2000, 2000


def med(f, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = f()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, out


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    occ = am.random_maze(N, N, 0.30, 2000)
    free = np.argwhere(occ == 0)
    src = free[len(free) // 2: len(free) // 2 + 1].astype(np.uint32)
    tctx, dctx = am.Context(0), am.Context(0, dense=True)
    gt, gd = am.Grid(occ, src, tctx), am.Grid(occ, src, dctx)
    gt.propagate(L)
    gd.propagate(L)

    def batched_tiles():
        gt.propagate(L)
        return gt.activity()

    def batched_dense():
        gd.propagate(L)
        return gd.activity()

    def iterative():
        gd.propagate(L, am.ITERATIVE)
        return gd.activity()

    def recursive():
        sm = np.zeros_like(occ)
        sm[src[:, 0], src[:, 1]] = 1
        a = sm.astype(np.uint32)  # ActivityMap::initial
        for _ in range(L):
            a = am.propagate_layer(a, occ, src, ctx=dctx)
        return a

    bt, a1 = med(batched_tiles, reps)
    bd, a2 = med(batched_dense, reps)
    it, a3 = med(iterative, reps)
    rc, a4 = med(recursive, max(1, reps // 3))
    equal = bool(np.array_equal(a1, a2) and np.array_equal(a1, a3) and np.array_equal(a1, a4))
    print(json.dumps({
        "grid": [N, N], "layers": L, "workload": "random_maze(2000, 2000, 0.30, seed 2000), 1 central source",
        "batched_tiles_ms": round(bt, 3), "batched_dense_ms": round(bd, 3), "iterative_ms": round(it, 3),
        "recursive_host_ms": round(rc, 3), "ratio_iterative_over_batched_dense": round(it / bd, 2),
        "ratio_recursive_over_batched_dense": round(rc / bd, 2), "maps_equal": equal,
        "paper_table1_s": {"gtx1080ti": [2.370, 117.314], "titan_v": [0.871, 109.299]}}))
    for g in (gt, gd):
        g.close()
    os._exit(0)


if __name__ == "__main__":
    main()
