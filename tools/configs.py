"""The other SURVEY.md §8(d) configurations on one GPU (C2, C3, C5, C4-fixed, E), each timed on the
device like bench.py's C4 line: python tools/configs.py  (GPU box).  Prints one JSON line per config."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2], out


def grid_solve(name, occ, src, tgt, cap, ctx):
    H, W = occ.shape
    g = am.Grid(occ, src, ctx)

    def run():
        r = g.propagate_auto(cap)
        off, pts, st = g.trace(tgt, am.EUCLIDEAN)
        return r, st
    t, (r, st) = timed(run)
    g.close()
    return {"config": name, "grid": [W, H], "sources": len(src), "targets": len(tgt), "time_to_solve_s": round(t, 5),
            "layers_used": r.layers_used, "cause": r.cause,
            "gcell_per_s": round(W * H * r.layers_used / t / 1e9, 1), "paths_ok": int((st == 0).sum())}


def main():
    ctx = am.Context(0)
    out = []
    # C2: 4096^2 Kruskal maze, 16 sources / 16 targets (perfect-maze corridors: cap at the cell count)
    occ = am.kruskal_maze(4096, 4096, 2)
    src, tgt = bench.sample_points(occ, 16, 2), bench.sample_points(occ, 16, 3)
    out.append(grid_solve("C2 4096^2 Kruskal maze", occ, src, tgt, 4096 * 4096, ctx))
    # C3: 16384^2 city grid, 64 sources / 1000 targets
    occ = am.city_grid(16384, 16384, 3)
    src, tgt = bench.sample_points(occ, 64, 3), bench.sample_points(occ, 1000, 4)
    out.append(grid_solve("C3 16384^2 city", occ, src, tgt, 4 * 16384, ctx))
    # C4-fixed and E: fixed L = 1024 on the C4 grid / an empty 23170^2 grid with a centred source
    occ4, src4, _ = bench.make_workload(am.random_maze)
    for name, occ, src in (("C4-fixed L=1024", occ4, src4),
                           ("E 23170^2 empty, centred source, L=1024",
                            np.zeros((23170, 23170), np.uint8), np.array([[11585, 11585]], np.uint32))):
        g = am.Grid(occ, src, ctx)
        t, _ = timed(lambda: g.propagate(1024))
        g.close()
        out.append({"config": name, "time_s": round(t, 5), "gcell_per_s": round(occ.size * 1024 / t / 1e9, 1)})
    # C5: 4096 x 256^2 random mazes (density 0.30, seeds 5000+i), 1 source and 8 targets each, cap 1024
    n = 4096
    mazes = np.stack([am.random_maze(256, 256, 0.30, 5000 + i) for i in range(n)])
    srcs = [bench.sample_points(mazes[i], 1, 5000 + i) for i in range(n)]
    tg = np.concatenate([np.column_stack([np.full(8, i, np.uint32), bench.sample_points(mazes[i], 8, 9000 + i)])
                         for i in range(n)]).astype(np.uint32)
    b = am.Batch(mazes, srcs, ctx)
    import torch
    h_pts = torch.empty((8 << 20, 2), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    def run5():
        used, cause, _ = b.propagate(auto_cap=1024)
        off, pts, st = b.trace(tg, am.EUCLIDEAN, out=h_pts)
        return used, st
    t, (used, st) = timed(run5)
    b.close()
    cells = int(n * 256 * 256 * np.asarray(used, np.int64).mean())
    out.append({"config": "C5 4096 x 256^2 batch, 1 source + 8 targets each, cap 1024", "time_to_solve_s": round(t, 5),
                "mazes_per_s": round(n / t, 1), "gcell_per_s": round(cells / t / 1e9, 1),
                "paths_ok": int((np.asarray(st) == 0).sum())})
    for o in out:
        print(json.dumps(o), flush=True)
    ctx.close()
    os._exit(0)


if __name__ == "__main__":
    main()
