"""Times propagate_auto on C4 in dense and active-tile modes (CUDA events on the library stream).

  python tools/solve_time.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_00540_b200 as am  # noqa: E402
from bench import AUTO_CAP, H, W, make_workload  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
occ, src, tgt = make_workload(am.random_maze)
out = {}
maps = {}
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["dense", "tiles"]
for mode in modes:
    ctx = am.Context(0, timing=True, dense=(mode == "dense"))
    g = am.Grid(occ, src, ctx)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    g.propagate_auto(AUTO_CAP)
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = g.propagate_auto(AUTO_CAP)
        b.record(stream)
        ctx.synchronize()
        times.append(a.elapsed_time(b))
    maps[mode] = g.activity()
    out[mode] = {"ms": min(times), "all_ms": times, "L": r.layers_used, "cause": r.cause,
                 "blocks": r.block_launches, "stencil_ms": r.stencil_ms,
                 "tiles_processed": r.tiles_processed, "tiles_total": r.tiles_total,
                 "gcell_s_dense_equiv": W * H * r.layers_used / (min(times) / 1000) / 1e9}
    g.close()
if len(maps) == 2:
    out["maps_equal"] = bool(np.array_equal(maps["dense"], maps["tiles"]))
print(json.dumps(out, indent=1))
os._exit(0)
