"""K5 (per-maze wave kernel) timing on the C5 workload: kernel time (CUDA events) vs the whole
am_batch_propagate call.  python tools/k5_probe.py [n]   (GPU box)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
mazes, srcs, tg, cap = bench.c5_workload(am, n)
ctx = am.Context(0, timing=True)
b = am.Batch(mazes, srcs, ctx)
for rep in range(4):
    t0 = time.perf_counter()
    used, cause, r = b.propagate(auto_cap=cap)
    t1 = time.perf_counter()
    print(f"rep {rep}: call {1e3 * (t1 - t0):.3f} ms, kernel {r.stencil_ms:.3f} ms, mean L {used.mean():.1f}",
          flush=True)
b.close()
ctx.close()
