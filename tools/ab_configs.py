"""A/B of library builds on the benchmark configurations: C4 / C2 / C3 propagate_auto + paths (median of
reps, host wall clock around the synchronous calls), bit-exactness via a map digest.
  ACTMAP_LIB=build_ab/x.so python tools/ab_configs.py [reps]   (GPU box)"""
import hashlib
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = am.Context(0, timing=True)
cfgs = [("C4", *bench.make_workload(am.random_maze), bench.AUTO_CAP), ("C2", *bench.c2_workload(am)),
        ("C3", *bench.c3_workload(am))]
for name, occ, src, tgt, cap in cfgs:
    g = am.Grid(occ, src, ctx)
    g.propagate_auto(cap)
    ts, ps = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = g.propagate_auto(cap)
        t1 = time.perf_counter()
        g.trace(tgt, am.EUCLIDEAN)
        t2 = time.perf_counter()
        ts.append(t1 - t0)
        ps.append(t2 - t1)
    dig = hashlib.sha1(g.activity().tobytes()).hexdigest()[:12]
    print(f"{name}: propagate {1e3 * statistics.median(ts):.3f} ms (stencil {r.stencil_ms:.3f} ms, "
          f"{r.block_launches} blocks), paths {1e3 * statistics.median(ps):.3f} ms, L_used {r.layers_used}, "
          f"digest {dig}", flush=True)
    g.close()
ctx.close()
