"""Grid creation from host memory on the C4 grid (the first step of an end-to-end solve): wall clock of
am_grid_create with the packed upload (upload.cu) and with a plain byte copy, and the device ops of one
creation (CUPTI).  Usage (GPU box):  python tools/create_time.py
"""
import collections
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    torch.cuda.set_device(0)
    occ, src, _ = bench.make_workload(am.random_maze)
    h_occ = torch.from_numpy(occ).pin_memory().numpy()
    ctx = am.Context(0)
    times = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = am.Grid(h_occ, src, ctx)
        ctx.synchronize()
        times.append(time.perf_counter() - t0)
        g.close()
    print(f"create (pinned source, {os.environ.get('AM_PACKED_UPLOAD', 'packed')}, threads "
          f"{os.environ.get('AM_HOST_THREADS', 'all')}): median {1000 * statistics.median(times[1:]):.2f} ms "
          f"min {1000 * min(times[1:]):.2f} ms", flush=True)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g = am.Grid(h_occ, src, ctx)
        ctx.synchronize()
    g.close()
    path = os.path.join(tempfile.mkdtemp(), "t.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and
          e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    ev.sort(key=lambda e: e["ts"])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        k = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:40]
        agg[k][0] += 1
        agg[k][1] += e["dur"]
    span = (ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]) / 1e3
    print(f"  device span {span:.2f} ms: " + ", ".join(f"{k} x{n} {us / 1e3:.3f} ms" for k, (n, us) in agg.items()))
    ctx.close()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "sweep":
        for env in ({}, {"AM_HOST_THREADS": "8"}, {"AM_HOST_THREADS": "4"}, {"AM_HOST_THREADS": "1"},
                    {"AM_PACKED_UPLOAD": "0"}):
            subprocess.run([sys.executable, __file__], env={**os.environ, **env}, check=False)
    else:
        main()
