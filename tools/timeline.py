"""Device timeline of one C4 propagate_auto (CUPTI via torch.profiler).

Reports, per op kind (kernel name / memcpy / memset), count and total device
time, and the idle gaps between consecutive device ops on the library stream:
the part of the solve that is neither kernel nor copy.  Usage (GPU box):
  python tools/timeline.py [timing(0|1)] [dense(0|1)]
"""
import collections
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    timing = bool(int(sys.argv[1])) if len(sys.argv) > 1 else False
    dense = bool(int(sys.argv[2])) if len(sys.argv) > 2 else False
    torch.cuda.set_device(0)
    occ, src, tgt = bench.make_workload(am.random_maze)
    ctx = am.Context(0, timing=timing, dense=dense)
    g = am.Grid(occ, src, ctx)
    g.propagate_auto(bench.AUTO_CAP)
    ctx.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        res = g.propagate_auto(bench.AUTO_CAP)
        ctx.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    dev.sort(key=lambda e: e["ts"])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in dev:
        k = e["name"].split("(")[0][:50] if e["cat"] == "kernel" else e["cat"] + ":" + e["name"][:30]
        agg[k][0] += 1
        agg[k][1] += e["dur"]
    span = dev[-1]["ts"] + dev[-1]["dur"] - dev[0]["ts"]
    busy = sum(e["dur"] for e in dev)
    gaps = collections.Counter()
    for a, b in zip(dev, dev[1:]):
        gap = b["ts"] - (a["ts"] + a["dur"])
        ka = a["name"].split("(")[0][:24] if a["cat"] == "kernel" else a["cat"]
        kb = b["name"].split("(")[0][:24] if b["cat"] == "kernel" else b["cat"]
        gaps[f"{ka} -> {kb}"] += max(gap, 0)
    print(f"timing={timing} dense={dense} L_used={res.layers_used} blocks={res.block_launches}")
    print(f"device span {span / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, idle {(span - busy) / 1e3:.2f} ms")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:55s} n={n:5d} total={us / 1e3:8.3f} ms mean={us / n:8.2f} us")
    print("idle gaps by transition:")
    for k, us in gaps.most_common(4):
        print(f"  {k:55s} {us / 1e3:8.3f} ms")
    ends = [e["ts"] + e["dur"] for e in dev if e["cat"] == "kernel" and ("block_tiles" in e["name"] or "bits_tiles" in e["name"])]
    if len(ends) > 10:
        step = [b - a for a, b in zip(ends, ends[1:])]  # per-block span: end-to-end spacing of consecutive blocks
        print("last 32 end spacings (us): " + " ".join(f"{x:.1f}" for x in step[-32:]))
        print("k_block_tiles end spacing by launch decile (mean us): " +
              " ".join(f"{sum(x) / len(x):.1f}" for x in (step[i * len(step) // 10:(i + 1) * len(step) // 10]
                                                          for i in range(10))))
    tk = [e["dur"] for e in dev if e["cat"] == "kernel" and ("block_tiles" in e["name"] or "bits_tiles" in e["name"])]
    if tk:
        q = sorted(tk)
        pct = lambda p: q[min(len(q) - 1, int(p * len(q)))]
        print(f"k_block_tiles durations: p10 {pct(0.1):.1f} p50 {pct(0.5):.1f} p90 {pct(0.9):.1f} max {q[-1]:.1f} us; "
              f"by launch index decile (mean us): " +
              " ".join(f"{sum(tk[i * len(tk) // 10:(i + 1) * len(tk) // 10]) / max(1, len(tk) // 10):.0f}"
                       for i in range(10)))
    gl = sorted(max(b["ts"] - (a["ts"] + a["dur"]), 0) for a, b in zip(dev, dev[1:]))
    big = [x for x in gl if x > 20]
    print(f"gaps: n={len(gl)} median={gl[len(gl) // 2]:.2f} us p99={gl[int(len(gl) * 0.99)]:.2f} us "
          f"max={gl[-1]:.1f} us; {len(big)} gaps > 20 us sum {sum(big) / 1e3:.3f} ms")
    g.close()
    ctx.close()
    os._exit(0)


if __name__ == "__main__":
    main()
