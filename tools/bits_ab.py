"""A/B timing of propagate_auto builds (ACTMAP_LIB=build_ab/<v>.so) on C4 / C2 / C3 / C4-fixed.

Per config: median of 5 solves (CUDA events on the library stream), L_used, cause, blocks, tiles, a
digest of the downloaded map (compare across builds), and the per-launch device-time profile of the
blocked kernel by launch decile (CUPTI, one extra solve).  Usage (GPU box):
  ACTMAP_LIB=build_ab/x.so python tools/bits_ab.py [c4,c2,c3,c4f]
"""
import collections
import hashlib
import json
import os
import sys
import tempfile

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def profile_launches(g, fn):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        g.ctx.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "t.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        k = e["name"].replace("(anonymous namespace)::", "").split("(")[0].split("<")[0].replace("void ", "")[-30:]
        agg[k][0] += 1
        agg[k][1] += e["dur"]
    blk = [e for e in ev if "tiles" in e["name"] and ("bits" in e["name"] or "block" in e["name"])]
    span = (ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]) / 1e3 if ev else 0
    ends = [e["ts"] + e["dur"] for e in blk]
    step = [b - a for a, b in zip(ends, ends[1:])]
    dec = [round(sum(step[i * len(step) // 10:(i + 1) * len(step) // 10]) / max(1, len(step) // 10), 1)
           for i in range(10)] if len(step) >= 10 else []
    dur = [e["dur"] for e in blk]
    ddec = [round(sum(dur[i * len(dur) // 10:(i + 1) * len(dur) // 10]) / max(1, len(dur) // 10), 1)
            for i in range(10)] if len(dur) >= 10 else []
    return {"span_ms": round(span, 3), "kernels": {k: [n, round(us / 1e3, 3)] for k, (n, us) in agg.items()},
            "end_spacing_us_by_decile": dec, "duration_us_by_decile": ddec}


def main():
    which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c4", "c2", "c3", "c4f"]
    torch.cuda.set_device(0)
    ctx = am.Context(0, timing=True)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    out = {"lib": os.environ.get("ACTMAP_LIB", "default")}
    cfgs = {}
    if "c4" in which or "c4f" in which:
        occ, src, _ = bench.make_workload(am.random_maze)
        if "c4" in which:
            cfgs["c4"] = (occ, src, 0, bench.AUTO_CAP)
        if "c4f" in which:
            cfgs["c4f"] = (occ, src, 1024, 0)
    if "c2" in which:
        occ, src, _, cap = bench.c2_workload(am)
        cfgs["c2"] = (occ, src, 0, cap)
    if "c3" in which:
        occ, src, _, cap = bench.c3_workload(am)
        cfgs["c3"] = (occ, src, 0, cap)
    for name, (occ, src, L, cap) in cfgs.items():
        g = am.Grid(occ, src, ctx)
        run = (lambda: g.propagate(L)) if L else (lambda: g.propagate_auto(cap))
        run()
        times = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r = run()
            b.record(stream)
            ctx.synchronize()
            times.append(a.elapsed_time(b))
        times.sort()
        digest = hashlib.sha1(g.activity().tobytes()).hexdigest()[:16]
        rec = {"ms": round(times[2], 3), "min_ms": round(times[0], 3), "L": r.layers_used, "cause": r.cause,
               "blocks": r.block_launches, "tiles": r.tiles_processed, "digest": digest}
        rec.update(profile_launches(g, run))
        out[name] = rec
        if os.environ.get("BITS_AB_FULL"):
            print(name, json.dumps(rec), flush=True)
        else:
            ks = " ".join(f"{k.split('::')[-1]}={v[1]}" for k, v in rec["kernels"].items())
            print(f"{name}: {rec['ms']} ms L={rec['L']} blocks={rec['blocks']} tiles={rec['tiles']} "
                  f"digest={rec['digest']} | {ks} | spacing {rec['end_spacing_us_by_decile']}", flush=True)
        g.close()
    ctx.close()


if __name__ == "__main__":
    main()
