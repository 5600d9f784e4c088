"""Benchmark of the oMAP hot path on B200 (BASELINE.json metric on config C4).

One step = one full solve of C4: a 23170x23170 random-obstacle
maze (density 0.40, seed 4), 64 sources, 4096 targets, propagate_auto to the
fixed point (auto_cap = 4*max dim) + Euclidean path extraction for every
target, paths copied to the host.  Inputs are resident in HBM when the timed
region starts (the 1 GiB activity field is far larger than L2, so no flush is
needed).  value = W*H*L_used / time-to-solve.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the CPU restatement of the reference planner
(oracle/, the reference ships no implementation) on the host cores, same
config and metric, one bounded fixed-L slice per step.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gcell-updates/s and time-to-solve (s) for 23k^2 maze; fraction of HBM roofline"
UNIT = "Gcell-updates/s"
W = H = 23170
DENSITY, GRID_SEED = 0.40, 4
N_SOURCES, N_TARGETS, PT_SEED = 64, 4096, 4
AUTO_CAP = 4 * max(W, H)
BYTES_PER_CELL_UPDATE = 9  # 4 B read + 4 B write of uint32 activity + 1 B mask (activity.hpp:51, grid.hpp:56)
LAYERS_PER_BLOCK = 8       # am::kK


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def sample_points(occ, n, seed, exclude=None):
    """n distinct free cells (deterministic); exclude: set of (r, c)."""
    rng = np.random.default_rng(seed)
    h, w = occ.shape
    out, seen = [], set(exclude or ())
    while len(out) < n:
        rs = rng.integers(0, h, 4 * n)
        cs = rng.integers(0, w, 4 * n)
        for r, c in zip(rs.tolist(), cs.tolist()):
            if occ[r, c] == 0 and (r, c) not in seen:
                seen.add((r, c))
                out.append((r, c))
                if len(out) == n:
                    break
    return np.array(out, np.uint32)


def make_workload(am):
    t0 = time.perf_counter()
    occ = am.random_maze(W, H, DENSITY, GRID_SEED)
    src = sample_points(occ, N_SOURCES, PT_SEED)
    tgt = sample_points(occ, N_TARGETS, PT_SEED + 1, exclude={tuple(x) for x in src.tolist()})
    log(f"workload generated in {time.perf_counter() - t0:.1f}s (obstacles {occ.mean():.4f})")
    return occ, src, tgt


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per block launch from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_block_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    def __init__(self, index):
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(occ, src, budget_s=12.0):
    """Oracle (CPU restatement, all host threads) on a bounded fixed-L slice of the same grid."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    threads = os.cpu_count() or 1
    sm = O.source_mask(occ, src)
    t0 = time.perf_counter()
    O.propagate(occ, sm, 1, threads=threads)
    one = time.perf_counter() - t0
    L = max(1, min(64, int(budget_s / max(one, 1e-3))))
    t0 = time.perf_counter()
    O.propagate(occ, sm, L, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": round(W * H * L / dt / 1e9, 4), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle propagate, full {W}x{H} C4 grid, fixed L={L} slice ({dt:.1f}s), threads={threads}"}


def run_reference(args, rank, world):
    """--impl reference: CPU restatement on the host cores (rank 0 only)."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    occ = O.random_maze(W, H, DENSITY, GRID_SEED)
    src = sample_points(occ, N_SOURCES, PT_SEED)
    sm = O.source_mask(occ, src)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.propagate(occ, sm, 1, threads=threads)
    one = time.perf_counter() - t0
    L = max(1, min(64, int(15.0 / max(one, 1e-3) / max(1, args.steps + args.warmup))))
    for _ in range(args.warmup):
        O.propagate(occ, sm, L, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.propagate(occ, sm, L, threads=threads)
        times.append(time.perf_counter() - t0)
    ms = 1000 * sum(times) / len(times)
    value = W * H * L / (ms / 1000) / 1e9
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"C4 {W}x{H} random_maze(0.40, seed 4), 64 sources; fixed L={L} slice per step",
                       "layers_per_step": L},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"fixed L={L} over the full grid per step"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local_rank):
    import torch

    import paper_2004_00540_b200 as am

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

    occ, src, tgt = make_workload(am)
    ctx = am.Context(local_rank, timing=True)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=f"cuda:{local_rank}")
    dev = torch.device(f"cuda:{local_rank}")
    d_occ = torch.from_numpy(occ).to(dev)
    d_src = torch.from_numpy(src.astype(np.int32)).to(dev)
    d_tgt = torch.from_numpy(tgt.astype(np.int32)).to(dev)
    torch.cuda.synchronize()
    grid = am.Grid.from_device(W, H, d_occ.data_ptr(), d_src.data_ptr(), len(src), ctx)
    n = len(tgt)
    d_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    d_status = torch.zeros(n, dtype=torch.int32, device=dev)

    # first solve sizes the point buffer (total points is a pure function of the workload)
    r = grid.propagate_auto(AUTO_CAP)
    off, st = grid.path_counts(tgt, am.EUCLIDEAN)
    total = int(off[-1])
    d_pts = torch.empty(2 * max(total, 1), dtype=torch.int32, device=dev)
    h_pts = torch.empty(2 * max(total, 1), dtype=torch.int32, pin_memory=True)
    h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    h_status = torch.empty(n, dtype=torch.int32, pin_memory=True)
    log(f"L_used={r.layers_used} cause={r.cause} computed={r.layers_computed} bits={r.cell_bits} "
        f"blocks={r.block_launches} paths: total points={total}, covered={(st == 0).sum()}/{n}")

    def step():
        rr = grid.propagate_auto(AUTO_CAP)
        ctx.trace_device(grid, d_tgt.data_ptr(), n, am.EUCLIDEAN, 0, d_off.data_ptr(), d_pts.data_ptr(), total,
                         d_status.data_ptr())
        with torch.cuda.stream(stream):
            h_pts.copy_(d_pts, non_blocking=True)
            h_off.copy_(d_off, non_blocking=True)
            h_status.copy_(d_status, non_blocking=True)
        return rr

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    # phase split for the report (untimed): propagate alone
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    rprop = grid.propagate_auto(AUTO_CAP)
    ev[1].record(stream)
    ctx.trace_device(grid, d_tgt.data_ptr(), n, am.EUCLIDEAN, 0, d_off.data_ptr(), d_pts.data_ptr(), total,
                     d_status.data_ptr())
    ev[2].record(stream)
    ctx.synchronize()
    prop_ms, path_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])

    launches0 = ctx.kernel_launches()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    stencil_ms, blocks, res = 0.0, 0, None
    for _ in range(args.steps):
        res = step()
        stencil_ms += res.stencil_ms
        blocks += res.block_launches
    t_end.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    launches = ctx.kernel_launches() - launches0
    clk = clocks.stop() if clocks else None
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    assert int((h_status == 0).sum()) == int((st == 0).sum())
    L = res.layers_used
    cell_updates = W * H * L
    value = world * cell_updates / (ms_step / 1000) / 1e9

    # roofline of the dominant kernel (k_block): algorithmic bytes per launch / mean launch time
    peak, peak_src = peaks()
    per_launch_ms = stencil_ms / max(blocks, 1)
    alg_bytes = BYTES_PER_CELL_UPDATE * W * H * LAYERS_PER_BLOCK
    achieved = alg_bytes / (per_launch_ms / 1000) / 1e9
    stencil_gcells = W * H * LAYERS_PER_BLOCK / (per_launch_ms / 1000) / 1e9

    # end-to-end through the C ABI with host buffers (H2D of the grid, D2H of map + paths inside the timing)
    e2e = None
    if rank == 0 or world > 1:
        h_occ = torch.from_numpy(occ).pin_memory().numpy()
        h_map = torch.empty((H, W), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        e2e_times = []
        for i in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g2 = am.Grid(h_occ, src, ctx)
            g2.propagate_auto(AUTO_CAP)
            off2, pts2, st2 = g2.trace(tgt, am.EUCLIDEAN)
            g2.activity(out=h_map)
            ctx.synchronize()
            dt = time.perf_counter() - t0
            g2.close()
            if i:
                e2e_times.append(dt)
        e2e_s = statistics.median(e2e_times)
        h2d = occ.nbytes + src.nbytes + tgt.nbytes * 2 + off2.nbytes + st2.nbytes
        d2h = h_map.nbytes + pts2.nbytes + off2.nbytes + st2.nbytes * 2
        e2e = {"value": round(world * cell_updates / e2e_s / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "time_to_solve_s": round(e2e_s, 4),
               "api": "am_grid_create(host) + am_propagate(auto) + am_path_counts + am_trace_paths + "
                      "am_activity_download (pinned host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(occ, src)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16x2" if res.cell_bits == 16 else "u32",
            "data": "synthetic",
            "config": {"workload": f"C4: {W}x{H} random_maze(density 0.40, seed 4), {N_SOURCES} sources, "
                                   f"{N_TARGETS} targets, propagate_auto(cap {AUTO_CAP}) + Euclidean paths to host",
                       "grid": [W, H], "sources": N_SOURCES, "targets": N_TARGETS, "auto_cap": AUTO_CAP,
                       "parallelism": "single GPU" if world == 1 else f"replicas x{world}",
                       "l2": "inputs larger than L2 (1.07 GB 16-bit field vs 126 MB L2), no flush"},
            "time_to_solve_s": round(ms_step / 1000, 4),
            "layers_used": L, "layers_computed": res.layers_computed, "termination": ["filled", "stalled", "cap"][res.cause],
            "phase_ms": {"propagate": round(prop_ms, 3), "paths": round(path_ms, 3),
                         "path_share": round(path_ms / max(prop_ms + path_ms, 1e-9), 4)},
            "stencil_gcell_per_s": round(stencil_gcells, 2),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 3), "traffic": ncu_traffic(),
                         "kernel": "am::k_block<16>", "algorithmic_bytes_per_launch": alg_bytes,
                         "mean_launch_ms": round(per_launch_ms, 4), "peak_source": peak_src,
                         "note": "9 B per cell-update (reference uint32 layout) x W*H x 8 layers per launch"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    # teardown order: torch's pinned-memory allocator records events on the context stream when these
    # buffers die, so release them (and sync) before the context and its stream go away
    del h_pts, h_off, h_status, d_pts, d_off, d_status
    torch.cuda.synchronize()
    ctx.synchronize()
    grid.close()
    return ctx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    keep = run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)  # skip interpreter teardown (ctx/stream vs torch caching allocators)


if __name__ == "__main__":
    main()
