"""Benchmark of the oMAP hot path on B200 (BASELINE.json metric on config C4).

One step = one full solve of C4: a 23170x23170 random-obstacle
maze (density 0.40, seed 4), 64 sources, 4096 targets, propagate_auto to the
fixed point (auto_cap = 4*max dim) + Euclidean path extraction for every
target, paths copied to the host.  Inputs are resident in HBM when the timed
region starts (the 1 GiB activity field is far larger than L2, so no flush is
needed).  value = W*H*L_used / time-to-solve.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--no-cpu-baseline] [--no-e2e] [--no-parity] [--no-configs]

After the timed region (rank 0, N=1) the line also carries
  * "parity": the benchmarked instance checked by the CPU oracle (the checker,
    never the thing measured): the closed-form law against a CPU BFS on every
    cell, the auto-L outcome predicted from the BFS, and 256 of the timed
    step's own paths against the oracle's reconstruction on the device map;
  * "configs": the other BASELINE.json configurations (C2, C3, C4-fixed L=1024,
    C5) timed the same way, each with its own parity flags.

--impl reference times the CPU restatement of the reference planner
(oracle/, the reference ships no implementation) on the host cores, same
config and metric: each step one fixed-L slice of layers over the full C4 grid
with preallocated buffers (the same measurement as the GPU arm's
cpu_baseline), plus full CPU solves of C1 and C2.
"""
import argparse
import gc
import json
import os
import shutil
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
CPU_SLICE_LAYERS = 8       # layers per CPU timing slice (both CPU legs)
PARITY_PATHS = 256         # paths of the timed step re-derived by the oracle


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ workloads
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


def points_for(occ, n_src, n_tgt, seed):
    src = sample_points(occ, n_src, seed)
    tgt = sample_points(occ, n_tgt, seed + 1, exclude={tuple(x) for x in src.tolist()})
    return src, tgt


def make_workload(gen):
    """C4; gen = a random_maze implementation (the product's am.random_maze or the oracle's -- equal, tested)."""
    t0 = time.perf_counter()
    occ = gen(W, H, DENSITY, GRID_SEED)
    src, tgt = points_for(occ, N_SOURCES, N_TARGETS, PT_SEED)
    log(f"workload generated in {time.perf_counter() - t0:.1f}s (obstacles {occ.mean():.4f})")
    return occ, src, tgt


def c1_workload(am):
    occ = am.random_maze(1024, 1024, 0.30, 1)
    src, tgt = points_for(occ, 1, 1, 1)
    return occ, src, tgt, 4 * 1024


def c2_workload(am):
    occ = am.kruskal_maze(4096, 4096, 2)
    src, tgt = points_for(occ, 16, 16, 2)
    return occ, src, tgt, 4096 * 4096  # perfect-maze corridors: cap at the cell count


def c3_workload(am):
    occ = am.city_grid(16384, 16384, 3)
    src, tgt = points_for(occ, 64, 1000, 3)
    return occ, src, tgt, 4 * 16384


def c5_workload(am, n=4096):
    """n x 256^2 random mazes (0.30, seeds 5000+i), 1 source + 8 targets each, cap 1024."""
    mazes = np.stack([am.random_maze(256, 256, 0.30, 5000 + i) for i in range(n)])
    srcs, tg = [], []
    for i in range(n):
        s, t = points_for(mazes[i], 1, 8, 5000 + 7 * i)
        srcs.append(s)
        tg.append(np.column_stack([np.full(8, i, np.uint32), t]))
    return mazes, srcs, np.concatenate(tg).astype(np.uint32), 1024


# ------------------------------------------------------------------ measurement helpers
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _dram_line(traffic, per_launch_ms, peak):
    """The physical side of the roofline: the ncu DRAM bytes of one launch over the live mean launch time.
    The modelled frac above counts the reference's per-layer uint32 traffic; the bit-plane kernel keeps its
    16 layers on chip, so this fraction says how close it runs to HBM itself."""
    if not traffic or not per_launch_ms:
        return None
    gbs = traffic / (per_launch_ms / 1000) / 1e9
    return {"achieved": round(gbs, 1), "frac": round(gbs / peak, 3), "unit": "GB/s",
            "basis": "ncu dram bytes per launch (profiles/ncu_traffic.json) / live mean launch time"}


def ncu_traffic(kind):
    """dram bytes (read + write) per launch of the dominant kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kind, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class NvmlSampler:
    """The same clocks and throttle reasons read through NVML (the library nvidia-smi queries) from a
    thread every 5 ms: the fallback when nvidia-smi's buffered output holds no sample of a short region."""
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        import threading
        self.rows, self.stop_ev, self.t = [], threading.Event(), None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop_ev.is_set():
                    try:
                        self.rows.append((time.time(), float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                          float(mx), int(reasons(h))))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.005)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None

    def stop(self):
        if self.t:
            self.stop_ev.set()
            self.t.join(timeout=2)
        return [(ts, sm, mx, [("Active" if r & b else "Not Active") for b in self.BITS.values()])
                for ts, sm, mx, r in self.rows]


class ClockSampler:
    def __init__(self, index):
        self.p = None
        self.nvml = NvmlSampler(index)
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            # line-buffered (stdbuf): nvidia-smi's block-buffered output is lost when it is terminated
            self.p = subprocess.Popen(
                (["stdbuf", "-oL"] if shutil.which("stdbuf") else []) + ["nvidia-smi", "-i", str(index),
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, window=None):
        """Median SM clock and throttle reasons of the samples taken inside `window` (wall-clock (t0, t1) of
        the timed region; the sampler starts before the warm-up so nvidia-smi is polling by then)."""
        nv_rows = self.nvml.stop()
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) < 8:
                        continue
                    try:
                        ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                        rows.append((ts, float(parts[1]), float(parts[2]), parts[4:8]))
                    except ValueError:
                        continue
        source = "nvidia-smi"
        inside = [r for r in rows if window is None or window[0] <= r[0] <= window[1]]
        nv_inside = [r for r in nv_rows if window is None or window[0] <= r[0] <= window[1]]
        if len(nv_inside) > len(inside):  # nvidia-smi polls every ~100 ms in practice; NVML every 5 ms
            rows, inside, source = nv_rows, nv_inside, "nvml (the library nvidia-smi reads), 5 ms"
        scope = "timed region"
        if not inside and rows and window is not None:  # region shorter than the polling interval
            mid = 0.5 * (window[0] + window[1])
            inside = [min(rows, key=lambda r: abs(r[0] - mid))]
            scope = "nearest sample to the timed region"
        if not inside:
            return None
        reasons = sorted({n for r in inside for n, v in zip(names, r[3]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(r[1] for r in inside), "sm_max_mhz": max(r[2] for r in inside),
                "reasons": reasons, "samples": len(inside), "scope": scope, "source": source}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ CPU side (oracle: checker + baseline only)
_ORACLE = None


def load_oracle():
    """The CPU restatement (oracle/), built for THIS host (-march=native) when gcc can; else the portable
    x86-64-v3 build.  Returns (module, isa)."""
    global _ORACLE
    if _ORACLE is None:
        isa = "x86-64-v3 (portable build)"
        try:
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "native"], check=True,
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=120)
            os.environ["ORACLE_LIB"] = os.path.join(ROOT, "oracle", "liboracle_native.so")
            isa = "-march=native (built on this host)"
        except Exception:
            pass
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        O.lib()
        _ORACLE = (O, isa)
    return _ORACLE


def cpu_slices(O, occ, src, layers, reps, threads):
    """Times `reps` slices of `layers` oracle layers (propagate_layer ping-pong over the full grid, buffers
    allocated and first-touched outside the timer).  Returns per-slice seconds."""
    sm = O.source_mask(occ, src)
    a = O.initial(occ, sm)
    b = np.zeros_like(a)
    O.propagate_layer(occ, sm, a, threads=threads, out=b)  # warm: page-in + OpenMP pool
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for _ in range(layers):
            O.propagate_layer(occ, sm, a, threads=threads, out=b)
            a, b = b, a
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(occ, src, L_used):
    """Oracle on all host threads: fixed-L slices of the full C4 grid, same measurement as
    the --impl reference arm; plus a single-thread layer."""
    O, isa = load_oracle()
    threads = os.cpu_count() or 1
    ts = cpu_slices(O, occ, src, CPU_SLICE_LAYERS, 3, threads)
    dt = statistics.median(ts)
    rate = W * H * CPU_SLICE_LAYERS / dt / 1e9
    single = W * H / statistics.median(cpu_slices(O, occ, src, 1, 1, 1)) / 1e9
    return {"value": round(rate, 4), "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
            "isa": isa, "single_thread_value": round(single, 4),
            "sample": f"oracle propagate_layer x {CPU_SLICE_LAYERS} layers over the full {W}x{H} C4 grid, "
                      f"median of 3 slices ({dt:.2f} s each), threads={threads}, buffers preallocated; "
                      f"single thread: one layer",
            "extrapolated_time_to_solve_s": round(W * H * L_used / (rate * 1e9), 1)}


def predicted_auto(O, occ, hops, cap):
    """propagate_auto's (L_used, cause) from the BFS alone (pin P3)."""
    reach = hops != O.UNREACH
    maxd = int(hops[reach].max())
    unreachable_free = bool(((occ == 0) & ~reach).any())
    lu, cause = (max(1, maxd), O.FILLED) if not unreachable_free else (maxd + 1, O.STALLED)
    if lu > cap:
        lu, cause = cap, (O.FILLED if (not unreachable_free and maxd <= cap) else O.CAP)
    return lu, cause


def check_grid(O, occ, src, amap, L, cap, tgt, off, pts, st, n_paths, hops=None):
    """Oracle check of one solved grid: law on every cell, auto outcome, and n_paths of the device paths
    (offsets / points / status of the traced targets) against oracle reconstruct_euclidean."""
    sm = O.source_mask(occ, src)
    if hops is None:
        hops = O.bfs_multi_source(occ, sm)
    bad, _ = O.check_activity(occ, amap, hops, L)
    out = {"cells_checked": int(occ.size), "law_violations": int(bad)}
    if cap is not None:
        out["auto_outcome_matches_bfs"] = predicted_auto(O, occ, hops, cap)[0] == L
    idx = np.linspace(0, len(tgt) - 1, min(n_paths, len(tgt))).astype(np.int64) if len(tgt) else []
    mism = 0
    for k in idx:
        ost, opts = O.reconstruct_euclidean(occ, sm, amap, tgt[k], cap=L + 2)
        if int(st[k]) != ost or (ost == 0 and not np.array_equal(pts[int(off[k]):int(off[k + 1])], opts)):
            mism += 1
    out["paths_checked"] = int(len(idx))
    out["path_mismatches"] = mism
    return out, hops


def parity_ok(p):
    return p["law_violations"] == 0 and p["path_mismatches"] == 0 and p.get("auto_outcome_matches_bfs", True)


def bench_config(world):
    return {"workload": f"C4: {W}x{H} random_maze(density 0.40, seed 4), {N_SOURCES} sources, "
                        f"{N_TARGETS} targets, propagate_auto(cap {AUTO_CAP}) + Euclidean paths to host",
            "grid": [W, H], "sources": N_SOURCES, "targets": N_TARGETS, "auto_cap": AUTO_CAP,
            "parallelism": "single GPU" if world == 1 else f"row slabs x{world} (K=8 halos through peer memory)",
            "l2": "inputs larger than L2 (1.07 GB 16-bit field vs 126 MB L2), no flush"}


def run_reference(args, rank, world):
    """--impl reference: CPU restatement on the host cores (rank 0 only)."""
    if rank != 0:
        return
    O, isa = load_oracle()
    occ, src, tgt = make_workload(O.random_maze)
    threads = os.cpu_count() or 1
    sm = O.source_mask(occ, src)
    times = cpu_slices(O, occ, src, CPU_SLICE_LAYERS, args.warmup + args.steps, threads)[args.warmup:]
    ms = 1000 * statistics.mean(times)
    value = W * H * CPU_SLICE_LAYERS / (ms / 1000) / 1e9
    hops = O.bfs_multi_source(occ, sm)
    L_used, _ = predicted_auto(O, occ, hops, AUTO_CAP)
    del hops
    # full CPU solves of the two configurations that finish in seconds on the host
    full = []
    c1 = O.random_maze(1024, 1024, 0.30, 1)
    s1, _ = points_for(c1, 1, 1, 1)
    for name, occ_c, src_c, cap in (("C1 1024^2 random 0.30, 1 source", c1, s1, 4 * 1024),
                                    ("C2 4096^2 Kruskal maze, 16 sources", O.kruskal_maze(4096, 4096, 2), None,
                                     4096 * 4096)):
        if src_c is None:
            src_c, _ = points_for(occ_c, 16, 16, 2)
        t0 = time.perf_counter()
        _, lu, cause = O.propagate_auto(occ_c, O.source_mask(occ_c, src_c), cap, threads=threads)
        dt = time.perf_counter() - t0
        full.append({"config": name, "time_to_solve_s": round(dt, 3), "layers_used": lu, "cause": cause,
                     "gcell_per_s": round(occ_c.size * lu / dt / 1e9, 3)})
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": bench_config(world),
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(), "isa": isa,
                             "sample": f"oracle propagate_layer x {CPU_SLICE_LAYERS} layers over the full C4 grid "
                                       f"per step (buffers preallocated; the reference has no buildable sources)",
                             "extrapolated_time_to_solve_s": round(W * H * L_used / (value * 1e9), 1),
                             "layers_used_bfs": L_used},
            "full_solves": full,
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
class Solver:
    """One timed step = propagate_auto to the fixed point + Euclidean paths of this rank's targets to the host.

    N == 1: the whole C4 grid on one GPU (inputs resident in HBM).
    N > 1, peer transport: row slabs (one per rank, halos through peer memory every block); each rank traces
    targets[rank::N] on the distributed map, its walkers reading across slab edges through the peers'
    published rows (no gather).  N > 1, NCCL transport: the map is all-gathered into a full-size field on
    every rank first."""

    def __init__(self, am, torch, ctx, occ, src, tgt, rank, world, local_rank, transport="peer"):
        self.am, self.torch, self.ctx, self.world, self.rank = am, torch, ctx, world, rank
        dev = torch.device(f"cuda:{local_rank}")
        self.stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=dev)
        self.peer = world > 1 and transport == "peer"
        my_tgt = tgt[rank::world]
        self.tgt = my_tgt
        self.d_tgt = torch.from_numpy(my_tgt.astype(np.int32)).to(dev)
        self.full = None
        if not self.peer:
            d_occ = torch.from_numpy(occ).to(dev)
            d_src = torch.from_numpy(src.astype(np.int32)).to(dev)
            torch.cuda.synchronize()
            self.full = am.Grid.from_device(W, H, d_occ.data_ptr(), d_src.data_ptr(), len(src), ctx)
            del d_occ, d_src
        self.slab = None
        self.transport = transport
        if world > 1:
            self.slab = make_slab(am, ctx, occ, src, rank, world, transport)
        n = len(my_tgt)
        self.n = n
        self.d_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        self.d_status = torch.zeros(n, dtype=torch.int32, device=dev)
        r = self.propagate()
        if self.peer:  # point counts come with the first trace (an upper-bound buffer), then the exact one
            self.total = max(n, 1) * (r.layers_computed + 2)
            self.d_pts = torch.empty(2 * self.total, dtype=torch.int32, device=dev)
            self.trace()
            ctx.synchronize()
            self.total = int(self.d_off[-1].item())
            self.covered = int((self.d_status == 0).sum().item())
        else:
            off, st = self.full.path_counts(my_tgt, am.EUCLIDEAN)
            self.total = int(off[-1])
            self.covered = int((st == 0).sum())
        self.h_pts = torch.empty(2 * max(self.total, 1), dtype=torch.int32, pin_memory=True)
        # N == 1: the walkers store the points straight into the pinned host buffer (device-mapped under UVA,
        # as the library's host-buffer trace call does), so the 47 MB cross PCIe while the paths are walked
        self.direct = not self.peer
        self.d_pts = self.h_pts if self.direct else torch.empty(2 * max(self.total, 1), dtype=torch.int32,
                                                                device=dev)
        self.h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
        self.h_status = torch.empty(n, dtype=torch.int32, pin_memory=True)
        log(f"[rank {rank}] L_used={r.layers_used} cause={r.cause} computed={r.layers_computed} bits={r.cell_bits} "
            f"blocks={r.block_launches} paths: points={self.total}, covered={self.covered}/{n}")

    def grid(self):
        return self.full if self.full is not None else self.slab

    def propagate(self):
        if self.slab is None:
            return self.full.propagate_auto(AUTO_CAP)
        r = self.slab.propagate_auto(AUTO_CAP)
        if not self.peer:
            gather(self.am, self.ctx, self.slab, self.full, self.transport)
        return r

    def trace(self):
        if self.peer:
            self.am.peer_trace_device(self.slab, self.d_tgt.data_ptr(), self.n, self.am.EUCLIDEAN, 0,
                                      self.d_off.data_ptr(), self.d_pts.data_ptr(), self.total,
                                      self.d_status.data_ptr())
        else:
            self.ctx.trace_device(self.full, self.d_tgt.data_ptr(), self.n, self.am.EUCLIDEAN, 0,
                                  self.d_off.data_ptr(), self.d_pts.data_ptr(), self.total, self.d_status.data_ptr())

    def step(self):
        r = self.propagate()
        self.trace()
        with self.torch.cuda.stream(self.stream):
            if not self.direct:
                self.h_pts.copy_(self.d_pts, non_blocking=True)
            self.h_off.copy_(self.d_off, non_blocking=True)
            self.h_status.copy_(self.d_status, non_blocking=True)
        return r

    def host_paths(self):
        """(offsets, points (total, 2), status) of the last step, copied out of the pinned buffers (a numpy view
        would keep torch's pinned block alive past the context's stream, which its allocator records on)."""
        self.ctx.synchronize()
        return (self.h_off.numpy().view(np.uint64).copy(),
                self.h_pts.numpy().view(np.uint32).reshape(-1, 2)[: self.total].copy(), self.h_status.numpy().copy())

    def close(self):
        self.torch.cuda.synchronize()
        self.ctx.synchronize()
        del self.h_pts, self.h_off, self.h_status, self.d_pts, self.d_off, self.d_status, self.d_tgt
        if self.slab is not None:
            self.slab.close()
        if self.full is not None:
            self.full.close()


def make_slab(am, ctx, occ, src, rank, world, transport):
    """This rank's row slab; peer transport: IPC handles shared with every rank (torch.distributed carries
    the 1 KB blobs), halos then move through peer memory with no NCCL call per block."""
    if transport == "nccl":
        r0, r1 = ctx.slab_rows(H)
        return am.Grid.slab(occ, src, r0, r1, ctx)
    import torch.distributed as dist

    r0, r1 = am.slab_rows(H, world, rank)
    slab = am.Grid.slab(occ, src, r0, r1, ctx)
    blobs = [None] * world
    dist.all_gather_object(blobs, am.peer_export(slab))
    am.peer_connect(slab, world, rank, blobs)
    return slab


def gather(am, ctx, slab, full, transport):
    if transport == "nccl":
        ctx.comm_gather(slab, full)
    else:
        am.peer_gather(slab, full)


def e2e_solve(am, ctx, occ, src, tgt, rank, world, h_map, h_pts, split=None, transport="peer"):
    """One end-to-end solve through the C ABI with host buffers (pinned): occupancy + sources H2D, propagate
    to the fixed point, every path to the host.  Returns (offsets, points, status, seconds); the full activity
    map is then downloaded too, outside that time (SURVEY.md §8d reports it separately), and split receives
    the create/H2D and map-D2H wall-clock."""
    my_tgt = tgt[rank::world]
    if world == 1:
        t0 = time.perf_counter()
        g = am.Grid(occ, src, ctx)
        t1 = time.perf_counter()
        g.propagate_auto(AUTO_CAP)
        off, pts, st = g.trace(my_tgt, am.EUCLIDEAN, out=h_pts)
        t2 = time.perf_counter()
        g.activity(out=h_map)
        t3 = time.perf_counter()
        g.close()
        if split is not None:
            split.setdefault("create_h2d", []).append(t1 - t0)
            split.setdefault("map_d2h", []).append(t3 - t2)
        return off, pts, st, t2 - t0
    t0 = time.perf_counter()
    s = make_slab(am, ctx, occ, src, rank, world, transport)
    r0, r1 = s.row0, s.row0 + s.height
    r = s.propagate_auto(AUTO_CAP)
    if transport == "peer":  # paths on the distributed map: targets up, points down (torch device buffers)
        import torch

        dev = torch.device(f"cuda:{ctx.device}")
        n = len(my_tgt)
        cap = max(n, 1) * (r.layers_computed + 2)
        d_t = torch.from_numpy(my_tgt.astype(np.int32)).to(dev)
        d_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        d_st = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        d_pts = torch.empty(2 * cap, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        am.peer_trace_device(s, d_t.data_ptr(), n, am.EUCLIDEAN, 0, d_off.data_ptr(), d_pts.data_ptr(), cap,
                             d_st.data_ptr())
        ctx.synchronize()
        off = d_off.cpu().numpy().view(np.uint64)
        total = int(off[-1])
        pts = h_pts[:total]
        pts[:] = d_pts[: 2 * total].cpu().numpy().view(np.uint32).reshape(-1, 2)
        st = d_st[:n].cpu().numpy()
        full = None
    else:
        full = am.Grid(occ, src, ctx)
        gather(am, ctx, s, full, transport)
        off, pts, st = full.trace(my_tgt, am.EUCLIDEAN, out=h_pts)
    t2 = time.perf_counter()
    s.activity(out=h_map[r0:r1])
    t3 = time.perf_counter()
    if split is not None:
        split.setdefault("map_d2h", []).append(t3 - t2)
    s.close()
    if full is not None:
        full.close()
    return off, pts, st, t2 - t0


def timed_median(fn, reps=3):
    fn()  # warm-up
    ts, out = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), out


def run_configs(am, torch, ctx, info_c4, occ4, src4, hops4, parity):
    """The other BASELINE.json configurations on one GPU, inputs resident in HBM, paths to pinned host
    memory, median of 3 solves after a warm-up (host wall clock around synchronous library calls)."""
    out = []
    O = load_oracle()[0] if parity else None
    h_pts = torch.empty((8 << 20, 2), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    def grid_cfg(name, occ, src, tgt, cap, fixed=None, hops=None):
        hh, ww = occ.shape
        g = am.Grid(occ, src, ctx)

        def run():
            r = g.propagate(fixed) if fixed else g.propagate_auto(cap)
            if not len(tgt):
                return r, np.zeros(1, np.uint64), h_pts[:0], np.zeros(0, np.int32)
            off, pts, st = g.trace(tgt, am.EUCLIDEAN, out=h_pts)
            return r, off, pts, st
        t, (r, off, pts, st) = timed_median(run)
        L = fixed or r.layers_used
        e = {"config": name, "grid": [ww, hh], "sources": len(src), "targets": len(tgt),
             "time_to_solve_s": round(t, 5), "layers_used": r.layers_used,
             "termination": ["filled", "stalled", "cap", "fixed"][r.cause if not fixed else 3],
             "dense_equivalent_gcell_per_s": round(ww * hh * L / t / 1e9, 1),
             "executed_gcell_per_s": round(r.cells_executed / t / 1e9, 1) if r.tiles_total else None,
             "engine": r.engine,
             "paths_covered": int((st == 0).sum())}
        if parity:
            p, _ = check_grid(O, occ, src, g.activity(), L, None if fixed else cap, tgt, off, pts, st, PARITY_PATHS,
                              hops)
            e["parity"] = p
            e["parity_ok"] = parity_ok(p)
        g.close()
        log(f"config {name}: {json.dumps(e)}")
        return e

    occ, src, tgt, cap = c1_workload(am)
    out.append(grid_cfg("C1 1024^2 random maze (0.30), 1 source / 1 target, auto", occ, src, tgt, cap))
    occ, src, tgt, cap = c2_workload(am)
    out.append(grid_cfg("C2 4096^2 Kruskal maze, 16 sources / 16 targets, auto", occ, src, tgt, cap))
    occ, src, tgt, cap = c3_workload(am)
    out.append(grid_cfg("C3 16384^2 city grid, 64 sources / 1000 targets, auto", occ, src, tgt, cap))
    del occ
    out.append(grid_cfg("C4-fixed: the C4 grid, fixed L=1024", occ4, src4, np.zeros((0, 2), np.uint32), None,
                        fixed=1024, hops=hops4))
    mazes, srcs, tg, cap = c5_workload(am)
    b = am.Batch(mazes, srcs, ctx)

    def run5():
        used, cause, r = b.propagate(auto_cap=cap)
        off, pts, st = b.trace(tg, am.EUCLIDEAN, out=h_pts)
        return used, cause, r, off, pts, st
    t, (used, cause, r, off, pts, st) = timed_median(run5)
    n = len(mazes)
    cells = int(256 * 256 * np.asarray(used, np.int64).sum())
    e = {"config": f"C5 {n} x 256^2 random mazes (0.30), 1 source + 8 targets each, cap {cap}",
         "time_to_solve_s": round(t, 5), "mazes_per_s": round(n / t, 1),
         "dense_equivalent_gcell_per_s": round(cells / t / 1e9, 1), "paths": int(len(tg)),
         "paths_covered": int((st == 0).sum()), "layers_used_max": int(np.max(used)),
         "layers_used_mean": round(float(np.mean(used)), 1)}
    if parity:
        maps = b.activity()
        bad = mism = wrong_auto = 0
        for i in range(n):
            sm = O.source_mask(mazes[i], srcs[i])
            hops = O.bfs_multi_source(mazes[i], sm)
            bad += O.check_activity(mazes[i], maps[i], hops, int(used[i]))[0]
            wrong_auto += predicted_auto(O, mazes[i], hops, cap) != (int(used[i]), int(cause[i]))
        for k, (i, rr, cc) in enumerate(tg):
            sm = O.source_mask(mazes[i], srcs[i])
            ost, opts = O.reconstruct_euclidean(mazes[i], sm, maps[i], (rr, cc), cap=int(used[i]) + 2)
            if int(st[k]) != ost or (ost == 0 and not np.array_equal(pts[int(off[k]):int(off[k + 1])], opts)):
                mism += 1
        p = {"mazes_checked": n, "cells_checked": int(mazes.size), "law_violations": int(bad),
             "auto_outcome_mismatches": int(wrong_auto), "paths_checked": int(len(tg)), "path_mismatches": mism}
        e["parity"] = p
        e["parity_ok"] = bad == 0 and mism == 0 and wrong_auto == 0
    b.close()
    log(f"config C5: {json.dumps(e)}")
    out.append(e)
    return out


def reduce_device(dist, local_rank):
    """Where the max-over-ranks timing reductions run (gloo: host tensors)."""
    return "cpu" if dist.get_backend() == "gloo" else f"cuda:{local_rank}"


def run_b200(args, rank, world, local_rank):
    import torch

    import paper_2004_00540_b200 as am

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

    occ, src, tgt = make_workload(am.random_maze)
    ctx = am.Context(local_rank, timing=True)
    if world > 1 and args.transport == "nccl":
        uid = [am.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])
    sol = Solver(am, torch, ctx, occ, src, tgt, rank, world, local_rank, args.transport)
    stream = sol.stream

    clocks = ClockSampler(local_rank) if rank == 0 else None  # polling well before the timed region
    for _ in range(args.warmup):
        sol.step()
    ctx.synchronize()
    # phase split for the report (untimed): propagate (+ gather) vs paths
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(stream)
    sol.propagate()
    ev[1].record(stream)
    sol.trace()
    ev[2].record(stream)
    ctx.synchronize()
    prop_ms, path_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    # the same trace again, alone: after a bit-plane run the field encoding runs on the map stream beside
    # the first trace (and is joined by it), so "paths" above is max(walk, encoding); this is the walk with
    # its points streamed to the host, and then the walk into device memory (no PCIe)
    ev[1].record(stream)
    sol.trace()
    ev[2].record(stream)
    ctx.synchronize()
    walk_ms = ev[1].elapsed_time(ev[2])
    walk_dev_ms = walk_ms
    if sol.direct:
        d_tmp = torch.empty_like(sol.h_pts, device=f"cuda:{local_rank}")
        ev[1].record(stream)
        ctx.trace_device(sol.full, sol.d_tgt.data_ptr(), sol.n, am.EUCLIDEAN, 0, sol.d_off.data_ptr(),
                         d_tmp.data_ptr(), sol.total, sol.d_status.data_ptr())
        ev[2].record(stream)
        ctx.synchronize()
        walk_dev_ms = ev[1].elapsed_time(ev[2])
        del d_tmp

    launches0 = ctx.kernel_launches()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    t_start.record(stream)
    stencil_ms, blocks, res, tiles_done, tiles_all, executed = 0.0, 0, None, 0, 0, 0
    for _ in range(args.steps):
        res = sol.step()
        stencil_ms += res.stencil_ms
        blocks += res.block_launches
        tiles_done += res.tiles_processed
        tiles_all += res.tiles_total
        executed += res.cells_executed
    t_end.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    wall1 = time.time()
    launches = ctx.kernel_launches() - launches0
    clk = clocks.stop((wall0, wall1)) if clocks else None
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64, device=reduce_device(dist, local_rank))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    assert int((sol.h_status == 0).sum()) == sol.covered
    L = res.layers_used
    cell_updates = W * H * L
    value = cell_updates / (ms_step / 1000) / 1e9  # whole job: the full grid's cell-updates per second

    # roofline of the dominant kernel: algorithmic bytes per launch / mean launch time (CUDA events bracketing the
    # runs of stencil launches on the library stream, inside the timed steps, so the gaps between launches count).
    # Active-tile mode: the launch is k_block_tiles and its work is the executed cell-updates of the processed tiles.
    peak, peak_src = peaks()
    rows_here = (sol.slab.height if sol.slab is not None else H)
    per_launch_ms = stencil_ms / max(blocks, 1)
    tile_mode = tiles_all > 0
    info = sol.grid().info()
    # executed cell-updates of the blocked launches (processed tiles x tile cells x layers per launch), counted
    # by the library; the engine names the kernel that ran them
    cells_per_launch = executed / max(blocks, 1)
    kernel = {"bits": "am::k_bits_tiles<false>", "tiles": "am::k_block_tiles<16>",
              "dense": "am::k_block<16>"}.get(res.engine, res.engine)
    tile_geom = {"bits": "32 rows x 128 cols (1-bit planes)"}.get(res.engine,
                                                                  f"{info['tile_rows']} rows x {info['tile_cols']} cols")
    alg_bytes = BYTES_PER_CELL_UPDATE * cells_per_launch
    achieved = alg_bytes / (per_launch_ms / 1000) / 1e9
    stencil_gcells = cells_per_launch / (per_launch_ms / 1000) / 1e9
    # the dense sweep (every tile every block) measured on its own: a fixed-L run of the plain k_block
    dense = None
    if rank == 0 and world == 1:
        dctx = am.Context(local_rank, timing=True, dense=True)
        dg = am.Grid(occ, src, dctx)
        best = None
        for _ in range(3):
            rr = dg.propagate(64)
            ms = rr.stencil_ms / max(rr.block_launches, 1)
            best = ms if best is None else min(best, ms)
        dg.close()
        dctx.close()
        dbytes = BYTES_PER_CELL_UPDATE * W * H * LAYERS_PER_BLOCK
        dense = {"kernel": "am::k_block<16> (dense, fixed L=64 on the C4 grid)", "mean_launch_ms": round(best, 4),
                 "gcell_per_s": round(W * H * LAYERS_PER_BLOCK / (best / 1000) / 1e9, 1),
                 "achieved": round(dbytes / (best / 1000) / 1e9, 1), "peak": peak, "unit": "GB/s",
                 "frac": round(dbytes / (best / 1000) / 1e9 / peak, 3), "traffic": ncu_traffic("dense")}

    # end-to-end through the C ABI with host buffers (H2D of the grid, D2H of map + paths inside the timing):
    # one warm-up solve, then the median of 3
    e2e = None
    if not args.no_e2e:
        h_occ = torch.from_numpy(occ).pin_memory().numpy()
        h_map = torch.empty((H, W), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        h_pts = torch.empty((16 << 20, 2), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        e2e_times, full_times, split = [], [], {}
        for i in range(4):
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            hb0 = ctx.h2d_bytes()
            t0 = time.perf_counter()
            off2, pts2, st2, dt = e2e_solve(am, ctx, h_occ, src, tgt, rank, world, h_map, h_pts, split if i else None,
                                            args.transport)
            ctx.synchronize()
            dfull = time.perf_counter() - t0  # including the full map download
            h2d_step = ctx.h2d_bytes() - hb0  # what the library copied host -> device (packed occupancy)
            if dist:
                t = torch.tensor([dt, dfull], dtype=torch.float64, device=reduce_device(dist, local_rank))
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt, dfull = (float(x) for x in t.tolist())
            if i:
                e2e_times.append(dt)
                full_times.append(dfull)
        e2e_s, full_s = statistics.median(e2e_times), statistics.median(full_times)
        h2d = h2d_step
        d2h = pts2.nbytes + off2.nbytes + st2.nbytes * 2
        e2e = {"value": round(cell_updates / e2e_s / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "time_to_solve_s": round(e2e_s, 4), "runs": len(e2e_times),
               "split_ms": {k: round(1000 * statistics.median(v), 2) for k, v in split.items()},
               "with_full_map_download": {"value": round(cell_updates / full_s / 1e9, 3),
                                          "time_to_solve_s": round(full_s, 4),
                                          "d2h_bytes_per_step": int(d2h + W * rows_here * 4)},
               "h2d_note": "counted by the library (am_stats.h2d_bytes): the occupancy crosses PCIe packed to 1 bit "
                           "per cell by host worker threads (upload.cu), plus sources, targets, offsets, status",
               "api": "am_grid_create(host occupancy + sources, pinned) + am_propagate(auto) + am_path_counts + "
                      "am_trace_paths (every path to pinned host memory); the uint32 activity map stays on the "
                      "device (the C++ ActivityMap fetches it lazily) and its download is reported separately" +
                      ("; per rank: slab grid, peer-memory halos, am_peer_gather" if world > 1 else "")}
        del h_occ, h_map, h_pts

    # ---- CPU leg (rank 0, N=1): the oracle as baseline and as the checker of what was just timed ----
    cpu = parity = configs = None
    hops4 = None
    solo = rank == 0 and world == 1
    if solo and not args.no_cpu_baseline:
        cpu = cpu_baseline(occ, src, L)
    if solo and not args.no_parity:
        O = load_oracle()[0]
        off_h, pts_h, st_h = sol.host_paths()
        parity, hops4 = check_grid(O, occ, src, sol.full.activity(), L, AUTO_CAP, sol.tgt, off_h, pts_h, st_h,
                                   PARITY_PATHS)
        parity["auto_outcome_matches_bfs"] = predicted_auto(O, occ, hops4, AUTO_CAP) == (L, res.cause)
        parity["ok"] = parity_ok(parity)
        parity["instance"] = "the timed C4 instance (bench.py's own grid, sources and targets)"
        log(f"parity: {json.dumps(parity)}")
    if solo and not args.no_configs:
        configs = run_configs(am, torch, ctx, info, occ, src, hops4, not args.no_parity)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": ("u32 bit planes (1 bit per cell), u16 field" if res.engine == "bits" else
                      "u16x2" if res.cell_bits == 16 else "u32"),
            "data": "synthetic",
            "config": bench_config(world),
            "time_to_solve_s": round(ms_step / 1000, 4),
            "layers_used": L, "layers_computed": res.layers_computed,
            "termination": ["filled", "stalled", "cap"][res.cause],
            "phase_ms": {"propagate": round(prop_ms, 3), "paths": round(path_ms, 3), "walk_alone": round(walk_ms, 3),
                         "walk_device_only": round(walk_dev_ms, 3),
                         "note": "paths = path counts + walks with every point streamed to pinned host memory, "
                                 "overlapped with the field encoding of the bit-plane run (map stream); "
                                 "walk_alone = the same calls without the encoding; walk_device_only = the walks "
                                 "into device memory (path extraction without the PCIe transfer)",
                         "walk_share_of_time_to_solve": round(walk_dev_ms / ms_step, 4),
                         "path_share": round(path_ms / max(prop_ms + path_ms, 1e-9), 4)},
            "stencil_gcell_per_s": round(stencil_gcells, 2),
            "propagate_gcell_per_s": round(cell_updates / (prop_ms / 1000) / 1e9, 1),
            "cell_updates": {"dense_equivalent_per_step": int(cell_updates),
                             "executed_per_step": int(executed // args.steps)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 3), "traffic": ncu_traffic(res.engine),
                         "kernel": kernel, "algorithmic_bytes_per_launch": int(alg_bytes),
                         "mean_launch_ms": round(per_launch_ms, 4), "peak_source": peak_src,
                         "layers_per_launch": res.block_layers,
                         "dram": _dram_line(ncu_traffic(res.engine), per_launch_ms, peak),
                         "note": "9 B per cell-update (reference uint32 layout, SURVEY 8d) x executed cell-updates "
                                 "per launch (processed tiles x tile cells x layers per launch); traffic = ncu dram "
                                 "read+write per launch (profiles/)"},
            "active_tiles": ({"processed": tiles_done // args.steps, "dense_equivalent": tiles_all // args.steps,
                              "fraction": round(tiles_done / max(tiles_all, 1), 4),
                              "tile": tile_geom} if tile_mode else None),
            "engine": res.engine,
            "dense_stencil": dense,
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
            "configs": configs,
        }
        print(json.dumps(line), flush=True)
    # teardown order: torch's pinned-memory allocator records events on the context stream when these
    # buffers die, so release them (and sync) before the context and its stream go away
    sol.close()
    del sol
    gc.collect()
    torch.cuda.synchronize()
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed instance")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2/C3/C4-fixed/C5 block")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N>1 halo transport: peer memory (CUDA IPC, default) or NCCL send/recv")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # AM_BENCH_SHARED_GPU=1 (code-path check only, the numbers mean nothing): every rank on cuda:0, gloo for
    # the host-side collectives; the peer transport's cross-rank dependencies are stream waits, so ranks may
    # share a GPU
    shared = os.environ.get("AM_BENCH_SHARED_GPU") == "1"
    if shared:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("gloo" if shared else "nccl")
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    sys.stdout.flush()
    sys.stderr.flush()


if __name__ == "__main__":
    main()
