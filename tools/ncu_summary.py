"""Summarise ncu captures into profiles/ (text + JSON the bench reads).

  python tools/ncu_summary.py gpurun_out/prof_block.ncu-rep profiles/r1_k_block  [--launches gpurun_out/launches.csv]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    launches = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    recs = raw(rep)
    lines, summary = [], {"report": rep, "kernels": []}
    for d in recs:
        name = d.get("Kernel Name", ("?", ""))[0]
        k = {"kernel": name}
        lines.append(f"== {name}")
        for key in KEYS:
            if key in d:
                v, u = d[key]
                lines.append(f"  {key:78s} {v:>14s} {u}")
                k[key] = [v, u]
        rb = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
        wb = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
        if rb is not None and wb is not None:
            k["dram_bytes_per_launch"] = rb + wb
            lines.append(f"  dram bytes per launch (read+write): {rb + wb:.4e}")
        summary["kernels"].append(k)
    if summary["kernels"]:
        summary["dram_bytes_per_launch"] = summary["kernels"][0].get("dram_bytes_per_launch")
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hi]
        ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows[hi + 1:]:
            if len(r) <= mi:
                continue
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
            a = agg[r[ki].split("(")[0]]
            a[0] += 1
            a[1] += float(r[mi].replace(",", "")) * scale
        tot = sum(v for _, v in agg.values())
        lines.append("== launch list (ncu gpu__time_duration, cold-cache serialised: compare shares)")
        summary["launch_shares"] = {}
        for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"  {name:60s} n={n:5d} total={us / 1e3:10.3f} ms share={us / tot:7.2%} mean={us / n:9.2f} us")
            summary["launch_shares"][name] = {"launches": n, "total_us": us, "share": us / tot}
    with open(out + ".txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
