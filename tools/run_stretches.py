"""k_bits_run stretches of one propagate_auto per config (AM_BITS_RUN_PRINT) and the kernel's device time
per block run in the cluster.  Usage (GPU box):  python tools/run_stretches.py [c4,c2,c3]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfgs = sys.argv[1] if len(sys.argv) > 1 else "c4,c2,c3"
code = f'''
import sys; sys.path.insert(0, {ROOT!r})
import bench, paper_2004_00540_b200 as am, torch
for c in {cfgs!r}.split(','):
    if c == 'c4':
        occ, src, _ = bench.make_workload(am.random_maze); cap = bench.AUTO_CAP
    else:
        occ, src, _, cap = getattr(bench, c + '_workload')(am)
    ctx = am.Context(0, timing=True); g = am.Grid(occ, src, ctx)
    g.propagate_auto(cap)
    sys.stderr.write('CFG ' + c + chr(10)); sys.stderr.flush()
    r = g.propagate_auto(cap); ctx.synchronize()
    print('END', c, r.block_launches, r.stencil_ms, flush=True)
    g.close(); ctx.close()
'''
out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "AM_BITS_RUN_PRINT": "1"},
                     capture_output=True, text=True)
print(out.stdout[-3000:])
if out.returncode:
    print(out.stderr[-3000:])
runs = [l for l in out.stderr.splitlines() if l.startswith(("bits run", "CFG"))]
tot = 0
for l in runs:
    if l.startswith("CFG"):
        continue
    a, b = map(int, re.findall(r"blocks (\d+)\.\.(\d+)", l)[0])
    tot += b - a
print(f"{len(runs)} stretch lines (both solves), blocks in stretches {tot}")
print("\n".join(runs[-40:]))
