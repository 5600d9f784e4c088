"""A/B timing of stencil builds: python tools/stencil_ab.py lib1.so lib2.so ...
Runs a fixed-L propagate on the C4 grid through each library (subprocess per lib)."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(lib, L=800, reps=3):
    code = f"""
import os, sys, time, json
sys.path.insert(0, {ROOT!r})
import numpy as np
import paper_2004_00540_b200 as am
occ = am.random_maze(23170, 23170, 0.40, 4)
ctx = am.Context(0, timing=True)
free = np.argwhere(occ[:64, :64] == 0)[:2]
g = am.Grid(occ, free, ctx)
g.propagate(64)
best = None
for _ in range({reps}):
    r = g.propagate({L})
    ms = r.stencil_ms / max(r.block_launches, 1)
    best = ms if best is None else min(best, ms)
print(json.dumps({{"lib": {lib!r}, "ms_per_block": best, "gcell_s": 23170*23170*8/(best/1000)/1e9}}))
os._exit(0)
"""
    env = dict(os.environ, ACTMAP_LIB=lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    return out.stdout.strip() or out.stderr[-2000:]


if __name__ == "__main__":
    for lib in sys.argv[1:]:
        print(one(lib), flush=True)
