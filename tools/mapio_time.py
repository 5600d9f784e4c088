"""Timing of the device map I/O at C4 size (23170^2): Moving AI text -> device scene
(H2D of the text + parse), scene -> grid, and PGM export of the solved map,
next to the plain occupancy upload they replace.  Usage (GPU box):
  python tools/mapio_time.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    torch.cuda.set_device(0)
    occ, src, tgt = bench.make_workload(am.random_maze)
    ctx = am.Context(0)
    text = am.emit_movingai(occ, ctx)
    h_text = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
    h_text.numpy()[:] = np.frombuffer(text, np.uint8)
    h_occ = torch.from_numpy(occ).pin_memory()
    print(f"text {len(text) / 1e6:.1f} MB, occupancy {occ.nbytes / 1e6:.1f} MB")
    lib = am.lib()
    import ctypes as C
    ptr = C.cast(C.c_void_p(h_text.data_ptr()), C.c_char_p)
    for rep in range(reps):
        t0 = time.perf_counter()
        info = am._ParseInfo()
        h = C.c_void_p()
        st = lib.am_scene_parse(ctx.handle, ptr, len(text), am.MOVINGAI, C.byref(h), C.byref(info))
        assert st == 0, info.error
        t1 = time.perf_counter()
        sc = am.Scene.__new__(am.Scene)
        sc.ctx, sc.handle, sc.width, sc.height = ctx, h, info.width, info.height
        sc.n_sources = sc.n_targets = 0
        g = sc.grid(sources=src)
        ctx.synchronize()
        t2 = time.perf_counter()
        g2 = am.Grid(h_occ.numpy(), src, ctx)
        ctx.synchronize()
        t3 = time.perf_counter()
        g.propagate_auto(bench.AUTO_CAP)
        t4 = time.perf_counter()
        pgm = g.export_pgm()
        t5 = time.perf_counter()
        hm = np.empty((occ.shape[0], occ.shape[1]), np.uint32)
        g.activity(out=hm)
        t6 = time.perf_counter()
        print(f"rep {rep}: parse(text H2D + device parse) {1e3 * (t1 - t0):.1f} ms "
              f"({len(text) / (t1 - t0) / 1e9:.1f} GB/s), scene->grid {1e3 * (t2 - t1):.1f} ms, "
              f"grid from pinned occupancy {1e3 * (t3 - t2):.1f} ms, solve {1e3 * (t4 - t3):.1f} ms, "
              f"export_pgm {1e3 * (t5 - t4):.1f} ms ({len(pgm) / 1e6:.0f} MB), "
              f"uint32 map download {1e3 * (t6 - t5):.1f} ms")
        g.close()
        g2.close()
        sc.close()
    ctx.close()
    os._exit(0)


if __name__ == "__main__":
    main()
