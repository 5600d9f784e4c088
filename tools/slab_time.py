"""In-process row slabs on one GPU (same driver as the NCCL path): C4 propagate time vs slab count.
  python tools/slab_time.py [n ...]   (GPU box).  Slabs run one after another on one device, so this
shows the per-block exchange / halo-scan overhead, not multi-GPU speed-up."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402
from tests.test_gpu_slabs import aligned_split  # noqa: E402


def main():
    ns = [int(a) for a in sys.argv[1:]] or [1, 2, 4]
    occ, src, _ = bench.make_workload(am.random_maze)
    H = occ.shape[0]
    ctx = am.Context(0)
    for n in ns:
        slabs = [am.Grid.slab(occ, src, a, b, ctx) for a, b in aligned_split(H, n)]
        best = None
        for _ in range(2):
            ctx.synchronize()
            t0 = time.perf_counter()
            r = am.slabs_propagate(slabs, auto_cap=bench.AUTO_CAP)
            ctx.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        print(f"slabs {n}: {best * 1e3:.1f} ms  L_used={r.layers_used} blocks={r.block_launches} "
              f"tiles={r.tiles_processed}", flush=True)
        for s in slabs:
            s.close()
    os._exit(0)


if __name__ == "__main__":
    main()
