"""Active-tile kernel scaling: launch time vs number of work items (tile pairs).

  python tools/tile_probe.py      (GPU box)
Answers whether k_block_tiles is bound by per-item latency (flat curve up to
the warp slots) or by SM throughput (linear in items).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    occ, src, _ = bench.make_workload(am.random_maze)
    ctx = am.Context(0)
    g = am.Grid(occ, src, ctx)
    nt = g.info()["tiles"]
    stride = int(os.environ.get("PROBE_STRIDE", 7919))  # 7919: spread over the grid (prime); 1: adjacent tiles
    sizes = [int(a) for a in sys.argv[1:]] or [1, 2, 8, 32, 148, 296, 592, 1000, 1184, 1500, 2368, 4736, 9472]
    for items in sizes:
        ms = g.bench_tile_kernel(items, stride, 30)
        print(f"items {items:6d} tiles {min(2 * items, nt):6d}: {ms * 1e3:8.2f} us/launch  "
              f"{ms * 1e3 / items:7.3f} us/item")
    g.close()
    ctx.close()
    os._exit(0)


if __name__ == "__main__":
    main()
