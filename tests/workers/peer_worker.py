"""One rank of the peer-memory slab transport (am_peer_*), launched by tests/test_gpu_peer.py through
torch.distributed.run (gloo on 127.0.0.1 carries only the 1 KB handle blobs).  Every rank builds the
same grid, propagates its row slab with halos exchanged through peer memory, assembles the full map with
am_peer_gather and writes its results to --out; the test compares them with the CPU oracle.

All ranks may share one GPU: the transport's cross-rank dependencies are stream waits on IPC events
(no kernel waits on another rank)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--gen", default="random")
    ap.add_argument("--w", type=int, required=True)
    ap.add_argument("--h", type=int, required=True)
    ap.add_argument("--density", type=float, default=0.3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sources", type=int, default=3)
    ap.add_argument("--layers", type=int, default=0)  # 0: auto
    ap.add_argument("--cap", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch.distributed as dist

    import paper_2004_00540_b200 as am

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    if a.gen == "comb":
        occ = am.comb_maze(a.w, a.h)
        src = np.array([[a.h - 1, 0]], np.uint32)
    else:
        occ = am.random_maze(a.w, a.h, a.density, a.seed)
        rng = np.random.default_rng(a.seed)
        free = np.argwhere(occ == 0)
        src = free[rng.choice(len(free), size=min(a.sources, len(free)), replace=False)].astype(np.uint32)
    ctx = am.Context(0)
    r0, r1 = am.slab_rows(a.h, world, rank)
    slab = am.Grid.slab(occ, src, r0, r1, ctx)
    blobs = [None] * world
    dist.all_gather_object(blobs, am.peer_export(slab))
    am.peer_connect(slab, world, rank, blobs)
    full = am.Grid(occ, src, ctx)
    # targets: every free cell on a sparse lattice (grid coordinates); this rank traces targets[rank::world]
    # on the distributed map (peer reads across slab edges), without gathering it
    import torch

    lat = np.argwhere(occ[::7, ::5] == 0) * np.array([7, 5])
    tgt = lat.astype(np.uint32)[rank::world]
    nt = len(tgt)
    dev = torch.device("cuda:0")
    d_tgt = torch.from_numpy(tgt.astype(np.int32).reshape(-1)).to(dev) if nt else torch.zeros(2, dtype=torch.int32, device=dev)
    d_off = torch.zeros(nt + 1, dtype=torch.int64, device=dev)
    d_st = torch.zeros(max(nt, 1), dtype=torch.int32, device=dev)
    res = []
    for rep in range(a.reps):
        r = slab.propagate(a.layers) if a.layers else slab.propagate_auto(a.cap)
        am.peer_gather(slab, full)
        res.append({"layers_used": r.layers_used, "cause": r.cause, "cell_bits": r.cell_bits,
                    "blocks": r.block_launches, "tiles": r.tiles_processed})
        if rank == 0:
            np.save(os.path.join(a.out, f"map_{rep}.npy"), full.activity())
        cap = max(nt, 1) * (r.layers_computed + 2)
        d_pts = torch.zeros(2 * cap, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        am.peer_trace_device(slab, d_tgt.data_ptr(), nt, am.EUCLIDEAN, 0, d_off.data_ptr(), d_pts.data_ptr(), cap,
                             d_st.data_ptr())
        ctx.synchronize()
        off = d_off.cpu().numpy().astype(np.int64)
        np.savez(os.path.join(a.out, f"paths_{rank}_{rep}.npz"), tgt=tgt, off=off, st=d_st.cpu().numpy()[:nt],
                 pts=d_pts.cpu().numpy().view(np.uint32)[: 2 * int(off[-1])].reshape(-1, 2))
    with open(os.path.join(a.out, f"rank{rank}.json"), "w") as f:
        json.dump({"rank": rank, "rows": [r0, r1], "results": res}, f)
    dist.barrier()
    full.close()
    slab.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
