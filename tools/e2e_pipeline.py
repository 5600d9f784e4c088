"""Serving-style throughput of the end-to-end C4 solve: two host threads, each with its own context
(stream + pool), solve back to back from pinned host buffers (occupancy H2D, propagate_auto, every
path to the host), so one solve's 0.54 GB upload overlaps the other's compute.  Compared with the
same solves run sequentially.  Usage (GPU box): python tools/e2e_pipeline.py [solves per thread]
"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_00540_b200 as am  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    torch.cuda.set_device(0)
    occ, src, tgt = bench.make_workload(am.random_maze)
    h_occ = torch.from_numpy(occ).pin_memory().numpy()
    ctxs = [am.Context(0), am.Context(0)]
    outs = [torch.empty((16 << 20, 2), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in ctxs]
    sig = []

    def solve(i):
        g = am.Grid(h_occ, src, ctxs[i])
        r = g.propagate_auto(bench.AUTO_CAP)
        off, pts, st = g.trace(tgt, am.EUCLIDEAN, out=outs[i])
        g.close()
        return r.layers_used, int(off[-1])

    for i in (0, 1):  # warm both contexts (pools, flag sets)
        sig.append(solve(i))
    t0 = time.perf_counter()
    for _ in range(k):
        sig.append(solve(0))
    seq = (time.perf_counter() - t0) / k

    def worker(i):
        for _ in range(k):
            sig.append(solve(i))

    th = [threading.Thread(target=worker, args=(i,)) for i in (0, 1)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    par = (time.perf_counter() - t0) / (2 * k)
    assert len(set(sig)) == 1, set(sig)
    cells = occ.size * sig[0][0]
    print(f'{{"sequential_ms_per_solve": {seq * 1e3:.1f}, "two_streams_ms_per_solve": {par * 1e3:.1f}, '
          f'"sequential_tcell_per_s": {cells / seq / 1e12:.1f}, "two_streams_tcell_per_s": {cells / par / 1e12:.1f}, '
          f'"solves": {2 * k}, "results_identical": true}}')
    for c in ctxs:
        c.close()
    os._exit(0)


if __name__ == "__main__":
    main()
