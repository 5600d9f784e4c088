"""Multi-rank row-slab protocol on CPU (gloo, world_size 2 and 3).

Mirrors the device driver (capi.cu drive_propagation + multigpu.cu
NcclTransport) with the oracle as the per-slab compute: K-row halo
send/recv between neighbouring ranks before every block, carrying the ring of
per-block minimum covered activities (merged with MIN on receipt: a block's
word is global after world-1 exchanges, checked against an all-reduce),
termination from those words, flag-only exchanges to flush the last blocks,
filled/stalled from an all-reduced zero check, exact rollback of the
overshoot.  The assembled map must equal the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.oracle_adapter import O

K = 8


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab_rows(h, n, r, tile_rows=32):
    """Mirror of am::slab_rows (am_host.hpp): cuts on tile-chunk multiples when every slab keeps two chunks."""
    def cut(k):
        b = h * k // n
        if 0 < k < n and h >= 2 * tile_rows * n:
            b = (b + tile_rows // 2) // tile_rows * tile_rows
        return b
    return cut(r), cut(r + 1)


def termination(start, count, m):
    vmin = None if m >= 0xFFFFFFFF else m + 1
    if vmin is not None and vmin < 2:
        return 0
    capped = count + 1 if vmin is None else min(vmin, count + 1)
    return start + count + 2 - capped


def worker(rank, world, port, occ, src, cap, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    H, W = occ.shape
    f, l = slab_rows(H, world, rank)
    Hl = l - f
    sm_full = O.source_mask(occ, src)
    # slab + K halo rows each side; rows outside the grid are obstacle padding (zero padding)
    ext_occ = np.ones((Hl + 2 * K, W), np.uint8)
    ext_sm = np.zeros((Hl + 2 * K, W), np.uint8)
    lo, hi = max(0, f - K), min(H, l + K)
    ext_occ[lo - (f - K):hi - (f - K)] = occ[lo:hi]
    ext_sm[lo - (f - K):hi - (f - K)] = sm_full[lo:hi]
    A = np.zeros((Hl + 2 * K, W), np.uint32)
    A[K:K + Hl] = O.initial(occ[f:l], sm_full[f:l])

    NS = 64  # kFlagSlots
    slots = np.full(NS, 0xFFFFFFFF, np.int64)
    hops = world - 1
    awaiting = []  # [slot, start, count, exchanges so far, all-reduced word (check)]
    ready = []

    def exchange(rows=True):
        nonlocal slots
        reqs = []
        up_recv = torch.zeros((K, W), dtype=torch.int64)
        dn_recv = torch.zeros((K, W), dtype=torch.int64)
        up_s = torch.full((NS,), 0xFFFFFFFF, dtype=torch.int64)
        dn_s = torch.full((NS,), 0xFFFFFFFF, dtype=torch.int64)
        mine = torch.from_numpy(slots.copy())
        if rank > 0:
            if rows:
                reqs.append(dist.isend(torch.from_numpy(A[K:2 * K].astype(np.int64)), rank - 1))
                reqs.append(dist.irecv(up_recv, rank - 1))
            reqs.append(dist.isend(mine, rank - 1))
            reqs.append(dist.irecv(up_s, rank - 1))
        if rank + 1 < world:
            if rows:
                reqs.append(dist.isend(torch.from_numpy(A[Hl:Hl + K].astype(np.int64)), rank + 1))
                reqs.append(dist.irecv(dn_recv, rank + 1))
            reqs.append(dist.isend(mine, rank + 1))
            reqs.append(dist.irecv(dn_s, rank + 1))
        for q in reqs:
            q.wait()
        if rows and rank > 0:
            A[0:K] = up_recv.numpy().astype(np.uint32)
        if rows and rank + 1 < world:
            A[K + Hl:] = dn_recv.numpy().astype(np.uint32)
        slots = np.minimum(slots, np.minimum(up_s.numpy(), dn_s.numpy()))  # launch_flags_merge
        for a in awaiting:
            a[3] += 1
        while awaiting and awaiting[0][3] >= hops:
            sl, start, count, _, check = awaiting.pop(0)
            assert slots[sl] == check, "the word is global after world-1 exchanges"
            ready.append((start, count, int(slots[sl])))

    done, lprime, nblock = 0, 0, 0

    def consume():
        nonlocal lprime
        while ready:
            start, count, m = ready.pop(0)
            t = termination(start, count, m)
            if t and not lprime:
                lprime = t

    while done < cap and not lprime:
        kk = K if cap - done >= K else 1
        exchange()
        consume()
        for _ in range(kk):
            A = O.propagate_layer(ext_occ, ext_sm, A)
        own = A[K:K + Hl]
        cov = own[own > 0]
        m = int(cov.min()) - 1 if cov.size else 0xFFFFFFFF
        sl = nblock % NS
        slots[sl] = m  # re-armed slot + this block's local minimum
        check = torch.tensor([m], dtype=torch.int64)
        dist.all_reduce(check, op=dist.ReduceOp.MIN)  # test-only reference value
        awaiting.append([sl, done, kk, 0, int(check.item())])
        if hops == 0:
            exchange(rows=False)
        done += kk
        nblock += 1
        consume()
    while awaiting:  # flush: flag-only exchanges
        exchange(rows=False)
    consume()
    own = A[K:K + Hl].copy()
    z = torch.tensor([int(((own == 0) & (occ[f:l] == 0)).any())], dtype=torch.int64)
    dist.all_reduce(z, op=dist.ReduceOp.MAX)
    if lprime:
        used, cause = (max(1, lprime - 1), O.FILLED) if not z.item() else (lprime, O.STALLED)
    else:
        used, cause = cap, (O.CAP if z.item() else O.FILLED)
    own[own > 0] -= np.uint32(done - used)
    parts = [torch.zeros(1)] * world
    gathered = [None] * world
    dist.all_gather_object(gathered, (f, own, used, cause))
    if rank == 0:
        full = np.zeros((H, W), np.uint32)
        for ff, o, _, _ in gathered:
            full[ff:ff + o.shape[0]] = o
        np.save(out_path, full)
        with open(out_path + ".meta", "w") as fh:
            fh.write(f"{used} {cause}")
    del parts
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_matches_oracle(world, tmp_path):
    for seed, (w, h), dens, ns, cap in [(1, (90, 70), 0.3, 3, 400), (2, (64, 61), 0.45, 2, 300),
                                         (3, (50, 40), 0.0, 1, 7)]:
        occ = O.random_maze(w, h, dens, seed)
        src = O.sample_free_cells(occ, ns, seed)
        out = os.path.join(str(tmp_path), f"map_{world}_{seed}.npy")
        mp.spawn(worker, args=(world, free_port(), occ, src, cap, out), nprocs=world, join=True)
        got = np.load(out)
        used, cause = map(int, open(out + ".meta").read().split())
        ref, rl, rc = O.propagate_auto(occ, O.source_mask(occ, src), cap)
        assert (used, cause) == (rl, rc), (world, seed)
        assert np.array_equal(got, ref), (world, seed)


def test_slab_rows_partition():
    for h in (23170, 4096, 100):
        for n in (1, 2, 3, 4, 8):
            rows = [slab_rows(h, n, r) for r in range(n)]
            assert rows[0][0] == 0 and rows[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            if h >= 64 * n:  # tile-aligned cuts, balanced to within one chunk
                assert all(a[1] % 32 == 0 for a in rows[:-1])
                assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 32
            else:
                assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1
