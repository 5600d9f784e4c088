"""Adapter exposing the CPU oracle (oracle/oracle.py) through the KAT interface."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

STATUS = {O.OK: "ok", O.EINVAL: "InvalidInputError", O.EUNCOVERED: "UncoveredTargetError",
          O.EINTERNAL: "Error"}


class OracleImpl:
    name = "oracle"

    def build_grid(self, w, h, obstacles):
        occ = np.zeros((h, w), np.uint8)
        for r, c in obstacles:
            occ[r, c] = 1
        return occ

    def sourceset_error(self, occ, src):
        try:
            O.source_mask(occ, src)
            return None
        except O.OracleError as e:
            return STATUS[e.code]

    def comb_maze(self, w, h):
        return O.comb_maze(w, h)

    def random_maze(self, w, h, d, s):
        return O.random_maze(w, h, d, s)

    def initial(self, occ, src):
        return O.initial(occ, O.source_mask(occ, src))

    def propagate_layer(self, occ, src, a):
        return O.propagate_layer(occ, O.source_mask(occ, src), a)

    def propagate(self, occ, src, L):
        return O.propagate(occ, O.source_mask(occ, src), L)

    def propagate_auto(self, occ, src, cap):
        return O.propagate_auto(occ, O.source_mask(occ, src), cap)

    def propagate_reference(self, occ, src, L):
        return O.propagate_reference(occ, O.source_mask(occ, src), L)

    def layer_bound(self, w, h):
        return O.layer_bound(w, h)

    def reconstruct_simple(self, occ, src, amap, t, seed):
        st, pts = O.reconstruct_simple(occ, O.source_mask(occ, src), amap, t, seed)
        return STATUS[st], pts

    def reconstruct_euclidean(self, occ, src, amap, t):
        st, pts = O.reconstruct_euclidean(occ, O.source_mask(occ, src), amap, t)
        return STATUS[st], pts

    def straighten(self, pts):
        return O.straighten(pts)

    def path_metrics(self, pts):
        return O.path_metrics(pts)

    def bfs(self, occ, src):
        return O.bfs_multi_source(occ, O.source_mask(occ, src))

    def dijkstra(self, occ, src):
        return O.dijkstra_octile(occ, O.source_mask(occ, src))

    def check_activity(self, occ, src, m, L):
        hops = O.bfs_multi_source(occ, O.source_mask(occ, src))
        return O.check_activity(occ, m, hops, L)[0]
