"""Adapter exposing the product (C ABI via paper_2004_00540_b200) through the KAT interface."""
import numpy as np

import paper_2004_00540_b200 as am

STATUS = {am.OK: "ok", am.EINVAL: "InvalidInputError", am.EUNCOVERED: "UncoveredTargetError",
          am.EINTERNAL: "Error"}


class ProductImpl:
    name = "product"

    def sourceset_error(self, occ, src):
        try:
            g = am.Grid(occ, src)
            g.close()
            return None
        except am.InvalidInputError:
            return "InvalidInputError"

    def comb_maze(self, w, h):
        return am.comb_maze(w, h)

    def random_maze(self, w, h, d, s):
        return am.random_maze(w, h, d, s)

    def propagate_layer(self, occ, src, a):
        return am.propagate_layer(a, occ, src)

    def propagate(self, occ, src, L):
        return am.propagate(occ, src, L)

    def propagate_auto(self, occ, src, cap):
        return am.propagate_auto(occ, src, cap)

    def propagate_reference(self, occ, src, L):
        return am.propagate_reference(occ, src, L)

    def layer_bound(self, w, h):
        return am.layer_bound(w, h)

    def _paths(self, occ, src, amap, t, method, seed):
        # trace on the device-propagated map when it matches, else on the uploaded map
        g = am.Grid(occ, src)
        try:
            g.upload_activity(amap, int(np.max(amap)))
            (st, pts), = g.paths([t], method, seed)
        finally:
            g.close()
        return STATUS[st], (pts if pts is not None else np.zeros((0, 2), np.uint32))

    def reconstruct_simple(self, occ, src, amap, t, seed):
        return self._paths(occ, src, amap, t, am.SIMPLE, seed)

    def reconstruct_euclidean(self, occ, src, amap, t):
        st, pts = self._paths(occ, src, amap, t, am.EUCLIDEAN, 0)
        if st == "ok":
            pts = am.straighten(pts, occ, am.STRICT)
        return st, pts

    def straighten(self, pts):
        return am.straighten(pts)

    def path_metrics(self, pts):
        return am.path_metrics(pts)
