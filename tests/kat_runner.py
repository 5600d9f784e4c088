"""Runs the SPEC.md worked examples (tests/golden/spec_kats.json) against an
implementation adapter.  The same fixtures check the CPU oracle (CPU suite)
and the product C-ABI on the GPU (gpu suite), so both are pinned to the
reference's own known answers rather than to each other.
"""
import json
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "spec_kats.json")
CAUSES = {"filled": 0, "stalled": 1, "cap": 2}


def load_kats():
    with open(GOLDEN) as f:
        return json.load(f)["kats"]


def occ_of(k):
    occ = np.zeros((k["h"], k["w"]), np.uint8)
    for r, c in k.get("obstacles", []):
        occ[r, c] = 1
    return occ


def srcs_of(k):
    return np.asarray(k["sources"], np.uint32).reshape(-1, 2)


def _map_for_paths(impl, k, occ, src):
    if "layers" in k:
        return impl.propagate(occ, src, k["layers"])
    m, _, _ = impl.propagate_auto(occ, src, k["auto_cap"])
    return m


def run_kat(impl, k):
    """Returns None on pass, or raises AssertionError.  Skips ops the adapter lacks."""
    op = k["op"]
    if not hasattr(impl, op):
        return "skip"
    if op == "build_grid":
        assert np.array_equal(impl.build_grid(k["w"], k["h"], k["obstacles"]), np.asarray(k["expect_occ"]))
    elif op == "sourceset":
        err = impl.sourceset_error(occ_of(k), srcs_of(k))
        assert err == k["expect_error"], err
    elif op == "comb_maze":
        occ = impl.comb_maze(k["w"], k["h"])
        assert np.array_equal(occ, np.asarray(k["expect_occ"]))
        assert int((occ == 0).sum()) == k["expect_free"]
    elif op == "random_maze":
        occ = impl.random_maze(k["w"], k["h"], k["density"], k["seed"])
        assert int(occ.sum()) == k["expect_obstacles"]
        assert np.array_equal(occ, impl.random_maze(k["w"], k["h"], k["density"], k["seed"]))
        if k["density"] > 0:
            assert not np.array_equal(occ, impl.random_maze(k["w"], k["h"], k["density"], k["seed"] + 1))
    elif op == "propagate_layer":
        out = impl.propagate_layer(occ_of(k), srcs_of(k), np.asarray(k["input"], np.uint32))
        assert np.array_equal(out, np.asarray(k["expect"])), out
    elif op == "propagate":
        out = impl.propagate(occ_of(k), srcs_of(k), k["layers"])
        assert np.array_equal(out, np.asarray(k["expect"])), out
    elif op == "propagate_auto":
        out, lu, cause = impl.propagate_auto(occ_of(k), srcs_of(k), k["auto_cap"])
        assert lu == k["expect_layers"], (lu, k["expect_layers"])
        assert cause == CAUSES[k["expect_cause"]], cause
        if "expect" in k:
            assert np.array_equal(out, np.asarray(k["expect"])), out
    elif op == "propagate_reference":
        out = impl.propagate_reference(occ_of(k), srcs_of(k), k["layers"])
        assert np.array_equal(out, np.asarray(k["expect"])), out
    elif op == "layer_bound":
        worst, lo, hi = impl.layer_bound(k["w"], k["h"])
        if "expect_worst" in k:
            assert worst == k["expect_worst"]
        if "expect_high" in k:
            assert hi == k["expect_high"] and lo == k["expect_low"]
    elif op in ("reconstruct_simple", "reconstruct_euclidean"):
        occ, src = occ_of(k), srcs_of(k)
        amap = _map_for_paths(impl, k, occ, src)
        seeds = k.get("seeds", [None])
        for seed in seeds:
            if op == "reconstruct_simple":
                st, pts = impl.reconstruct_simple(occ, src, amap, k["target"], seed)
            else:
                st, pts = impl.reconstruct_euclidean(occ, src, amap, k["target"])
            if "expect_error" in k:
                assert st == k["expect_error"], st
                continue
            assert st == "ok", st
            pts = np.asarray(pts).reshape(-1, 2)
            if "expect_points" in k:
                assert pts.tolist() == k["expect_points"], pts.tolist()
            if "expect_steps" in k:
                assert len(pts) - 1 == k["expect_steps"]
            if "expect_length" in k:
                _, length = impl.path_metrics(pts)
                assert math.isclose(length, k["expect_length"], rel_tol=0, abs_tol=1e-12)
    elif op == "straighten":
        out = impl.straighten(np.asarray(k["points"], np.uint32))
        assert np.asarray(out).tolist() == k["expect_points"]
    elif op == "path_metrics":
        steps, length = impl.path_metrics(np.asarray(k["points"], np.uint32))
        assert steps == k["expect_steps"]
        assert math.isclose(length, k["expect_length"], rel_tol=0, abs_tol=1e-12)
    elif op == "bfs":
        out = impl.bfs(occ_of(k), srcs_of(k))
        assert np.array_equal(out, np.asarray(k["expect"], np.uint64).astype(np.uint32)), out
    elif op == "dijkstra":
        a, b = impl.dijkstra(occ_of(k), srcs_of(k))
        for (r, c), (ea, eb) in zip(k["cells"], k["expect_pairs"]):
            assert (int(a[r, c]), int(b[r, c])) == (ea, eb)
    elif op == "check_activity":
        occ, src = occ_of(k), srcs_of(k)
        if k["layers"] == 0:
            m = impl.initial(occ, src)
        else:
            m = impl.propagate(occ, src, k["layers"])
        if k.get("fault"):
            m = m.copy()
            m[tuple(k["fault"])] += 1
        assert impl.check_activity(occ, src, m, k["layers"]) == k["expect_violations"]
    else:
        raise AssertionError(f"unknown op {op}")
    return None
