"""Generate tests/golden/spec_kats.json from the worked examples in the reference SPEC.

The reference ships no implementation, so its own known-answer
tests are the examples written into /root/reference/SPEC.md.  This script
transcribes them: every expected value below is either a literal from the SPEC
line cited next to it or the closed form the SPEC states for that example
(e.g. SPEC.md:121 "closed form v = L+1 - Chebyshev distance on empty grid").
Nothing here calls the oracle or the product, so the fixtures pin both.

Run: python tests/golden/make_golden.py   (writes spec_kats.json beside itself)
"""
import json
import math
import os


def cheb(a, b):
    return max(abs(a[0] - b[0]), abs(a[1] - b[1]))


def empty(w, h):
    return [[0] * w for _ in range(h)]


def law_map_empty(w, h, sources, L):
    """activity.hpp:12-14 on an obstacle-free grid: max(0, L+1 - min Chebyshev)."""
    return [[max(0, L + 1 - min(cheb((r, c), s) for s in sources)) for c in range(w)] for r in range(h)]


kats = []


def add(name, cite, **kw):
    kw.update(name=name, spec=cite)
    kats.append(kw)


# ---- grid module ------------------------------------------------------------
add("build_grid_3x3_empty", "SPEC.md:47", op="build_grid", w=3, h=3, obstacles=[], expect_occ=empty(3, 3))
add("build_grid_full_block_sourceset_fails", "SPEC.md:49", op="sourceset", w=2, h=2,
    obstacles=[[0, 0], [0, 1], [1, 0], [1, 1]], sources=[[0, 0]], expect_error="InvalidInputError")
# SPEC.md:56 + grid.hpp:65-69: rows 1 and 3 are walls, first gap at column 0, next at width-1
comb55 = empty(5, 5)
for r, gap in ((1, 0), (3, 4)):
    comb55[r] = [0 if c == gap else 1 for c in range(5)]
add("comb_maze_5x5", "SPEC.md:56", op="comb_maze", w=5, h=5, expect_occ=comb55, expect_free=17)
add("comb_maze_2x2", "SPEC.md:57", op="comb_maze", w=2, h=2, expect_occ=[[0, 0], [0, 1]], expect_free=3)
add("random_maze_zero_density", "SPEC.md:65", op="random_maze", w=64, h=64, density=0.0, seed=7,
    expect_obstacles=0)
add("random_maze_density_03", "SPEC.md:62,66", op="random_maze", w=64, h=64, density=0.3, seed=42,
    expect_obstacles=round(0.3 * 64 * 64))

# ---- propagate module -------------------------------------------------------
add("propagate_layer_1x1", "SPEC.md:112", op="propagate_layer", w=1, h=1, obstacles=[], sources=[[0, 0]],
    input=[[1]], expect=[[2]])
add("propagate_layer_3x3_center", "SPEC.md:113", op="propagate_layer", w=3, h=3, obstacles=[],
    sources=[[1, 1]], input=[[0, 0, 0], [0, 1, 0], [0, 0, 0]], expect=[[1, 1, 1], [1, 2, 1], [1, 1, 1]])
add("propagate_layer_3x3_obstacle", "SPEC.md:114", op="propagate_layer", w=3, h=3, obstacles=[[0, 1]],
    sources=[[1, 1]], input=[[0, 0, 0], [0, 1, 0], [0, 0, 0]], expect=[[1, 0, 1], [1, 2, 1], [1, 1, 1]])
add("propagate_9x9_L4", "SPEC.md:121", op="propagate", w=9, h=9, obstacles=[], sources=[[4, 4]], layers=4,
    expect=law_map_empty(9, 9, [(4, 4)], 4))
add("propagate_auto_9x9", "SPEC.md:130", op="propagate_auto", w=9, h=9, obstacles=[], sources=[[4, 4]],
    auto_cap=100, expect_layers=4, expect_cause="filled", expect=law_map_empty(9, 9, [(4, 4)], 4))
# a fully walled-off free region stops by cause (b) with that region at 0.
walled = [[0, 0, 0, 0, 0], [0, 0, 0, 0, 0], [1, 1, 1, 1, 1], [0, 0, 0, 0, 0], [0, 0, 0, 0, 0]]
add("propagate_auto_walled", "SPEC.md:132", op="propagate_auto", w=5, h=5,
    obstacles=[[r, c] for r in range(5) for c in range(5) if walled[r][c]], sources=[[0, 0]], auto_cap=100,
    # d from (0,0) on rows 0-1 is Chebyshev; coverage fixed after 4 layers; stalled at layer 5
    expect_layers=5, expect_cause="stalled",
    expect=[[6 - max(r, c) for c in range(5)] if r < 2 else [0] * 5 for r in range(5)])
add("propagate_reference_obstacle_adjacent", "SPEC.md:140", op="propagate_reference", w=3, h=3,
    obstacles=[[1, 2]], sources=[[1, 1]], layers=2, expect=[[2, 2, 2], [2, 3, 0], [2, 2, 2]])
for n in (5, 9, 33):  # SPEC.md:503 acceptance 6(a)
    add(f"auto_empty_center_{n}", "SPEC.md:503", op="propagate_auto", w=n, h=n, obstacles=[],
        sources=[[n // 2, n // 2]], auto_cap=4 * n, expect_layers=n // 2, expect_cause="filled")
add("layer_bound_9x9", "SPEC.md:148", op="layer_bound", w=9, h=9, expect_worst=49)
add("layer_bound_1x1", "SPEC.md:149", op="layer_bound", w=1, h=1, expect_worst=1)
add("layer_bound_1000", "SPEC.md:150", op="layer_bound", w=1000, h=1000, expect_high=2000, expect_low=1500)

# ---- reconstruct module -----------------------------------------------------
add("reconstruct_simple_9x9_corner", "SPEC.md:198", op="reconstruct_simple", w=9, h=9, obstacles=[],
    sources=[[4, 4]], layers=4, target=[0, 0], seeds=[0, 1, 2, 3, 4, 99], expect_steps=4)
add("reconstruct_euclidean_diag", "SPEC.md:207", op="reconstruct_euclidean", w=5, h=5, obstacles=[],
    sources=[[0, 0]], layers=8, target=[2, 2], expect_points=[[2, 2], [1, 1], [0, 0]],
    expect_length=2 * math.sqrt(2))
# diagonal-only passage (two obstacles touching corner-wise) -> fallback step.
add("reconstruct_euclidean_diag_passage", "SPEC.md:209", op="reconstruct_euclidean", w=4, h=4,
    obstacles=[[0, 1], [1, 0]], sources=[[0, 0]], layers=6, target=[3, 3],
    expect_points=[[3, 3], [2, 2], [1, 1], [0, 0]], expect_steps=3)
add("straighten_single_corner", "SPEC.md:216", op="straighten", points=[[0, 0], [0, 1], [1, 1]],
    expect_points=[[0, 0], [1, 1]])
add("straighten_collinear", "SPEC.md:217", op="straighten", points=[[0, 0], [0, 1], [0, 2]],
    expect_points=[[0, 0], [0, 1], [0, 2]])
add("straighten_two_pass", "SPEC.md:218", op="straighten", points=[[0, 0], [0, 1], [1, 1], [1, 2], [2, 2]],
    expect_points=[[0, 0], [1, 1], [2, 2]])
add("path_metrics_single", "SPEC.md:225", op="path_metrics", points=[[0, 0]], expect_steps=0, expect_length=0.0)
add("path_metrics_diag", "SPEC.md:226", op="path_metrics", points=[[0, 0], [1, 1]], expect_steps=1,
    expect_length=math.sqrt(2))
add("path_metrics_mixed", "SPEC.md:227", op="path_metrics", points=[[0, 0], [0, 1], [1, 2]], expect_steps=2,
    expect_length=1 + math.sqrt(2))
# SPEC.md:408 (cli plan): "S.\n.T", auto, euclidean -> one path, 1 step, length sqrt(2)
add("plan_2x2_scene", "SPEC.md:408", op="reconstruct_euclidean", w=2, h=2, obstacles=[], sources=[[0, 0]],
    auto_cap=4, target=[1, 1], expect_points=[[1, 1], [0, 0]], expect_length=math.sqrt(2))
# --layers 1 on a 9x9 grid, distant target -> uncovered
add("uncovered_target_L1", "SPEC.md:410", op="reconstruct_euclidean", w=9, h=9, obstacles=[], sources=[[0, 0]],
    layers=1, target=[8, 8], expect_error="UncoveredTargetError")
add("obstacle_target_rejected", "SPEC.md:196", op="reconstruct_simple", w=3, h=3, obstacles=[[2, 2]],
    sources=[[0, 0]], layers=4, target=[2, 2], seeds=[0], expect_error="InvalidInputError")

# ---- oracle module ----------------------------------------------------------
add("bfs_3x3_center", "SPEC.md:275", op="bfs", w=3, h=3, obstacles=[], sources=[[1, 1]],
    expect=[[1, 1, 1], [1, 0, 1], [1, 1, 1]])
add("bfs_two_corners", "SPEC.md:276", op="bfs", w=5, h=5, obstacles=[], sources=[[0, 0], [4, 4]],
    expect=[[min(cheb((r, c), (0, 0)), cheb((r, c), (4, 4))) for c in range(5)] for r in range(5)])
add("bfs_walled_cell", "SPEC.md:277", op="bfs", w=3, h=3, obstacles=[[0, 1], [1, 0], [1, 1]], sources=[[2, 2]],
    expect=[[4294967295, 4294967295, 2], [4294967295, 4294967295, 1], [2, 1, 0]])
add("dijkstra_octile_closed_forms", "SPEC.md:284-286", op="dijkstra", w=5, h=5, obstacles=[], sources=[[0, 0]],
    cells=[[2, 2], [0, 3], [1, 2]], expect_pairs=[[0, 2], [3, 0], [1, 1]])
add("check_activity_fault", "SPEC.md:294", op="check_activity", w=9, h=9, obstacles=[], sources=[[4, 4]],
    layers=4, fault=[2, 3], expect_violations=1)
add("check_activity_base", "SPEC.md:295", op="check_activity", w=9, h=9, obstacles=[], sources=[[4, 4]],
    layers=0, fault=None, expect_violations=0)

if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_kats.json")
    with open(out, "w") as f:
        json.dump({"source": "/root/reference/SPEC.md worked examples", "kats": kats}, f, indent=1)
    print(f"wrote {len(kats)} KATs to {out}")
