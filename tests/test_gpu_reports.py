"""RunReport path entries from the drop-in planner session against the oracle.

`b200::Planner::target_reports` (include/actmap/b200.hpp; reference record
report.hpp:35-42 / TargetReport) fills target, covered, reached source, steps,
Euclidean length and points from one device trace.  Each entry is compared
here with the CPU oracle's reconstruct_euclidean / reconstruct_simple
(reconstruct.hpp:38-47) and path_metrics (reconstruct.hpp:26-32) on the same
grid and map, and the map / L_used / cause with the oracle's propagate_auto.
The report is read back through the JSON the C++ side serialised
(serialize_run_report), so the record a caller would store is what is checked."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.oracle_adapter import O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2004_00540_b200")
THREADS = os.cpu_count() or 1


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "planner_reports")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "planner_reports.cpp"), "-L", LIBDIR, "-lactmap_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_planner_reports_tool_compiles(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libactmap_b200.so")):
        pytest.skip("library not built")
    assert os.path.exists(build(tmp_path))


CASES = [  # (generator, w, h, seed, n_src, n_tgt, method, tie seed)
    ("random", 700, 500, 21, 3, 300, 1, 0),
    ("random", 700, 500, 21, 3, 300, 0, 5),
    ("kruskal", 513, 385, 7, 2, 200, 1, 0),
    ("city", 1200, 900, 3, 4, 250, 1, 0),
    ("random", 333, 1, 2, 1, 50, 1, 0),  # one row
]


@pytest.mark.gpu
@pytest.mark.parametrize("gen,w,h,seed,ns,nt,method,tie", CASES)
def test_target_reports_match_oracle(tmp_path, gen, w, h, seed, ns, nt, method, tie):
    if gen == "random":
        occ = O.random_maze(w, h, 0.35, seed)
    elif gen == "kruskal":
        occ = O.kruskal_maze(w, h, seed)
    else:
        occ = O.city_grid(w, h, seed)
    src = O.sample_free_cells(occ, ns, seed)
    sm = O.source_mask(occ, src)
    tgt = O.sample_free_cells(occ, nt, seed + 1, exclude=sm)
    cap = 4 * max(w, h) + 8
    paths = {n: os.path.join(str(tmp_path), n) for n in ("occ", "src", "tgt")}
    np.ascontiguousarray(occ, np.uint8).tofile(paths["occ"])
    np.ascontiguousarray(src, np.uint32).tofile(paths["src"])
    np.ascontiguousarray(tgt, np.uint32).tofile(paths["tgt"])
    exe = build(tmp_path)
    out = subprocess.run([exe, str(w), str(h), paths["occ"], paths["src"], paths["tgt"], str(method), str(tie),
                          str(cap)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    rep = json.loads(out.stdout)

    amap, lu, cause = O.propagate_auto(occ, sm, cap, threads=THREADS)
    assert rep["layers_used"] == lu
    assert rep["termination"] == ["filled", "stalled", "cap"][cause]
    assert rep["max_activity"] == lu + 1
    assert len(rep["paths"]) == len(tgt)
    n_cov = 0
    for e, t in zip(rep["paths"], tgt):
        assert tuple(e["target"]) == tuple(int(x) for x in t)
        if method == 1:
            st, pts = O.reconstruct_euclidean(occ, sm, amap, t, cap=lu + 2)
        else:
            st, pts = O.reconstruct_simple(occ, sm, amap, t, tie, cap=lu + 2)
        assert e["covered"] == (st == O.OK), (tuple(t), st)
        if st != O.OK:
            assert e["reached_source"] is None and e["steps"] == 0 and e["points"] == []
            continue
        n_cov += 1
        steps, length = O.path_metrics(pts)
        assert np.array_equal(np.asarray(e["points"], np.uint32).reshape(-1, 2), pts), tuple(t)
        assert e["steps"] == steps
        assert e["euclidean_length"] == length  # same summation order: exact
        assert tuple(e["reached_source"]) == tuple(int(x) for x in pts[-1])
    assert n_cov > 0
