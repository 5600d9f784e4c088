"""GPU part of the map / scene text suite: the device parser / emitters / PGM
export (csrc/mapio.cu, through the C ABI) against the CPU restatement
(oracle/mapio.py) -- byte-exact text, identical occupancy / sources / targets,
identical error positions; plus size-independent round trips at full size."""
import numpy as np
import pytest

from tests.mapio_cases import (M, MOVINGAI_BAD, MOVINGAI_KATS, SCENE_BAD, SCENE_KATS, movingai_text, mutate,
                               oracle_parse, scene_text)
from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")
pytestmark = pytest.mark.gpu


def dev_parse(fmt, text):
    try:
        sc = am.Scene(text, fmt)
    except am.ParseError as e:
        return ("parse", e.line, e.column)
    except am.InvalidInputError:
        return ("invalid",)
    try:
        return ("ok", sc.download())
    finally:
        sc.close()


def same(got, exp, fmt):
    if got[0] != exp[0]:
        return False
    if got[0] != "ok":
        return got == exp
    occ, src, tgt = got[1]
    if fmt == am.MOVINGAI:
        return np.array_equal(occ, exp[1]) and len(src) == 0 and len(tgt) == 0
    eo, es, et = exp[1]
    return (np.array_equal(occ, eo) and [tuple(x) for x in src.tolist()] == es
            and [tuple(x) for x in tgt.tolist()] == et)


@pytest.mark.parametrize("text,rows", MOVINGAI_KATS)
def test_movingai_examples(text, rows):
    assert am.parse_movingai(text).tolist() == rows


@pytest.mark.parametrize("text,pos", MOVINGAI_BAD)
def test_movingai_errors(text, pos):
    with pytest.raises(am.ParseError) as e:
        am.parse_movingai(text)
    assert (e.value.line, e.value.column) == pos


@pytest.mark.parametrize("text,rows,src,tgt", SCENE_KATS)
def test_scene_examples(text, rows, src, tgt):
    occ, s, t = am.parse_ascii_scene(text)
    assert occ.tolist() == rows
    assert [tuple(x) for x in s.tolist()] == src and [tuple(x) for x in t.tolist()] == tgt


@pytest.mark.parametrize("text,pos", SCENE_BAD)
def test_scene_errors(text, pos):
    with pytest.raises(am.ParseError) as e:
        am.parse_ascii_scene(text)
    assert (e.value.line, e.value.column) == pos


def test_scene_without_source():
    with pytest.raises(am.InvalidInputError) as e:
        am.parse_ascii_scene(b"..\n.T\n")
    assert not isinstance(e.value, am.ParseError)


@pytest.mark.parametrize("fmt", [am.MOVINGAI, am.ASCII_SCENE])
def test_mutations_match_oracle(fmt):
    """Seeded body + header mutations: same grid or the same error position as the oracle."""
    rng = np.random.default_rng(7 + fmt)
    occ = O.random_maze(19, 9, 0.3, 5)
    occ[0, 0] = occ[8, 18] = occ[4, 4] = 0
    if fmt == am.MOVINGAI:
        base, fn = movingai_text(occ), M.parse_movingai
    else:
        base, fn = scene_text(occ, [(0, 0), (4, 4)], [(8, 18)]), M.parse_ascii_scene
    kinds = {}
    for i in range(400):
        t = mutate(base, rng)
        if rng.integers(0, 4) == 0:
            t = mutate(t, rng)
        exp, got = oracle_parse(fn, t), dev_parse(fmt, t)
        assert same(got, exp, fmt), (i, t, got[:3] if got[0] != "ok" else "ok", exp[:3] if exp[0] != "ok" else "ok")
        kinds[exp[0]] = kinds.get(exp[0], 0) + 1
    assert kinds.get("parse", 0) > 100 and kinds.get("ok", 0) >= 10


@pytest.mark.parametrize("w,h", [(1, 1), (1, 300), (300, 1), (37, 23), (129, 257), (1000, 3), (4097, 5)])
def test_emit_parse_round_trip_matches_oracle(w, h):
    occ = O.random_maze(w, h, 0.3, w * 7 + h)
    t = am.emit_movingai(occ)
    assert t == M.emit_movingai(occ)
    assert np.array_equal(am.parse_movingai(t), occ)
    assert np.array_equal(am.parse_movingai(movingai_text(occ, crlf=True, trailing=False)), occ)
    free = np.argwhere(occ == 0)
    if len(free) >= 3:
        src = [tuple(int(v) for v in free[0]), tuple(int(v) for v in free[-1])]
        tgt = [tuple(int(v) for v in free[len(free) // 2])]
        s = am.emit_ascii_scene(occ, src, tgt)
        assert s == M.emit_ascii_scene(occ, src, tgt)
        o2, s2, t2 = am.parse_ascii_scene(s)
        assert np.array_equal(o2, occ) and [tuple(x) for x in s2.tolist()] == sorted(src)
        assert [tuple(x) for x in t2.tolist()] == tgt
        assert am.emit_ascii_scene(o2, s2, t2) == s  # idempotent after one normalisation


def test_scene_grid_solves_like_host_grid():
    occ = O.random_maze(300, 200, 0.3, 12)
    src_a = O.sample_free_cells(occ, 3, 1)
    src = [tuple(int(v) for v in x) for x in src_a]
    tgt = [tuple(int(v) for v in x) for x in O.sample_free_cells(occ, 5, 2, exclude=O.source_mask(occ, src_a))]
    sc = am.Scene(scene_text(occ, src, tgt), am.ASCII_SCENE)
    assert (sc.width, sc.height, sc.n_sources, sc.n_targets) == (300, 200, 3, 5)
    assert sc.obstacles == int(occ.sum())
    g1 = sc.grid()
    r1 = g1.propagate_auto(2000)
    g2 = am.Grid(occ, src)
    r2 = g2.propagate_auto(2000)
    assert (r1.layers_used, r1.cause) == (r2.layers_used, r2.cause)
    assert np.array_equal(g1.activity(), g2.activity())
    _, s_dev, t_dev = sc.download()
    o1, p1, s1 = g1.trace(t_dev)
    o2, p2, s2 = g2.trace(t_dev)
    assert np.array_equal(o1, o2) and np.array_equal(p1, p2) and np.array_equal(s1, s2)
    # caller sources override the file's
    g3 = sc.grid(sources=[tgt[0]])
    g3.propagate(5)
    assert g3.activity()[tgt[0]] == 6
    for g in (g1, g2, g3):
        g.close()
    sc.close()


@pytest.mark.parametrize("w,h,layers", [(1, 1, 1), (9, 9, 9), (64, 33, 200), (300, 200, 700), (513, 77, 1)])
def test_pgm_matches_oracle(w, h, layers):
    occ = O.random_maze(w, h, 0.25, w + h)
    src = O.sample_free_cells(occ, 2 if w * h > 1 else 1, 3)
    g = am.Grid(occ, src)
    g.propagate(layers)
    vals = g.activity()
    assert g.export_pgm() == M.export_pgm(vals)
    assert am.export_pgm(vals) == M.export_pgm(vals)
    g.close()


def test_pgm_large_map_matches_oracle():
    """4096^2 maze, 64 sources, fixed point (16-bit samples): device export == oracle export of the downloaded map."""
    occ = O.random_maze(4096, 4096, 0.35, 77)
    src = O.sample_free_cells(occ, 64, 78)
    g = am.Grid(occ, src)
    r = g.propagate_auto(4 * 4096)
    vals = g.activity()
    assert int(vals.max()) == r.layers_used + 1 > 255
    assert g.export_pgm() == M.export_pgm(vals)
    g.close()


def test_pgm_rounding_and_zero():
    v = np.array([[0, 1, 300, 599, 600, 2**31 - 1]], np.uint32)
    assert am.export_pgm(v) == M.export_pgm(v)
    assert am.export_pgm(np.zeros((3, 5), np.uint32)) == b"P5\n5 3\n255\n" + bytes(15)
    assert am.export_pgm(np.array([[2]], np.uint32)) == b"P5\n1 1\n255\n\xff"
    rng = np.random.default_rng(3)
    for mx in (1, 7, 255, 256, 1000, 65535, 65536, 123456789):
        v = rng.integers(0, mx + 1, size=(17, 23), dtype=np.uint64).astype(np.uint32)
        v[0, 0] = mx
        assert am.export_pgm(v) == M.export_pgm(v), mx


def test_full_size_movingai_round_trip():
    """C4-sized (23170^2) map text: device parse == the generator's occupancy, and the
    device emitter reproduces the text byte for byte (size-independent round trip)."""
    occ = am.random_maze(23170, 23170, 0.40, 4)
    text = am.emit_movingai(occ)
    assert len(text) == len(b"type octile\nheight 23170\nwidth 23170\nmap\n") + 23170 * 23171
    # spot-check the emitted rows against the occupancy
    off = len(b"type octile\nheight 23170\nwidth 23170\nmap\n")
    body = np.frombuffer(text, np.uint8, offset=off).reshape(23170, 23171)
    assert (body[:, -1] == 10).all()
    assert np.array_equal(body[::997, :-1] == ord("@"), occ[::997] != 0)
    sc = am.Scene(text, am.MOVINGAI)
    assert (sc.width, sc.height, sc.obstacles) == (23170, 23170, int(occ.sum(dtype=np.uint64)))
    back, _, _ = sc.download()
    assert np.array_equal(back, occ)
    sc.close()


def test_c_abi_rejections():
    """Capacity, format and handle checks of the text / PGM entry points (status codes, no crash)."""
    import ctypes as C
    L, ctx = am.lib(), am.default_context()
    occ = np.zeros((3, 4), np.uint8)
    n = C.c_uint64(0)
    args = (ctx.handle, am.MOVINGAI, 4, 3, occ.ctypes.data_as(C.c_void_p), None, 0, None, 0)
    assert L.am_emit_text(*args, None, 0, C.byref(n)) == am.OK and n.value == len(b"type octile\nheight 3\nwidth 4\nmap\n") + 15
    small = np.empty(n.value - 1, np.uint8)
    assert L.am_emit_text(*args, small.ctypes.data_as(C.c_void_p), n.value - 1, C.byref(n)) == am.EINVAL
    assert L.am_emit_text(ctx.handle, 7, 4, 3, occ.ctypes.data_as(C.c_void_p), None, 0, None, 0, None, 0,
                          C.byref(n)) == am.EINVAL
    info, h = am._ParseInfo(), C.c_void_p()
    assert L.am_scene_parse(ctx.handle, b"S.", 2, 9, C.byref(h), C.byref(info)) == am.EINVAL
    v = np.array([[1, 2]], np.uint32)
    assert L.am_export_pgm(ctx.handle, 2, 1, v.ctypes.data_as(C.c_void_p), None, 0, C.byref(n)) == am.OK
    out = np.empty(n.value - 1, np.uint8)
    assert L.am_export_pgm(ctx.handle, 2, 1, v.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                           n.value - 1, C.byref(n)) == am.EINVAL
    g = am.Grid(occ, [(0, 0)])
    assert L.am_activity_export_pgm(ctx.handle, g.handle, None, 0, C.byref(n)) == am.EINVAL  # no map yet
    g.propagate(2)
    assert g.export_pgm() == M.export_pgm(g.activity())
    sc = am.Scene(b"S.\n.T\n")
    with pytest.raises(am.InvalidInputError):
        sc.grid(sources=[(0, 5)])  # out of bounds source
    g.close()
    sc.close()
