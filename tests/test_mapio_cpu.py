"""CPU part of the map / scene text suite: the oracle (oracle/mapio.py) against the
SPEC.md mapio examples, and the host-side Moving AI header parser of the product
library (am_movingai_header, no device work) against the oracle on 1000 seeded
header mutations."""
import numpy as np
import pytest

from tests.mapio_cases import (M, MOVINGAI_BAD, MOVINGAI_KATS, SCENE_BAD, SCENE_KATS, movingai_text, mutate,
                               oracle_parse, scene_text)
from tests.oracle_adapter import O

am = pytest.importorskip("paper_2004_00540_b200")


@pytest.mark.parametrize("text,rows", MOVINGAI_KATS)
def test_oracle_movingai_examples(text, rows):
    assert M.parse_movingai(text).tolist() == rows


@pytest.mark.parametrize("text,pos", MOVINGAI_BAD)
def test_oracle_movingai_errors(text, pos):
    with pytest.raises(M.ParseError) as e:
        M.parse_movingai(text)
    assert (e.value.line, e.value.column) == pos


@pytest.mark.parametrize("text,rows,src,tgt", SCENE_KATS)
def test_oracle_scene_examples(text, rows, src, tgt):
    occ, s, t = M.parse_ascii_scene(text)
    assert occ.tolist() == rows and s == src and t == tgt


@pytest.mark.parametrize("text,pos", SCENE_BAD)
def test_oracle_scene_errors(text, pos):
    with pytest.raises(M.ParseError) as e:
        M.parse_ascii_scene(text)
    assert (e.value.line, e.value.column) == pos
    with pytest.raises(M.InvalidInput):  # at least one S
        M.parse_ascii_scene(b"..\n.T\n")


def test_oracle_round_trips():
    occ = O.random_maze(37, 23, 0.35, 9)
    assert np.array_equal(M.parse_movingai(M.emit_movingai(occ)), occ)
    assert M.emit_movingai(occ) == movingai_text(occ)
    src, tgt = [(0, 1), (5, 5)], [(7, 2)]
    occ[0, 1] = occ[5, 5] = occ[7, 2] = 0
    t = M.emit_ascii_scene(occ, src, tgt)
    assert t == scene_text(occ, src, tgt)
    o2, s2, t2 = M.parse_ascii_scene(t)
    assert np.array_equal(o2, occ) and s2 == sorted(src) and t2 == tgt
    # idempotent after one normalisation
    norm = M.emit_ascii_scene(*M.parse_ascii_scene(b"S..\r\n.#T\r\n\r\n"))
    assert M.emit_ascii_scene(*M.parse_ascii_scene(norm)) == norm


def test_oracle_pgm_examples():
    # SPEC.md:359-361
    assert M.export_pgm(np.array([[2]], np.uint32)) == b"P5\n1 1\n255\n\xff"
    assert M.export_pgm(np.zeros((2, 3), np.uint32)) == b"P5\n3 2\n255\n" + bytes(6)
    # 9x9 empty grid, centre source, L=9: brightness decreases with BFS distance
    occ = np.zeros((9, 9), np.uint8)
    sm = O.source_mask(occ, [(4, 4)])
    vals = O.propagate(occ, sm, 9)
    body = np.frombuffer(M.export_pgm(vals)[len(b"P5\n9 9\n255\n"):], np.uint8).reshape(9, 9)
    d = O.bfs_multi_source(occ, sm)
    for a in range(81):
        for b in range(81):
            if d.flat[a] < d.flat[b]:
                assert body.flat[a] > body.flat[b]
    # 16-bit samples, big-endian, round-half-up
    v = np.array([[0, 1, 300, 599, 600]], np.uint32)
    out = M.export_pgm(v)
    assert out.startswith(b"P5\n5 1\n65535\n")
    q = np.frombuffer(out[len(b"P5\n5 1\n65535\n"):], ">u2")
    assert q.tolist() == [(2 * x * 65535 + 600) // 1200 for x in [0, 1, 300, 599, 600]]


def test_header_parser_matches_oracle_on_mutations():
    """Structured errors only, same position as the oracle."""
    rng = np.random.default_rng(2024)
    base = movingai_text(O.random_maze(13, 11, 0.3, 3))
    n_err = 0
    for i in range(1000):
        t = mutate(base, rng, header_only=True)
        exp = oracle_parse(M.movingai_header, t)
        try:
            got = ("ok", am.movingai_header(t))
        except am.ParseError as e:
            got = ("parse", e.line, e.column)
        assert got == exp, (i, t[:60], got, exp)
        n_err += got[0] != "ok"
    assert n_err > 300


def test_header_parser_valid():
    assert am.movingai_header(b"type octile\nheight 881\nwidth 767\nmap\n") == (767, 881, 37)
    assert am.movingai_header(b"type octile\r\nheight 3\r\nwidth 2\r\nmap\r\n..") == (2, 3, 37)
