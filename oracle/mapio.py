"""CPU restatement of the reference's map / scene text I/O -- TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module (as the checker); the product path parses
on the device (paper_2004_00540_b200/csrc/mapio.cu) and never calls it.

Follows /root/reference/proj/core/include/actmap/mapio.hpp:12-38 and the
mapio module of /root/reference/SPEC.md:323-390, plus the pins the reference
leaves open:
  P11 line ends '\\n' or '\\r\\n'; final newline optional; trailing empty lines
      ignored; a '\\r' anywhere else is an unknown byte.
  P12 Moving AI header: `type octile`, `height H`, `width W`, `map` in this
      order, tokens separated by spaces / tabs, H and W decimal in 1..65535.
  P13 PGM sample = round-half-up(v * maxval / max), header "P5\\n<W> <H>\\n<maxval>\\n",
      16-bit samples big-endian.
Plain Python loops: meant for the small fixtures and fuzz cases of the tests.
Parity pinned by the SPEC.md examples (tests/test_mapio_cpu.py).
"""
from __future__ import annotations

import numpy as np

MAX_DIM = 65535  # grid.hpp:14


class ParseError(Exception):
    """errors.hpp:23-38 -- message plus 1-based (line, column)."""

    def __init__(self, msg, line, column):
        super().__init__(f"{msg} (line {line}, column {column})")
        self.line, self.column = line, column


class InvalidInput(Exception):
    """errors.hpp:17 -- rejected input without a text position."""


def _lines(body: bytes):
    """P11: split on '\\n', strip one trailing '\\r', drop the empty tail and trailing empty lines."""
    parts = body.split(b"\n")
    if parts and parts[-1] == b"":
        parts.pop()  # text ended with a newline (or was empty)
    parts = [p[:-1] if p.endswith(b"\r") else p for p in parts]
    n_lines = len(parts)
    while parts and parts[-1] == b"":
        parts.pop()
    return parts, n_lines


def movingai_header(text: bytes):
    """mapio.hpp:19-22 header rules (P12) -> (width, height, body offset)."""
    keys = (b"type", b"height", b"width", b"map")
    pos = 0
    dims = []
    for ln, key in enumerate(keys, start=1):
        if pos >= len(text):
            raise ParseError(f"missing `{key.decode()}` line", ln, 1)
        e = text.find(b"\n", pos)
        raw = text[pos:] if e < 0 else text[pos:e]
        pos = len(text) if e < 0 else e + 1
        if raw.endswith(b"\r"):
            raw = raw[:-1]
        toks, i = [], 0
        while i < len(raw):
            while i < len(raw) and raw[i] in b" \t":
                i += 1
            if i >= len(raw):
                break
            b = i
            while i < len(raw) and raw[i] not in b" \t":
                i += 1
            toks.append((raw[b:i], b + 1))
        want = 1 if key == b"map" else 2
        if not toks or toks[0][0] != key:
            raise ParseError(f"expected `{key.decode()}`", ln, toks[0][1] if toks else 1)
        if len(toks) != want:
            raise ParseError("wrong value count", ln, toks[want][1] if len(toks) > want else len(raw) + 1)
        if key == b"type" and toks[1][0] != b"octile":
            raise ParseError("map type must be `octile`", ln, toks[1][1])
        if key in (b"height", b"width"):
            t, c = toks[1]
            for j, ch in enumerate(t):
                if not 48 <= ch <= 57:
                    raise ParseError("not a decimal number", ln, c + j)
            v = int(t)
            if not 1 <= v <= MAX_DIM:
                raise ParseError("outside 1..65535", ln, c)
            dims.append(v)
    return dims[1], dims[0], pos


_MAI = {ord("."): 0, ord("G"): 0, ord("@"): 1, ord("O"): 1, ord("T"): 1, ord("S"): 1, ord("W"): 1}
_ASC = {ord("."): 0, ord("#"): 1, ord("S"): 0, ord("T"): 0}


def _rows(lines, w, first_line, table):
    """Row checks in file order: first unknown byte, else length mismatch."""
    occ = np.zeros((len(lines), w), dtype=np.uint8)
    for r, row in enumerate(lines):
        for c, ch in enumerate(row[:w]):
            if ch not in table:
                raise ParseError(f"unexpected byte 0x{ch:02x}", first_line + r, c + 1)
            occ[r, c] = table[ch]
        if len(row) != w:
            raise ParseError("row length", first_line + r, min(len(row), w) + 1)
    return occ


def parse_movingai(text: bytes) -> np.ndarray:
    """mapio.hpp:19-23 -> occupancy (H, W) uint8, nonzero = obstacle."""
    w, h, off = movingai_header(text)
    lines, n_lines = _lines(text[off:])
    # rows inside the header's height (empty ones included) are checked first
    body_all = text[off:].split(b"\n")
    if body_all and body_all[-1] == b"":
        body_all.pop()
    body_all = [p[:-1] if p.endswith(b"\r") else p for p in body_all]
    occ = _rows(body_all[:h], w, 5, _MAI)
    if n_lines < h:
        raise ParseError(f"body has {n_lines} rows, the header says {h}", 5 + n_lines, 1)
    for i in range(h, len(body_all)):
        if body_all[i]:
            raise ParseError("more rows than the header's height", 5 + i, 1)
    return occ


def emit_movingai(occ) -> bytes:
    """mapio.hpp:25-26: canonical '.' / '@' re-emission."""
    occ = np.asarray(occ)
    h, w = occ.shape
    out = [f"type octile\nheight {h}\nwidth {w}\nmap\n".encode()]
    for r in range(h):
        out.append(bytes(64 if occ[r, c] else 46 for c in range(w)) + b"\n")
    return b"".join(out)


def parse_ascii_scene(text: bytes):
    """mapio.hpp:28-30 -> (occupancy, sources [(r, c)], targets [(r, c)]) in row-major order."""
    lines, _ = _lines(text)
    if not lines:
        raise ParseError("no rows", 1, 1)
    w = len(lines[0])
    if w == 0:
        raise ParseError("empty first row", 1, 1)
    if w > MAX_DIM:
        raise ParseError("row longer than 65535 cells", 1, MAX_DIM + 1)
    if len(lines) > MAX_DIM:
        raise ParseError("more than 65535 rows", MAX_DIM + 1, 1)
    occ = _rows(lines, w, 1, _ASC)
    src = [(r, c) for r, row in enumerate(lines) for c, ch in enumerate(row) if ch == ord("S")]
    tgt = [(r, c) for r, row in enumerate(lines) for c, ch in enumerate(row) if ch == ord("T")]
    if not src:
        raise InvalidInput("no source ('S') cell")
    return occ, src, tgt


def emit_ascii_scene(occ, sources, targets) -> bytes:
    """mapio.hpp:32: '.', '#', then 'T' targets, then 'S' sources (a cell in both reads 'S')."""
    occ = np.asarray(occ)
    h, w = occ.shape
    grid = [[35 if occ[r, c] else 46 for c in range(w)] for r in range(h)]
    for r, c in targets:
        grid[r][c] = 84
    for r, c in sources:
        grid[r][c] = 83
    return b"".join(bytes(row) + b"\n" for row in grid)


def export_pgm(vals) -> bytes:
    """mapio.hpp:35-38 + P13 (numpy, any size)."""
    v = np.asarray(vals, dtype=np.uint64)
    h, w = v.shape
    mx = int(v.max()) if v.size else 0
    maxval = 65535 if mx > 255 else 255
    if mx:
        q = (2 * v * maxval + mx) // (2 * mx)
    else:
        q = np.zeros_like(v)
    head = f"P5\n{w} {h}\n{maxval}\n".encode()
    body = q.astype(np.uint8).tobytes() if maxval == 255 else q.astype(">u2").tobytes()
    return head + body
