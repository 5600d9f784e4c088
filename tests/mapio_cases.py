"""Shared inputs of the map / scene text tests: SPEC.md mapio examples and seeded
mutations of valid Moving AI maps and ASCII scenes ("rejects
every mutation of a valid header in a fuzz suite (no crashes, structured errors
only)")."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import mapio as M  # noqa: E402  (oracle/mapio.py)

# (text, expected occupancy rows or error line)
MOVINGAI_KATS = [
    (b"type octile\nheight 2\nwidth 2\nmap\n.@\n@.\n", [[0, 1], [1, 0]]),
    (b"type octile\nheight 2\nwidth 2\nmap\n.@\n@.", [[0, 1], [1, 0]]),
    (b"type octile\r\nheight 2\r\nwidth 2\r\nmap\r\n.@\r\n@.\r\n", [[0, 1], [1, 0]]),
    (b"type octile\nheight 1\nwidth 7\nmap\n.G@OTSW\n", [[0, 0, 1, 1, 1, 1, 1]]),
    (b"type octile\nheight 2\nwidth 2\nmap\n.@\n@.\n\n\n", [[0, 1], [1, 0]]),
    (b"type  octile\nheight\t2\nwidth 2\nmap\n..\n..\n", [[0, 0], [0, 0]]),
]
# header / body height mismatch -> a ParseError naming the line
MOVINGAI_BAD = [
    (b"type octile\nheight 3\nwidth 2\nmap\n..\n..\n", (7, 1)),
    (b"type octile\nheight 1\nwidth 2\nmap\n..\n..\n", (6, 1)),
    (b"type octile\nheight 2\nwidth 2\nmap\n...\n..\n", (5, 3)),
    (b"type octile\nheight 2\nwidth 2\nmap\n.\n..\n", (5, 2)),
    (b"type octile\nheight 2\nwidth 2\nmap\n..\n.x\n", (6, 2)),
    (b"type octile\nheight 2\nwidth 2\nmap\n..\n\n..\n", (6, 1)),
    (b"type octile\nheight 2\nwidth 2\nmap\n.\r.\n..\n", (5, 2)),
    (b"type octagon\nheight 2\nwidth 2\nmap\n..\n..\n", (1, 6)),
    (b"type octile\nwidth 2\nheight 2\nmap\n..\n..\n", (2, 1)),
    (b"type octile\nheight 0\nwidth 2\nmap\n", (2, 8)),
    (b"type octile\nheight 2\nwidth 65536\nmap\n", (3, 7)),
    (b"type octile\nheight 2x\nwidth 2\nmap\n", (2, 9)),
    (b"type octile\nheight 2\nwidth 2\n", (4, 1)),
    (b"type octile\nheight 2\nwidth 2\nmap extra\n..\n..\n", (4, 5)),
    (b"", (1, 1)),
]
SCENE_KATS = [
    (b"S.\n.T", [[0, 0], [0, 0]], [(0, 0)], [(1, 1)]),
    (b"S#\n#T", [[0, 1], [1, 0]], [(0, 0)], [(1, 1)]),
    (b"S.\r\n.T\r\n\r\n", [[0, 0], [0, 0]], [(0, 0)], [(1, 1)]),
    (b"..S\n#T#\nS.T\n", [[0, 0, 0], [1, 0, 1], [0, 0, 0]], [(0, 2), (2, 0)], [(1, 1), (2, 2)]),
]
SCENE_BAD = [
    (b"S.\n.T.\n", (2, 3)),
    (b"S.\n.\n", (2, 2)),
    (b"S.\n\n..\n", (2, 1)),
    (b"S?\n", (1, 2)),
    (b"\n\n", (1, 1)),
    (b"", (1, 1)),
    (b"\nS.\n", (1, 1)),
]


def movingai_text(occ, crlf=False, trailing=True):
    nl = b"\r\n" if crlf else b"\n"
    h, w = occ.shape
    rows = [bytes(np.where(occ[r] != 0, ord("@"), ord(".")).astype(np.uint8)) for r in range(h)]
    head = nl.join([b"type octile", b"height %d" % h, b"width %d" % w, b"map"]) + nl
    return head + nl.join(rows) + (nl if trailing else b"")


def scene_text(occ, src, tgt):
    g = np.where(occ != 0, ord("#"), ord(".")).astype(np.uint8)
    for r, c in tgt:
        g[r, c] = ord("T")
    for r, c in src:
        g[r, c] = ord("S")
    return b"".join(bytes(row) + b"\n" for row in g)


def mutate(text: bytes, rng, header_only=False):
    """One seeded mutation: replace / insert / delete a byte, or duplicate / drop a line."""
    b = bytearray(text)
    limit = text.find(b"map") + 4 if header_only and b"map" in text else len(b)
    limit = max(1, min(limit, len(b)))
    kind = rng.integers(0, 5)
    i = int(rng.integers(0, limit))
    alphabet = b".@#ST\n\r GOW0123456789 abcdefghijklmnopqrstuvwxyz\t-+x"
    ch = alphabet[int(rng.integers(0, len(alphabet)))]
    if kind == 0 and b:
        b[min(i, len(b) - 1)] = ch
    elif kind == 1:
        b.insert(i, ch)
    elif kind == 2 and b:
        del b[min(i, len(b) - 1)]
    else:
        lines = bytes(b).split(b"\n")
        j = int(rng.integers(0, len(lines)))
        if kind == 3:
            lines.insert(j, lines[j])
        else:
            del lines[j]
        b = bytearray(b"\n".join(lines))
    return bytes(b)


def oracle_parse(fn, text):
    """('ok', value) | ('parse', line, col) | ('invalid',)"""
    try:
        return ("ok", fn(text))
    except M.ParseError as e:
        return ("parse", e.line, e.column)
    except M.InvalidInput:
        return ("invalid",)
