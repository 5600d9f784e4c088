"""ctypes view of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs -- never by the
product package.  See actmap_oracle.h for what each function restates and
how the oracle is pinned (SPEC.md KATs + closed-form law + sentinel kernel).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ORACLE_LIB: an alternative build of the same sources (bench.py builds `make native`, -march=native, on the
# host it times; the default .so is portable x86-64-v3)
_LIB_PATH = os.environ.get("ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")

OK, EINVAL, EUNCOVERED, EINTERNAL = 0, 1, 2, 6
UNREACH = 0xFFFFFFFF
MAX_LAYERS = 2147483646
FILLED, STALLED, CAP = 0, 1, 2
STRICT, PERMISSIVE = 0, 1
BATCHED, ITERATIVE = 0, 1

_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no reference build system)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


def _declare(L):
    u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double
    sig = {
        "or_splitmix64": (u64, [_u64p]),
        "or_random_maze": (i32, [u32, u32, dbl, u64, _u8p]),
        "or_comb_maze": (i32, [u32, u32, _u8p]),
        "or_kruskal_maze": (i32, [u32, u32, u64, _u8p]),
        "or_city_grid": (i32, [u32, u32, u64, _u8p]),
        "or_sample_free_cells": (i32, [u32, u32, _u8p, u64, u64, _u8p, _u32p]),
        "or_source_mask": (i32, [u32, u32, _u8p, _u32p, u64, _u8p]),
        "or_initial": (i32, [u32, u32, _u8p, _u8p, _u32p]),
        "or_propagate_layer": (i32, [u32, u32, _u8p, _u8p, _u32p, _u32p, i32]),
        "or_propagate": (i32, [u32, u32, _u8p, _u8p, u32, i32, i32, _u32p]),
        "or_propagate_auto": (i32, [u32, u32, _u8p, _u8p, u32, i32, _u32p, _u32p, C.POINTER(C.c_int)]),
        "or_propagate_reference": (i32, [u32, u32, _u8p, _u8p, u32, _u32p]),
        "or_layer_bound": (None, [u32, u32, _u64p, _u32p, _u32p]),
        "or_zero_free_cells": (u64, [u32, u32, _u8p, _u32p]),
        "or_bfs_multi_source": (i32, [u32, u32, _u8p, _u8p, _u32p]),
        "or_bfs_from": (i32, [u32, u32, _u8p, u32, u32, _u32p]),
        "or_dijkstra_octile": (i32, [u32, u32, _u8p, _u8p, i32, _i64p, _i64p]),
        "or_check_activity": (u64, [u32, u32, _u8p, _u32p, _u32p, u32, _u32p, u32]),
        "or_reconstruct_simple": (i32, [u32, u32, _u8p, _u8p, _u32p, u32, u32, u64, _u32p, u64, _u64p]),
        "or_reconstruct_euclidean": (i32, [u32, u32, _u8p, _u8p, _u32p, u32, u32, i32, _u32p, u64, _u64p]),
        "or_straighten": (i32, [_u32p, u64, _u8p, u32, u32, i32, _u32p, _u64p]),
        "or_path_metrics": (None, [_u32p, u64, _u64p, C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _p(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle status {code} {what}")
        self.code = code


def _chk(st, what=""):
    if st != OK:
        raise OracleError(st, what)


# ---------------------------------------------------------------- generators
def random_maze(w, h, density, seed):
    occ = np.empty((h, w), np.uint8)
    _chk(lib().or_random_maze(w, h, density, seed, _p(occ, _u8p)), "random_maze")
    return occ


def comb_maze(w, h):
    occ = np.empty((h, w), np.uint8)
    _chk(lib().or_comb_maze(w, h, _p(occ, _u8p)), "comb_maze")
    return occ


def kruskal_maze(w, h, seed):
    occ = np.empty((h, w), np.uint8)
    _chk(lib().or_kruskal_maze(w, h, seed, _p(occ, _u8p)), "kruskal_maze")
    return occ


def city_grid(w, h, seed):
    occ = np.empty((h, w), np.uint8)
    _chk(lib().or_city_grid(w, h, seed, _p(occ, _u8p)), "city_grid")
    return occ


def sample_free_cells(occ, n, seed, exclude=None):
    occ = _u8(occ)
    h, w = occ.shape
    out = np.empty((n, 2), np.uint32)
    ex = None if exclude is None else _u8(exclude)
    _chk(lib().or_sample_free_cells(w, h, _p(occ, _u8p), n, seed, _p(ex, _u8p), _p(out, _u32p)), "sample")
    return out


def source_mask(occ, sources):
    occ = _u8(occ)
    h, w = occ.shape
    src = _u32(np.asarray(sources, dtype=np.uint32).reshape(-1, 2))
    m = np.empty((h, w), np.uint8)
    _chk(lib().or_source_mask(w, h, _p(occ, _u8p), _p(src, _u32p), len(src), _p(m, _u8p)), "source_mask")
    return m


# ---------------------------------------------------------------- propagation
def initial(occ, srcmask):
    occ, sm = _u8(occ), _u8(srcmask)
    h, w = occ.shape
    out = np.empty((h, w), np.uint32)
    lib().or_initial(w, h, _p(occ, _u8p), _p(sm, _u8p), _p(out, _u32p))
    return out


def propagate_layer(occ, srcmask, act, threads=1, out=None):
    """out: optional preallocated (h, w) uint32 C-contiguous buffer (no allocation inside a timed loop)."""
    occ, sm, a = _u8(occ), _u8(srcmask), _u32(act)
    h, w = occ.shape
    if out is None or out.shape != (h, w) or out.dtype != np.uint32 or not out.flags.c_contiguous:
        out = np.empty((h, w), np.uint32)
    _chk(lib().or_propagate_layer(w, h, _p(occ, _u8p), _p(sm, _u8p), _p(a, _u32p), _p(out, _u32p), threads))
    return out


def propagate(occ, srcmask, layers, mode=BATCHED, threads=1):
    occ, sm = _u8(occ), _u8(srcmask)
    h, w = occ.shape
    out = np.empty((h, w), np.uint32)
    _chk(lib().or_propagate(w, h, _p(occ, _u8p), _p(sm, _u8p), layers, mode, threads, _p(out, _u32p)), "propagate")
    return out


def propagate_auto(occ, srcmask, auto_cap, threads=1):
    occ, sm = _u8(occ), _u8(srcmask)
    h, w = occ.shape
    out = np.empty((h, w), np.uint32)
    lu = C.c_uint32(0)
    cause = C.c_int(0)
    _chk(lib().or_propagate_auto(w, h, _p(occ, _u8p), _p(sm, _u8p), auto_cap, threads, _p(out, _u32p),
                                 C.byref(lu), C.byref(cause)), "propagate_auto")
    return out, lu.value, cause.value


def propagate_reference(occ, srcmask, layers):
    occ, sm = _u8(occ), _u8(srcmask)
    h, w = occ.shape
    out = np.empty((h, w), np.uint32)
    _chk(lib().or_propagate_reference(w, h, _p(occ, _u8p), _p(sm, _u8p), layers, _p(out, _u32p)), "reference")
    return out


def layer_bound(w, h):
    worst, lo, hi = C.c_uint64(0), C.c_uint32(0), C.c_uint32(0)
    lib().or_layer_bound(w, h, C.byref(worst), C.byref(lo), C.byref(hi))
    return worst.value, lo.value, hi.value


def zero_free_cells(occ, vals):
    occ, v = _u8(occ), _u32(vals)
    h, w = occ.shape
    return lib().or_zero_free_cells(w, h, _p(occ, _u8p), _p(v, _u32p))


# ---------------------------------------------------------------- oracles
def bfs_multi_source(occ, srcmask):
    occ, sm = _u8(occ), _u8(srcmask)
    h, w = occ.shape
    out = np.empty((h, w), np.uint32)
    lib().or_bfs_multi_source(w, h, _p(occ, _u8p), _p(sm, _u8p), _p(out, _u32p))
    return out


def bfs_from(occ, row, col):
    occ = _u8(occ)
    h, w = occ.shape
    out = np.empty((h, w), np.uint32)
    _chk(lib().or_bfs_from(w, h, _p(occ, _u8p), row, col, _p(out, _u32p)), "bfs_from")
    return out


def dijkstra_octile(occ, srcmask, rule=STRICT):
    occ, sm = _u8(occ), _u8(srcmask)
    h, w = occ.shape
    a = np.empty((h, w), np.int64)
    b = np.empty((h, w), np.int64)
    lib().or_dijkstra_octile(w, h, _p(occ, _u8p), _p(sm, _u8p), rule, _p(a, _i64p), _p(b, _i64p))
    return a, b


def check_activity(occ, vals, hops, layers, max_samples=16):
    occ, v, hp = _u8(occ), _u32(vals), _u32(hops)
    h, w = occ.shape
    s = np.zeros((max_samples, 2), np.uint32)
    bad = lib().or_check_activity(w, h, _p(occ, _u8p), _p(v, _u32p), _p(hp, _u32p), layers, _p(s, _u32p),
                                  max_samples)
    return bad, [tuple(x) for x in s[: min(bad, max_samples)]]


# ---------------------------------------------------------------- paths
def _path_cap(vals):
    return int(np.max(vals)) + 2 if vals.size else 2


def reconstruct_simple(occ, srcmask, vals, target, seed, cap=None):
    """cap: point capacity (defaults to max(vals)+2; pass layers+2 on big maps)."""
    occ, sm, v = _u8(occ), _u8(srcmask), _u32(vals)
    h, w = occ.shape
    cap = cap or _path_cap(v)
    pts = np.empty((cap, 2), np.uint32)
    n = C.c_uint64(0)
    st = lib().or_reconstruct_simple(w, h, _p(occ, _u8p), _p(sm, _u8p), _p(v, _u32p), int(target[0]),
                                     int(target[1]), seed, _p(pts, _u32p), cap, C.byref(n))
    return st, pts[: n.value].copy()


def reconstruct_euclidean(occ, srcmask, vals, target, rule=STRICT, cap=None):
    occ, sm, v = _u8(occ), _u8(srcmask), _u32(vals)
    h, w = occ.shape
    cap = cap or _path_cap(v)
    pts = np.empty((cap, 2), np.uint32)
    n = C.c_uint64(0)
    st = lib().or_reconstruct_euclidean(w, h, _p(occ, _u8p), _p(sm, _u8p), _p(v, _u32p), int(target[0]),
                                        int(target[1]), rule, _p(pts, _u32p), cap, C.byref(n))
    return st, pts[: n.value].copy()


def straighten(points, occ=None, rule=STRICT):
    pts = _u32(np.asarray(points, dtype=np.uint32).reshape(-1, 2))
    out = np.empty_like(pts)
    n = C.c_uint64(0)
    if occ is None:
        lib().or_straighten(_p(pts, _u32p), len(pts), None, 0, 0, rule, _p(out, _u32p), C.byref(n))
    else:
        o = _u8(occ)
        lib().or_straighten(_p(pts, _u32p), len(pts), _p(o, _u8p), o.shape[1], o.shape[0], rule,
                            _p(out, _u32p), C.byref(n))
    return out[: n.value].copy()


def path_metrics(points):
    pts = _u32(np.asarray(points, dtype=np.uint32).reshape(-1, 2))
    steps, length = C.c_uint64(0), C.c_double(0)
    lib().or_path_metrics(_p(pts, _u32p), len(pts), C.byref(steps), C.byref(length))
    return steps.value, length.value
