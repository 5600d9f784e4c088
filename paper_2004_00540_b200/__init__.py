"""B200-native oMAP hot path (arXiv 2004.00540) -- Python mirror of the actmap:: API.

Thin ctypes layer over the C ABI in ``include/actmap_b200.h`` (library
``libactmap_b200.so``, built in-tree for sm_100a).  Names, argument meaning and
error behaviour follow the reference planner API
(/root/reference/proj/core/include/actmap/propagate.hpp, reconstruct.hpp,
grid.hpp, errors.hpp).  All compute runs in the CUDA library; there is no
CPU fallback -- importing works without a GPU, the first device call raises
``Error`` if the extension or the device is missing.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACTMAP_LIB") or os.path.join(_HERE, "libactmap_b200.so")  # override: A/B kernel builds

OK, EINVAL, EUNCOVERED, ECUDA, EOOM, ENCCL, EINTERNAL = 0, 1, 2, 3, 4, 5, 6
FILLED, STALLED, CAP, FIXED = 0, 1, 2, 3          # AutoStop (propagate.hpp:45-49) + fixed
BATCHED, ITERATIVE = 0, 1                          # Mode (propagate.hpp:22)
SIMPLE, EUCLIDEAN = 0, 1                           # Method (report.hpp:15)
STRICT, PERMISSIVE = 0, 1                          # CornerRule (reconstruct.hpp:14)
MOVINGAI, ASCII_SCENE = 0, 1                      # text formats (mapio.hpp:19-33)
CTX_TIMING = 1
CTX_DENSE = 2
K_MAX_LAYERS = 2147483646                          # propagate.hpp:15-16
K_MAX_GRID_DIM = 65535                             # grid.hpp:14


class Error(RuntimeError):
    """actmap::Error (errors.hpp:10)."""


class InvalidInputError(Error):
    """actmap::InvalidInputError (errors.hpp:17)."""


class UncoveredTargetError(Error):
    """actmap::UncoveredTargetError (errors.hpp:41)."""


class ParseError(InvalidInputError):
    """actmap::ParseError (errors.hpp:23-38): malformed map / scene text, 1-based position."""

    def __init__(self, msg: str, line: int, column: int):
        super().__init__(f"{msg} (line {line}, column {column})")
        self.line = line
        self.column = column


class _PropResult(C.Structure):
    _fields_ = [("layers_used", C.c_uint32), ("cause", C.c_uint32), ("layers_computed", C.c_uint32),
                ("cell_bits", C.c_uint32), ("block_launches", C.c_uint64), ("layer_launches", C.c_uint64),
                ("stencil_ms", C.c_double), ("tiles_processed", C.c_uint64), ("tiles_total", C.c_uint64),
                ("cells_executed", C.c_uint64), ("engine", C.c_uint32), ("block_layers", C.c_uint32)]


class _GridInfo(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("width", "height", "pitch", "rows", "bands", "segments", "seg_len",
                                           "halo", "cell_bits", "layers_used", "layers_computed", "tile_rows",
                                           "tile_cols", "tiles")]


class _CtxOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("flags", C.c_uint32)]


class _ParseInfo(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("n_sources", C.c_uint64),
                ("n_targets", C.c_uint64), ("obstacles", C.c_uint64), ("error_line", C.c_uint64),
                ("error_column", C.c_uint64), ("error", C.c_char * 160)]


class _Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("pool_reserved", C.c_uint64), ("pool_used", C.c_uint64),
                ("h2d_bytes", C.c_uint64)]


_lib = None
_lock = threading.RLock()
_vp, _u8p, _u32p, _u64p, _i32p = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), \
    C.POINTER(C.c_int32)


def lib():
    """Loads libactmap_b200.so (raises Error if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Error(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        st, u32, u64 = C.c_int, C.c_uint32, C.c_uint64
        sig = {
            "am_ctx_create": (st, [C.POINTER(_CtxOpts), C.POINTER(_vp)]),
            "am_ctx_destroy": (None, [_vp]),
            "am_last_error": (C.c_char_p, [_vp]),
            "am_ctx_stats": (st, [_vp, C.POINTER(_Stats)]),
            "am_ctx_synchronize": (st, [_vp]),
            "am_ctx_trim": (st, [_vp]),
            "am_bench_tile_kernel": (st, [_vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_float)]),
            "am_ctx_get_stream": (st, [_vp, C.POINTER(_vp)]),
            "am_grid_create": (st, [_vp, u32, u32, _vp, _vp, u64, C.POINTER(_vp)]),
            "am_grid_create_device": (st, [_vp, u32, u32, _vp, _vp, u64, C.POINTER(_vp)]),
            "am_grid_destroy": (st, [_vp, _vp]),
            "am_grid_clone": (st, [_vp, _vp, C.POINTER(_vp)]),
            "am_grid_get_info": (st, [_vp, C.POINTER(_GridInfo)]),
            "am_propagate": (st, [_vp, _vp, u32, u32, u32, C.POINTER(_PropResult)]),
            "am_activity_download": (st, [_vp, _vp, _vp]),
            "am_activity_download_device": (st, [_vp, _vp, _vp]),
            "am_activity_upload": (st, [_vp, _vp, _vp, u32]),
            "am_path_counts": (st, [_vp, _vp, _vp, u64, u32, u64, _vp, _vp]),
            "am_trace_paths": (st, [_vp, _vp, _vp, u64, u32, u64, _vp, _vp, u64, _vp]),
            "am_trace_paths_device": (st, [_vp, _vp, _vp, u64, u32, u64, _vp, _vp, u64, _vp]),
            "am_propagate_layer": (st, [_vp, u32, u32, _vp, _vp, u64, _vp, _vp]),
            "am_propagate_reference": (st, [_vp, u32, u32, _vp, _vp, u64, u32, _vp]),
            "am_grid_create_slab": (st, [_vp, u32, u32, u32, u32, _vp, _vp, u64, C.POINTER(_vp)]),
            "am_slabs_propagate": (st, [_vp, C.POINTER(_vp), u32, u32, u32, u32, C.POINTER(_PropResult)]),
            "am_slabs_gather": (st, [_vp, C.POINTER(_vp), u32, _vp]),
            "am_comm_unique_id": (st, [_vp]),
            "am_comm_init": (st, [_vp, u32, u32, _vp]),
            "am_comm_slab_rows": (st, [_vp, u32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
            "am_comm_gather": (st, [_vp, _vp, _vp]),
            "am_slab_rows": (st, [u32, u32, u32, C.POINTER(u32), C.POINTER(u32)]),
            "am_peer_export": (st, [_vp, _vp, _vp]),
            "am_peer_connect": (st, [_vp, _vp, u32, u32, _vp]),
            "am_peer_gather": (st, [_vp, _vp, _vp]),
            "am_peer_trace_paths_device": (st, [_vp, _vp, _vp, u64, u32, u64, _vp, _vp, u64, _vp]),
            "am_batch_create": (st, [_vp, u32, u32, u32, _vp, _vp, _vp, C.POINTER(_vp)]),
            "am_batch_destroy": (st, [_vp, _vp]),
            "am_batch_propagate": (st, [_vp, _vp, u32, u32, _vp, _vp, C.POINTER(_PropResult)]),
            "am_batch_download": (st, [_vp, _vp, _vp]),
            "am_batch_path_counts": (st, [_vp, _vp, _vp, u64, u32, u64, _vp, _vp]),
            "am_batch_trace_paths": (st, [_vp, _vp, _vp, u64, u32, u64, _vp, _vp, u64, _vp]),
            "am_movingai_header": (st, [C.c_char_p, u64, C.POINTER(_ParseInfo), _u64p]),
            "am_scene_parse": (st, [_vp, C.c_char_p, u64, u32, C.POINTER(_vp), C.POINTER(_ParseInfo)]),
            "am_scene_destroy": (st, [_vp, _vp]),
            "am_scene_download": (st, [_vp, _vp, _vp, _vp, _vp]),
            "am_grid_create_scene": (st, [_vp, _vp, _vp, u64, C.POINTER(_vp)]),
            "am_emit_text": (st, [_vp, u32, u32, u32, _vp, _vp, u64, _vp, u64, _vp, u64, _u64p]),
            "am_activity_export_pgm": (st, [_vp, _vp, _vp, u64, _u64p]),
            "am_export_pgm": (st, [_vp, u32, u32, _vp, _vp, u64, _u64p]),
            "am_random_maze": (st, [u32, u32, C.c_double, u64, _vp]),
            "am_comb_maze": (st, [u32, u32, _vp]),
            "am_kruskal_maze": (st, [u32, u32, u64, _vp]),
            "am_city_grid": (st, [u32, u32, u64, _vp]),
            "am_straighten": (st, [_vp, u64, _vp, u32, u32, u32, _vp, _u64p]),
            "am_path_metrics": (st, [_vp, u64, _u64p, C.POINTER(C.c_double)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _raise(st, ctx, what):
    msg = what
    if ctx is not None and ctx.handle:
        err = lib().am_last_error(ctx.handle)
        if err:
            msg = f"{what}: {err.decode(errors='replace')}"
    if st == EINVAL:
        raise InvalidInputError(msg)
    if st == EUNCOVERED:
        raise UncoveredTargetError(msg)
    raise Error(f"{msg} (status {st})")


def _check(st, ctx, what):
    if st != OK:
        _raise(st, ctx, what)


class Context:
    """One CUDA device + stream (am_ctx).  Externally synchronised."""

    def __init__(self, device: int = 0, timing: bool = False, dense: bool = False):
        h = C.c_void_p()
        opts = _CtxOpts(device, (CTX_TIMING if timing else 0) | (CTX_DENSE if dense else 0))
        st = lib().am_ctx_create(C.byref(opts), C.byref(h))
        if st != OK:
            raise Error(f"cannot create a B200 context on device {device} (status {st})")
        self.handle = h
        self.device = device
        self._owned = weakref.WeakSet()  # grids / batches: closed before the context
        _live_contexts.add(self)

    def _own(self, obj):
        self._owned.add(obj)

    def close(self):
        if self.handle:
            for o in list(self._owned):
                o.close()
            lib().am_ctx_destroy(self.handle)
            self.handle = None

    def pool_bytes(self) -> tuple[int, int]:
        """(reserved, in use) device bytes of the context's memory pool."""
        s = _Stats()
        _check(lib().am_ctx_stats(self.handle, C.byref(s)), self, "stats")
        return s.pool_reserved, s.pool_used

    def h2d_bytes(self) -> int:
        """Host-to-device bytes this context has copied so far (am_stats.h2d_bytes)."""
        s = _Stats()
        _check(lib().am_ctx_stats(self.handle, C.byref(s)), self, "stats")
        return s.h2d_bytes

    def trim(self):
        """Return the pool's cached (unused) device memory to the driver (am_ctx_trim)."""
        _check(lib().am_ctx_trim(self.handle), self, "trim")

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def kernel_launches(self) -> int:
        s = _Stats()
        _check(lib().am_ctx_stats(self.handle, C.byref(s)), self, "stats")
        return s.kernel_launches

    def synchronize(self):
        _check(lib().am_ctx_synchronize(self.handle), self, "synchronize")

    def stream_ptr(self) -> int:
        """cudaStream_t of this context (wrap with torch.cuda.ExternalStream for events)."""
        s = C.c_void_p()
        _check(lib().am_ctx_get_stream(self.handle, C.byref(s)), self, "stream")
        return s.value or 0

    # ---- multi-GPU (one process per GPU, NCCL) ----
    def comm_init(self, nranks: int, rank: int, unique_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().am_comm_init(self.handle, nranks, rank, C.cast(buf, C.c_void_p)), self, "comm_init")

    def slab_rows(self, height: int):
        a, b = C.c_uint32(0), C.c_uint32(0)
        _check(lib().am_comm_slab_rows(self.handle, height, C.byref(a), C.byref(b)), self, "slab_rows")
        return a.value, b.value

    def comm_gather(self, slab: "Grid", full: "Grid"):
        _check(lib().am_comm_gather(self.handle, slab.handle, full.handle), self, "comm_gather")
        full.layers = slab.layers

    def trace_device(self, grid: "Grid", d_tgt: int, n: int, method: int, seed: int, d_offsets: int, d_pts: int,
                     cap: int, d_status: int):
        """am_trace_paths_device: device pointers in, no host round trip."""
        _check(lib().am_trace_paths_device(self.handle, grid.handle, C.c_void_p(d_tgt), n, method, seed,
                                           C.c_void_p(d_offsets), C.c_void_p(d_pts), cap, C.c_void_p(d_status)),
               self, "trace_device")


_default = None
_live_contexts = weakref.WeakSet()


@atexit.register
def _close_contexts():
    """Destroy every live context (its grids first) while the CUDA runtime is still up: a context left to the
    garbage collector at interpreter teardown would release its stream and pool after torch / cudart shut down."""
    for c in list(_live_contexts):
        try:
            c.close()
        except Exception:
            pass


def default_context() -> Context:
    global _default
    with _lock:
        if _default is None:
            _default = Context(int(os.environ.get("ACTMAP_DEVICE", "0")))
        return _default


def _occ(occupancy):
    occ = np.ascontiguousarray(occupancy, dtype=np.uint8)
    if occ.ndim != 2:
        raise InvalidInputError("occupancy must be a 2-D (height, width) array")
    return occ


def _rc(points):
    a = np.ascontiguousarray(np.asarray(points, dtype=np.uint32).reshape(-1, 2))
    return a


class PropResult:
    def __init__(self, r: _PropResult):
        self.layers_used = r.layers_used
        self.cause = r.cause
        self.layers_computed = r.layers_computed
        self.cell_bits = r.cell_bits
        self.block_launches = r.block_launches
        self.layer_launches = r.layer_launches
        self.stencil_ms = r.stencil_ms
        self.tiles_processed = r.tiles_processed
        self.tiles_total = r.tiles_total
        self.cells_executed = r.cells_executed
        self.engine = ("dense", "tiles", "bits", "batch")[r.engine] if r.engine < 4 else str(r.engine)
        self.block_layers = r.block_layers


class Grid:
    """GridMap + SourceSet resident on the device (am_grid), plus its activity map."""

    def __init__(self, occupancy, sources, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.occ = _occ(occupancy)
        self.height, self.width = self.occ.shape
        src = _rc(sources)
        h = C.c_void_p()
        _check(lib().am_grid_create(self.ctx.handle, self.width, self.height, _ptr(self.occ), _ptr(src), len(src),
                                    C.byref(h)), self.ctx, "SourceSet/grid")
        self.handle = h
        self.ctx._own(self)
        self.layers = 0

    @classmethod
    def from_device(cls, width, height, d_occ_ptr: int, d_src_ptr: int, n_src: int, ctx: Context | None = None):
        """Inputs already resident in HBM (device pointers)."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.occ = None
        self.width, self.height = width, height
        h = C.c_void_p()
        _check(lib().am_grid_create_device(self.ctx.handle, width, height, C.c_void_p(d_occ_ptr),
                                           C.c_void_p(d_src_ptr), n_src, C.byref(h)), self.ctx, "grid")
        self.handle = h
        self.ctx._own(self)
        self.layers = 0
        return self

    @classmethod
    def slab(cls, occupancy_full, sources, row0: int, row1: int, ctx: Context | None = None):
        """Rows [row0, row1) of the full grid as a row slab (multi-GPU decomposition)."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        occ = _occ(occupancy_full)
        self.occ = None
        self.height, self.width = row1 - row0, occ.shape[1]
        src = _rc(sources)
        h = C.c_void_p()
        _check(lib().am_grid_create_slab(self.ctx.handle, occ.shape[1], occ.shape[0], row0, row1, _ptr(occ),
                                         _ptr(src), len(src), C.byref(h)), self.ctx, "slab")
        self.handle = h
        self.ctx._own(self)
        self.layers = 0
        self.row0, self.row1 = row0, row1
        return self

    def close(self):
        if getattr(self, "handle", None):
            lib().am_grid_destroy(self.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = _GridInfo()
        _check(lib().am_grid_get_info(self.handle, C.byref(i)), self.ctx, "info")
        return {n: getattr(i, n) for n, _ in _GridInfo._fields_}

    def propagate(self, layers: int, mode: int = BATCHED) -> PropResult:
        if layers < 1:
            raise InvalidInputError("propagate: L must be >= 1")
        r = _PropResult()
        _check(lib().am_propagate(self.ctx.handle, self.handle, layers, 0, mode, C.byref(r)), self.ctx, "propagate")
        self.layers = r.layers_used
        return PropResult(r)

    def propagate_auto(self, auto_cap: int) -> PropResult:
        r = _PropResult()
        _check(lib().am_propagate(self.ctx.handle, self.handle, 0, auto_cap, BATCHED, C.byref(r)), self.ctx,
               "propagate_auto")
        self.layers = r.layers_used
        return PropResult(r)

    def activity(self, out=None) -> np.ndarray:
        if out is None:
            out = np.empty((self.height, self.width), np.uint32)
        _check(lib().am_activity_download(self.ctx.handle, self.handle, _ptr(out)), self.ctx, "download")
        return out

    def activity_to_device(self, d_ptr: int):
        _check(lib().am_activity_download_device(self.ctx.handle, self.handle, C.c_void_p(d_ptr)), self.ctx,
               "download")

    def upload_activity(self, values, layers_applied: int):
        v = np.ascontiguousarray(values, dtype=np.uint32)
        if v.shape != (self.height, self.width):
            raise InvalidInputError("activity/grid dimension mismatch")
        _check(lib().am_activity_upload(self.ctx.handle, self.handle, _ptr(v), layers_applied), self.ctx, "upload")
        self.layers = layers_applied

    def bench_tile_kernel(self, items: int, stride: int = 1, reps: int = 20) -> float:
        """Mean launch time (ms) of the active-tile kernel on `items` tile pairs (am_bench_tile_kernel)."""
        ms = C.c_float()
        _check(lib().am_bench_tile_kernel(self.ctx.handle, self.handle, items, stride, reps, C.byref(ms)), self.ctx,
               "bench tile kernel")
        return ms.value

    def path_counts(self, targets, method=EUCLIDEAN, seed=0):
        t = _rc(targets)
        off = np.zeros(len(t) + 1, np.uint64)
        st = np.zeros(len(t), np.int32)
        _check(lib().am_path_counts(self.ctx.handle, self.handle, _ptr(t), len(t), method, seed, _ptr(off),
                                    _ptr(st)), self.ctx, "path counts")
        return off, st

    def trace(self, targets, method=EUCLIDEAN, seed=0, out=None):
        """Batched path extraction: returns (offsets, points (total, 2), status).

        out: optional preallocated (e.g. pinned) uint32 array of shape (>= total, 2) for the points."""
        t = _rc(targets)
        off, st = self.path_counts(t, method, seed)
        total = int(off[-1])
        if out is not None and out.dtype == np.uint32 and out.ndim == 2 and out.shape[1] == 2 and \
                out.shape[0] >= max(total, 1) and out.flags.c_contiguous:
            pts = out
        else:
            pts = np.empty((max(total, 1), 2), np.uint32)
        _check(lib().am_trace_paths(self.ctx.handle, self.handle, _ptr(t), len(t), method, seed, _ptr(off),
                                    _ptr(pts), total, _ptr(st)), self.ctx, "trace")
        return off, pts[:total], st

    def paths(self, targets, method=EUCLIDEAN, seed=0):
        off, pts, st = self.trace(targets, method, seed)
        out = []
        for i in range(len(st)):
            if st[i] != OK:
                out.append((int(st[i]), None))
                continue
            p = pts[off[i]:off[i + 1]]
            keep = p[:, 0] != 0xFFFFFFFF
            out.append((OK, p[keep]))
        return out

    def export_pgm(self) -> bytes:
        """export_pgm (mapio.hpp:35-38) of this grid's map, rescaled on the device."""
        n = C.c_uint64(0)
        _check(lib().am_activity_export_pgm(self.ctx.handle, self.handle, None, 0, C.byref(n)), self.ctx, "pgm")
        buf = np.empty(n.value, dtype=np.uint8)
        _check(lib().am_activity_export_pgm(self.ctx.handle, self.handle, _ptr(buf), n.value, C.byref(n)), self.ctx,
               "pgm")
        return buf.tobytes()


class Batch:
    """Many independent small mazes solved in one device run (config C5)."""

    def __init__(self, occupancy, sources, ctx: Context | None = None):
        """occupancy: (n, h, w) uint8; sources: list of (k_i, 2) arrays of maze-local (row, col)."""
        self.ctx = ctx or default_context()
        occ = np.ascontiguousarray(occupancy, dtype=np.uint8)
        if occ.ndim != 3:
            raise InvalidInputError("occupancy must be (n, height, width)")
        self.n, self.height, self.width = occ.shape
        if len(sources) != self.n:
            raise InvalidInputError("one source list per maze")
        src_off = np.zeros(self.n + 1, np.uint64)
        src_off[1:] = np.cumsum([len(np.asarray(s).reshape(-1, 2)) for s in sources])
        src = np.ascontiguousarray(np.concatenate([np.asarray(s, np.uint32).reshape(-1, 2) for s in sources]),
                                   dtype=np.uint32)
        h = C.c_void_p()
        _check(lib().am_batch_create(self.ctx.handle, self.n, self.width, self.height, _ptr(occ), _ptr(src_off),
                                     _ptr(src), C.byref(h)), self.ctx, "batch")
        self.handle = h
        self.ctx._own(self)

    def close(self):
        if getattr(self, "handle", None):
            lib().am_batch_destroy(self.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def propagate(self, layers: int = 0, auto_cap: int = 0):
        """layers>0: fixed L for every maze; else auto with auto_cap.  -> (layers_used[n], cause[n], PropResult)."""
        lu = np.zeros(self.n, np.uint32)
        cause = np.zeros(self.n, np.uint32)
        r = _PropResult()
        _check(lib().am_batch_propagate(self.ctx.handle, self.handle, layers, auto_cap, _ptr(lu), _ptr(cause),
                                        C.byref(r)), self.ctx, "batch propagate")
        return lu, cause, PropResult(r)

    def activity(self) -> np.ndarray:
        out = np.empty((self.n, self.height, self.width), np.uint32)
        _check(lib().am_batch_download(self.ctx.handle, self.handle, _ptr(out)), self.ctx, "batch download")
        return out

    def trace(self, targets, method=EUCLIDEAN, seed=0, out=None):
        """targets: (k, 3) (maze, row, col) -> (offsets, points (maze-local), status).

        out: optional preallocated (e.g. pinned) uint32 array of shape (>= total, 2) for the points."""
        t = np.ascontiguousarray(np.asarray(targets, np.uint32).reshape(-1, 3))
        off = np.zeros(len(t) + 1, np.uint64)
        st = np.zeros(len(t), np.int32)
        _check(lib().am_batch_path_counts(self.ctx.handle, self.handle, _ptr(t), len(t), method, seed, _ptr(off),
                                          _ptr(st)), self.ctx, "batch counts")
        total = int(off[-1])
        if out is not None and out.dtype == np.uint32 and out.ndim == 2 and out.shape[1] == 2 and \
                out.shape[0] >= max(total, 1) and out.flags.c_contiguous:
            pts = out
        else:
            pts = np.empty((max(total, 1), 2), np.uint32)
        _check(lib().am_batch_trace_paths(self.ctx.handle, self.handle, _ptr(t), len(t), method, seed, _ptr(off),
                                          _ptr(pts), total, _ptr(st)), self.ctx, "batch trace")
        return off, pts[:total], st


def comm_unique_id() -> bytes:
    """128-byte NCCL id for am_comm_init (create on one rank, share with all)."""
    buf = (C.c_uint8 * 128)()
    st = lib().am_comm_unique_id(C.cast(buf, C.c_void_p))
    if st != OK:
        raise Error(f"am_comm_unique_id failed (status {st})")
    return bytes(buf)


def slabs_propagate(slabs, layers: int = 0, auto_cap: int = 0, mode: int = BATCHED) -> PropResult:
    """In-process row-slab group on one context: layers>0 fixed L, else auto with auto_cap."""
    arr = (C.c_void_p * len(slabs))(*[s.handle for s in slabs])
    r = _PropResult()
    ctx = slabs[0].ctx
    _check(lib().am_slabs_propagate(ctx.handle, arr, len(slabs), layers, auto_cap, mode, C.byref(r)), ctx,
           "slabs_propagate")
    for s in slabs:
        s.layers = r.layers_used
    return PropResult(r)


PEER_BLOB_BYTES = 1024  # AM_PEER_BLOB_BYTES


def slab_rows(height: int, nranks: int, rank: int):
    """Rows [row0, row1) of slab `rank` of `nranks` (am_slab_rows)."""
    a, b = C.c_uint32(0), C.c_uint32(0)
    st = lib().am_slab_rows(height, nranks, rank, C.byref(a), C.byref(b))
    if st != OK:
        raise InvalidInputError(f"slab_rows({height}, {nranks}, {rank})")
    return a.value, b.value


def peer_export(slab: Grid) -> bytes:
    """This rank's slab handles for the peer-memory transport (share with every rank, then peer_connect)."""
    buf = (C.c_uint8 * PEER_BLOB_BYTES)()
    _check(lib().am_peer_export(slab.ctx.handle, slab.handle, C.cast(buf, C.c_void_p)), slab.ctx, "peer_export")
    return bytes(buf)


def peer_connect(slab: Grid, nranks: int, rank: int, blobs):
    """Connect this rank's slab to the others (blobs: every rank's peer_export, in rank order); am_propagate on
    the slab then exchanges halos through peer memory."""
    if len(blobs) != nranks or any(len(b) != PEER_BLOB_BYTES for b in blobs):
        raise InvalidInputError("peer_connect: one blob of PEER_BLOB_BYTES per rank")
    buf = (C.c_uint8 * (PEER_BLOB_BYTES * nranks)).from_buffer_copy(b"".join(blobs))
    _check(lib().am_peer_connect(slab.ctx.handle, slab.handle, nranks, rank, C.cast(buf, C.c_void_p)), slab.ctx,
           "peer_connect")


def peer_gather(slab: Grid, full: Grid):
    """Every rank's slab into `full` (full-size grid on this rank) by peer-to-peer copies."""
    _check(lib().am_peer_gather(slab.ctx.handle, slab.handle, full.handle), slab.ctx, "peer_gather")
    full.layers = slab.layers


def peer_trace_device(slab: Grid, d_tgt: int, n: int, method: int, seed: int, d_offsets: int, d_pts: int,
                      cap: int, d_status: int):
    """am_peer_trace_paths_device: trace targets (device pointers, grid coordinates) on the map distributed
    over the connected slabs, reading across slab edges through peer memory.  Every rank must call it."""
    _check(lib().am_peer_trace_paths_device(slab.ctx.handle, slab.handle, C.c_void_p(d_tgt), n, method, seed,
                                            C.c_void_p(d_offsets), C.c_void_p(d_pts), cap, C.c_void_p(d_status)),
           slab.ctx, "peer_trace")


def slabs_gather(slabs, full: Grid):
    arr = (C.c_void_p * len(slabs))(*[s.handle for s in slabs])
    ctx = slabs[0].ctx
    _check(lib().am_slabs_gather(ctx.handle, arr, len(slabs), full.handle), ctx, "slabs_gather")
    full.layers = slabs[0].layers


# ---------------------------------------------------------------- free functions
def propagate_layer(activity, occupancy, sources, threads: int = 1, ctx: Context | None = None) -> np.ndarray:
    """propagate.hpp:37-38."""
    ctx = ctx or default_context()
    occ = _occ(occupancy)
    a = np.ascontiguousarray(activity, dtype=np.uint32)
    if a.shape != occ.shape:
        raise InvalidInputError("propagate_layer: activity/grid dimension mismatch")
    src = _rc(sources)
    out = np.empty_like(a)
    _check(lib().am_propagate_layer(ctx.handle, occ.shape[1], occ.shape[0], _ptr(occ), _ptr(src), len(src), _ptr(a),
                                    _ptr(out)), ctx, "propagate_layer")
    return out


def propagate(occupancy, sources, layers: int, mode: int = BATCHED, threads: int = 1,
              ctx: Context | None = None) -> np.ndarray:
    """propagate.hpp:40-43."""
    if layers < 1 or layers > K_MAX_LAYERS:
        raise InvalidInputError("propagate: L out of range")
    g = Grid(occupancy, sources, ctx)
    try:
        g.propagate(layers, mode)
        return g.activity()
    finally:
        g.close()


def propagate_auto(occupancy, sources, auto_cap: int, threads: int = 1, ctx: Context | None = None):
    """propagate.hpp:57-61 -> (map, layers_used, cause)."""
    if auto_cap < 1 or auto_cap > K_MAX_LAYERS:
        raise InvalidInputError("propagate_auto: auto_cap out of range")
    g = Grid(occupancy, sources, ctx)
    try:
        r = g.propagate_auto(auto_cap)
        return g.activity(), r.layers_used, r.cause
    finally:
        g.close()


def propagate_reference(occupancy, sources, layers: int, ctx: Context | None = None) -> np.ndarray:
    """propagate.hpp:63-68 (INT32_MIN sentinel kernel)."""
    ctx = ctx or default_context()
    occ = _occ(occupancy)
    src = _rc(sources)
    out = np.empty(occ.shape, np.uint32)
    _check(lib().am_propagate_reference(ctx.handle, occ.shape[1], occ.shape[0], _ptr(occ), _ptr(src), len(src),
                                        layers, _ptr(out)), ctx, "propagate_reference")
    return out


def layer_bound(width: int, height: int):
    """propagate.hpp:70-79 -> (worst_case, heuristic_low, heuristic_high)."""
    mx, mn = max(width, height), min(width, height)
    return mx * ((mn + 1) // 2) + mn // 2, (3 * mx + 1) // 2, 2 * mx


def _reconstruct(activity, occupancy, sources, target, method, seed, ctx, layers_applied=None):
    occ = _occ(occupancy)
    g = Grid(occ, sources, ctx)
    try:
        a = np.ascontiguousarray(activity, dtype=np.uint32)
        g.upload_activity(a, int(layers_applied if layers_applied is not None else a.max(initial=0)))
        (st, pts), = g.paths([target], method, seed)
    finally:
        g.close()
    if st == EUNCOVERED:
        raise UncoveredTargetError(f"uncovered target {tuple(target)}: increase L or target unreachable")
    if st == EINVAL:
        raise InvalidInputError(f"invalid target {tuple(target)}")
    if st != OK:
        raise Error("activity map has no ascending neighbour on the path")
    return pts


def reconstruct_simple(activity, occupancy, sources, target, seed: int, ctx: Context | None = None) -> np.ndarray:
    """reconstruct.hpp:38-40 (device trace on the given map)."""
    return _reconstruct(activity, occupancy, sources, target, SIMPLE, seed, ctx)


def reconstruct_euclidean(activity, occupancy, sources, target, rule: int = STRICT,
                          ctx: Context | None = None) -> np.ndarray:
    """reconstruct.hpp:45-47 (device trace, then straighten)."""
    pts = _reconstruct(activity, occupancy, sources, target, EUCLIDEAN, 0, ctx)
    return straighten(pts, occupancy, rule)


def straighten(points, occupancy=None, rule: int = STRICT) -> np.ndarray:
    """reconstruct.hpp:49-58."""
    p = _rc(points)
    out = np.empty_like(p)
    n = C.c_uint64(0)
    if occupancy is None:
        _check(lib().am_straighten(_ptr(p), len(p), None, 0, 0, rule, _ptr(out), C.byref(n)), None, "straighten")
    else:
        occ = _occ(occupancy)
        _check(lib().am_straighten(_ptr(p), len(p), _ptr(occ), occ.shape[1], occ.shape[0], rule, _ptr(out),
                                   C.byref(n)), None, "straighten")
    return out[: n.value].copy()


def path_metrics(points):
    """reconstruct.hpp:26-32 -> (steps, euclidean_length)."""
    p = _rc(points)
    s, length = C.c_uint64(0), C.c_double(0.0)
    _check(lib().am_path_metrics(_ptr(p), len(p), C.byref(s), C.byref(length)), None, "path_metrics")
    return s.value, length.value


# ---------------------------------------------------------------- map / scene text (mapio.hpp)
def _text(text) -> bytes:
    return text.encode() if isinstance(text, str) else bytes(text)


def _parse_fail(st, info: _ParseInfo, ctx):
    msg = info.error.decode(errors="replace")
    if st == EINVAL and info.error_line:
        raise ParseError(msg, int(info.error_line), int(info.error_column))
    if st == EINVAL and msg:
        raise InvalidInputError(msg)
    _raise(st, ctx, "parse")


class Scene:
    """A parsed map / scene resident on the device (am_scene): occupancy plus, for
    ASCII scenes, the 'S' sources and 'T' targets (mapio.hpp:13-17)."""

    def __init__(self, text, fmt: int = ASCII_SCENE, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        t = _text(text)
        info = _ParseInfo()
        h = C.c_void_p()
        st = lib().am_scene_parse(self.ctx.handle, t, len(t), fmt, C.byref(h), C.byref(info))
        if st != OK:
            _parse_fail(st, info, self.ctx)
        self.handle = h
        self.ctx._own(self)
        self.width, self.height = info.width, info.height
        self.n_sources, self.n_targets, self.obstacles = info.n_sources, info.n_targets, info.obstacles

    def close(self):
        if getattr(self, "handle", None):
            lib().am_scene_destroy(self.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def download(self):
        """(occupancy (H, W) uint8, sources (n, 2) uint32, targets (m, 2) uint32), row-major order."""
        occ = np.empty((self.height, self.width), dtype=np.uint8)
        src = np.empty((self.n_sources, 2), dtype=np.uint32)
        tgt = np.empty((self.n_targets, 2), dtype=np.uint32)
        _check(lib().am_scene_download(self.ctx.handle, self.handle, _ptr(occ), _ptr(src), _ptr(tgt)), self.ctx,
               "scene download")
        return occ, src, tgt

    def grid(self, sources=None) -> Grid:
        """Grid straight from the device-resident scene; sources override the file's 'S' cells."""
        g = Grid.__new__(Grid)
        g.ctx = self.ctx
        g.occ = None
        g.width, g.height = self.width, self.height
        h = C.c_void_p()
        if sources is None:
            st = lib().am_grid_create_scene(self.ctx.handle, self.handle, None, 0, C.byref(h))
        else:
            src = _rc(sources)
            st = lib().am_grid_create_scene(self.ctx.handle, self.handle, _ptr(src), len(src), C.byref(h))
        _check(st, self.ctx, "SourceSet/grid")
        g.handle = h
        self.ctx._own(g)
        g.layers = 0
        return g


def movingai_header(text):
    """Host-side Moving AI header check: (width, height, body offset) or ParseError."""
    t = _text(text)
    info = _ParseInfo()
    off = C.c_uint64(0)
    st = lib().am_movingai_header(t, len(t), C.byref(info), C.byref(off))
    if st != OK:
        _parse_fail(st, info, None)
    return info.width, info.height, off.value


def parse_movingai(text, ctx: Context | None = None) -> np.ndarray:
    """parse_movingai (mapio.hpp:23): the occupancy grid (nonzero = obstacle)."""
    sc = Scene(text, MOVINGAI, ctx)
    try:
        return sc.download()[0]
    finally:
        sc.close()


def parse_ascii_scene(text, ctx: Context | None = None):
    """parse_ascii_scene (mapio.hpp:30): (occupancy, sources, targets)."""
    sc = Scene(text, ASCII_SCENE, ctx)
    try:
        return sc.download()
    finally:
        sc.close()


def _emit(fmt, occupancy, sources, targets, ctx):
    ctx = ctx or default_context()
    occ = _occ(occupancy)
    h, w = occ.shape
    src = _rc(sources if sources is not None else np.zeros((0, 2)))
    tgt = _rc(targets if targets is not None else np.zeros((0, 2)))
    n = C.c_uint64(0)
    args = (ctx.handle, fmt, w, h, _ptr(occ), _ptr(src), len(src), _ptr(tgt), len(tgt))
    _check(lib().am_emit_text(*args, None, 0, C.byref(n)), ctx, "emit")
    buf = np.empty(n.value, dtype=np.uint8)
    _check(lib().am_emit_text(*args, _ptr(buf), n.value, C.byref(n)), ctx, "emit")
    return buf.tobytes()


def emit_movingai(occupancy, ctx: Context | None = None) -> bytes:
    """emit_movingai (mapio.hpp:26): canonical `.` / `@` text."""
    return _emit(MOVINGAI, occupancy, None, None, ctx)


def emit_ascii_scene(occupancy, sources, targets=(), ctx: Context | None = None) -> bytes:
    """emit_ascii_scene (mapio.hpp:32)."""
    return _emit(ASCII_SCENE, occupancy, sources, targets, ctx)


def export_pgm(values, ctx: Context | None = None) -> bytes:
    """export_pgm (mapio.hpp:35-38) of a host map (H, W) uint32."""
    ctx = ctx or default_context()
    v = np.ascontiguousarray(values, dtype=np.uint32)
    if v.ndim != 2:
        raise InvalidInputError("activity map must be a 2-D (height, width) array")
    h, w = v.shape
    n = C.c_uint64(0)
    _check(lib().am_export_pgm(ctx.handle, w, h, _ptr(v), None, 0, C.byref(n)), ctx, "pgm")
    buf = np.empty(n.value, dtype=np.uint8)
    _check(lib().am_export_pgm(ctx.handle, w, h, _ptr(v), _ptr(buf), n.value, C.byref(n)), ctx, "pgm")
    return buf.tobytes()


def random_maze(width: int, height: int, density: float, seed: int) -> np.ndarray:
    """grid.hpp:72-76."""
    occ = np.empty((height, width), np.uint8)
    _check(lib().am_random_maze(width, height, density, seed, _ptr(occ)), None, "random_maze")
    return occ


def kruskal_maze(width: int, height: int, seed: int) -> np.ndarray:
    """C2 workload: perfect maze on the odd lattice (randomised Kruskal, splitmix64)."""
    occ = np.empty((height, width), np.uint8)
    _check(lib().am_kruskal_maze(width, height, seed, _ptr(occ)), None, "kruskal_maze")
    return occ


def city_grid(width: int, height: int, seed: int) -> np.ndarray:
    """C3 workload: city blocks U[32,96] with streets U[3,8], 10% plazas, 1% clutter."""
    occ = np.empty((height, width), np.uint8)
    _check(lib().am_city_grid(width, height, seed, _ptr(occ)), None, "city_grid")
    return occ


def comb_maze(width: int, height: int) -> np.ndarray:
    """grid.hpp:65-70."""
    occ = np.empty((height, width), np.uint8)
    _check(lib().am_comb_maze(width, height, _ptr(occ)), None, "comb_maze")
    return occ
