"""Python host mirror of the reference's hot-path interface, over the C-ABI.

Same names and argument meaning as the reference's C++ entry points
(proj/include/plmss/{orderfield,segmentation,marching}.hpp); device memory
comes from torch (plumbing only). Every call runs on the B200 through
``libplmss_b200.so``; there is no CPU fallback — a missing library or a
missing CUDA device raises immediately.

Error behaviour mirrors the reference exceptions: std::invalid_argument ->
ValueError, std::logic_error -> RuntimeError, std::out_of_range -> IndexError,
io.hpp FormatError -> FormatError, IoError -> IoError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# PLMSS_B200_LIB: an alternative build of the same library (the checked
# build, libplmss_b200_checked.so, tools/checked_run.py)
LIB_PATH = os.environ.get("PLMSS_B200_LIB") or os.path.join(PKG, "libplmss_b200.so")

KEY_F32, KEY_F64, KEY_RANK = 0, 1, 2
ASCENDING, DESCENDING, BOTH = 0, 1, 2
(OPT_COMBINE_PATH, OPT_PIPELINE_PATH, OPT_TMA, OPT_SPECULATIVE_SWEEPS, OPT_PASS_A_SPLIT, OPT_HOP_CUBE,
 OPT_IDS_IN_COUNT) = 1, 2, 3, 4, 5, 6, 7

class FormatError(RuntimeError):
    """io.hpp:22-24: malformed input (sizes, magic, unknown dtype)."""


class IoError(RuntimeError):
    """io.hpp:27-29: underlying read/write failure."""


_ERR = {1: ValueError, 2: RuntimeError, 3: IndexError, 4: RuntimeError, 5: MemoryError, 6: FormatError, 7: IoError}
DTYPES = {"f32le": 0, "f64le": 1, "u8": 2, "u16le": 3, "i16le": 4}

HEADER_FUNCTIONS = [
    "plmss_b200_tet_table", "plmss_b200_last_error", "plmss_b200_version", "plmss_b200_ctx_create",
    "plmss_b200_ctx_destroy", "plmss_b200_ctx_scratch_bytes", "plmss_b200_ctx_set_timing",
    "plmss_b200_ctx_stage_ms", "plmss_b200_compute_order", "plmss_b200_segment", "plmss_b200_seed_hops",
    "plmss_b200_combine_ms", "plmss_b200_index_separators", "plmss_b200_emit_separators",
    "plmss_b200_materialize_separators", "plmss_b200_emit_boundaries", "plmss_b200_pipeline",
    "plmss_b200_result", "plmss_b200_copy", "plmss_b200_ctx_set_option", "plmss_b200_pipeline_host",
    "plmss_b200_synth", "plmss_b200_launch_count", "plmss_b200_ctx_stats", "plmss_b200_count_by_cell_ranges",
    "plmss_b200_compress_sweep", "plmss_b200_segment_slab", "plmss_b200_weld_points", "plmss_b200_read_volume",
    "plmss_b200_write_labels", "plmss_b200_write_surface_obj", "plmss_b200_synth_layers",
    "plmss_b200_slab_segment", "plmss_b200_slab_resolve", "plmss_b200_slab_ids", "plmss_b200_slab_emit",
    "plmss_b200_materialize_separators_chunked", "plmss_b200_write_separators_obj", "plmss_b200_ctx_release",
    "plmss_b200_pipeline_host_batch",
]

GEOMETRY_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_double),
                            C.POINTER(C.c_int64), C.POINTER(C.c_int64))


class PlmssResult(C.Structure):
    _fields_ = [
        ("d_desc", C.c_void_p), ("d_asc", C.c_void_p), ("d_ms", C.c_void_p), ("d_maxima", C.c_void_p),
        ("d_minima", C.c_void_p), ("d_region_keys", C.c_void_p), ("d_tris", C.c_void_p),
        ("n_vertices", C.c_int64), ("n_maxima", C.c_int64), ("n_minima", C.c_int64),
        ("n_regions", C.c_int64), ("n_tris", C.c_int64), ("sweeps", C.c_int32),
    ]


class PlmssHostVolume(C.Structure):
    """plmss_host_volume (include/plmss_b200.h): one volume of a host batch."""
    _fields_ = [
        ("h_field", C.c_void_p), ("h_desc", C.c_void_p), ("h_asc", C.c_void_p), ("h_ms", C.c_void_p),
        ("h_maxima", C.c_void_p), ("h_minima", C.c_void_p), ("h_region_keys", C.c_void_p), ("h_tris", C.c_void_p),
        ("tri_capacity", C.c_int64), ("result", PlmssResult), ("status", C.c_int32),
    ]


class PlmssSlabInfo(C.Structure):
    """plmss_slab_info (include/plmss_b200.h): z-slab stage outputs."""
    _fields_ = [
        ("n_maxima", C.c_int64), ("n_minima", C.c_int64), ("d_maxima", C.c_void_p), ("d_minima", C.c_void_p),
        ("d_boundary", C.c_void_p), ("n_keys", C.c_int64), ("d_keys", C.c_void_p), ("n_regions", C.c_int64),
        ("d_region_keys", C.c_void_p), ("n_tris", C.c_int64), ("d_tris", C.c_void_p), ("sweeps", C.c_int32),
        ("dense", C.c_int32),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load libplmss_b200.so (in-tree build). Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.plmss_b200_last_error.restype = C.c_char_p
        L.plmss_b200_version.restype = C.c_char_p
        L.plmss_b200_ctx_create.argtypes = [i32, vp, C.POINTER(vp)]
        L.plmss_b200_ctx_destroy.argtypes = [vp]
        L.plmss_b200_ctx_destroy.restype = None
        L.plmss_b200_ctx_scratch_bytes.argtypes = [vp]
        L.plmss_b200_ctx_scratch_bytes.restype = C.c_size_t
        L.plmss_b200_ctx_release.argtypes = [vp]
        L.plmss_b200_ctx_set_timing.argtypes = [vp, i32]
        L.plmss_b200_ctx_stage_ms.argtypes = [vp, vp]
        L.plmss_b200_ctx_stats.argtypes = [vp, vp]
        L.plmss_b200_ctx_set_option.argtypes = [vp, i32, i64]
        L.plmss_b200_compute_order.argtypes = [vp, i32, vp, i64, vp]
        L.plmss_b200_segment.argtypes = [vp, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp]
        L.plmss_b200_seed_hops.argtypes = [vp, vp, i32, vp, vp, vp]
        L.plmss_b200_combine_ms.argtypes = [vp, i64, vp, vp, vp, vp, vp]
        L.plmss_b200_index_separators.argtypes = [vp, vp, i32, vp, vp, vp]
        L.plmss_b200_count_by_cell_ranges.argtypes = [vp, vp, i32, vp, vp, i32, vp]
        L.plmss_b200_segment_slab.argtypes = [vp, vp, i32, vp, i32, i32, vp, vp, vp]
        L.plmss_b200_compress_sweep.argtypes = [vp, vp, vp, vp, i64, vp, vp]
        L.plmss_b200_emit_separators.argtypes = [vp, vp, i32, vp, vp, i64, vp]
        L.plmss_b200_materialize_separators.argtypes = [vp, vp, vp, vp, i32, vp, i64, vp, vp, vp]
        L.plmss_b200_emit_boundaries.argtypes = [vp, vp, vp, vp, i32, vp, i32, i64, vp, vp, vp, vp, vp, vp, vp]
        L.plmss_b200_pipeline.argtypes = [vp, vp, vp]
        L.plmss_b200_result.argtypes = [vp, C.POINTER(PlmssResult)]
        L.plmss_b200_copy.argtypes = [vp, vp, vp, i64, i32]
        L.plmss_b200_pipeline_host.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, C.POINTER(PlmssResult)]
        L.plmss_b200_pipeline_host_batch.argtypes = [vp, vp, C.POINTER(PlmssHostVolume), i64]
        L.plmss_b200_synth.argtypes = [vp, vp, i32, vp, i32, C.c_double, C.c_uint64, i32, vp]
        L.plmss_b200_synth_layers.argtypes = [vp, vp, i32, vp, i32, C.c_double, C.c_uint64, i64, i64, vp]
        L.plmss_b200_weld_points.argtypes = [vp, vp, i64, vp, i64, C.POINTER(i64)]
        L.plmss_b200_read_volume.argtypes = [vp, C.c_char_p, vp, i32, i32, vp]
        L.plmss_b200_write_labels.argtypes = [vp, C.c_char_p, i32, vp, vp, i64]
        L.plmss_b200_write_surface_obj.argtypes = [vp, C.c_char_p, vp, i64, vp, vp, i64, i32]
        L.plmss_b200_materialize_separators_chunked.argtypes = [vp, vp, vp, vp, i32, vp, i64, i64, GEOMETRY_SINK, vp]
        L.plmss_b200_write_separators_obj.argtypes = [vp, C.c_char_p, vp, vp, vp, i32, vp, i64]
        SI = C.POINTER(PlmssSlabInfo)
        L.plmss_b200_slab_segment.argtypes = [vp, vp, i64, i64, vp, SI]
        L.plmss_b200_slab_resolve.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, SI]
        L.plmss_b200_slab_ids.argtypes = [vp, vp, i64, SI]
        L.plmss_b200_slab_emit.argtypes = [vp, vp, SI]
        L.plmss_b200_tet_table.argtypes = [vp, vp]
        L.plmss_b200_tet_table.restype = None
        L.plmss_b200_launch_count.restype = C.c_ulonglong
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise _ERR.get(status, RuntimeError)(lib().plmss_b200_last_error().decode())


def tet_table():
    """Host copy of the device recipe table (no GPU needed)."""
    rows = np.zeros(52, np.uint32)
    cases = np.zeros(32, np.uint16)
    lib().plmss_b200_tet_table(rows.ctypes.data, cases.ctypes.data)
    return rows, cases


def launch_count() -> int:
    """Kernel launches issued by libplmss_b200 so far (process-wide)."""
    return int(lib().plmss_b200_launch_count())


def _dims(d) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(d, dtype=np.int64).reshape(3))
    return a


def _vec3(v, default):
    return np.ascontiguousarray(np.asarray(default if v is None else v, dtype=np.float64).reshape(3))


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("plmss_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch


class Context:
    """Device + stream + scratch arena (plmss_ctx). By default the context
    issues work on torch's current stream so torch events time it."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        h = C.c_void_p()
        # torch's default stream has handle 0, which the C-ABI reads as "make
        # your own non-blocking stream": library kernels would then race with
        # the torch ops that produce their inputs. Pass cudaStreamLegacy (0x1)
        # instead so both sides share one ordered stream.
        handle = stream.cuda_stream or 1
        _check(lib().plmss_b200_ctx_create(device, C.c_void_p(handle), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().plmss_b200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, on: bool):
        _check(lib().plmss_b200_ctx_set_timing(self.h, int(on)))

    def stage_ms(self):
        out = np.zeros(8, np.float32)
        _check(lib().plmss_b200_ctx_stage_ms(self.h, out.ctypes.data))
        return out

    def stats(self):
        out = np.zeros(8, np.int64)
        _check(lib().plmss_b200_ctx_stats(self.h, out.ctypes.data))
        return out

    def set_option(self, option: int, value: int):
        _check(lib().plmss_b200_ctx_set_option(self.h, option, value))

    def scratch_bytes(self) -> int:
        return lib().plmss_b200_ctx_scratch_bytes(self.h)

    def release(self):
        """Free the scratch arena (results of earlier calls become invalid)."""
        _check(lib().plmss_b200_ctx_release(self.h))


_default: dict = {}


def default_context(device: int = 0) -> Context:
    ctx = _default.get(device)
    if ctx is None:
        ctx = _default[device] = Context(device)
    return ctx


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _as_u32(t):
    """int32 device storage holding uint32 values -> int64 values."""
    torch = _torch()
    return t.to(torch.int64) & 0xFFFFFFFF


# --------------------------------------------------------------- order ----
def compute_order(values, ctx: Optional[Context] = None):
    """compute_order (orderfield.hpp:35): int64 ranks of (value, id)."""
    torch = _torch()
    ctx = ctx or default_context()
    v = values.contiguous()
    kt = KEY_F32 if v.dtype == torch.float32 else KEY_F64
    if v.dtype not in (torch.float32, torch.float64):
        raise ValueError("values must be float32 or float64")
    rank = torch.empty(v.numel(), dtype=torch.int64, device=v.device)
    _check(lib().plmss_b200_compute_order(ctx.h, kt, _ptr(v), v.numel(), _ptr(rank)))
    return rank


# -------------------------------------------------------- segmentation ----
@dataclass
class SegmentationResult:
    """Mirror of plmss::SegmentationResult (segmentation.hpp:35-58); label
    arrays are int32 device tensors holding uint32 vertex ids."""
    desc: object = None
    asc: object = None
    maxima: object = None
    minima: object = None
    ms_region: object = None
    region_keys: object = None  # int64: asc << 32 | desc
    sweeps: int = 0
    dims: tuple = ()

    def num_regions(self) -> int:
        return 0 if self.region_keys is None else int(self.region_keys.numel())


def _key_type(keys):
    torch = _torch()
    if keys.dtype == torch.float32:
        return KEY_F32
    if keys.dtype == torch.float64:
        return KEY_F64
    if keys.dtype == torch.int64:
        return KEY_RANK
    raise ValueError("keys must be float32, float64 values or int64 ranks")


def seed_hops(dims, keys, ctx: Optional[Context] = None):
    """detail::seed_hops_both (segmentation.hpp:108-113): step-1 hop targets."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    n = int(np.prod(d))
    k = keys.contiguous().view(-1)
    if k.numel() != n:
        raise ValueError("order field size does not match complex")
    desc = torch.empty(n, dtype=torch.int32, device=k.device)
    asc = torch.empty(n, dtype=torch.int32, device=k.device)
    _check(lib().plmss_b200_seed_hops(ctx.h, d.ctypes.data, _key_type(k), _ptr(k), _ptr(desc), _ptr(asc)))
    return desc, asc


def segment(dims, keys, direction: int = BOTH, workers: int = 1, ctx: Optional[Context] = None) -> SegmentationResult:
    """segment (segmentation.hpp:74-76). `keys`: float32/float64 scalar
    values (compared as (value, id)) or int64 OrderField ranks. `workers` is
    accepted for signature parity and must be >= 1, as in the reference."""
    torch = _torch()
    if workers < 1:
        raise ValueError("workers must be >= 1")
    ctx = ctx or default_context()
    d = _dims(dims)
    n = int(np.prod(d))
    k = keys.contiguous().view(-1)
    if k.numel() != n:
        raise ValueError("order field size does not match complex")
    dev = k.device
    want_desc, want_asc = direction != ASCENDING, direction != DESCENDING
    desc = torch.empty(n, dtype=torch.int32, device=dev) if want_desc else None
    asc = torch.empty(n, dtype=torch.int32, device=dev) if want_asc else None
    mx = torch.empty(n, dtype=torch.int32, device=dev) if want_desc else None
    mn = torch.empty(n, dtype=torch.int32, device=dev) if want_asc else None
    nmax, nmin, sweeps = C.c_int64(), C.c_int64(), C.c_int32()
    _check(lib().plmss_b200_segment(ctx.h, d.ctypes.data, _key_type(k), _ptr(k), direction, _ptr(desc), _ptr(asc),
                                    _ptr(mx), _ptr(mn), C.byref(nmax), C.byref(nmin), C.byref(sweeps)))
    return SegmentationResult(desc=desc, asc=asc, maxima=None if mx is None else mx[: nmax.value],
                              minima=None if mn is None else mn[: nmin.value], sweeps=sweeps.value,
                              dims=tuple(int(x) for x in d))


def combine_ms(seg: SegmentationResult, workers: int = 1, ctx: Optional[Context] = None) -> SegmentationResult:
    """combine_ms (segmentation.hpp:80): fills ms_region and region_keys."""
    torch = _torch()
    if seg.desc is None or seg.asc is None:
        raise ValueError("combine_ms needs both ascending and descending labels")
    ctx = ctx or default_context()
    n = seg.desc.numel()
    ms = torch.empty(n, dtype=torch.int32, device=seg.desc.device)
    keys = torch.empty(n, dtype=torch.int64, device=seg.desc.device)
    r = C.c_int64()
    _check(lib().plmss_b200_combine_ms(ctx.h, n, _ptr(seg.asc), _ptr(seg.desc), _ptr(ms), _ptr(keys), C.byref(r)))
    seg.ms_region = ms
    seg.region_keys = keys[: r.value]
    return seg


# -------------------------------------------------------------- marching ---
def _label_type(labels):
    torch = _torch()
    if labels.dtype == torch.int32:
        return 0
    if labels.dtype == torch.int64:
        return 1
    raise ValueError("labels must be int32 (uint32 ids) or int64")


def index_separators(dims, labels, workers: int = 1, ctx: Optional[Context] = None):
    """index_separators (marching.hpp:101-102): per-cell codes + total."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    lab = labels.contiguous().view(-1)
    if lab.numel() != int(np.prod(d)):
        raise ValueError("label field size does not match vertex count")
    ncells = 6 * int((d[0] - 1) * (d[1] - 1) * (d[2] - 1))
    codes = torch.empty(max(ncells, 1), dtype=torch.uint8, device=lab.device)
    total = C.c_int64()
    _check(lib().plmss_b200_index_separators(ctx.h, d.ctypes.data, _label_type(lab), _ptr(lab), _ptr(codes),
                                             C.byref(total)))
    return codes[:ncells], total.value


def emit_separators(dims, labels, workers: int = 1, ctx: Optional[Context] = None):
    """emit_separators (marching.hpp:115-117) as compact records in the
    reference order: int64 tensor (T, 2) = [cell << 6 | row, lo | hi << 32]
    for int32 labels, (T, 3) = [cell << 6 | row, lo, hi] for int64 labels."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    lab = labels.contiguous().view(-1)
    if lab.numel() != int(np.prod(d)):
        raise ValueError("label field size does not match vertex count")
    lt = _label_type(lab)
    width = 2 if lt == 0 else 3
    _, total = index_separators(d, lab, ctx=ctx)
    out = torch.empty((max(total, 1), width), dtype=torch.int64, device=lab.device)
    t = C.c_int64()
    _check(lib().plmss_b200_emit_separators(ctx.h, d.ctypes.data, lt, _ptr(lab), _ptr(out), total, C.byref(t)))
    return out[: t.value]


def materialize_separators(dims, records, spacing=None, origin=None, ctx: Optional[Context] = None):
    """Reference SeparatingMesh layout (marching.hpp:65-76) from records:
    points (3T, 3) float64, indices (identity soup), regions (T, 2) int64,
    source_cells (T,) int64."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    recs = records.contiguous()
    T = recs.shape[0]
    lt = 0 if recs.shape[1] == 2 else 1
    dev = recs.device
    pts = torch.empty((max(3 * T, 1), 3), dtype=torch.float64, device=dev)
    reg = torch.empty((max(T, 1), 2), dtype=torch.int64, device=dev)
    src = torch.empty(max(T, 1), dtype=torch.int64, device=dev)
    sp, og = _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0))
    _check(lib().plmss_b200_materialize_separators(ctx.h, d.ctypes.data, sp.ctypes.data, og.ctypes.data, lt,
                                                   _ptr(recs), T, _ptr(pts), _ptr(reg), _ptr(src)))
    return dict(points=pts[: 3 * T], indices=torch.arange(3 * T, device=dev), regions=reg[:T], source_cells=src[:T])


def materialize_separators_chunked(dims, records, sink, chunk: int = 1 << 22, spacing=None, origin=None,
                                   ctx: Optional[Context] = None):
    """The SeparatingMesh arrays of `records` streamed chunk by chunk (never
    held whole): sink(first, points (3k, 3) f64, regions (k, 2) i64,
    source_cells (k,) i64) is called per chunk of k triangles with numpy
    views of pinned host buffers, valid only during the call; a truthy
    return value stops the stream (RuntimeError)."""
    ctx = ctx or default_context()
    d = _dims(dims)
    recs = records.contiguous()
    T = recs.shape[0]
    lt = 0 if recs.shape[1] == 2 else 1
    sp, og = _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0))
    err = []

    def _cb(_user, first, count, p, r, c):
        try:
            pts = np.ctypeslib.as_array(p, shape=(3 * count, 3))
            reg = np.ctypeslib.as_array(r, shape=(count, 2))
            src = np.ctypeslib.as_array(c, shape=(count,))
            return 1 if sink(first, pts, reg, src) else 0
        except Exception as e:  # noqa: BLE001  (re-raised below)
            err.append(e)
            return 2

    cb = GEOMETRY_SINK(_cb)
    st = lib().plmss_b200_materialize_separators_chunked(ctx.h, d.ctypes.data, sp.ctypes.data, og.ctypes.data, lt,
                                                        _ptr(recs), T, chunk, cb, None)
    if err:
        raise err[0]
    _check(st)


def write_separators_obj(path, dims, records, spacing=None, origin=None, ctx: Optional[Context] = None):
    """io.cpp:268-299 write_surface_obj of emit_separators' mesh, streamed
    from the compact records (plmss_b200_write_separators_obj)."""
    ctx = ctx or default_context()
    d = _dims(dims)
    recs = records.contiguous()
    lt = 0 if recs.shape[1] == 2 else 1
    sp, og = _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0))
    _check(lib().plmss_b200_write_separators_obj(ctx.h, os.fsencode(str(path)), d.ctypes.data, sp.ctypes.data,
                                                 og.ctypes.data, lt, _ptr(recs), recs.shape[0]))


def emit_boundaries(dims, labels, region_filter=None, workers: int = 1, spacing=None, origin=None,
                    ctx: Optional[Context] = None):
    """emit_boundaries (marching.hpp:123-126), reference order and layout."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    lab = labels.contiguous().view(-1)
    if lab.numel() != int(np.prod(d)):
        raise ValueError("label field size does not match vertex count")
    lt = _label_type(lab)
    sp, og = _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0))
    hf = 0 if region_filter is None else 1
    flt = 0 if region_filter is None else int(region_filter)
    nf, npnt = C.c_int64(), C.c_int64()
    L = lib()
    _check(L.plmss_b200_emit_boundaries(ctx.h, d.ctypes.data, sp.ctypes.data, og.ctypes.data, lt, _ptr(lab), hf, flt,
                                        None, None, None, None, None, C.byref(nf), C.byref(npnt)))
    F, P = nf.value, npnt.value
    dev = lab.device
    faces = torch.empty((max(F, 1), 3), dtype=torch.int32, device=dev)
    tags = torch.empty(max(F, 1), dtype=lab.dtype, device=dev)
    cells = torch.empty(max(F, 1), dtype=torch.int64, device=dev)
    pts = torch.empty((max(P, 1), 3), dtype=torch.float64, device=dev)
    idx = torch.empty(max(3 * F, 1), dtype=torch.int64, device=dev)
    _check(L.plmss_b200_emit_boundaries(ctx.h, d.ctypes.data, sp.ctypes.data, og.ctypes.data, lt, _ptr(lab), hf, flt,
                                        _ptr(faces), _ptr(tags), _ptr(cells), _ptr(pts), _ptr(idx), C.byref(nf),
                                        C.byref(npnt)))
    tg = tags[:F].to(torch.int64)
    if lt == 0:
        tg = tg & 0xFFFFFFFF
    regions = torch.stack([tg, torch.full_like(tg, -1)], dim=1)
    return dict(faces=faces[:F], points=pts[:P], indices=idx[: 3 * F], regions=regions, source_cells=cells[:F])


def select_labels(seg: SegmentationResult, mode: str):
    """select_labels (marching.hpp:132-133): 'ascending', 'descending',
    'morse_smale' or 'union' (asc then desc)."""
    if mode == "ascending":
        if seg.asc is None:
            raise RuntimeError("ascending labels missing")
        return [seg.asc]
    if mode == "descending":
        if seg.desc is None:
            raise RuntimeError("descending labels missing")
        return [seg.desc]
    if mode == "morse_smale":
        if seg.ms_region is None:
            raise RuntimeError("combine_ms has not been run")
        return [seg.ms_region]
    if mode == "union":
        if seg.asc is None or seg.desc is None:
            raise RuntimeError("union needs both directions")
        return [seg.asc, seg.desc]
    raise RuntimeError("unknown segmentation mode")


# ------------------------------------------------------- fused pipeline ---
@dataclass
class PipelineResult:
    n_vertices: int
    n_maxima: int
    n_minima: int
    n_regions: int
    n_tris: int
    sweeps: int
    raw: PlmssResult = field(repr=False, default=None)


def pipeline(dims, field_f32, ctx: Optional[Context] = None) -> PipelineResult:
    """run_benchmark's MorseSmale pass (bench.cpp:66-87) on a device-resident
    float32 field: asc, desc, extrema, dense MS ids + region table, separator
    records. Results stay in the context (see fetch())."""
    ctx = ctx or default_context()
    d = _dims(dims)
    f = field_f32
    if f.numel() != int(np.prod(d)):
        raise ValueError("field size does not match dims")
    _check(lib().plmss_b200_pipeline(ctx.h, d.ctypes.data, _ptr(f)))
    return result(ctx)


def result(ctx: Context) -> PipelineResult:
    r = PlmssResult()
    _check(lib().plmss_b200_result(ctx.h, C.byref(r)))
    return PipelineResult(r.n_vertices, r.n_maxima, r.n_minima, r.n_regions, r.n_tris, r.sweeps, r)


def fetch(ctx: Context, res: PipelineResult, names=("desc", "asc", "ms", "maxima", "minima", "region_keys", "tris")):
    """Copy pipeline outputs from the context into fresh torch tensors."""
    torch = _torch()
    r = res.raw
    spec = {
        "desc": (r.d_desc, r.n_vertices, torch.int32, 1),
        "asc": (r.d_asc, r.n_vertices, torch.int32, 1),
        "ms": (r.d_ms, r.n_vertices, torch.int32, 1),
        "maxima": (r.d_maxima, r.n_maxima, torch.int32, 1),
        "minima": (r.d_minima, r.n_minima, torch.int32, 1),
        "region_keys": (r.d_region_keys, r.n_regions, torch.int64, 1),
        "tris": (r.d_tris, r.n_tris, torch.int64, 2),
    }
    out = {}
    for name in names:
        ptr, n, dt, w = spec[name]
        t = torch.empty((n, w) if w > 1 else n, dtype=dt, device=f"cuda:{ctx.device}")
        if n:
            _check(lib().plmss_b200_copy(ctx.h, _ptr(t), C.c_void_p(ptr), t.numel() * t.element_size(), 0))
        out[name] = t
    return out


class _DevArray:
    """__cuda_array_interface__ of context-owned device memory (zero-copy)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3}


def result_view(ctx: Context, res: PipelineResult, name: str):
    """Zero-copy torch view of one pipeline output inside the context (valid
    until the context's next call): no second device copy of e.g. cfg3's
    86 GB of separator records."""
    torch = _torch()
    r = res.raw
    spec = {"desc": (r.d_desc, (r.n_vertices,), "<i4"), "asc": (r.d_asc, (r.n_vertices,), "<i4"),
            "ms": (r.d_ms, (r.n_vertices,), "<i4"), "maxima": (r.d_maxima, (r.n_maxima,), "<i4"),
            "minima": (r.d_minima, (r.n_minima,), "<i4"), "region_keys": (r.d_region_keys, (r.n_regions,), "<i8"),
            "tris": (r.d_tris, (r.n_tris, 2), "<i8")}
    ptr, shape, ts = spec[name]
    if not ptr or 0 in shape:
        return torch.empty(shape, dtype=torch.int32 if ts == "<i4" else torch.int64, device=f"cuda:{ctx.device}")
    return torch.as_tensor(_DevArray(ptr, shape, ts), device=f"cuda:{ctx.device}")


def result_digests(ctx: Context, res: PipelineResult, names=("desc", "asc", "ms", "maxima", "minima",
                                                               "region_keys", "tris"), piece_bytes: int = 1 << 30):
    """Chunked SHA-256 (digest.py) of pipeline outputs in the context, read
    back to the host in pieces (the full-size parity tests: cfg3's records
    alone are 86 GB, more than a second device copy would leave room for)."""
    from .digest import BLOCK, ChunkedSha256

    r = res.raw
    spec = {"desc": (r.d_desc, 4 * r.n_vertices), "asc": (r.d_asc, 4 * r.n_vertices),
            "ms": (r.d_ms, 4 * r.n_vertices), "maxima": (r.d_maxima, 4 * r.n_maxima),
            "minima": (r.d_minima, 4 * r.n_minima), "region_keys": (r.d_region_keys, 8 * r.n_regions),
            "tris": (r.d_tris, 16 * r.n_tris)}
    out = {}
    for name in names:
        ptr, nbytes = spec[name]
        h = ChunkedSha256()
        for off in range(0, nbytes, piece_bytes):
            k = min(piece_bytes, nbytes - off)
            buf = np.empty(k, np.uint8)
            _check(lib().plmss_b200_copy(ctx.h, buf.ctypes.data, C.c_void_p(ptr + off), k, 1))
            h.update(buf)
            h.drain(4 * max(piece_bytes // BLOCK, 1))  # bound host memory
        out[name] = h.hexdigest()
    return out


def pipeline_host(dims, h_field: np.ndarray, ctx: Optional[Context] = None, want=("desc", "asc", "ms", "maxima",
                                                                                  "minima", "region_keys", "tris"),
                  out_buffers: Optional[dict] = None):
    """End-to-end call over host buffers (H2D of the field, D2H of every
    requested output). out_buffers may hold preallocated (pinned) arrays."""
    ctx = ctx or default_context()
    d = _dims(dims)
    n = int(np.prod(d))
    f = np.ascontiguousarray(h_field, dtype=np.float32).reshape(-1)
    if f.size != n:
        raise ValueError("field size does not match dims")
    bufs = dict(out_buffers or {})
    for name in ("desc", "asc", "ms"):
        if name in want and name not in bufs:
            bufs[name] = np.empty(n, np.uint32)
    for name in ("maxima", "minima"):
        if name in want and name not in bufs:
            bufs[name] = np.empty(n, np.uint32)
    if "region_keys" in want and "region_keys" not in bufs:
        bufs["region_keys"] = np.empty(n, np.uint64)
    tri_cap = 0
    if "tris" in want:
        if "tris" not in bufs:
            raise ValueError("pass out_buffers['tris'] (uint64 array of shape (cap, 2)) to fetch separators")
        tri_cap = bufs["tris"].shape[0]
    r = PlmssResult()

    def p(name):
        b = bufs.get(name) if name in want else None
        return C.c_void_p(b.ctypes.data) if b is not None else C.c_void_p(0)

    _check(lib().plmss_b200_pipeline_host(ctx.h, d.ctypes.data, f.ctypes.data, p("desc"), p("asc"), p("ms"),
                                          p("maxima"), p("minima"), p("region_keys"), p("tris"), tri_cap,
                                          C.byref(r)))
    res = PipelineResult(r.n_vertices, r.n_maxima, r.n_minima, r.n_regions, r.n_tris, r.sweeps, r)
    out = {k: v for k, v in bufs.items() if k in want}
    for name, cnt in (("maxima", r.n_maxima), ("minima", r.n_minima), ("region_keys", r.n_regions),
                      ("tris", r.n_tris)):
        if name in out:
            out[name] = out[name][:cnt]
    return res, out


def pipeline_host_batch(dims, volumes, ctx: Optional[Context] = None):
    """plmss_b200_pipeline_host_batch: a sequence of host volumes, each a dict
    with "field" (float32 numpy, ideally pinned) and optional numpy output
    buffers "desc", "asc", "ms" (uint32 N), "maxima", "minima" (uint32),
    "region_keys" (uint64), "tris" (uint64 (T, 2)); double-buffered so one
    volume's download overlaps the next one's upload and compute. Returns the
    PipelineResult counts per volume."""
    ctx = ctx or default_context()
    d = _dims(dims)
    arr = (PlmssHostVolume * len(volumes))()
    keep = []
    for v, vol in zip(arr, volumes):
        f = np.ascontiguousarray(vol["field"], dtype=np.float32).reshape(-1)
        keep.append(f)
        v.h_field = f.ctypes.data
        for k in ("desc", "asc", "ms", "maxima", "minima", "region_keys", "tris"):
            b = vol.get(k)
            setattr(v, "h_" + k, b.ctypes.data if b is not None else None)
        t = vol.get("tris")
        v.tri_capacity = 0 if t is None else t.shape[0]
    _check(lib().plmss_b200_pipeline_host_batch(ctx.h, d.ctypes.data, arr, len(volumes)))
    return [PipelineResult(v.result.n_vertices, v.result.n_maxima, v.result.n_minima, v.result.n_regions,
                           v.result.n_tris, v.result.sweeps, None) for v in arr]


def synth_field(dims, kind: str = "gaussians", gaussians=None, noise_amp: float = 0.0, seed: int = 0,
                levels: int = 0, ctx: Optional[Context] = None):
    """Seeded synthetic float32 field on the device (harness utility)."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    n = int(np.prod(d))
    f = torch.empty(n, dtype=torch.float32, device=f"cuda:{ctx.device}")
    g = np.ascontiguousarray(np.zeros((0, 5)) if gaussians is None else gaussians, dtype=np.float64)
    k = {"gaussians": 0, "uniform": 1}[kind]
    _check(lib().plmss_b200_synth(ctx.h, d.ctypes.data, k, g.ctypes.data, g.shape[0], noise_amp, seed, levels,
                                  _ptr(f)))
    return f


def synth_layers(dims, z0: int, nz: int, kind: str = "gaussians", gaussians=None, noise_amp: float = 0.0,
                 seed: int = 0, ctx: Optional[Context] = None):
    """Vertex layers [z0, z0 + nz) of the synth_field volume (a rank's slab
    plus its halo layers; no quantisation)."""
    torch = _torch()
    ctx = ctx or default_context()
    d = _dims(dims)
    f = torch.empty(int(d[0]) * int(d[1]) * int(nz), dtype=torch.float32, device=f"cuda:{ctx.device}")
    g = np.ascontiguousarray(np.zeros((0, 5)) if gaussians is None else gaussians, dtype=np.float64)
    k = {"gaussians": 0, "uniform": 1}[kind]
    _check(lib().plmss_b200_synth_layers(ctx.h, d.ctypes.data, k, g.ctypes.data, g.shape[0], noise_amp, seed,
                                         int(z0), int(nz), _ptr(f)))
    return f


# ---------------------------------------------------------------------------
# Callers either side of the path: volume ingest, the
# reference file formats, point welding.

def weld_points(points, indices, ctx: Optional[Context] = None):
    """marching.cpp:400-417 on the device: merge bitwise-identical points
    ((n, 3) float64), the first occurrence keeping its place; indices (int64)
    are remapped in place. Returns (points[:unique], indices)."""
    ctx = ctx or default_context()
    if points.dtype != _torch().float64 or indices.dtype != _torch().int64:
        raise ValueError("weld_points needs float64 points and int64 indices")
    pts, idx = points.contiguous(), indices.contiguous()
    u = C.c_int64()
    _check(lib().plmss_b200_weld_points(ctx.h, _ptr(pts), pts.shape[0] if pts.numel() else 0, _ptr(idx),
                                        idx.numel(), C.byref(u)))
    if idx.data_ptr() != indices.data_ptr():
        indices.copy_(idx)
    if pts.data_ptr() != points.data_ptr():
        points.copy_(pts)
    return points[: u.value], indices


def read_volume(path, dims, dtype: str = "f32le", out: str = "f32", ctx: Optional[Context] = None):
    """io.cpp:90-124: a raw little-endian volume (x fastest) streamed into a
    device tensor — float32 (the pipeline's input) or float64 (the reference's
    ScalarField values)."""
    torch = _torch()
    ctx = ctx or default_context()
    if dtype not in DTYPES:
        raise FormatError(f"unknown dtype '{dtype}' (expected f32le, f64le, u8, u16le, or i16le)")
    d = _dims(dims)
    n = int(np.prod(d)) if (d > 0).all() else 0
    t = torch.empty(max(n, 1), dtype=torch.float64 if out == "f64" else torch.float32, device=f"cuda:{ctx.device}")
    _check(lib().plmss_b200_read_volume(ctx.h, os.fsencode(str(path)), d.ctypes.data, DTYPES[dtype],
                                        1 if out == "f64" else 0, _ptr(t)))
    return t[:n]


def write_labels(path, asc, desc, ctx: Optional[Context] = None):
    """io.cpp:216-235: "PLMSSLBL", u32 1, u64 n, (u64 asc, u64 desc) per
    vertex, from device label arrays (uint32 or int64)."""
    ctx = ctx or default_context()
    a, b = asc.contiguous(), desc.contiguous()
    if a.shape != b.shape or a.dtype != b.dtype:
        raise ValueError("label output needs matching ascending and descending arrays")
    lt = _label_type(a)
    _check(lib().plmss_b200_write_labels(ctx.h, os.fsencode(str(path)), lt, _ptr(a), _ptr(b), a.numel()))


def write_surface_obj(path, points, indices, regions, verts_per_prim: int = 3, ctx: Optional[Context] = None):
    """io.cpp:268-299: the reference's OBJ text from device arrays (points
    (n, 3) float64, indices int64, regions (m, 2) int64)."""
    ctx = ctx or default_context()
    pts, idx, reg = points.contiguous(), indices.contiguous(), regions.contiguous()
    n_prims = reg.shape[0] if reg.numel() else 0
    _check(lib().plmss_b200_write_surface_obj(ctx.h, os.fsencode(str(path)), _ptr(pts),
                                              pts.shape[0] if pts.numel() else 0, _ptr(idx), _ptr(reg), n_prims,
                                              verts_per_prim))
