"""CPU oracle for the PLMSS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs import this package, and only as the checker. The
product (``paper_2303_15491_b200``) never imports it.

Two independent CPU implementations share one numpy-level API:

* :class:`Restatement` — ``plmss_oracle.c``, a plain-C restatement of the
  reference algorithm (each function cites the reference file:line);
* :class:`Reference` — the reference library itself, compiled unchanged from
  ``/root/reference/proj/src`` into ``oracle/_ref/libplmss_ref.so`` (namespace
  ``plmss_ref``) by ``oracle/Makefile``.

The restatement is pinned against the reference's golden vectors and against
:class:`Reference` in ``tests/test_oracle_pin.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libplmss_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libplmss_ref.so")
REF_SRC = "/root/reference/proj"

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
# one separator triangle record (plmss_tri of include/plmss_b200.h / orc_tri)
TRI_DTYPE = np.dtype([("cellrow", "<u8"), ("lo", "<u4"), ("hi", "<u4")])
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(reference: bool = True) -> None:
    """Build the restatement (always) and the compiled reference (only where
    /root/reference exists — i.e. in the build container; the .so travels)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if reference and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _dims(d):
    return np.ascontiguousarray(np.asarray(d, dtype=np.int64).reshape(3))


def _vec3(v, default):
    return np.ascontiguousarray(np.asarray(default if v is None else v, dtype=np.float64).reshape(3))


class Restatement:
    """ctypes front-end of plmss_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(reference=False)
        L = self.lib = C.CDLL(path)
        L.orc_compute_order.restype = C.c_int64
        L.orc_compute_order.argtypes = [_f64p, C.c_int64, _i64p]
        L.orc_seed_hops.restype = None
        L.orc_seed_hops.argtypes = [_i64p, C.c_void_p, C.c_int, _i64p, _i64p]
        L.orc_compress.restype = C.c_int
        L.orc_compress.argtypes = [C.c_int64, _i64p, _i64p]
        L.orc_extrema.restype = C.c_int64
        L.orc_extrema.argtypes = [C.c_int64, _i64p, C.c_void_p]
        L.orc_combine_ms.restype = C.c_int64
        L.orc_combine_ms.argtypes = [C.c_int64, _i64p, _i64p, _i64p, C.c_void_p]
        L.orc_tetra_code.restype = C.c_int
        L.orc_tetra_code.argtypes = [_i64p, C.c_void_p]
        L.orc_triangle_code.restype = C.c_int
        L.orc_triangle_code.argtypes = [_i64p]
        L.orc_tetra_case.restype = C.c_int
        L.orc_tetra_case.argtypes = [C.c_int, C.c_void_p]
        L.orc_triangle_case.restype = C.c_int
        L.orc_triangle_case.argtypes = [C.c_int, C.c_void_p]
        L.orc_num_cells.restype = C.c_int64
        L.orc_num_cells.argtypes = [_i64p]
        L.orc_cell.restype = C.c_int
        L.orc_cell.argtypes = [_i64p, C.c_int64, _i64p]
        L.orc_index_separators.restype = C.c_int64
        L.orc_index_separators.argtypes = [_i64p, _i64p, C.c_void_p]
        L.orc_emit_geometry.restype = None
        L.orc_emit_geometry.argtypes = [_i64p, _f64p, _f64p, _i64p, _u8p, _f64p, _i64p, _i64p]
        L.orc_emit_boundaries.restype = None
        L.orc_emit_boundaries.argtypes = [_i64p, _f64p, _f64p, _i64p, C.c_int, C.c_int64, _i64p] + [C.c_void_p] * 5

        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        L.orc_synth.restype = C.c_int
        L.orc_synth.argtypes = [_i64p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int64,
                                C.c_int64, f32p]
        L.orc_seed_hops_f32.restype = C.c_int64
        L.orc_seed_hops_f32.argtypes = [_i64p, f32p, u32p, u32p]
        L.orc_compress_u32.restype = C.c_int
        L.orc_compress_u32.argtypes = [C.c_int64, u32p, u32p]
        L.orc_extrema_u32.restype = C.c_int64
        L.orc_extrema_u32.argtypes = [C.c_int64, u32p, C.c_void_p]
        L.orc_combine_ms_u32.restype = C.c_int64
        L.orc_combine_ms_u32.argtypes = [C.c_int64, u32p, u32p, u32p, C.c_void_p, C.c_int64]
        L.orc_separator_records.restype = C.c_int64
        L.orc_separator_records.argtypes = [_i64p, u32p, C.c_int64, C.c_int64, C.c_void_p]

    # -- full-size grids (plmss_oracle_big.c) ----------------------------------
    def synth(self, cfg, z0=0, nz=None):
        """The BASELINE config's field (include/plmss_synth.h), layers [z0, z0+nz)."""
        d = _dims(cfg.dims)
        nz = int(d[2]) if nz is None else int(nz)
        out = np.empty(int(d[0]) * int(d[1]) * nz, np.float32)
        g = np.ascontiguousarray(cfg.gaussians() if cfg.kind == "gaussians" else np.zeros((0, 5)), np.float64)
        st = self.lib.orc_synth(d, 0 if cfg.kind == "gaussians" else 1, g.ctypes.data, g.shape[0], cfg.noise,
                                cfg.seed, cfg.levels, z0, nz, out)
        if st != 0:
            raise ValueError("orc_synth: bad layer range")
        return out

    def segment_u32(self, dims, f32):
        """seed_hops_both + compression on float32 values, uint32 labels."""
        d = _dims(dims)
        f = np.ascontiguousarray(f32, dtype=np.float32).ravel()
        desc = np.empty(f.size, np.uint32)
        asc = np.empty(f.size, np.uint32)
        bad = self.lib.orc_seed_hops_f32(d, f, desc, asc)
        if bad >= 0:
            raise ValueError(f"non-finite scalar value at vertex {bad}")
        sweeps = self.lib.orc_compress_u32(f.size, desc, asc)
        return dict(desc=desc, asc=asc, maxima=self.extrema_u32(desc), minima=self.extrema_u32(asc), sweeps=sweeps)

    def extrema_u32(self, labels):
        k = self.lib.orc_extrema_u32(labels.size, labels, None)
        out = np.empty(max(k, 1), np.uint32)
        self.lib.orc_extrema_u32(labels.size, labels, out.ctypes.data)
        return out[:k]

    def combine_ms_u32(self, asc, desc):
        """(ms uint32, sorted region keys uint64 = asc << 32 | desc)."""
        ms = np.empty(asc.size, np.uint32)
        r = self.lib.orc_combine_ms_u32(asc.size, asc, desc, ms, None, 0)
        keys = np.empty(max(r, 1), np.uint64)
        self.lib.orc_combine_ms_u32(asc.size, asc, desc, ms, keys.ctypes.data, r)
        return ms, keys[:r]

    def separator_records(self, dims, labels_u32, cz0, cz1):
        """(cell << 6 | row, lo, hi) records of cube layers [cz0, cz1),
        structured array of TRI_DTYPE, reference emission order."""
        d = _dims(dims)
        lab = np.ascontiguousarray(labels_u32, dtype=np.uint32).ravel()
        k = self.lib.orc_separator_records(d, lab, cz0, cz1, None)
        out = np.empty(max(k, 1), TRI_DTYPE)
        self.lib.orc_separator_records(d, lab, cz0, cz1, out.ctypes.data)
        return out[:k]

    # -- order / segmentation -------------------------------------------------
    def compute_order(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        rank = np.empty(v.size, np.int64)
        bad = self.lib.orc_compute_order(v, v.size, rank)
        if bad >= 0:
            raise ValueError(f"non-finite scalar value at vertex {bad}")
        return rank

    def seed_hops(self, dims, values=None, rank=None):
        d = _dims(dims)
        n = int(np.prod(d))
        desc = np.empty(n, np.int64)
        asc = np.empty(n, np.int64)
        if rank is not None:
            keys = np.ascontiguousarray(rank, dtype=np.int64).ravel()
            kind = 1
        else:
            keys = np.ascontiguousarray(values, dtype=np.float64).ravel()
            kind = 0
        assert keys.size == n
        self.lib.orc_seed_hops(d, keys.ctypes.data, kind, desc, asc)
        return desc, asc

    def segment(self, dims, values=None, rank=None):
        desc, asc = self.seed_hops(dims, values=values, rank=rank)
        sweeps = self.lib.orc_compress(desc.size, desc, asc)
        return dict(desc=desc, asc=asc, maxima=self.extrema(desc), minima=self.extrema(asc), sweeps=sweeps)

    def extrema(self, labels):
        lab = np.ascontiguousarray(labels, dtype=np.int64)
        k = self.lib.orc_extrema(lab.size, lab, None)
        out = np.empty(k, np.int64)
        self.lib.orc_extrema(lab.size, lab, out.ctypes.data)
        return out

    def combine_ms(self, asc, desc):
        a = np.ascontiguousarray(asc, dtype=np.int64)
        d = np.ascontiguousarray(desc, dtype=np.int64)
        ms = np.empty(a.size, np.int64)
        keys = np.empty(2 * max(a.size, 1), np.int64)
        r = self.lib.orc_combine_ms(a.size, a, d, ms, keys.ctypes.data)
        return ms, keys[: 2 * r].reshape(r, 2)

    # -- marching -------------------------------------------------------------
    def tetra_code(self, labels4):
        loc = np.zeros(4, np.int32)
        c = self.lib.orc_tetra_code(np.ascontiguousarray(labels4, dtype=np.int64), loc.ctypes.data)
        return c, loc

    def triangle_code(self, labels3):
        return self.lib.orc_triangle_code(np.ascontiguousarray(labels3, dtype=np.int64))

    def tetra_case(self, code):
        buf = np.zeros(12 * 5, np.uint8)
        k = self.lib.orc_tetra_case(code, buf.ctypes.data)
        return buf[: 5 * k].reshape(k, 5)

    def triangle_case(self, code):
        buf = np.zeros(3 * 4, np.uint8)
        k = self.lib.orc_triangle_case(code, buf.ctypes.data)
        return buf[: 4 * k].reshape(k, 4)

    def num_cells(self, dims):
        return self.lib.orc_num_cells(_dims(dims))

    def cell(self, dims, c):
        out = np.zeros(4, np.int64)
        ar = self.lib.orc_cell(_dims(dims), c, out)
        return out[:ar]

    def index_separators(self, dims, labels):
        d = _dims(dims)
        lab = np.ascontiguousarray(labels, dtype=np.int64).ravel()
        codes = np.empty(self.num_cells(d), np.uint8)
        total = self.lib.orc_index_separators(d, lab, codes.ctypes.data)
        return codes, total

    def emit_separators(self, dims, labels, spacing=None, origin=None):
        d = _dims(dims)
        lab = np.ascontiguousarray(labels, dtype=np.int64).ravel()
        codes, total = self.index_separators(d, lab)
        ar = 3 if int((d >= 2).sum()) == 3 else 2
        pts = np.zeros(3 * ar * max(total, 1), np.float64)
        reg = np.zeros(2 * max(total, 1), np.int64)
        src = np.zeros(max(total, 1), np.int64)
        self.lib.orc_emit_geometry(d, _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0)), lab, codes, pts, reg, src)
        return dict(
            codes=codes,
            points=pts[: 3 * ar * total].reshape(ar * total, 3),
            indices=np.arange(ar * total, dtype=np.int64),
            regions=reg[: 2 * total].reshape(total, 2),
            source_cells=src[:total],
            arity=ar,
        )

    def emit_boundaries(self, dims, labels, region_filter=None, spacing=None, origin=None):
        d = _dims(dims)
        lab = np.ascontiguousarray(labels, dtype=np.int64).ravel()
        sp, og = _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0))
        hf = 0 if region_filter is None else 1
        flt = 0 if region_filter is None else int(region_filter)
        sizes = np.zeros(2, np.int64)
        self.lib.orc_emit_boundaries(d, sp, og, lab, hf, flt, sizes, None, None, None, None, None)
        nf, npnt = int(sizes[0]), int(sizes[1])
        ar = 3 if int((d >= 2).sum()) == 3 else 2
        faces = np.zeros(ar * max(nf, 1), np.int64)
        tags = np.zeros(max(nf, 1), np.int64)
        cells = np.zeros(max(nf, 1), np.int64)
        pts = np.zeros(3 * max(npnt, 1), np.float64)
        idx = np.zeros(ar * max(nf, 1), np.int64)
        self.lib.orc_emit_boundaries(d, sp, og, lab, hf, flt, sizes, faces.ctypes.data, tags.ctypes.data,
                                     cells.ctypes.data, pts.ctypes.data, idx.ctypes.data)
        regions = np.stack([tags[:nf], np.full(nf, -1, np.int64)], axis=1)
        return dict(faces=faces[: ar * nf].reshape(nf, ar), points=pts[: 3 * npnt].reshape(npnt, 3),
                    indices=idx[: ar * nf], regions=regions, source_cells=cells[:nf], arity=ar)


class ReferenceError_(RuntimeError):
    pass


class RefFormatError(RuntimeError):
    """plmss::FormatError raised by the compiled reference (io.hpp:22-24)."""


class RefIoError(RuntimeError):
    """plmss::IoError raised by the compiled reference (io.hpp:27-29)."""


_KIND = {1: ValueError, 2: RuntimeError, 3: IndexError, 4: RuntimeError, 6: RefFormatError, 7: RefIoError}


class Reference:
    """ctypes front-end of the reference library compiled unchanged
    (oracle/_ref/libplmss_ref.so), through oracle/ref_capi.cpp. The same class
    also fronts build/libplmss_dropin_harness.so (reference API -> B200)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.cap_last_error.restype = C.c_char_p
        L.cap_compute_order.argtypes = [_f64p, C.c_int64, _i64p]
        L.cap_segment.argtypes = [_i64p, _i64p, C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.cap_seg_size.restype = C.c_int64
        L.cap_seg_size.argtypes = [C.c_void_p, C.c_int]
        L.cap_seg_copy.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.cap_seg_free.argtypes = [C.c_void_p]
        L.cap_oracle_walk.argtypes = [_i64p, _i64p, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_int64)]
        L.cap_tetra_code.argtypes = [_i64p, C.c_void_p, C.c_void_p]
        L.cap_triangle_code.argtypes = [_i64p, C.c_void_p]
        L.cap_tetra_case.argtypes = [C.c_int, C.c_void_p]
        L.cap_triangle_case.argtypes = [C.c_int, C.c_void_p]
        L.cap_emit.argtypes = [_i64p, _f64p, _f64p, _i64p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int64,
                               C.POINTER(C.c_void_p)]
        L.cap_mesh_sizes.argtypes = [C.c_void_p, _i64p]
        L.cap_mesh_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.cap_mesh_free.argtypes = [C.c_void_p]
        L.cap_run_benchmark.argtypes = [_i64p, _f64p, C.c_int, C.c_int, C.c_int, _f64p]
        L.cap_run_once.argtypes = [_i64p, np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS"), C.c_int,
                                   C.c_int, _f64p, _i64p]
        if hasattr(L, "cap_seed_hops"):
            L.cap_seed_hops.argtypes = [_i64p, _i64p, C.c_int64, C.c_int, C.c_int64, C.c_int64] + [C.c_void_p] * 8
            L.cap_compress_sweep.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                             C.c_void_p]
        if hasattr(L, "cap_records_chunk"):
            L.cap_records_chunk.argtypes = [_i64p, _i64p, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_void_p),
                                            C.POINTER(C.c_int64)]
            L.cap_records_copy.argtypes = [C.c_void_p, C.c_void_p]
            L.cap_records_copy.restype = None
            L.cap_records_free.argtypes = [C.c_void_p]
            L.cap_records_free.restype = None
            L.cap_records_geometry.argtypes = [C.c_void_p] * 4
            L.cap_records_geometry.restype = None
        if hasattr(L, "cap_weld"):
            L.cap_weld.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
            L.cap_read_volume.argtypes = [C.c_char_p, _i64p, C.c_char_p, C.c_void_p]
            L.cap_write_labels.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int64]
            L.cap_write_obj.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                        C.c_int]

    # ---- callers either side of the path (io.cpp, marching.cpp:400-417)
    def weld_points(self, points, indices):
        """Reference weld_points on an (n, 3) soup; returns (points, indices)."""
        p = np.array(points, dtype=np.float64, order="C").reshape(-1, 3).copy()
        i = np.array(indices, dtype=np.int64).ravel().copy()
        u = C.c_int64()
        self._check(self.lib.cap_weld(p.ctypes.data, p.shape[0], i.ctypes.data, i.size, C.byref(u)))
        return p[: u.value], i

    def read_volume(self, path, dims, dtype="f32le"):
        d = _dims(dims)
        n = int(np.prod(d)) if (d > 0).all() else 0
        out = np.zeros(max(n, 1), np.float64)
        self._check(self.lib.cap_read_volume(os.fsencode(str(path)), d, dtype.encode(), out.ctypes.data))
        return out[:n]

    def write_labels(self, path, asc, desc):
        a = np.ascontiguousarray(asc, dtype=np.int64)
        b = np.ascontiguousarray(desc, dtype=np.int64)
        self._check(self.lib.cap_write_labels(os.fsencode(str(path)), a.ctypes.data, b.ctypes.data, a.size))

    def write_surface_obj(self, path, points, indices, regions, verts_per_prim=3):
        p = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        i = np.ascontiguousarray(indices, dtype=np.int64).ravel()
        r = np.ascontiguousarray(regions, dtype=np.int64).reshape(-1, 2)
        self._check(self.lib.cap_write_obj(os.fsencode(str(path)), p.ctypes.data, p.shape[0], i.ctypes.data,
                                           r.ctypes.data, r.shape[0], verts_per_prim))

    def detail_seed_hops(self, dims, rank, mode, begin=0, end=None):
        """detail::seed_hops (mode 0 descending / 1 ascending) or
        seed_hops_both (mode 2) over [begin, end) (segmentation.hpp:90-113):
        (desc, asc, active, extrema1, extrema2); unset label entries are -1."""
        d = _dims(dims)
        r = np.ascontiguousarray(rank, dtype=np.int64).ravel()
        n = r.size
        end = n if end is None else end
        out = [np.empty(n, np.int64) for _ in range(5)]
        cnt = [C.c_int64() for _ in range(3)]
        self._check(self.lib.cap_seed_hops(d, r, n, mode, begin, end, out[0].ctypes.data, out[1].ctypes.data,
                                           out[2].ctypes.data, C.byref(cnt[0]), out[3].ctypes.data, C.byref(cnt[1]),
                                           out[4].ctypes.data, C.byref(cnt[2])))
        return out[0], out[1], out[2][: cnt[0].value], out[3][: cnt[1].value], out[4][: cnt[2].value]

    def detail_compress_sweep(self, desc, asc, active):
        """One detail::compress_sweep(_both) in place (asc None: single)."""
        act = np.ascontiguousarray(active, dtype=np.int64)
        nxt = np.empty(max(act.size, 1), np.int64)
        k = C.c_int64()
        self._check(self.lib.cap_compress_sweep(desc.ctypes.data, None if asc is None else asc.ctypes.data, desc.size,
                                                act.ctypes.data, act.size, nxt.ctypes.data, C.byref(k)))
        return nxt[: k.value]

    def records_chunk(self, dims, labels_slab, cz0, cz1, workers=1, geometry=False):
        """Reference separator records (TRI_DTYPE) of cube layers [cz0, cz1)
        of a (X, Y, Z) grid; labels_slab = int64 labels of vertex layers
        [cz0, cz1] (ref_capi.cpp cap_records_chunk)."""
        d = _dims(dims)
        lab = np.ascontiguousarray(labels_slab, dtype=np.int64).ravel()
        assert lab.size == int(d[0]) * int(d[1]) * (cz1 - cz0 + 1)
        k = C.c_int64()
        h = C.c_void_p()
        self._check(self.lib.cap_records_chunk(d, lab, cz0, cz1, workers, C.byref(h), C.byref(k)))
        try:
            out = np.empty(max(k.value, 1), TRI_DTYPE)
            self.lib.cap_records_copy(h, out.ctypes.data)
            if geometry:  # + the reference SeparatingMesh arrays of the chunk
                n = k.value
                pts = np.empty((max(3 * n, 1), 3), np.float64)
                reg = np.empty((max(n, 1), 2), np.int64)
                cel = np.empty(max(n, 1), np.int64)
                self.lib.cap_records_geometry(h, pts.ctypes.data, reg.ctypes.data, cel.ctypes.data)
                return out[:n], dict(points=pts[: 3 * n], regions=reg[:n], source_cells=cel[:n])
        finally:
            self.lib.cap_records_free(h)
        return out[: k.value]

    def run_once(self, dims, values_f32, workers, mode=2):
        """One reference pipeline pass (bench.cpp:62-87); returns (phase
        seconds dict, regions, primitives)."""
        v = np.ascontiguousarray(values_f32, dtype=np.float32).ravel()
        ph = np.zeros(5, np.float64)
        cnt = np.zeros(2, np.int64)
        self._check(self.lib.cap_run_once(_dims(dims), v, workers, mode, ph, cnt))
        return dict(zip(["order", "segmentation", "combine", "index", "geometry"], ph.tolist())), int(cnt[0]), \
            int(cnt[1])

    def _check(self, st):
        if st != 0:
            raise _KIND.get(st, RuntimeError)(self.lib.cap_last_error().decode())

    def compute_order(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        rank = np.empty(v.size, np.int64)
        self._check(self.lib.cap_compute_order(v, v.size, rank))
        return rank

    def segment(self, dims, rank, direction=2, workers=1, combine=False):
        d = _dims(dims)
        r = np.ascontiguousarray(rank, dtype=np.int64).ravel()
        h = C.c_void_p()
        self._check(self.lib.cap_segment(d, r, r.size, direction, workers, int(combine), C.byref(h)))
        try:
            out = {}
            for i, name in enumerate(["desc", "asc", "maxima", "minima", "ms_region", "region_keys", "sweeps"]):
                k = self.lib.cap_seg_size(h, i)
                buf = np.empty(max(k, 1), np.int64)
                self.lib.cap_seg_copy(h, i, buf.ctypes.data)
                out[name] = buf[:k]
            out["region_keys"] = out["region_keys"].reshape(-1, 2)
            out["sweeps"] = int(out["sweeps"][0])
            return out
        finally:
            self.lib.cap_seg_free(h)

    def oracle_walk(self, dims, rank, v, direction):
        r = np.ascontiguousarray(rank, dtype=np.int64).ravel()
        out = C.c_int64()
        self._check(self.lib.cap_oracle_walk(_dims(dims), r, r.size, v, direction, C.byref(out)))
        return out.value

    def tetra_code(self, labels4):
        code = C.c_int32()
        loc = np.zeros(4, np.int32)
        self._check(self.lib.cap_tetra_code(np.ascontiguousarray(labels4, dtype=np.int64), C.byref(code),
                                            loc.ctypes.data))
        return code.value, loc

    def triangle_code(self, labels3):
        code = C.c_int32()
        self._check(self.lib.cap_triangle_code(np.ascontiguousarray(labels3, dtype=np.int64), C.byref(code)))
        return code.value

    def tetra_case(self, code):
        buf = np.zeros(12 * 5, np.uint8)
        k = self.lib.cap_tetra_case(code, buf.ctypes.data)
        return buf[: 5 * k].reshape(k, 5)

    def triangle_case(self, code):
        buf = np.zeros(3 * 4, np.uint8)
        k = self.lib.cap_triangle_case(code, buf.ctypes.data)
        return buf[: 4 * k].reshape(k, 4)

    def _emit(self, dims, labels, kind, workers, region_filter, spacing, origin):
        d = _dims(dims)
        lab = np.ascontiguousarray(labels, dtype=np.int64).ravel()
        h = C.c_void_p()
        hf = 0 if region_filter is None else 1
        flt = 0 if region_filter is None else int(region_filter)
        self._check(self.lib.cap_emit(d, _vec3(spacing, (1, 1, 1)), _vec3(origin, (0, 0, 0)), lab, lab.size, kind,
                                      workers, hf, flt, C.byref(h)))
        try:
            s = np.zeros(5, np.int64)
            self.lib.cap_mesh_sizes(h, s)
            nprim, npnt, ar, ncodes = (int(x) for x in s[:4])
            pts = np.zeros(3 * max(npnt, 1), np.float64)
            idx = np.zeros(ar * max(nprim, 1), np.int64)
            reg = np.zeros(2 * max(nprim, 1), np.int64)
            src = np.zeros(max(nprim, 1), np.int64)
            codes = np.zeros(max(ncodes, 1), np.uint8)
            self.lib.cap_mesh_copy(h, pts.ctypes.data, idx.ctypes.data, reg.ctypes.data, src.ctypes.data,
                                   codes.ctypes.data)
            return dict(points=pts[: 3 * npnt].reshape(npnt, 3), indices=idx[: ar * nprim],
                        regions=reg[: 2 * nprim].reshape(nprim, 2), source_cells=src[:nprim], arity=ar,
                        codes=codes[:ncodes], plan_total=int(s[4]))
        finally:
            self.lib.cap_mesh_free(h)

    def emit_separators(self, dims, labels, workers=1, spacing=None, origin=None):
        return self._emit(dims, labels, 0, workers, None, spacing, origin)

    def emit_boundaries(self, dims, labels, region_filter=None, workers=1, spacing=None, origin=None):
        return self._emit(dims, labels, 1, workers, region_filter, spacing, origin)

    def run_benchmark(self, dims, values, workers, repeats=3, mode=2):
        """Reference protocol (proj/src/bench.cpp:46-103), one worker count;
        returns the trimmed-mean phase times in seconds."""
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        out = np.zeros(5, np.float64)
        self._check(self.lib.cap_run_benchmark(_dims(dims), v, workers, repeats, mode, out))
        return dict(zip(["order", "segmentation", "combine", "index", "geometry"], out.tolist()))
