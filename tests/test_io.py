"""Callers either side of the path: volume ingest
(io.cpp:90-124), the label and OBJ writers (io.cpp:216-235, 268-299) and point
welding (marching.cpp:400-417). The B200 side (device arrays through the
C-ABI) must produce the reference's values and byte-identical files; the
reference is the compiled reference library (oracle/_ref)."""
import os

import numpy as np
import pytest

from conftest import load_case

DTYPES = {"f32le": "<f4", "f64le": "<f8", "u8": "u1", "u16le": "<u2", "i16le": "<i2"}


def _volume(rng, n, dt):
    if dt == "f32le":
        return (rng.standard_normal(n) * 10).astype("<f4")
    if dt == "f64le":
        return rng.standard_normal(n).astype("<f8")
    info = np.iinfo(np.dtype(DTYPES[dt]))
    return rng.integers(info.min, int(info.max) + 1, size=n).astype(DTYPES[dt])


def _soup(seed=3):
    """A separator-like soup with duplicates, +-0.0 and a NaN payload."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 4, size=(40, 3)).astype(np.float64) * 0.5
    base[5] = [-0.0, 0.0, 1.0]
    base[6] = [0.0, 0.0, 1.0]
    base[7] = [np.nan, 1.0, 2.0]
    pts = base[rng.integers(0, 40, size=300)]
    idx = rng.integers(0, 300, size=600).astype(np.int64)
    return pts, idx


# ------------------------------------------------------ oracle pinning (CPU)
def test_reference_label_file_layout(reference, tmp_path):
    asc = np.array([3, 1, 4, 1, 5], np.int64)
    desc = np.array([9, 2, 6, 5, 3], np.int64)
    p = tmp_path / "l.bin"
    reference.write_labels(p, asc, desc)
    b = p.read_bytes()
    assert b[:8] == b"PLMSSLBL" and int.from_bytes(b[8:12], "little") == 1
    assert int.from_bytes(b[12:20], "little") == 5
    rec = np.frombuffer(b[20:], "<u8").reshape(5, 2)
    assert np.array_equal(rec[:, 0], asc) and np.array_equal(rec[:, 1], desc)


@pytest.mark.parametrize("dt", list(DTYPES))
def test_reference_read_volume_values(reference, tmp_path, dt):
    dims = (5, 4, 3)
    v = _volume(np.random.default_rng(1), 60, dt)
    p = tmp_path / "v.raw"
    v.tofile(p)
    assert np.array_equal(reference.read_volume(p, dims, dt), v.astype(np.float64), equal_nan=True)


def test_reference_weld_first_occurrence(reference):
    pts, idx = _soup()
    wp, wi = reference.weld_points(pts, idx)
    # restatement: bitwise keys, first occurrence order
    keys = [p.tobytes() for p in pts]
    first = {}
    for i, k in enumerate(keys):
        first.setdefault(k, len(first))
    order = sorted(first, key=first.get)
    assert np.array_equal(wp.view(np.uint64), np.array([np.frombuffer(k, "<f8") for k in order]).view(np.uint64))
    assert np.array_equal(wi, np.array([first[keys[i]] for i in idx]))


# ----------------------------------------------------------------- B200 (GPU)
def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("dt", list(DTYPES))
def test_read_volume_matches_reference(plmss, gpu, reference, tmp_path, dt):
    dims = (37, 29, 23)  # several staging chunks would need GBs; exercised by the big case below
    v = _volume(np.random.default_rng(11), int(np.prod(dims)), dt)
    p = tmp_path / "v.raw"
    v.tofile(p)
    ref = reference.read_volume(p, dims, dt)
    got = plmss.read_volume(p, dims, dt, out="f64", ctx=gpu).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    if dt != "f64le":
        g32 = plmss.read_volume(p, dims, dt, out="f32", ctx=gpu).cpu().numpy()
        assert np.array_equal(g32.astype(np.float64), ref)
    else:
        with pytest.raises(ValueError):
            plmss.read_volume(p, dims, dt, out="f32", ctx=gpu)


@pytest.mark.gpu
def test_read_volume_streams_chunks(plmss, gpu, tmp_path):
    dims = (512, 256, 160)  # 80 MiB of f32: two staging chunks
    v = (np.arange(int(np.prod(dims)), dtype=np.uint32) * 2654435761 % 1000003).astype("<f4")
    p = tmp_path / "big.raw"
    v.tofile(p)
    got = plmss.read_volume(p, dims, "f32le", ctx=gpu).cpu().numpy()
    assert np.array_equal(got, v)


@pytest.mark.gpu
def test_read_volume_errors_match_reference(plmss, gpu, reference, tmp_path):
    import oracle

    p = tmp_path / "short.raw"
    np.zeros(10, "<f4").tofile(p)
    with pytest.raises(oracle.RefFormatError) as r:
        reference.read_volume(p, (3, 3, 3), "f32le")
    with pytest.raises(plmss.FormatError) as g:
        plmss.read_volume(p, (3, 3, 3), "f32le", ctx=gpu)
    assert str(g.value) == str(r.value)
    with pytest.raises(oracle.RefFormatError) as r:
        reference.read_volume(p, (3, 3, 3), "f16")
    with pytest.raises(plmss.FormatError) as g:
        plmss.read_volume(p, (3, 3, 3), "f16", ctx=gpu)
    assert str(g.value) == str(r.value)
    with pytest.raises(plmss.IoError):
        plmss.read_volume(tmp_path / "missing.raw", (3, 3, 3), "f32le", ctx=gpu)
    with pytest.raises(plmss.FormatError):
        plmss.read_volume(p, (0, 3, 3), "f32le", ctx=gpu)


@pytest.mark.gpu
@pytest.mark.parametrize("width", ["u32", "i64"])
def test_write_labels_byte_identical(plmss, gpu, reference, tmp_path, width):
    import torch

    g = load_case("gauss_17x13x11")
    dims = tuple(int(x) for x in g["dims"])
    seg = plmss.segment(dims, _dev(g["field"]), ctx=gpu)
    asc, desc = seg.asc, seg.desc
    if width == "i64":
        asc, desc = asc.to(torch.int64), desc.to(torch.int64)
    mine, ref = tmp_path / "mine.bin", tmp_path / "ref.bin"
    plmss.write_labels(mine, asc, desc, ctx=gpu)
    reference.write_labels(ref, g["asc"], g["desc"])
    assert mine.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("weld", [False, True])
def test_write_surface_obj_byte_identical(plmss, gpu, reference, tmp_path, weld):
    g = load_case("gauss_17x13x11")
    dims = tuple(int(x) for x in g["dims"])
    res = plmss.pipeline(dims, _dev(g["field"]), ctx=gpu)
    out = plmss.fetch(gpu, res)
    m = plmss.materialize_separators(dims, out["tris"], spacing=(0.5, 1.0, 3.0), origin=(1.0, -2.0, 0.25),
                                     ctx=gpu)
    pts, idx, reg = m["points"], m["indices"], m["regions"]
    if weld:
        pts, idx = plmss.weld_points(pts.clone(), idx.clone(), ctx=gpu)
    mine, ref = tmp_path / "mine.obj", tmp_path / "ref.obj"
    plmss.write_surface_obj(mine, pts, idx, reg, ctx=gpu)
    reference.write_surface_obj(ref, pts.cpu().numpy(), idx.cpu().numpy(), reg.cpu().numpy())
    assert mine.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
def test_write_surface_obj_segments_and_open_regions(plmss, gpu, reference, tmp_path):
    rng = np.random.default_rng(5)
    pts = rng.standard_normal((50, 3)) * 1e3
    pts[3] = [-0.0, 1e-310, np.inf]
    idx = rng.integers(0, 50, size=80).astype(np.int64)
    reg = np.repeat(rng.integers(-1, 4, size=(10, 2)), 4, axis=0).astype(np.int64)
    reg[::7, 1] = -1
    mine, ref = tmp_path / "mine.obj", tmp_path / "ref.obj"
    plmss.write_surface_obj(mine, _dev(pts), _dev(idx), _dev(reg), verts_per_prim=2, ctx=gpu)
    reference.write_surface_obj(ref, pts, idx, reg, verts_per_prim=2)
    assert mine.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
def test_weld_points_matches_reference(plmss, gpu, reference):
    pts, idx = _soup()
    rp, ri = reference.weld_points(pts, idx)
    gp, gi = plmss.weld_points(_dev(pts), _dev(idx), ctx=gpu)
    assert np.array_equal(gp.cpu().numpy().view(np.uint64), rp.view(np.uint64))
    assert np.array_equal(gi.cpu().numpy(), ri)


@pytest.mark.gpu
def test_weld_points_on_separators(plmss, gpu, reference):
    for name in ("gauss_17x13x11", "noise_12x12x12", "quant_24x20x16"):
        g = load_case(name)
        dims = tuple(int(x) for x in g["dims"])
        res = plmss.pipeline(dims, _dev(g["field"]), ctx=gpu)
        out = plmss.fetch(gpu, res)
        m = plmss.materialize_separators(dims, out["tris"], ctx=gpu)
        rp, ri = reference.weld_points(m["points"].cpu().numpy(), m["indices"].cpu().numpy())
        gp, gi = plmss.weld_points(m["points"].clone(), m["indices"].clone(), ctx=gpu)
        assert gp.shape[0] < m["points"].shape[0]
        assert np.array_equal(gp.cpu().numpy().view(np.uint64), rp.view(np.uint64)), name
        assert np.array_equal(gi.cpu().numpy(), ri), name


@pytest.mark.gpu
def test_weld_points_errors(plmss, gpu):
    import torch

    pts = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    bad = torch.tensor([0, 4], dtype=torch.int64, device="cuda")
    with pytest.raises(IndexError):
        plmss.weld_points(pts, bad, ctx=gpu)
    p, i = plmss.weld_points(torch.zeros((0, 3), dtype=torch.float64, device="cuda"),
                             torch.zeros(0, dtype=torch.int64, device="cuda"), ctx=gpu)
    assert p.shape[0] == 0 and i.numel() == 0


# ------------------------------------ streamed separator geometry (f)3 --
@pytest.mark.gpu
@pytest.mark.parametrize("case,scaled_dims", [("gauss_17x13x11", None), ("noise_12x12x12", None),
                                              (None, (96, 80, 64))])
def test_write_separators_obj_byte_identical(plmss, gpu, reference, tmp_path, case, scaled_dims):
    """write_surface_obj(emit_separators(...)) of the reference, streamed from
    the records (the 96x80x64 case spans several point / face chunks)."""
    if case:
        g = load_case(case)
        dims = tuple(int(x) for x in g["dims"])
        f = g["field"]
    else:
        from paper_2303_15491_b200.configs import CONFIGS, host_field, scaled

        cfg = scaled(CONFIGS["cfg1"], scaled_dims)
        dims, f = cfg.dims, host_field(cfg)
    res = plmss.pipeline(dims, _dev(f), ctx=gpu)
    out = plmss.fetch(gpu, res)
    sp, og = (0.5, 1.0, 3.0), (1.0, -2.0, 0.25)
    mine, ref = tmp_path / "mine.obj", tmp_path / "ref.obj"
    plmss.write_separators_obj(mine, dims, out["tris"], spacing=sp, origin=og, ctx=gpu)
    e = reference.emit_separators(dims, out["ms"].cpu().numpy().view(np.uint32).astype(np.int64), spacing=sp,
                                  origin=og)
    reference.write_surface_obj(ref, e["points"], e["indices"], e["regions"])
    assert res.n_tris > (0 if case else 932067)  # > one points chunk for the large case
    assert mine.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
def test_materialize_chunked_equals_whole(plmss, gpu, reference):
    g = load_case("gauss_17x13x11")
    dims = tuple(int(x) for x in g["dims"])
    res = plmss.pipeline(dims, _dev(g["field"]), ctx=gpu)
    out = plmss.fetch(gpu, res)
    whole = plmss.materialize_separators(dims, out["tris"], spacing=(2.0, 1.0, 0.5), ctx=gpu)
    got = {"points": [], "regions": [], "source_cells": []}
    firsts = []

    def sink(first, pts, reg, src):
        firsts.append(first)
        got["points"].append(pts.copy())
        got["regions"].append(reg.copy())
        got["source_cells"].append(src.copy())

    plmss.materialize_separators_chunked(dims, out["tris"], sink, chunk=997, spacing=(2.0, 1.0, 0.5), ctx=gpu)
    assert firsts == list(range(0, res.n_tris, 997))
    for k in got:
        assert np.array_equal(np.concatenate(got[k]), whole[k].cpu().numpy()), k
    # a sink that stops the stream
    with pytest.raises(RuntimeError):
        plmss.materialize_separators_chunked(dims, out["tris"], lambda *a: True, chunk=997, ctx=gpu)
