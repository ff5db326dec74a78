"""GPU parity: the B200 path (through the C-ABI) against the reference's
golden outputs (tests/golden, produced by the compiled reference) and the CPU
restatement oracle, bit for bit. Tolerance: none — all outputs are integer
ids or correctly rounded doubles."""
import hashlib

import numpy as np
import pytest

from conftest import golden_cases, load_case

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def u32(t):
    return (t.to(dtype=__import__("torch").int64) & 0xFFFFFFFF).cpu().numpy()


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# --------------------------------------------------------------- step 1 --
@pytest.mark.parametrize("name", golden_cases())
def test_seed_hops_all_key_types(plmss, gpu, restatement, name):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    f = g["field"]
    d_ref, a_ref = restatement.seed_hops(dims, values=f.astype(np.float64))
    rank = restatement.compute_order(f.astype(np.float64))
    for keys in (dev(f), dev(f.astype(np.float64)), dev(rank)):
        d, a = plmss.seed_hops(dims, keys, ctx=gpu)
        assert np.array_equal(u32(d), d_ref) and np.array_equal(u32(a), a_ref)


def test_seed_hops_signed_zero_and_ties(plmss, gpu, restatement):
    rng = np.random.default_rng(7)
    for dims in [(2, 2, 2), (3, 2, 5), (17, 13, 11), (33, 4, 9)]:
        n = int(np.prod(dims))
        f = rng.integers(-1, 2, size=n).astype(np.float32) * 0.0  # only +-0.0: pure SoS
        f[rng.random(n) < 0.3] = 1.0
        d_ref, a_ref = restatement.seed_hops(dims, values=f.astype(np.float64))
        d, a = plmss.seed_hops(dims, dev(f), ctx=gpu)
        assert np.array_equal(u32(d), d_ref) and np.array_equal(u32(a), a_ref)


# --------------------------------------------------------- segmentation --
@pytest.mark.parametrize("name", golden_cases())
def test_segment_matches_reference(plmss, gpu, name):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    seg = plmss.segment(dims, dev(g["field"]), ctx=gpu)
    for k in ("desc", "asc", "maxima", "minima"):
        assert np.array_equal(u32(getattr(seg, k)), g[k]), k


@pytest.mark.parametrize("direction", [0, 1])
def test_single_direction_matches_fused(plmss, gpu, direction):
    g = load_case("gauss_17x13x11")
    dims = tuple(int(x) for x in g["dims"])
    seg = plmss.segment(dims, dev(g["field"]), direction=direction, ctx=gpu)
    if direction == 0:
        assert seg.desc is None and np.array_equal(u32(seg.asc), g["asc"])
        assert np.array_equal(u32(seg.minima), g["minima"])
    else:
        assert seg.asc is None and np.array_equal(u32(seg.desc), g["desc"])


def reference_noise(dims, seed):
    """synth_field(Noise) of the reference (synth.cpp:57-60): doubles from
    mt19937_64 — used by acceptance criterion 2."""
    from paper_2303_15491_b200.configs import MT19937_64

    r = MT19937_64(seed)
    return np.array([r.uniform01() for _ in range(int(np.prod(dims)))])


def test_acceptance_criterion_2_hundred_seeds(plmss, gpu, restatement):
    """acceptance.cpp:94-117: 100 seeds, sides 8..32, labels equal the oracle."""
    for seed in range(100):
        side = 8 + seed % 25
        dims = (side, side, side)
        vals = reference_noise(dims, seed) if seed < 20 else np.random.default_rng(seed).random(side ** 3)
        ref = restatement.segment(dims, values=vals)
        seg = plmss.segment(dims, dev(vals), ctx=gpu)  # float64 keys
        assert np.array_equal(u32(seg.desc), ref["desc"]), seed
        assert np.array_equal(u32(seg.asc), ref["asc"]), seed


def test_non_finite_input_raises(plmss, gpu):
    f = np.zeros(4 * 4 * 4, np.float32)
    f[37] = np.nan
    f[41] = np.inf
    with pytest.raises(ValueError, match="non-finite scalar value at vertex 37"):
        plmss.segment((4, 4, 4), dev(f), ctx=gpu)


def test_bad_sizes_raise(plmss, gpu):
    with pytest.raises(ValueError, match="does not match"):
        plmss.segment((4, 4, 4), dev(np.zeros(10, np.float32)), ctx=gpu)
    with pytest.raises(ValueError, match="3-D"):
        plmss.segment((4, 4, 1), dev(np.zeros(16, np.float32)), ctx=gpu)
    with pytest.raises(ValueError, match="workers"):
        plmss.segment((4, 4, 4), dev(np.zeros(64, np.float32)), workers=0, ctx=gpu)


# ------------------------------------------------------------ combine_ms --
@pytest.mark.parametrize("path", [0, 1, 2])
@pytest.mark.parametrize("name", golden_cases())
def test_combine_ms_matches_reference(plmss, gpu, name, path):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    gpu.set_option(1, path)
    try:
        seg = plmss.combine_ms(plmss.segment(dims, dev(g["field"]), ctx=gpu), ctx=gpu)
    finally:
        gpu.set_option(1, 0)
    assert np.array_equal(u32(seg.ms_region), g["ms_region"])
    keys = seg.region_keys.cpu().numpy().astype(np.uint64)
    got = np.stack([(keys >> np.uint64(32)).astype(np.int64), (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)], 1)
    assert np.array_equal(got, g["region_keys"])


# -------------------------------------------------------------- marching --
@pytest.mark.parametrize("name", golden_cases())
def test_codes_and_separators_match_reference(plmss, gpu, name):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    ms = dev(g["ms_region"].astype(np.int32))
    codes, total = plmss.index_separators(dims, ms, ctx=gpu)
    assert np.array_equal(codes.cpu().numpy(), g["codes"])
    assert total == int(g["sep_n"])
    recs = plmss.emit_separators(dims, ms, ctx=gpu)
    cells = (recs[:, 0] >> 6).cpu().numpy()
    assert np.all(np.diff(cells) >= 0)  # cell-major reference order
    m = plmss.materialize_separators(dims, recs, ctx=gpu)
    for k in ("points", "regions", "source_cells"):
        arr = m[k].cpu().numpy()
        if f"sep_{k}" in g:
            assert np.array_equal(arr, g[f"sep_{k}"]), k
        assert sha(arr) == str(g[f"sep_{k}_sha256"]), k
    m = plmss.materialize_separators(dims, recs, spacing=(2.0, 1.0, 3.0), origin=(0.5, -1.25, 0.0), ctx=gpu)
    for k in ("points", "regions", "source_cells"):
        assert sha(m[k].cpu().numpy()) == str(g[f"sepsp_{k}_sha256"]), k


@pytest.mark.parametrize("name", ["noise_12x12x12", "ties_9x8x7", "quant_24x20x16"])
def test_union_mode_fields(plmss, gpu, name):
    """Asc / Desc modes label by extremum vertex ids (marching.cpp:328-347)."""
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    for tag in ("asc", "desc"):
        lab = dev(g[tag].astype(np.int32))
        m = plmss.materialize_separators(dims, plmss.emit_separators(dims, lab, ctx=gpu), ctx=gpu)
        assert len(m["source_cells"]) == int(g[f"sep_{tag}_n"])
        for k in ("points", "regions", "source_cells"):
            assert sha(m[k].cpu().numpy()) == str(g[f"sep_{tag}_{k}_sha256"]), (tag, k)


def test_int64_labels_path(plmss, gpu, restatement):
    rng = np.random.default_rng(3)
    dims = (7, 6, 5)
    n = int(np.prod(dims))
    lab = (rng.integers(0, 5, size=n) * 1000003 - 2 ** 40).astype(np.int64)  # negative, > 32 bit
    ref = restatement.emit_separators(dims, lab, spacing=(0.5, 2.0, 1.0), origin=(1.0, 0.0, -3.0))
    codes, total = plmss.index_separators(dims, dev(lab), ctx=gpu)
    assert np.array_equal(codes.cpu().numpy(), ref["codes"]) and total == len(ref["source_cells"])
    recs = plmss.emit_separators(dims, dev(lab), ctx=gpu)
    m = plmss.materialize_separators(dims, recs, spacing=(0.5, 2.0, 1.0), origin=(1.0, 0.0, -3.0), ctx=gpu)
    for k in ("points", "regions", "source_cells"):
        assert np.array_equal(m[k].cpu().numpy(), ref[k]), k
    b = plmss.emit_boundaries(dims, dev(lab), ctx=gpu)
    rb = restatement.emit_boundaries(dims, lab)
    for k in ("points", "indices", "regions", "source_cells"):
        assert np.array_equal(b[k].cpu().numpy(), rb[k]), k


@pytest.mark.parametrize("name", golden_cases())
def test_boundaries_match_reference(plmss, gpu, name):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    for tag, lab in (("bnd_asc", g["asc"]), ("bnd_ms", g["ms_region"])):
        b = plmss.emit_boundaries(dims, dev(lab.astype(np.int32)), ctx=gpu)
        assert len(b["source_cells"]) == int(g[f"{tag}_n"])
        for k in ("points", "indices", "regions", "source_cells"):
            arr = b[k].cpu().numpy()
            if f"{tag}_{k}" in g:
                assert np.array_equal(arr, g[f"{tag}_{k}"]), (tag, k)
            assert sha(arr) == str(g[f"{tag}_{k}_sha256"]), (tag, k)


def test_boundaries_region_filter(plmss, gpu, restatement):
    g = load_case("ties_9x8x7")
    dims = tuple(int(x) for x in g["dims"])
    lab = g["asc"]
    for flt in sorted(set(lab.tolist()))[:5] + [10 ** 9]:
        b = plmss.emit_boundaries(dims, dev(lab.astype(np.int32)), region_filter=flt, ctx=gpu)
        rb = restatement.emit_boundaries(dims, lab, region_filter=flt)
        for k in ("points", "indices", "regions", "source_cells"):
            assert np.array_equal(b[k].cpu().numpy(), rb[k]), (flt, k)


# ---------------------------------------------------------- order field --
def test_compute_order(plmss, gpu, restatement):
    rng = np.random.default_rng(11)
    for vals in (rng.random(5000), rng.integers(0, 7, 5000).astype(np.float64),
                 np.array([2.0, 2.0, 1.0]), np.array([5.0]), np.array([0.0, -0.0, 0.0, -1.0, 1e30, -1e-300])):
        for dt in (np.float64, np.float32):
            v = vals.astype(dt)
            ref = restatement.compute_order(v.astype(np.float64))
            got = plmss.compute_order(dev(v), ctx=gpu).cpu().numpy()
            assert np.array_equal(got, ref)
    with pytest.raises(ValueError, match="vertex 1"):
        plmss.compute_order(dev(np.array([0.0, np.inf, np.nan])), ctx=gpu)


# ------------------------------------------------------- fused pipeline --
# path: 0 fused (dense rank-product region bitmap), 1 staged kernels,
#       2 fused with the hash-set region keys (the path for n_max * n_min >= 2^32),
#       3 fused with pass A split into the hop-code and brick kernels,
#       (paths 0-3 with the per-vertex equality-mask hops, 4-7 with the
#       cube-shared hops, the default)
#       4 fused with the cube-shared steepest hops, 5 = 3 + 4,
#       6 fused with the ids written by the count pass (the default), 7 = 6 +
#       hash-set keys; paths 0-5 run the interleaved token / count passes and
#       the in-place id pass; 8 = the mark pass (region bitmap first, ids
#       written by the token pass, count pass interleaved: IDS_IN_COUNT 2)
@pytest.mark.parametrize("path", [0, 1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("name", golden_cases())
def test_pipeline_matches_reference(plmss, gpu, name, path):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    gpu.set_option(2, 1 if path == 1 else 0)  # PIPELINE_PATH: 0 fused, 1 staged
    gpu.set_option(1, 2 if path in (2, 7) else 0)  # COMBINE_PATH: 2 hash
    gpu.set_option(plmss.OPT_PASS_A_SPLIT, 1 if path in (3, 5) else 0)
    gpu.set_option(plmss.OPT_HOP_CUBE, 1 if path in (4, 5, 6, 7, 8) else 0)
    gpu.set_option(plmss.OPT_IDS_IN_COUNT, 2 if path == 8 else (1 if path in (6, 7) else 0))
    try:
        res = plmss.pipeline(dims, dev(g["field"]), ctx=gpu)
    finally:
        gpu.set_option(2, 0)
        gpu.set_option(1, 0)
        gpu.set_option(plmss.OPT_PASS_A_SPLIT, 0)
        gpu.set_option(plmss.OPT_HOP_CUBE, 1)  # the default
        gpu.set_option(plmss.OPT_IDS_IN_COUNT, 1)  # the default
    out = plmss.fetch(gpu, res)
    for k, gk in (("desc", "desc"), ("asc", "asc"), ("ms", "ms_region"), ("maxima", "maxima"), ("minima", "minima")):
        assert np.array_equal(u32(out[k]), g[gk]), k
    assert res.n_regions == len(g["region_keys"]) and res.n_tris == int(g["sep_n"])
    keys = out["region_keys"].cpu().numpy().astype(np.uint64)
    assert np.array_equal((keys >> np.uint64(32)).astype(np.int64), g["region_keys"][:, 0])
    assert np.array_equal((keys & np.uint64(0xFFFFFFFF)).astype(np.int64), g["region_keys"][:, 1])
    m = plmss.materialize_separators(dims, out["tris"], ctx=gpu)
    for k in ("points", "regions", "source_cells"):
        assert sha(m[k].cpu().numpy()) == str(g[f"sep_{k}_sha256"]), k


def test_pipeline_host_e2e(plmss, gpu):
    g = load_case("gauss_17x13x11")
    dims = tuple(int(x) for x in g["dims"])
    tris = np.empty((int(g["sep_n"]), 2), np.uint64)
    res, out = plmss.pipeline_host(dims, g["field"], ctx=gpu, out_buffers={"tris": tris})
    assert np.array_equal(out["desc"].astype(np.int64), g["desc"])
    assert np.array_equal(out["ms"].astype(np.int64), g["ms_region"])
    keys = out["region_keys"]
    assert np.array_equal((keys >> np.uint64(32)).astype(np.int64), g["region_keys"][:, 0])
    assert res.n_tris == len(out["tris"])


# Fused pipeline across brick boundaries: partial bricks (dims not multiples
# of 32), multi-brick chains, tie-heavy and white-noise fields (the latter
# with many extrema), both region-key modes; oracle = the C restatement.
def _field(kind, dims, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    if kind == "noise":
        return rng.random(n).astype(np.float32)
    if kind == "ties":
        return rng.integers(0, 4, n).astype(np.float32)
    from paper_2303_15491_b200.configs import CONFIGS, host_field, scaled

    return host_field(scaled(CONFIGS["cfg2"], dims))


@pytest.mark.parametrize("path", [0, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("dims,kind", [((97, 66, 40), "gauss"), ((33, 33, 33), "noise"), ((64, 31, 65), "ties"),
                                       ((128, 96, 70), "gauss"), ((70, 40, 36), "noise"), ((36, 20, 33), "ties")])
def test_pipeline_brick_geometry(plmss, gpu, restatement, dims, kind, path):
    f = _field(kind, dims, sum(dims))
    gpu.set_option(1, 2 if path in (2, 7) else 0)
    gpu.set_option(plmss.OPT_PASS_A_SPLIT, 1 if path in (3, 5) else 0)
    gpu.set_option(plmss.OPT_HOP_CUBE, 1 if path in (4, 5, 6, 7, 8) else 0)
    gpu.set_option(plmss.OPT_IDS_IN_COUNT, 2 if path == 8 else (1 if path in (6, 7) else 0))
    try:
        res = plmss.pipeline(dims, dev(f), ctx=gpu)
    finally:
        gpu.set_option(1, 0)
        gpu.set_option(plmss.OPT_PASS_A_SPLIT, 0)
        gpu.set_option(plmss.OPT_HOP_CUBE, 1)  # the default
        gpu.set_option(plmss.OPT_IDS_IN_COUNT, 1)  # the default
    out = plmss.fetch(gpu, res)
    s = restatement.segment(dims, values=f.astype(np.float64))
    ms, keys = restatement.combine_ms(s["asc"], s["desc"])
    for k, ref in (("desc", s["desc"]), ("asc", s["asc"]), ("ms", ms), ("maxima", s["maxima"]),
                   ("minima", s["minima"])):
        assert np.array_equal(u32(out[k]), ref), k
    rk = out["region_keys"].cpu().numpy().astype(np.uint64)
    assert np.array_equal((rk >> np.uint64(32)).astype(np.int64), keys[:, 0])
    assert np.array_equal((rk & np.uint64(0xFFFFFFFF)).astype(np.int64), keys[:, 1])
    e = restatement.emit_separators(dims, ms)
    assert res.n_tris == len(e["source_cells"])
    m = plmss.materialize_separators(dims, out["tris"], ctx=gpu)
    assert np.array_equal(m["source_cells"].cpu().numpy(), e["source_cells"])
    assert np.array_equal(m["regions"].cpu().numpy(), e["regions"])
    assert np.array_equal(m["points"].cpu().numpy(), e["points"])


# Chains through many bricks (a ramp along x crosses 128 bricks) and the
# fallback when the terminal forest has not converged after the speculative
# sweeps: the sweeps continue and passes C and D are redone.
@pytest.mark.parametrize("spec", [1, 2, 0])
def test_pipeline_long_forest_chains(plmss, gpu, restatement, spec):
    dims = (4096, 6, 5)
    x = np.arange(dims[0], dtype=np.float64)[None, None, :]
    y = np.arange(dims[1], dtype=np.float64)[None, :, None]
    z = np.arange(dims[2], dtype=np.float64)[:, None, None]
    f = (x + 1e-3 * np.sin(y + 2 * z) + 0 * z).astype(np.float32).reshape(-1)
    gpu.set_option(plmss.OPT_SPECULATIVE_SWEEPS, spec)
    try:
        res = plmss.pipeline(dims, dev(f), ctx=gpu)
    finally:
        gpu.set_option(plmss.OPT_SPECULATIVE_SWEEPS, 1)
    out = plmss.fetch(gpu, res)
    s = restatement.segment(dims, values=f.astype(np.float64))
    ms, keys = restatement.combine_ms(s["asc"], s["desc"])
    for k, ref in (("desc", s["desc"]), ("asc", s["asc"]), ("ms", ms)):
        assert np.array_equal(u32(out[k]), ref), k
    e = restatement.emit_separators(dims, ms)
    assert res.n_tris == len(e["source_cells"])
    assert res.sweeps >= 1
    m = plmss.materialize_separators(dims, out["tris"], ctx=gpu)
    assert np.array_equal(m["source_cells"].cpu().numpy(), e["source_cells"])
    assert np.array_equal(m["regions"].cpu().numpy(), e["regions"])


@pytest.mark.gpu
def test_library_is_ordered_after_torch_default_stream(plmss, gpu):
    """Inputs produced by torch ops on the default stream, then a library call
    with no host sync in between (the z-slab path's pattern,
    distributed.py): the context must run on the same stream as torch."""
    import torch

    from paper_2303_15491_b200 import api

    dims = (192, 160, 128)
    n = dims[0] * dims[1] * dims[2]
    g = torch.Generator(device="cuda").manual_seed(7)
    base = torch.randint(0, 1 << 20, (n,), device="cuda", generator=g)
    torch.cuda.synchronize()
    got = []
    for _ in range(3):
        lab = torch.sort(base)[0] // 4096  # slow enough to still run when the library starts
        got.append(api.index_separators(dims, lab, ctx=gpu)[1])
        del lab
    torch.cuda.synchronize()
    lab = torch.sort(base)[0] // 4096
    torch.cuda.synchronize()
    want = api.index_separators(dims, lab, ctx=gpu)[1]
    assert want > 0 and got == [want] * 3
    r = api.emit_separators(dims, torch.sort(base)[0] // 4096, ctx=gpu)
    assert r.shape[0] == want



def test_pipeline_host_batch_matches_single_calls(plmss, gpu):
    """plmss_b200_pipeline_host_batch (two internal contexts, alternate
    volumes) returns every volume's outputs exactly as pipeline_host."""
    from paper_2303_15491_b200.configs import CONFIGS, host_field, scaled

    vols, refs = [], []
    for i, dims in enumerate([(40, 36, 33), (40, 36, 33), (40, 36, 33), (40, 36, 33), (40, 36, 33)]):
        f = host_field(scaled(CONFIGS["cfg2" if i % 2 else "cfg1"], dims))
        res, out = plmss.pipeline_host(dims, f, ctx=gpu,
                                       out_buffers={"tris": np.empty((4000000, 2), np.uint64)})
        refs.append((res, out))
        v = {"field": f, "desc": np.empty(f.size, np.uint32), "asc": np.empty(f.size, np.uint32),
             "ms": np.empty(f.size, np.uint32), "tris": np.empty((res.n_tris, 2), np.uint64)}
        vols.append(v)
    rb = plmss.pipeline_host_batch((40, 36, 33), vols, ctx=gpu)
    for (res, out), v, r in zip(refs, vols, rb):
        assert (r.n_tris, r.n_regions, r.n_maxima) == (res.n_tris, res.n_regions, res.n_maxima)
        for k in ("desc", "asc", "ms"):
            assert np.array_equal(v[k], out[k]), k
        assert np.array_equal(v["tris"], out["tris"][: res.n_tris])


@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 2, 2), (2, 3, 2), (2, 2, 3), (33, 2, 2), (2, 2, 65), (4, 33, 2),
                                  (65, 3, 34)])
def test_pipeline_degenerate_extents(plmss, gpu, restatement, dims):
    """Extents of 2 (one cube layer), single partial bricks and bricks cut
    to one vertex in some axis, against the restatement."""
    rng = np.random.default_rng(sum(dims))
    f = rng.integers(0, 3, int(np.prod(dims))).astype(np.float32)
    res = plmss.pipeline(dims, dev(f), ctx=gpu)
    out = plmss.fetch(gpu, res)
    s = restatement.segment(dims, values=f.astype(np.float64))
    ms, keys = restatement.combine_ms(s["asc"], s["desc"])
    for k, ref in (("desc", s["desc"]), ("asc", s["asc"]), ("ms", ms)):
        assert np.array_equal(u32(out[k]), ref), k
    e = restatement.emit_separators(dims, ms)
    assert res.n_tris == len(e["source_cells"])
    if res.n_tris:
        m = plmss.materialize_separators(dims, out["tris"], ctx=gpu)
        assert np.array_equal(m["source_cells"].cpu().numpy(), e["source_cells"])
        assert np.array_equal(m["points"].cpu().numpy(), e["points"])
